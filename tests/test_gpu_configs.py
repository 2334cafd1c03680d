"""GPU: whole BASELINE configs word for word against the reference (SURVEY
§8(d)): C3 (CryptoNets-style, 28x28x1) and C4 (CIFAR-shaped with the degree-2
ReLU surrogate, 32x32x3), each on a full set of 4096 encrypted synthetic
images at net-n8192-d8 -- the same inputs, keys and seeds on both sides, the
reference running on every host core. C4's reference pass takes about a
minute on a 16-core host."""
import os

import numpy as np
import pytest

import bench
import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_full_config_matches_reference(ref, config):
    p = hb.preset_params("net-n8192-d8")
    spec = bench.c3_spec(hb) if config == "c3" else bench.c4_spec(hb)
    threads = os.cpu_count() or 1
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(1)
    y = hb.forward_encrypted(spec, eng.encrypt_tensor(data, seed=11, shape=spec.input), eng, seed=13)
    r = ref.RefEngine.from_params(p).keygen(1)
    ry, _ = r.forward_encrypted(spec, r.encrypt_tensor(data, spec.input, seed=11, threads=threads), seed=13,
                                threads=threads)
    assert (y.level, y.scale) == ry.info()[1:]
    assert np.array_equal(y.words(), ry.words())
    # and the decrypted logits agree with the plain model within the reference's tolerance
    plain = ref.forward_plain(spec, data[:64])
    dec = eng.decrypt_tensor(y, p.n // 2)[:64]
    assert np.max(np.abs(dec - plain)) < 1e-2


def test_c5_ring_slice_matches_reference(ref):
    """C5's ring (large-n16384-d24, 25 limbs, 8192 slots) on a slice of its
    stack: conv 11x11 (K = 363: the tcgen05 path for every limb) -> relu-poly2
    (key switch at N = 2^14, level 23, 49 digits) -> avg_pool 2 -> dense(1),
    on a 4x4x3 crop with 8 filters (the full AlexNet layers are too slow for
    the reference)."""
    p = hb.preset_params("large-n16384-d24")
    spec = hb.ModelSpec(hb.Shape.spatial(4, 4, 3))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.conv2d(8, 11, 11), hb.LayerSpec.activation("relu-poly2"), hb.LayerSpec.avg_pool2d(2),
                   hb.LayerSpec.dense(1)]
    spec = hb.glorot_weights(spec, 5)
    threads = os.cpu_count() or 1
    data = np.random.default_rng(7).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(3)
    eng.profile_reset()
    eng.profile(True)
    y = hb.forward_encrypted(spec, eng.encrypt_tensor(data, seed=21, shape=spec.input), eng, seed=23)
    eng.synchronize()
    eng.profile(False)
    assert "k_conv_tc" in eng.profile_read()
    r = ref.RefEngine.from_params(p).keygen(3)
    ry, _ = r.forward_encrypted(spec, r.encrypt_tensor(data, spec.input, seed=21, threads=threads), seed=23,
                                threads=threads)
    assert (y.level, y.scale) == ry.info()[1:]
    assert np.array_equal(y.words(), ry.words())


def narrow_alexnet(image):
    """alexnet32_preset's layer sequence (model.hpp:189-219) -- conv 11x11 /
    5x5 / 3x3 / 3x3, six relu-poly2 activations, four pools, three zero-pads,
    three dense layers, sigmoid: all 23 levels of large-n16384-d24 -- with
    narrow channels (8/16/16/16, dense 32/32/1) so the reference finishes in
    about a minute on 16 host cores."""
    m = hb.ModelSpec(hb.Shape.spatial(image, image, 3))
    m.activations["relu-poly2"] = hb.relu_default_surrogate()
    act = lambda: hb.LayerSpec.activation("relu-poly2")  # noqa: E731
    L = hb.LayerSpec
    m.layers = [L.conv2d(8, 11, 11), act(), L.avg_pool2d(2), L.conv2d(16, 5, 5), act(),
                L.avg_pool2d(2), L.zero_pad2d(1), L.conv2d(16, 3, 3), act(),
                L.avg_pool2d(2), L.zero_pad2d(1), L.conv2d(16, 3, 3), act(),
                L.zero_pad2d(1), L.avg_pool2d(2), L.dense(32), act(),
                L.dense(32), act(), L.dense(1), L.sigmoid()]
    m.ensure_param_slots()
    return hb.glorot_weights(m, 1)


def test_c5_full_depth_stack_matches_reference(ref):
    """C5's whole layer sequence at full depth (levels 24 -> 1) on an 8x8x3
    crop, row-streamed with one-column tiles and run whole: both equal the
    reference word for word, and the decrypted logit (through the exact
    sigmoid) matches the plain model."""
    p = hb.preset_params("large-n16384-d24")
    spec = narrow_alexnet(8)
    threads = os.cpu_count() or 1
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(1)
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    streamed = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_ALWAYS, tile=1), x, eng, seed=13)
    whole = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_NEVER), x, eng, seed=13)
    assert np.array_equal(streamed.words(), whole.words())
    r = ref.RefEngine.from_params(p).keygen(1)
    ry, _ = r.forward_encrypted(spec, r.encrypt_tensor(data, spec.input, seed=11, threads=threads), seed=13,
                                threads=threads)
    assert (streamed.level, streamed.scale) == ry.info()[1:] and streamed.level == 1
    assert np.array_equal(streamed.words(), ry.words())
    # the plain path applies the trailing sigmoid; the encrypted pass stops at the logits (layers.hpp:8-9)
    plain = ref.forward_plain(spec, data[:64])
    dec = eng.decrypt_tensor(streamed, p.n // 2)[:64]
    assert np.max(np.abs(1.0 / (1.0 + np.exp(-dec)) - plain)) < 1e-3
