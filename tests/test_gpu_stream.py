"""GPU: the row-streamed forward pass (stream.cpp) against the
whole-tensor pass and the reference, word for word.

Streaming changes only which ciphertexts are resident when (rings of rows,
tile transients, lazily produced zero-pad margins); every output word must
be the reference's. The models here are chosen so the rings wrap (more rows
than the window), tiles are ragged, pads feed convs and pools, and a pool
follows a pad (alexnet32_preset layers 14-15)."""
import os

import numpy as np
import pytest

import bench
import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu


def tall_spec():
    """A tall narrow map so each ring holds fewer rows than the tensor:
    conv 3x3 -> relu-poly2 -> pool 2 -> pad 1 -> conv 3x3 -> relu-poly2 ->
    pad 1 -> pool 2 -> dense(2); depth 9 on a 10-limb chain."""
    spec = hb.ModelSpec(hb.Shape.spatial(16, 6, 3))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    act = lambda: hb.LayerSpec.activation("relu-poly2")  # noqa: E731
    spec.layers = [hb.LayerSpec.conv2d(4, 3, 3), act(), hb.LayerSpec.avg_pool2d(2), hb.LayerSpec.zero_pad2d(1),
                   hb.LayerSpec.conv2d(5, 3, 3), act(), hb.LayerSpec.zero_pad2d(1), hb.LayerSpec.avg_pool2d(2),
                   hb.LayerSpec.dense(2)]
    return hb.glorot_weights(spec, 6)


def tall_params():
    return hb.CkksParams(4096, hb.find_chain(4096, [60] + [40] * 9), 2.0 ** 40, 3.2, False)


@pytest.mark.parametrize("tile", [0, 1, 2])
def test_streamed_tall_model_matches_reference(ref, tile):
    p = tall_params()
    spec = tall_spec()
    data = np.random.default_rng(17).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(2)
    x = eng.encrypt_tensor(data, seed=31, shape=spec.input)
    whole = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_NEVER), x, eng, seed=41)
    m = eng.model(spec).set_streaming(hb.Model.STREAM_ALWAYS, tile=tile)
    secs = []
    streamed = hb.forward_encrypted(m, x, eng, seed=41, layer_seconds=secs)
    assert (streamed.level, streamed.scale) == (whole.level, whole.scale)
    assert np.array_equal(streamed.words(), whole.words())
    assert len(secs) == len(spec.layers) and all(s >= 0 for s in secs) and sum(secs) > 0
    threads = os.cpu_count() or 1
    r = ref.RefEngine.from_params(p).keygen(2)
    ry, _ = r.forward_encrypted(spec, r.encrypt_tensor(data, spec.input, seed=31, threads=threads), seed=41,
                                threads=threads)
    assert (streamed.level, streamed.scale) == ry.info()[1:]
    assert np.array_equal(streamed.words(), ry.words())


def test_memory_budget_triggers_streaming_with_identical_words():
    """Mode 0 with a device budget below the whole-tensor peak streams on its
    own and still yields the same words (C4 stack at 16x16, net-n8192-d8)."""
    p = hb.preset_params("net-n8192-d8")
    spec = bench.c4_spec(hb, 16)
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(1)
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    whole = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_NEVER), x, eng, seed=13)
    # conv1 output at 16x16x16, level 7: 4096 cells x 1 MiB = 4 GiB; plan with 14 GiB
    budget = 14 << 30
    m = eng.model(spec).set_streaming(hb.Model.STREAM_AUTO, mem_budget=budget)
    eng.profile_reset()
    eng.profile(True)
    y = hb.forward_encrypted(m, x, eng, seed=13)
    eng.synchronize()
    eng.profile(False)
    assert np.array_equal(y.words(), whole.words())


def test_streamed_alexnet_crop_matches_whole_tensor_pass():
    """Every alexnet32_preset layer kind on C5's ring (large-n16384-d24) on an
    8x8x3 crop: conv 11x11 / 5x5 / 3x3 on tcgen05, activations at levels 23..2,
    pads feeding convs, the pool after a pad -- streamed with one-column
    tiles against the whole-tensor pass."""
    p = hb.preset_params("large-n16384-d24")
    spec = hb.glorot_weights(hb.alexnet32_preset(image=8), 1)
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(1)
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    whole = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_NEVER), x, eng, seed=13)
    streamed = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_ALWAYS, tile=1), x, eng, seed=13)
    assert (streamed.level, streamed.scale) == (whole.level, whole.scale)
    assert np.array_equal(streamed.words(), whole.words())


def test_streamed_cryptonets_matches_reference(ref):
    """C3 forced through the streaming executor: the leading pad
    runs whole, then a stride-2 valid conv + square stage is row-streamed with
    ragged two-column tiles; every output word equals the reference's."""
    p = hb.preset_params("net-n8192-d8")
    spec = bench.c3_spec(hb)
    threads = os.cpu_count() or 1
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(1)
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    y = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_ALWAYS, tile=2), x, eng, seed=13)
    r = ref.RefEngine.from_params(p).keygen(1)
    ry, _ = r.forward_encrypted(spec, r.encrypt_tensor(data, spec.input, seed=11, threads=threads), seed=13,
                                threads=threads)
    assert (y.level, y.scale) == ry.info()[1:]
    assert np.array_equal(y.words(), ry.words())
