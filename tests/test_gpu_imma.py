"""GPU: the integer-tensor-core linear layers (csrc/conv_imma.cu).

The byte-sliced mma.sync path must give the same words as the reference's
sequential mul_scalar_mac accumulation (ckks.hpp:448-465). Small cases are
compared with the compiled reference directly; the sizes where the reference
is too slow (K > 6144 taps, where the int32 class sums are folded, weights
beyond the signed-digit range) are compared word-for-word with the
gather-MAC kernels (HECNN_NO_IMMA=1), which tests/test_gpu_parity.py pins to
the reference."""
import os

import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu

SWEEP_BITS = [60] + [40] * 8


def _words(p, cells, level, seed):
    rng = np.random.default_rng(seed)
    w = np.empty((cells, 2, level + 1, p.n), dtype=np.uint64)
    for i in range(level + 1):
        w[:, :, i, :] = rng.integers(0, p.primes[i], size=(cells, 2, p.n), dtype=np.uint64)
    return w


def _forward(eng, spec, words, level, scale, imma):
    """One forward pass with the tensor-core path on or off (the switch is read
    when a model builds its per-level weight caches, so each call uses a fresh
    model)."""
    old = os.environ.get("HECNN_NO_IMMA")
    os.environ["HECNN_NO_IMMA"] = "0" if imma else "1"
    try:
        m = eng.model(spec)
        x = eng.tensor_from_words(words, level, scale)
        x.set_shape(spec.input, 1)
        y = hb.forward_encrypted(m, x, eng)
        return y.words(), y.level, y.scale
    finally:
        if old is None:
            del os.environ["HECNN_NO_IMMA"]
        else:
            os.environ["HECNN_NO_IMMA"] = old


def _compare(p, spec, seed=3, level=None):
    eng = hb.CkksEngine(p).keygen(1)
    level = p.top_level if level is None else level
    words = _words(p, spec.input.positions(), level, seed)
    a = _forward(eng, spec, words, level, p.scale, True)
    b = _forward(eng, spec, words, level, p.scale, False)
    assert a[1] == b[1] and a[2] == b[2]
    assert np.array_equal(a[0], b[0])


def test_imma_conv_matches_reference(ref):
    """K = 450 taps (15 tensor-core steps, last one ragged), same padding,
    OC = 6 (one padded channel tile), chain [60, 40 x 8]: 40-bit limbs on the
    u8 x u8 kernel, the 60-bit limb on the signed-digit kernel."""
    p = hb.CkksParams(1024, hb.find_chain(1024, SWEEP_BITS), 2.0 ** 40, 3.2, False)
    spec = hb.ModelSpec(hb.Shape.spatial(5, 5, 18))
    spec.layers = [hb.LayerSpec.conv2d(6, 5, 5), hb.LayerSpec.dense(3)]
    ref.init_random_weights(spec, 9)
    eng = hb.CkksEngine(p).keygen(2)
    r = ref.RefEngine.from_params(p).keygen(2)
    rng = np.random.default_rng(4)
    data = rng.uniform(-1, 1, size=(2, 5 * 5 * 18))
    tx = eng.encrypt_tensor(data, seed=5, shape=spec.input)
    rx = r.encrypt_tensor(data, spec.input, seed=5)
    ty = hb.forward_encrypted(spec, tx, eng, seed=6)
    ry, _ = r.forward_encrypted(spec, rx, seed=6)
    assert ty.level == ry.info()[1] and ty.scale == ry.info()[2]
    assert np.array_equal(ty.words(), ry.words())


def test_imma_dense_fold_long_k():
    """K = 6500 > 6144: both kernels fold their int32 class sums mid-way."""
    p = hb.preset_params("nn-n4096-d8")
    spec = hb.ModelSpec(hb.Shape.flattened(6500))
    spec.layers = [hb.LayerSpec.dense(20)]
    hb.glorot_weights(spec, 7)
    _compare(p, spec)


def test_imma_wide_weights_fall_back_exactly():
    """|round(w * Delta)| >= 2^47 leaves the signed-digit range: the 60-bit limb
    goes back to the gather-MAC, the 40-bit limbs stay on the tensor cores."""
    p = hb.preset_params("nn-n4096-d8")
    spec = hb.ModelSpec(hb.Shape.flattened(40))
    spec.layers = [hb.LayerSpec.dense(5)]
    hb.glorot_weights(spec, 2)
    spec.weights[0] = spec.weights[0] * 4.0e3
    _compare(p, spec)


@pytest.mark.parametrize("oc,kh,cin", [(10, 3, 3), (33, 3, 4), (16, 1, 32), (48, 2, 9)])
def test_imma_conv_shapes(oc, kh, cin):
    """Channel tiles with padding and odd pairing, K = 27 / 36 / 32 / 36."""
    p = hb.preset_params("nn-n4096-d8")
    spec = hb.ModelSpec(hb.Shape.spatial(6, 6, cin))
    spec.layers = [hb.LayerSpec.conv2d(oc, kh, kh)]
    hb.glorot_weights(spec, oc)
    _compare(p, spec, level=5)
