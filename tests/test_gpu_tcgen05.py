"""GPU: the conv layers on the 5th-generation tensor cores (csrc/conv_tc.cu,
tcgen05.mma kind::i8 with TMEM accumulators, K >= 256 taps; the 40-bit limbs
as u8 x u8 byte planes, the 60-bit limb as signed weight digits x u8).

The kernel must give the reference's words (mul_scalar_mac summed over the
taps, ckks.hpp:448-465 via layers.hpp:174-211). Checked directly against the
compiled reference at small N, and at the large-n16384-d24 ring (the C5
shapes, where the reference is too slow) against the gather-MAC kernels
(HECNN_NO_IMMA=1, pinned to the reference by test_gpu_parity.py). Each case
also checks from the launch profile that k_conv_tc actually ran."""
import os

import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu

SWEEP_BITS = [60] + [40] * 8


def _run(eng, spec, x, env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        eng.profile_reset()
        eng.profile(True)
        y = hb.forward_encrypted(eng.model(spec), x, eng, seed=6)
        eng.synchronize()
        eng.profile(False)
        return y, eng.profile_read()
    finally:
        for k, v in old.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v


@pytest.mark.parametrize("oc,k,cin,valid", [(100, 3, 40, False), (48, 9, 5, True), (7, 5, 12, False)])
def test_tcgen05_conv_matches_reference(ref, oc, k, cin, valid):
    """K = 360 / 405 / 300 taps (ragged last step), 1-3 channel tiles with
    padded channels, same and valid padding, n = 1024, chain [60, 40 x 8]."""
    p = hb.CkksParams(1024, hb.find_chain(1024, SWEEP_BITS), 2.0 ** 40, 3.2, False)
    side = 6 if not valid else 10
    spec = hb.ModelSpec(hb.Shape.spatial(side, side, cin))
    spec.layers = [hb.LayerSpec.conv2d(oc, k, k, valid=valid)]
    ref.init_random_weights(spec, oc + k)
    eng = hb.CkksEngine(p).keygen(2)
    r = ref.RefEngine.from_params(p).keygen(2)
    data = np.random.default_rng(4).uniform(-1, 1, size=(3, side * side * cin))
    tx = eng.encrypt_tensor(data, seed=5, shape=spec.input)
    rx = r.encrypt_tensor(data, spec.input, seed=5)
    ty, prof = _run(eng, spec, tx, {})
    assert "k_conv_tc" in prof, "the tcgen05 conv did not run"
    assert "k_conv_tc_wide" in prof, "the 60-bit limb did not run on tcgen05"
    ry, _ = r.forward_encrypted(spec, rx, seed=6)
    assert ty.level == ry.info()[1] and ty.scale == ry.info()[2]
    assert np.array_equal(ty.words(), ry.words())


def test_tcgen05_conv_c5_ring_matches_gather_mac():
    """AlexNet conv3-like layer (3x3, 64 -> 96) at large-n16384-d24, level 18:
    every 40-bit limb on tcgen05, compared with the gather-MAC kernels."""
    p = hb.preset_params("large-n16384-d24")
    eng = hb.CkksEngine(p).keygen(1)
    spec = hb.ModelSpec(hb.Shape.spatial(3, 3, 64))
    spec.layers = [hb.LayerSpec.conv2d(96, 3, 3)]
    hb.glorot_weights(spec, 5)
    level = 18
    rng = np.random.default_rng(8)
    words = np.empty((9 * 64, 2, level + 1, p.n), dtype=np.uint64)
    for i in range(level + 1):
        words[:, :, i, :] = rng.integers(0, p.primes[i], size=(9 * 64, 2, p.n), dtype=np.uint64)
    x = eng.tensor_from_words(words, level, p.scale)
    x.set_shape(spec.input, p.n // 2)
    a, prof = _run(eng, spec, x, {"HECNN_NO_IMMA": "0"})
    assert "k_conv_tc" in prof and "k_conv_tc_wide" in prof
    b, prof_b = _run(eng, spec, x, {"HECNN_NO_IMMA": "1"})
    assert "k_conv_tc" not in prof_b
    assert (a.level, a.scale) == (b.level, b.scale)
    assert np.array_equal(a.words(), b.words())
