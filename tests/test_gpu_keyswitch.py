"""GPU: the key switch of the 60-bit limb 0 computed through limbs 1..3
(keyswitch.cu "aux": exact integer convolution of the digits with INTT_q0 of
the evaluation key, recovered by a 3-prime CRT) against the reference and the
C restatement, word for word, at the ring degrees and levels where it runs
(N = 2^13, 2^14; levels 3..top) -- raw key switch (hecnn_key_switch, C
oracle or_key_switch), mul and square (the reference), with keys both
generated on the device and imported from the reference."""
import ctypes
import os

import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _orc():
    L = ctypes.CDLL(os.path.join(ROOT, "oracle", "liboracle.so"))
    L.or_relin_digits.restype = ctypes.c_size_t
    return L


def _p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))


@pytest.mark.parametrize("preset,levels", [("net-n8192-d8", (8, 5, 3)), ("large-n16384-d24", (23, 9, 3))])
def test_mul_square_through_aux_limbs(ref, preset, levels):
    p = hb.preset_params(preset)
    eng = hb.CkksEngine(p).keygen(3)
    r = ref.RefEngine.from_params(p).keygen(3)
    for level in levels:
        x = np.stack([r.sample_uniform(level, 100 + 2 * level + k) for k in range(2)])[None]
        y = np.stack([r.sample_uniform(level, 300 + 2 * level + k) for k in range(2)])[None]
        tx, ty = eng.tensor_from_words(x, level, p.scale), eng.tensor_from_words(y, level, p.scale)
        want, _ = r.mul(x[0], y[0], level, p.scale, p.scale)
        assert np.array_equal(eng.mul(tx, ty).words()[0], want), f"mul at level {level}"
        want_sq, _ = r.square(x[0], level, p.scale)
        assert np.array_equal(eng.square(tx).words()[0], want_sq), f"square at level {level}"


def test_raw_key_switch_with_imported_keys(ref):
    """hecnn_key_switch (mode 0) on uniform d2 with the reference's evaluation
    key imported into the engine, against the C restatement or_key_switch."""
    p = hb.preset_params("net-n8192-d8")
    r = ref.RefEngine.from_params(p).keygen(5)
    s, b, a, evk = r.export_keys()
    eng = hb.CkksEngine(p)
    eng.import_keys(secret=s, pk_b=b, pk_a=a, evk=evk)
    orc = _orc()
    n, top = p.n, p.top_level
    primes = np.array(p.primes, dtype=np.uint64)
    roots = np.zeros((top + 1, n), np.uint64)
    iroots = np.zeros(n, np.uint64)
    ninv = ctypes.c_uint64()
    for i, q in enumerate(p.primes):
        assert orc.or_ntt_tables(ctypes.c_size_t(n), ctypes.c_uint64(q), _p(roots[i]), _p(iroots), ctypes.byref(ninv)) == 0
    for level in (7, 3):
        d2 = r.sample_uniform(level, 77 + level)
        got = eng.key_switch(d2[None], level)[0]
        want = np.zeros((2, level + 1, n), np.uint64)
        evk_c = np.ascontiguousarray(evk)
        orc.or_key_switch(ctypes.c_size_t(n), _p(primes), ctypes.c_size_t(top), _p(roots), ctypes.c_size_t(level),
                          _p(np.ascontiguousarray(d2)), _p(evk_c), _p(want))
        assert np.array_equal(got, want), f"key switch at level {level}"


@pytest.mark.parametrize("preset,level", [("net-n8192-d8", 7), ("large-n16384-d24", 23), ("large-n16384-d24", 2)])
def test_key_switch_crt_extremes(ref, preset, level):
    """The CRT digits (k_crt_digits) at the edges of [0, Q): coefficients
    with x = Q - 1 (residues q_i - 1: the quotient estimate sum_i w_i/q_i sits
    just below an integer and the exact fix-up decides), x = 0, x = 1 and a
    single-limb residue, the rest uniform -- the key switch against the C
    restatement with the reference's keys."""
    p = hb.preset_params(preset)
    r = ref.RefEngine.from_params(p).keygen(5)
    s, b, a, evk = r.export_keys()
    eng = hb.CkksEngine(p)
    eng.import_keys(secret=s, pk_b=b, pk_a=a, evk=evk)
    orc = _orc()
    n, top = p.n, p.top_level
    primes = np.array(p.primes, dtype=np.uint64)
    roots = np.zeros((top + 1, n), np.uint64)
    iroots = np.zeros(n, np.uint64)
    ninv = ctypes.c_uint64()
    for i, q in enumerate(p.primes):
        assert orc.or_ntt_tables(ctypes.c_size_t(n), ctypes.c_uint64(q), _p(roots[i]), _p(iroots), ctypes.byref(ninv)) == 0
    d2 = r.sample_uniform(level, 91 + level)
    q = primes[: level + 1, None]
    d2[:, 0:64] = q - 1                      # x = Q - 1
    d2[:, 64:128] = 0                        # x = 0
    d2[:, 128:192] = 1                       # x = 1
    d2[:, 192:256] = 0
    d2[0, 192:256] = 1                       # x = Q/q_0 * [(Q/q_0)^-1 mod q_0]
    got = eng.key_switch(d2[None], level)[0]
    want = np.zeros((2, level + 1, n), np.uint64)
    orc.or_key_switch(ctypes.c_size_t(n), _p(primes), ctypes.c_size_t(top), _p(roots), ctypes.c_size_t(level),
                      _p(np.ascontiguousarray(d2)), _p(np.ascontiguousarray(evk)), _p(want))
    assert np.array_equal(got, want)
