"""CPU: pin the C restatement (oracle/hecnn_oracle.c) against the reference's
golden vectors (tests/golden/golden.npz, produced by the compiled reference)
and its own known answers; when the reference oracle library is present,
also against the live reference on fresh seeded inputs."""
import ctypes
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))
_u64p = ctypes.POINTER(ctypes.c_uint64)


@pytest.fixture(scope="module")
def orc():
    path = os.path.join(ROOT, "oracle", "liboracle.so")
    if not os.path.exists(path):
        import subprocess
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "liboracle.so"], check=True)
    L = ctypes.CDLL(path)
    L.or_relin_digits.restype = ctypes.c_size_t
    return L


def p(a, t=ctypes.c_uint64):
    return a.ctypes.data_as(ctypes.POINTER(t))


def tables(orc, n, q):
    roots, iroots = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
    ninv = ctypes.c_uint64()
    assert orc.or_ntt_tables(ctypes.c_size_t(n), ctypes.c_uint64(q), p(roots), p(iroots), ctypes.byref(ninv)) == 0
    return roots, iroots, ninv.value


def fwd(orc, q, a):
    a = np.ascontiguousarray(a, dtype=np.uint64).copy()
    roots, _, _ = tables(orc, a.size, q)
    orc.or_ntt_forward(ctypes.c_size_t(a.size), ctypes.c_uint64(q), p(roots), p(a))
    return a


def inv(orc, q, a):
    a = np.ascontiguousarray(a, dtype=np.uint64).copy()
    _, iroots, ninv = tables(orc, a.size, q)
    orc.or_ntt_inverse(ctypes.c_size_t(a.size), ctypes.c_uint64(q), p(iroots), ctypes.c_uint64(ninv), p(a))
    return a


def test_toy_ring_known_answers(orc):
    """test_ring.cpp:83-125 on Z_17[X]/(X^8+1)."""
    n, q = 8, 17
    xh = np.zeros(n, np.uint64)
    xh[4] = 1
    f = fwd(orc, q, xh)
    prod = inv(orc, q, (f * f) % q)
    assert prod[0] == 16 and not prod[1:].any()            # X^4 * X^4 = -1
    assert np.array_equal(fwd(orc, q, G["t8_a"]), G["t8_ntt"])
    rng = np.random.default_rng(3)
    for _ in range(20):                                    # NTT product == schoolbook oracle
        a, b = rng.integers(0, q, n, dtype=np.uint64), rng.integers(0, q, n, dtype=np.uint64)
        want = np.zeros(n, np.uint64)
        orc.or_naive_negacyclic(ctypes.c_size_t(n), ctypes.c_uint64(q), p(a), p(b), p(want))
        got = inv(orc, q, (fwd(orc, q, a) * fwd(orc, q, b)) % q)
        assert np.array_equal(got, want)


def test_ntt_golden(orc):
    primes = [int(v) for v in G["r256_primes"]]
    for i, q in enumerate(primes):
        assert np.array_equal(fwd(orc, q, G["r256_poly"][i]), G["r256_ntt"][i])
        assert np.array_equal(inv(orc, q, G["r256_poly"][i]), G["r256_intt"][i])
        assert np.array_equal(inv(orc, q, G["r256_ntt"][i]), G["r256_poly"][i])


def test_rescale_golden(orc):
    pr = np.ascontiguousarray(G["r256_primes"])
    out = np.zeros((3, 256), np.uint64)
    orc.or_rescale(ctypes.c_size_t(256), p(pr), ctypes.c_size_t(3), p(np.ascontiguousarray(G["r256_poly"])), p(out))
    assert np.array_equal(out, G["r256_rescale"])


def test_crt_digits_golden(orc):
    pr = np.ascontiguousarray(G["r256_primes"])
    D = orc.or_relin_digits(p(pr), ctypes.c_size_t(3))
    assert D == 9  # ceil(ceil(60 + 3*40 - eps) / 20)
    dig = np.zeros((D, 256), np.uint32)
    orc.or_crt_digits(ctypes.c_size_t(256), p(pr), ctypes.c_size_t(3), p(np.ascontiguousarray(G["r256_poly"])),
                      ctypes.c_size_t(D), p(dig, ctypes.c_uint32))
    # the digits reassemble the reference's exact CRT value (reconstruct_mod_q)
    crt = G["r256_crt"]
    for j in range(0, 256, 17):
        want = sum(int(w) << (64 * k) for k, w in enumerate(crt[j]))
        got = sum(int(dig[t, j]) << (20 * t) for t in range(D))
        assert got == want


def _mul(orc, x, y, top_primes, evk, level):
    pr = np.ascontiguousarray(top_primes)
    out = np.zeros((2, level, 256), np.uint64)
    orc.or_mul(ctypes.c_size_t(256), p(pr), ctypes.c_size_t(len(pr) - 1), ctypes.c_size_t(level),
               p(np.ascontiguousarray(x)), None if y is None else p(np.ascontiguousarray(y)),
               p(np.ascontiguousarray(evk)), p(out))
    return out


def test_mul_square_golden(orc):
    assert np.array_equal(_mul(orc, G["r256_x"], G["r256_y"], G["r256_primes"], G["r256_evk"], 3), G["r256_mul"])
    assert np.array_equal(_mul(orc, G["r256_x"], None, G["r256_primes"], G["r256_evk"], 3), G["r256_square"])


def test_mul_const_golden(orc):
    primes = [int(v) for v in G["r256_primes"]]
    u = float(G["r256_mulc_u"])
    c = int(np.floor(0.5 * u + 0.5))  # roundl: half away from zero (0.5 * u is an exact x.5)
    res = np.array([c % q for q in primes], np.uint64)
    out = np.zeros((2, 3, 256), np.uint64)
    orc.or_mul_const(ctypes.c_size_t(256), p(np.ascontiguousarray(G["r256_primes"])), ctypes.c_size_t(3),
                     p(np.ascontiguousarray(G["r256_x"])), p(res), p(out))
    assert np.array_equal(out, G["r256_mulc"])


def test_scalar_mac_golden(orc):
    """C1's dense(1): acc = 0.75 x (Delta = 2^20), + 0.125 at scale 2^40, rescale."""
    primes = [int(v) for v in G["chain_toy-n16"]]
    w = np.array([[round(0.75 * 2 ** 20) % q for q in primes]], np.uint64)
    bias = np.array([round(0.125 * 2 ** 40) % q for q in primes], np.uint64)
    src = np.array([0], np.int32)
    out = np.zeros((2, 3, 16), np.uint64)
    orc.or_scalar_mac(ctypes.c_size_t(16), p(np.array(primes, np.uint64)), ctypes.c_size_t(3),
                      p(np.ascontiguousarray(G["c1_in"])), p(src, ctypes.c_int), ctypes.c_size_t(1), p(w), p(bias),
                      p(out))
    assert np.array_equal(out, G["c1_dense_out"][0])


def test_oracle_against_live_reference(orc, ref):
    """Fresh seeds at the survey's C2 chain (n=4096, [60, 40 x 8]) against the reference itself."""
    import paper_1911_11377_b200 as hb
    n, bits = 1024, [60, 40, 40, 40, 40]
    pr = hb.find_chain(n, bits)
    r = ref.RefEngine(n, pr, 2.0 ** 40).keygen(3)
    s, b, a, evk = r.export_keys()
    poly = r.sample_uniform(4, 99)
    for i, q in enumerate(pr):
        assert np.array_equal(fwd(orc, q, poly[i]), r.ntt_forward(i, poly[i]))
    x = np.stack([r.sample_uniform(4, 7), r.sample_uniform(4, 8)])
    y = np.stack([r.sample_uniform(4, 9), r.sample_uniform(4, 10)])
    prs = np.array(pr, np.uint64)
    out = np.zeros((2, 4, n), np.uint64)
    orc.or_mul(ctypes.c_size_t(n), p(prs), ctypes.c_size_t(4), ctypes.c_size_t(4), p(x), p(y), p(evk), p(out))
    want, _ = r.mul(x, y, 4, 2.0 ** 40, 2.0 ** 40)
    assert np.array_equal(out, want)
