"""GPU parity: every device kernel path against the compiled reference
(oracle/_ref/libhecnn_ref.so) on identical params, seeds and inputs.
Integer work must be word-for-word identical; doubles (scale ledger) must be
bit-identical too. Mirrors the reference's own test structure
(proj/tests/test_ring.cpp, test_ckks.cpp, test_activation.cpp, test_nn.cpp)."""
import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu

SWEEP_BITS = [60] + [40] * 8  # SURVEY §8(d) C2 chain


def params(n, bits, log2_scale=40, degenerate=False):
    return hb.CkksParams(n, hb.find_chain(n, bits), 2.0 ** log2_scale, 3.2, degenerate)


def engines(ref, p, seed=1, keys=True):
    eng = hb.CkksEngine(p)
    r = ref.RefEngine.from_params(p)
    if keys:
        eng.keygen(seed)
        r.keygen(seed)
    return eng, r


# ---------------------------------------------------------------- ring tier

@pytest.mark.parametrize("n,bits", [(8, [30, 20]), (16, [40, 21, 21, 21]), (32, [40, 30]), (1024, [60, 40, 40]),
                                    (4096, SWEEP_BITS), (8192, SWEEP_BITS), (16384, SWEEP_BITS[:4]),
                                    (32768, SWEEP_BITS[:3]), (65536, SWEEP_BITS[:3])])
def test_ntt_forward_inverse_match_reference(ref, n, bits):
    p = params(n, bits, log2_scale=min(bits) - 2)
    eng, r = engines(ref, p, keys=False)
    level = len(bits) - 1
    polys = np.stack([r.sample_uniform(level, 1000 + i) for i in range(3)])
    got = eng.ntt_forward(polys, level)
    want = np.stack([np.stack([r.ntt_forward(i, polys[c, i]) for i in range(level + 1)]) for c in range(3)])
    assert np.array_equal(got, want)
    back = eng.ntt_inverse(got, level)
    assert np.array_equal(back, polys)
    want_inv = np.stack([np.stack([r.ntt_inverse(i, polys[c, i]) for i in range(level + 1)]) for c in range(3)])
    assert np.array_equal(eng.ntt_inverse(polys, level), want_inv)


def test_toy_ring_known_answers(ref):
    """test_ring.cpp:83-96: X^4 * X^4 == -1 in Z_17[X]/(X^8+1) via NTT pointwise."""
    p = hb.CkksParams(8, [17], 2.0, 3.2)
    eng = hb.CkksEngine(p)
    xh = np.zeros((1, 1, 8), dtype=np.uint64)
    xh[0, 0, 4] = 1
    f = eng.ntt_forward(xh, 0)
    prod = eng.poly_pointwise_mul(f, f, 0)
    sq = eng.ntt_inverse(prod, 0)
    assert sq[0, 0, 0] == 16 and not sq[0, 0, 1:].any()


@pytest.mark.parametrize("n,bits", [(16, [50, 30, 30]), (4096, SWEEP_BITS), (8192, [60, 40, 40, 40])])
def test_rescale_matches_reference(ref, n, bits):
    p = params(n, bits, log2_scale=25)
    eng, r = engines(ref, p, keys=False)
    level = len(bits) - 1
    polys = np.stack([r.sample_uniform(level, 77 + i) for i in range(4)])
    got = eng.rescale_poly(polys, level)
    want = np.stack([r.rescale_poly(polys[i], level) for i in range(4)])
    assert np.array_equal(got, want)


def test_rescale_errors(ref):
    eng = hb.CkksEngine(params(16, [50, 30, 30], 25))
    with pytest.raises(ValueError, match="already at last level"):
        eng.rescale_poly(np.zeros((1, 1, 16), dtype=np.uint64), 0)


# ---------------------------------------------------------------- keys / encryption

@pytest.mark.parametrize("preset", ["toy-n16", "test-n4096-d4"])
def test_keygen_word_identical(ref, preset):
    p = hb.preset_params(preset)
    eng, r = engines(ref, p, seed=5)
    s, b, a, evk = r.export_keys()
    assert np.array_equal(eng.export_secret_key(), s)
    gb, ga = eng.export_public_key()
    assert np.array_equal(gb, b) and np.array_equal(ga, a)
    assert np.array_equal(eng.export_eval_key(), evk)


def test_keygen_degenerate(ref):
    p = hb.preset_params("toy-n16", degenerate_noise=True)
    eng, r = engines(ref, p, seed=3)
    s, b, a, evk = r.export_keys()
    assert np.array_equal(eng.export_secret_key(), s) and not s.any()
    assert np.array_equal(eng.export_eval_key(), evk)


@pytest.mark.parametrize("preset,batch", [("toy-n16", 8), ("test-n4096-d4", 2048)])
def test_encrypt_tensor_word_identical(ref, preset, batch):
    p = hb.preset_params(preset)
    eng, r = engines(ref, p, seed=7)
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, size=(batch, 5))
    shape = hb.Shape.flattened(5)
    got = eng.encrypt_tensor(x, seed=11, shape=shape)
    want = r.encrypt_tensor(x, shape, seed=11)
    assert np.array_equal(got.words(), want.words())
    assert got.scale == want.info()[2] and got.level == want.info()[1]
    dec = eng.decrypt_tensor(got, batch)
    assert np.array_equal(dec, r.decrypt_tensor(want, batch))


def test_encrypt_degenerate_gives_plaintext(ref):
    """test_ckks.cpp:145-155: zero randomness -> ct = (m, 0)."""
    p = hb.preset_params("toy-n16", degenerate_noise=True)
    eng, r = engines(ref, p, seed=5)
    vals = [0.5, -0.25, 0.125, 1.0, -1.0, 0.75, -0.5, 0.3]
    t = eng.encrypt_tensor(np.array(vals)[:, None], seed=9)
    w = t.words()[0]
    m = r.encode(vals, p.top_level)
    assert np.array_equal(w[0], m) and not w[1].any()


# ---------------------------------------------------------------- HE mul / square / key switch

def _fresh(r, count, seed0=100):
    rng = np.random.default_rng(seed0)
    return np.stack([r.encrypt(rng.uniform(-1, 1, r.n // 2), seed0 + i) for i in range(count)])


@pytest.mark.parametrize("preset", ["toy-n16", "test-n4096-d4", "nn-n4096-d8"])
def test_mul_and_square_word_identical(ref, preset):
    p = hb.preset_params(preset)
    eng, r = engines(ref, p, seed=1)
    L = p.top_level
    xs, ys = _fresh(r, 3, 10), _fresh(r, 3, 20)
    tx, ty = eng.tensor_from_words(xs, L, p.scale), eng.tensor_from_words(ys, L, p.scale)
    prod = eng.mul(tx, ty)
    sq = eng.square(tx)
    pw, sw = prod.words(), sq.words()
    for i in range(3):
        want, s = r.mul(xs[i], ys[i], L, p.scale, p.scale)
        assert np.array_equal(pw[i], want)
        assert prod.scale == s
        want_sq, s2 = r.square(xs[i], L, p.scale)
        assert np.array_equal(sw[i], want_sq)
        assert sq.scale == s2
    # square == mul(x, x) bit-exact (test_ckks.cpp:258-264)
    assert np.array_equal(eng.mul(tx, tx).words(), sw)


def test_mul_at_lower_levels_and_uniform_residues(ref):
    """Uniform-random residues exercise every CRT/digit path (SURVEY C2 inputs)."""
    p = params(4096, SWEEP_BITS)
    eng, r = engines(ref, p, seed=1)
    for level in (8, 5, 1):
        x = np.stack([r.sample_uniform(level, 1000 + 4 * i + k) for i in range(2) for k in range(2)]).reshape(2, 2, level + 1, 4096)
        y = np.stack([r.sample_uniform(level, 2000 + 4 * i + k) for i in range(2) for k in range(2)]).reshape(2, 2, level + 1, 4096)
        got = eng.mul(eng.tensor_from_words(x, level, p.scale), eng.tensor_from_words(y, level, p.scale)).words()
        for i in range(2):
            want, _ = r.mul(x[i], y[i], level, p.scale, p.scale)
            assert np.array_equal(got[i], want), f"level {level} ct {i}"


@pytest.mark.parametrize("n", [16384, 32768])
def test_mul_large_degree(ref, n):
    p = params(n, SWEEP_BITS[:4])
    eng, r = engines(ref, p, seed=2)
    L = 3
    x = np.stack([r.sample_uniform(L, 5 + k) for k in range(2)])[None]
    y = np.stack([r.sample_uniform(L, 9 + k) for k in range(2)])[None]
    got = eng.mul(eng.tensor_from_words(x, L, p.scale), eng.tensor_from_words(y, L, p.scale)).words()[0]
    want, _ = r.mul(x[0], y[0], L, p.scale, p.scale)
    assert np.array_equal(got, want)


def test_mul_errors(ref):
    p = hb.preset_params("toy-n16")
    eng, r = engines(ref, p, seed=1)
    x = eng.tensor_from_words(_fresh(r, 1), p.top_level, p.scale)
    low = eng.mod_switch(x, 0)
    with pytest.raises(ValueError, match="mul: at last level, no room to rescale"):
        eng.square(low)
    with pytest.raises(ValueError, match="level mismatch"):
        eng.mul(x, eng.mod_switch(x, 1))
    with pytest.raises(ValueError, match="mod_switch: cannot raise level"):
        eng.mod_switch(low, 2)


def test_rescale_mul_const_add_const(ref):
    p = hb.preset_params("test-n4096-d4")
    eng, r = engines(ref, p, seed=4)
    L = p.top_level
    xs = _fresh(r, 2, 30)
    t = eng.tensor_from_words(xs, L, p.scale)
    rs = eng.rescale(t)
    for i in range(2):
        want, s = r.rescale(xs[i], L, p.scale)
        assert np.array_equal(rs.words()[i], want) and rs.scale == s
    u = p.scale * p.primes[L] / p.scale
    mc = eng.mul_const(t, 0.5, u)
    for i in range(2):
        want, s = r.mul_const(xs[i], L, p.scale, 0.5, u)
        assert np.array_equal(mc.words()[i], want) and mc.scale == s


@pytest.mark.parametrize("coeffs", [[0.0, 0.5, 0.000469841857369822], [0.0, 0.0, 1.0], [0.1, -0.3, 0.2, 0.05],
                                    [0.25, 1.0, 0.5, -0.1, 0.02],
                                    # degree 9: more terms than the fused rescale-and-add epilogue takes
                                    [0.05, 0.5, 0.1, 0.0, -0.02, 0.0, 0.003, 0.0, -0.0004, 0.00002]])
def test_eval_activation_word_identical(ref, coeffs):
    p = hb.preset_params("nn-n4096-d8")
    eng, r = engines(ref, p, seed=6)
    L = p.top_level
    xs = _fresh(r, 2, 40)
    act = hb.PolyActivation(list(coeffs), 100.0)
    out = eng.eval_activation(act, eng.tensor_from_words(xs, L, p.scale))
    for i in range(2):
        want, lv, s = r.eval_activation(coeffs, 100.0, xs[i], L, p.scale)
        assert out.level == lv and out.scale == s
        assert np.array_equal(out.words()[i], want)


# ---------------------------------------------------------------- network

def _run_both(ref, p, spec, batch, keyseed, encseed, fwdseed, data=None):
    eng, r = engines(ref, p, seed=keyseed)
    rng = np.random.default_rng(encseed)
    if data is None:
        data = rng.uniform(0, 1, size=(batch, spec.input.positions()))
    tx = eng.encrypt_tensor(data, seed=encseed, shape=spec.input)
    rx = r.encrypt_tensor(data, spec.input, seed=encseed)
    assert np.array_equal(tx.words(), rx.words())
    secs = []
    ty = hb.forward_encrypted(spec, tx, eng, seed=fwdseed, layer_seconds=secs)
    ry, _ = r.forward_encrypted(spec, rx, seed=fwdseed)
    return eng, r, ty, ry, data


def test_c1_toy_dense_square_activation(ref):
    """toy-n16, dense(1) w=0.75 b=0.125 + relu-poly2, 8 slots."""
    p = hb.preset_params("toy-n16")
    spec = hb.ModelSpec(hb.Shape.flattened(1))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.dense(1), hb.LayerSpec.activation("relu-poly2")]
    spec.weights = [np.array([0.75]), None]
    spec.biases = [np.array([0.125]), None]
    data = (-1 + 0.25 * np.arange(8))[:, None]
    eng, r, ty, ry, _ = _run_both(ref, p, spec, 8, 42, 7, 9, data)
    assert ty.level == ry.info()[1] == 0
    assert ty.scale == ry.info()[2]
    assert np.array_equal(ty.words(), ry.words())
    assert np.array_equal(eng.decrypt_tensor(ty, 8), r.decrypt_tensor(ry, 8))


def test_tiny_preset_forward_word_identical(ref):
    """tiny_preset (model.hpp:223-235) at nn-n4096-d8 with reference Glorot weights."""
    p = hb.preset_params("nn-n4096-d8")
    spec = hb.tiny_preset()
    ref.init_random_weights(spec, 3)
    eng, r, ty, ry, data = _run_both(ref, p, spec, 4, 7, 11, 13)
    assert np.array_equal(ty.words(), ry.words())
    dec = eng.decrypt_tensor(ty, 4)
    assert np.array_equal(dec, r.decrypt_tensor(ry, 4))
    plain = ref.forward_plain(spec, data)
    assert np.max(np.abs(dec - plain)) < 1e-2


def test_cnn_with_pad_pool_dense(ref):
    """Small CryptoNets/CIFAR-shaped stack exercising zero-pad fresh encryptions,
    strided valid conv, same conv, avg-pool, dense and square activation."""
    p = params(1024, SWEEP_BITS)
    spec = hb.ModelSpec(hb.Shape.spatial(6, 6, 2))
    spec.activations["sq"] = hb.PolyActivation([0.0, 0.0, 1.0], 10.0)
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.zero_pad2d(1), hb.LayerSpec.conv2d(3, 3, 3, stride=2, valid=True),
                   hb.LayerSpec.activation("sq"), hb.LayerSpec.conv2d(4, 3, 3), hb.LayerSpec.activation("relu-poly2"),
                   hb.LayerSpec.avg_pool2d(2), hb.LayerSpec.dense(3), hb.LayerSpec.sigmoid()]
    ref.init_random_weights(spec, 5)
    eng, r, ty, ry, data = _run_both(ref, p, spec, 16, 3, 4, 5)
    assert ty.level == ry.info()[1] and ty.scale == ry.info()[2]
    assert np.array_equal(ty.words(), ry.words())


def test_forward_errors(ref):
    p = hb.preset_params("toy-n16")
    eng = hb.CkksEngine(p).keygen(1)
    spec = hb.ModelSpec(hb.Shape.flattened(2))
    spec.activations["a"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.dense(2), hb.LayerSpec.activation("a"), hb.LayerSpec.dense(1)]
    hb.glorot_weights(spec, 1)
    x = eng.encrypt_tensor(np.zeros((2, 2)), seed=1, shape=hb.Shape.flattened(2))
    with pytest.raises(ValueError, match=r"depth budget exhausted at layer 2 \(dense\)"):
        hb.forward_encrypted(spec, x, eng)
    bad = eng.encrypt_tensor(np.zeros((2, 3)), seed=1, shape=hb.Shape.flattened(3))
    with pytest.raises(ValueError, match=r"input shape \(3\) != model input \(2\)"):
        hb.forward_encrypted(spec, bad, eng)
