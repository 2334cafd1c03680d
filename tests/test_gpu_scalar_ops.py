"""GPU parity of CkksEngine's scalar fast path and plaintext operands
(ckks.hpp:283-311, 372-472) -- make_scalar_plain, make_zero_ciphertext,
add_inplace, mul_scalar_mac, add_scalar_inplace, add_plain, mul_plain_raw,
mul_plain -- against the compiled reference, word for word, on every cell of
a tensor (the way the reference's layer kernels, layers.hpp:174-293, chain
them: zero accumulator -> scalar MACs -> bias -> rescale)."""
import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu

BITS = [60] + [40] * 8


def setup(ref, n=4096):
    p = hb.CkksParams(n, hb.find_chain(n, BITS), 2.0 ** 40, 3.2, False)
    eng = hb.CkksEngine(p).keygen(1)
    r = ref.RefEngine.from_params(p).keygen(1)
    return p, eng, r


def fresh(r, p, seed, cells):
    rng = np.random.default_rng(seed)
    cts = [r.encrypt(rng.uniform(-1, 1, p.n // 2), seed=seed * 100 + k) for k in range(cells)]
    return np.stack(cts)  # [cells][2][top+1][n]


@pytest.mark.parametrize("c,scale,level", [(0.75, 2.0 ** 40, 8), (-1.5, 2.0 ** 40, 3), (1e-3, 2.0 ** 30, 0),
                                           (-123.25, 2.0 ** 40, 5)])
def test_make_scalar_plain_matches_reference(ref, c, scale, level):
    p, eng, r = setup(ref)
    sp = eng.make_scalar_plain(c, scale, level)
    assert np.array_equal(sp.residues, r.scalar_plain(c, scale, level))
    assert (sp.scale, sp.level) == (scale, level)


def test_scalar_mac_chain_matches_reference(ref):
    """A conv/dense output cell (layers.hpp:196-207): zero accumulator at
    x.scale * Delta, two scalar MACs, the bias, then rescale -- one scalar for
    every cell and one per cell."""
    p, eng, r = setup(ref)
    top = p.top_level
    cells = 3
    xs = fresh(r, p, 7, cells)
    ys = fresh(r, p, 8, cells)
    x = eng.tensor_from_words(xs, top, p.scale)
    y = eng.tensor_from_words(ys, top, p.scale)
    acc_scale = p.scale * p.scale
    acc = eng.make_zero_ciphertext(top, acc_scale, cells)
    assert not acc.words().any() and (acc.level, acc.scale) == (top, acc_scale)
    w1 = [0.5, -0.25, 1.75]
    eng.mul_scalar_mac(acc, x, eng.make_scalar_plain(0.3, p.scale, top))
    eng.mul_scalar_mac(acc, y, [eng.make_scalar_plain(w, p.scale, top) for w in w1])
    eng.add_scalar_inplace(acc, -0.125)
    out = eng.rescale(acc)
    for k in range(cells):
        z = np.zeros_like(xs[k])
        a = r.scalar_mac(z, xs[k], top, acc_scale, p.scale, 0.3, p.scale)
        a = r.scalar_mac(a, ys[k], top, acc_scale, p.scale, w1[k], p.scale, b=-0.125)
        assert np.array_equal(acc.words()[k], a)
        want, s = r.rescale(a, top, acc_scale)
        assert np.array_equal(out.words()[k], want) and out.scale == s


def test_add_inplace_matches_add(ref):
    p, eng, r = setup(ref)
    xs, ys = fresh(r, p, 3, 2), fresh(r, p, 4, 2)
    x = eng.tensor_from_words(xs, p.top_level, p.scale)
    y = eng.tensor_from_words(ys, p.top_level, p.scale)
    want = eng.add(x, y).words()
    eng.add_inplace(x, y)
    assert np.array_equal(x.words(), want)


@pytest.mark.parametrize("op", [0, 1, 2])
@pytest.mark.parametrize("constant", [False, True])
def test_plaintext_ops_match_reference(ref, op, constant):
    """add_plain / mul_plain_raw / mul_plain with an encode_real plaintext (NTT
    product) or an encode_const one (scalar multiply)."""
    p, eng, r = setup(ref)
    level = 6
    xs = fresh(r, p, 11, 2)[:, :, : level + 1]
    x = eng.tensor_from_words(xs, level, p.scale)
    slots = np.random.default_rng(5).uniform(-1, 1, p.n // 2)
    pscale = p.scale if op == 0 else 2.0 ** 30
    m = eng.encode_const(float(slots[0]), pscale, level) if constant else eng.encode_real(slots, pscale, level)
    got = [eng.add_plain, eng.mul_plain_raw, eng.mul_plain][op](x, m)
    for k in range(2):
        want, lv, s = r.plain_op(op, xs[k], level, p.scale, slots, pscale, constant)
        assert (got.level, got.scale) == (lv, s)
        assert np.array_equal(got.words()[k], want)


def test_scalar_op_errors_carry_reference_texts(ref):
    p, eng, r = setup(ref)
    xs = fresh(r, p, 2, 1)
    x = eng.tensor_from_words(xs, p.top_level, p.scale)
    acc = eng.make_zero_ciphertext(p.top_level - 1, p.scale * p.scale)
    with pytest.raises(ValueError, match="mul_scalar_mac: level mismatch"):
        eng.mul_scalar_mac(acc, x, eng.make_scalar_plain(1.0, p.scale, p.top_level))
    acc = eng.make_zero_ciphertext(p.top_level, p.scale)
    with pytest.raises(ValueError, match="mul_scalar_mac: scale mismatch"):
        eng.mul_scalar_mac(acc, x, eng.make_scalar_plain(1.0, p.scale, p.top_level))
    m = eng.encode_const(1.0, p.scale, 3)
    with pytest.raises(ValueError, match="add_plain: level mismatch"):
        eng.add_plain(x, m)
    with pytest.raises(ValueError, match="mul_plain: level mismatch"):
        eng.mul_plain(x, m)
    x0 = eng.tensor_from_words(xs[:, :, :1], 0, p.scale)
    with pytest.raises(ValueError, match="mul_plain: at last level, no room to rescale"):
        eng.mul_plain(x0, eng.encode_const(1.0, p.scale, 0))
