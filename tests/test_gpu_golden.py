"""GPU vs the reference's committed golden vectors (tests/golden/golden.npz):
the same checks as test_gpu_parity.py but independent of the live reference
library, plus the reference's frozen logit (test_nn.cpp:233-252) through the
encrypted path."""
import os

import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


def r256():
    p = hb.CkksParams(256, [int(v) for v in G["r256_primes"]], 2.0 ** 40)
    eng = hb.CkksEngine(p).keygen(1)
    return p, eng


def test_keys_golden():
    p, eng = r256()
    assert np.array_equal(eng.export_secret_key(), G["r256_s"])
    b, a = eng.export_public_key()
    assert np.array_equal(b, G["r256_pk_b"]) and np.array_equal(a, G["r256_pk_a"])
    assert np.array_equal(eng.export_eval_key(), G["r256_evk"])
    toy = hb.CkksEngine(hb.CkksParams(16, [int(v) for v in G["chain_toy-n16"]], 2.0 ** 20)).keygen(42)
    assert np.array_equal(toy.export_eval_key(), G["toy_evk"])


def test_ring_ops_golden():
    p, eng = r256()
    poly = G["r256_poly"][None]
    assert np.array_equal(eng.ntt_forward(poly, 3)[0], G["r256_ntt"])
    assert np.array_equal(eng.ntt_inverse(poly, 3)[0], G["r256_intt"])
    assert np.array_equal(eng.rescale_poly(poly, 3)[0], G["r256_rescale"])


def test_scheme_ops_golden():
    p, eng = r256()
    x = eng.tensor_from_words(G["r256_x"][None], 3, p.scale)
    y = eng.tensor_from_words(G["r256_y"][None], 3, p.scale)
    m = eng.mul(x, y)
    assert np.array_equal(m.words()[0], G["r256_mul"]) and m.scale == float(G["r256_mul_scale"])
    s = eng.square(x)
    assert np.array_equal(s.words()[0], G["r256_square"]) and s.scale == float(G["r256_square_scale"])
    mc = eng.mul_const(x, 0.5, float(G["r256_mulc_u"]))
    assert np.array_equal(mc.words()[0], G["r256_mulc"]) and mc.scale == float(G["r256_mulc_scale"])
    a = eng.eval_activation(hb.PolyActivation([0.0, 0.5, 0.000469841857369822], 100.0), x)
    assert a.level == int(G["r256_act_level"]) and a.scale == float(G["r256_act_scale"])
    assert np.array_equal(a.words()[0], G["r256_act"])


def test_c1_golden():
    p = hb.CkksParams(16, [int(v) for v in G["chain_toy-n16"]], 2.0 ** 20)
    eng = hb.CkksEngine(p).keygen(42)
    spec = hb.ModelSpec(hb.Shape.flattened(1))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.dense(1), hb.LayerSpec.activation("relu-poly2")]
    spec.weights = [np.array([0.75]), None]
    spec.biases = [np.array([0.125]), None]
    data = (-1 + 0.25 * np.arange(8))[:, None]
    x = eng.encrypt_tensor(data, seed=7, shape=spec.input)
    assert np.array_equal(x.words(), G["c1_in"])
    y = hb.forward_encrypted(spec, x, eng, seed=9)
    assert y.level == int(G["c1_out_level"]) and y.scale == float(G["c1_out_scale"])
    assert np.array_equal(y.words(), G["c1_out"])
    assert np.array_equal(eng.decrypt_tensor(y, 8), G["c1_dec"])


def test_frozen_logit_through_encrypted_path():
    """tiny_preset, init_random_weights(2024), x ~ Rng(7): plain logit is frozen at
    -0.2619418027202618 (test_nn.cpp:251); the encrypted path must agree < 1e-2
    (the reference's end-to-end tolerance, test_nn.cpp:362-378)."""
    spec = hb.tiny_preset()
    for i in range(len(spec.layers)):
        if f"tiny_w{i}" in G:
            spec.weights[i] = G[f"tiny_w{i}"]
            spec.biases[i] = G[f"tiny_b{i}"]
    assert float(G["tiny_plain_logit"][0]) == pytest.approx(-0.2619418027202618, abs=1e-12)
    eng = hb.CkksEngine(hb.preset_params("nn-n4096-d8")).keygen(7)
    x = eng.encrypt_tensor(G["tiny_x"][None, :], seed=11, shape=spec.input)
    y = hb.forward_encrypted(spec, x, eng, seed=13)
    got = eng.decrypt_tensor(y, 1)[0, 0]
    assert abs(got - (-0.2619418027202618)) < 1e-2
