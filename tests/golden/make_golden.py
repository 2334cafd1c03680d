"""Generate tests/golden/golden.npz from the compiled REFERENCE (oracle/_ref).

Run here (where /root/reference exists and oracle/_ref was built):
    python tests/golden/make_golden.py
The fixtures pin the CPU oracle (tests/test_oracle.py) and the GPU engine
(tests/test_gpu_golden.py) on boxes where the reference cannot be rebuilt.
Everything below is produced by the reference's own code paths (keygen,
encrypt, NTT, rescale, mul, square, mul_plain, forward_encrypted,
encode/decode, randomness); nothing is computed by the product.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import paper_1911_11377_b200 as hb  # noqa: E402  (spec builders only)
from oracle import ref  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")


def main():
    g = {}
    # ---- preset chains (RingParams::create)
    for p in hb.builtin_presets():
        g[f"chain_{p.name}"] = np.array(ref.find_chain(p.n, p.prime_bits), dtype=np.uint64)

    # ---- toy-n16: keys + C1 (dense(1) w=.75 b=.125 + relu-poly2 on 8 slots)
    toy = hb.CkksParams(16, [int(v) for v in g["chain_toy-n16"]], 2.0 ** 20)
    r = ref.RefEngine.from_params(toy).keygen(42)
    s, b, a, evk = r.export_keys()
    g.update(toy_s=s, toy_pk_b=b, toy_pk_a=a, toy_evk=evk)
    spec = hb.ModelSpec(hb.Shape.flattened(1))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.dense(1), hb.LayerSpec.activation("relu-poly2")]
    spec.weights = [np.array([0.75]), None]
    spec.biases = [np.array([0.125]), None]
    data = (-1 + 0.25 * np.arange(8))[:, None]
    x = r.encrypt_tensor(data, spec.input, seed=7)
    y, _ = r.forward_encrypted(spec, x, seed=9)
    cells, lvl, sc = y.info()
    g.update(c1_in=x.words(), c1_out=y.words(), c1_out_level=np.array(lvl), c1_out_scale=np.array(sc),
             c1_in_scale=np.array(x.info()[2]), c1_dec=r.decrypt_tensor(y, 8))
    # dense(1) alone: the scalar-MAC + bias + rescale step of C1
    d1 = hb.ModelSpec(hb.Shape.flattened(1))
    d1.layers = [hb.LayerSpec.dense(1)]
    d1.weights = [np.array([0.75])]
    d1.biases = [np.array([0.125])]
    yd, _ = r.forward_encrypted(d1, x, seed=9)
    g.update(c1_dense_out=yd.words(), c1_dense_scale=np.array(yd.info()[2]))

    # ---- ring ops at n=256, chain [60,40,40,40]
    n = 256
    primes = ref.find_chain(n, [60, 40, 40, 40])
    p = hb.CkksParams(n, primes, 2.0 ** 40)
    g["r256_primes"] = np.array(primes, dtype=np.uint64)
    r = ref.RefEngine.from_params(p).keygen(1)
    poly = r.sample_uniform(3, 1000)
    g["r256_poly"] = poly
    g["r256_ntt"] = np.stack([r.ntt_forward(i, poly[i]) for i in range(4)])
    g["r256_intt"] = np.stack([r.ntt_inverse(i, poly[i]) for i in range(4)])
    g["r256_rescale"] = r.rescale_poly(poly, 3)
    g["r256_crt"] = r.reconstruct(poly, 3, 4)
    s, b, a, evk = r.export_keys()
    g.update(r256_s=s, r256_pk_b=b, r256_pk_a=a, r256_evk=evk)
    rng = np.random.default_rng(2)
    xs = r.encrypt(rng.uniform(-1, 1, n // 2), 11)
    ys = r.encrypt(rng.uniform(-1, 1, n // 2), 12)
    g.update(r256_x=xs, r256_y=ys)
    m, ms = r.mul(xs, ys, 3, p.scale, p.scale)
    sq, ss = r.square(xs, 3, p.scale)
    g.update(r256_mul=m, r256_mul_scale=np.array(ms), r256_square=sq, r256_square_scale=np.array(ss))
    u = p.scale * primes[3] / p.scale
    mc, mcs = r.mul_const(xs, 3, p.scale, 0.5, u)
    g.update(r256_mulc=mc, r256_mulc_scale=np.array(mcs), r256_mulc_u=np.array(u))
    act, alv, asc = r.eval_activation([0.0, 0.5, 0.000469841857369822], 100.0, xs, 3, p.scale)
    g.update(r256_act=act, r256_act_level=np.array(alv), r256_act_scale=np.array(asc))
    vals = rng.uniform(-1, 1, n // 2)
    g["r256_vals"] = vals
    g["r256_encode"] = r.encode(vals, 3)
    g["r256_decode"] = r.decode(g["r256_encode"], 3, p.scale)
    rr, e0, e1 = r.encryption_randomness(123)
    g.update(r256_rand_r=rr, r256_rand_e0=e0, r256_rand_e1=e1)
    g["r256_dec_x"] = r.decrypt(xs, 3, p.scale)

    # ---- toy ring n=8, q=17 (test_ring.cpp:10-16)
    t8 = ref.RefEngine(8, [17], 2.0)
    a8 = t8.sample_uniform(0, 5)[0]
    g.update(t8_a=a8, t8_ntt=t8.ntt_forward(0, a8))

    # ---- frozen plain logit input (test_nn.cpp:233-252): tiny_preset, weights 2024, x ~ Rng(7)
    tiny = hb.tiny_preset()
    ref.init_random_weights(tiny, 2024)
    for i, (w, bb) in enumerate(zip(tiny.weights, tiny.biases)):
        if w is not None:
            g[f"tiny_w{i}"] = w
            g[f"tiny_b{i}"] = bb
    g["tiny_x"] = ref.rng_uniform(7, tiny.input.positions())
    g["tiny_plain_logit"] = ref.forward_plain(tiny, g["tiny_x"][None, :])[0]

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes,", len(g), "arrays")


if __name__ == "__main__":
    main()
