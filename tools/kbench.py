#!/usr/bin/env python
"""Kernel-level microbenchmarks for tuning (one GPU): NTT/INTT, key switch,
HE square and the conv gather-MAC at the C4 / C5 shapes, with per-kernel
CUDA-event timings and achieved modmul-eq/s against the live integer probe.
Prints one JSON object. Not part of the driver contract (bench.py is)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1911_11377_b200 as hb  # noqa: E402


def timed(eng, fn, reps=3):
    fn()
    eng.synchronize()
    eng.profile_reset()
    eng.profile(True)
    t0 = time.perf_counter()
    for _ in range(reps):
        out = fn()
    eng.synchronize()
    wall = (time.perf_counter() - t0) / reps
    eng.profile(False)
    prof = eng.profile_read()
    return wall, {k: {"ms": v["ms"] / reps, "gmm_s": v["ops"] / max(v["ms"], 1e-9) / 1e6,
                      "gb_s": v["bytes"] / max(v["ms"], 1e-9) / 1e6} for k, v in prof.items()}, out


def uniform_words(p, cells, level, seed=5):
    rng = np.random.default_rng(seed)
    w = np.empty((cells, 2, level + 1, p.n), dtype=np.uint64)
    for i in range(level + 1):
        w[:, :, i, :] = rng.integers(0, p.primes[i], size=(cells, 2, p.n), dtype=np.uint64)
    return w


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--which", default="ntt,ks,square,conv,large")
    args = ap.parse_args()
    which = set(args.which.split(","))
    res = {}
    p = hb.preset_params("net-n8192-d8")
    eng = hb.CkksEngine(p).keygen(1)
    res["int_peak_gmm_s"] = eng.modmul_peak() / 1e9
    L = p.top_level
    if "ntt" in which:
        x = eng.tensor_from_words(uniform_words(p, 512, L), L, p.scale)
        import ctypes
        d = ctypes.c_void_p(x.device_ptr())
        f = lambda: hb._check(hb.lib().hecnn_ntt_forward(eng.ctx, d, L, 1024))  # noqa: E731
        g = lambda: hb._check(hb.lib().hecnn_ntt_inverse(eng.ctx, d, L, 1024))  # noqa: E731
        res["ntt_fwd_8192"] = timed(eng, f)[1]
        res["ntt_inv_8192"] = timed(eng, g)[1]
    if "rescale" in which:
        # C4 conv1's rescale shape: 16384 ciphertexts, level 8 -> 7 (one of the HBM-bound streams)
        x = eng.tensor_from_words(uniform_words(p, 4096, L), L, p.scale)
        res["rescale_l8_4096"] = timed(eng, lambda: eng.rescale(x))[1]
        y = eng.tensor_from_words(uniform_words(p, 4096, L), L, p.scale)
        res["add_l8_4096"] = timed(eng, lambda: eng.add(x, y))[1]
    if "ks" in which or "square" in which:
        lv = 7
        x = eng.tensor_from_words(uniform_words(p, 512, lv), lv, p.scale)
        if "square" in which:
            wall, prof, _ = timed(eng, lambda: eng.square(x))
            res["square_l7_512"] = {"ms_per_ct": wall * 1e3 / 512, "kernels": prof}
    if "conv" in which:
        spec = hb.ModelSpec(hb.Shape.spatial(32, 32, 3))
        spec.layers = [hb.LayerSpec.conv2d(16, 3, 3)]
        hb.glorot_weights(spec, 4)
        m = eng.model(spec)
        xin = eng.tensor_from_words(uniform_words(p, 3072, L), L, p.scale)
        xin.set_shape(spec.input, 4096)
        wall, prof, _ = timed(eng, lambda: hb.forward_encrypted(m, xin, eng))
        res["conv1_c4"] = {"ms": wall * 1e3, "kernels": prof}
    if "conv5" in which:
        # AlexNet conv2 shape (5x5, 96 -> 256) at its C5 level, on an 8x8 spatial tile
        pl = hb.preset_params("large-n16384-d24")
        el = hb.CkksEngine(pl).keygen(1)
        spec = hb.ModelSpec(hb.Shape.spatial(8, 8, 96))
        spec.layers = [hb.LayerSpec.conv2d(256, 5, 5)]
        hb.glorot_weights(spec, 4)
        m5 = el.model(spec)
        lv = 20
        xin = el.tensor_from_words(uniform_words(pl, 8 * 8 * 96, lv), lv, pl.scale)
        xin.set_shape(spec.input, 8192)
        wall, prof, _ = timed(el, lambda: hb.forward_encrypted(m5, xin, el), reps=1)
        res["conv_alexnet2_l20"] = {"ms": wall * 1e3, "kernels": prof}
    if "large" in which:
        pl = hb.preset_params("large-n16384-d24")
        el = hb.CkksEngine(pl).keygen(1)
        lv = 23
        x = el.tensor_from_words(uniform_words(pl, 32, lv), lv, pl.scale)
        wall, prof, _ = timed(el, lambda: el.square(x), reps=2)
        res["square_large_l23_32"] = {"ms_per_ct": wall * 1e3 / 32, "kernels": prof}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
