"""Debug helper: streamed vs whole-tensor forward on growing prefixes of a model."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1911_11377_b200 as hb

p = hb.CkksParams(4096, hb.find_chain(4096, [60] + [40] * 9), 2.0 ** 40, 3.2, False)
eng = hb.CkksEngine(p).keygen(2)
A = lambda: hb.LayerSpec.activation("relu-poly2")
full = [hb.LayerSpec.conv2d(4, 3, 3), A(), hb.LayerSpec.avg_pool2d(2), hb.LayerSpec.zero_pad2d(1),
        hb.LayerSpec.conv2d(5, 3, 3), A(), hb.LayerSpec.zero_pad2d(1), hb.LayerSpec.avg_pool2d(2)]
for H, W in [(4, 4), (16, 6)]:
    for n in range(1, len(full) + 1):
        spec = hb.ModelSpec(hb.Shape.spatial(H, W, 3))
        spec.activations["relu-poly2"] = hb.relu_default_surrogate()
        spec.layers = list(full[:n])
        spec = hb.glorot_weights(spec, 6)
        data = np.random.default_rng(17).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
        x = eng.encrypt_tensor(data, seed=31, shape=spec.input)
        w = hb.forward_encrypted(eng.model(spec).set_streaming(2), x, eng, seed=41)
        for tile in (0, 1):
            try:
                s = hb.forward_encrypted(eng.model(spec).set_streaming(1, tile=tile), x, eng, seed=41)
            except Exception as e:
                print(H, W, n, tile, "ERR", e); continue
            ww, sw = w.words(), s.words()
            ok = ww.shape == sw.shape and np.array_equal(ww, sw)
            bad = [] if ok or ww.shape != sw.shape else sorted(set(np.nonzero((ww != sw).any(axis=(1, 2, 3)))[0].tolist()))
            print(H, W, n, tile, "OK" if ok else f"DIFF shape {ww.shape} {sw.shape} levels {(w.level, s.level)} scale {(w.scale, s.scale)} badcells {bad[:20]} n={len(bad)}", flush=True)
