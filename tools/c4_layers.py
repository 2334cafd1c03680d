"""Per-layer device seconds and per-kernel totals of one warm C4 forward pass
(net-n8192-d8, 4096 images, 32x32x3). Not part of the bench contract."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1911_11377_b200 as hb

p = hb.preset_params("net-n8192-d8")
spec = bench.c4_spec(hb)
eng = hb.CkksEngine(p).keygen(1)
data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
m = eng.model(spec)
for it in range(3):
    secs = []
    if it == 2:
        eng.profile_reset()
        eng.profile(True)
    y = hb.forward_encrypted(m, x, eng, seed=13, layer_seconds=secs)
    eng.synchronize()
eng.profile(False)
prof = eng.profile_read()
print(json.dumps({"layer_s": [round(s, 5) for s in secs], "total_s": sum(secs),
                  "kernels_ms": {k: round(v["ms"], 3) for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}},
                 indent=1))
