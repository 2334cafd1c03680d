"""C5's whole AlexNet stack (alexnet32_preset: 4 convs, 6 relu-poly2
activations, 4 pools, 3 zero-pads, 3 dense, sigmoid) on a 4x4x3 crop at
large-n16384-d24 with 8,192 slots: the device's row-streamed forward pass
(one-column tiles) against the reference's forward_encrypted on all host
cores, every output word and the scale ledger. A one-off check (the
reference needs ~5 minutes); prints one JSON line."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_1911_11377_b200 as hb
from oracle import ref

p = hb.preset_params("large-n16384-d24")
spec = hb.glorot_weights(hb.alexnet32_preset(image=4), 1)
data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
eng = hb.CkksEngine(p).keygen(1)
x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
t0 = time.perf_counter()
y = hb.forward_encrypted(eng.model(spec).set_streaming(hb.Model.STREAM_ALWAYS, tile=1), x, eng, seed=13)
eng.synchronize()
dev_s = time.perf_counter() - t0
threads = os.cpu_count() or 1
r = ref.RefEngine.from_params(p).keygen(1)
rx = r.encrypt_tensor(data, spec.input, seed=11, threads=threads)
t0 = time.perf_counter()
ry, secs = r.forward_encrypted(spec, rx, seed=13, threads=threads)
ref_s = time.perf_counter() - t0
print(json.dumps({"crop": "4x4x3", "preset": "large-n16384-d24", "layers": len(spec.layers),
                  "device_s": dev_s, "reference_s": ref_s, "threads": threads,
                  "level_scale_equal": (y.level, y.scale) == tuple(ry.info()[1:]),
                  "words_equal": bool(np.array_equal(y.words(), ry.words())),
                  "out_level": y.level, "reference_layer_s": [round(float(v), 2) for v in secs]}))
