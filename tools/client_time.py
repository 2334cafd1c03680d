#!/usr/bin/env python
"""Client-side timing (one GPU): encrypt_tensor of the C4 input set (4096
images x 3072 positions, net-n8192-d8) and of the C5 32x32 set (8192 images x
3072 positions, large-n16384-d24), and decrypt_tensor of the logits. Encode
runs on the host (long-double FFT, bit-identical to the reference's
encode_real, all host threads), overlapped chunk by chunk with the device
encryption (engine.cpp encrypt_pipelined). Prints one JSON object."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import bench
import paper_1911_11377_b200 as hb

res = {}
for name, preset, spec in (("c4", "net-n8192-d8", bench.c4_spec(hb)),
                           ("c5_32", "large-n16384-d24", hb.glorot_weights(hb.alexnet32_preset(32), 1))):
    p = hb.preset_params(preset)
    eng = hb.CkksEngine(p).keygen(1)
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    eng.synchronize()
    del x
    t0 = time.perf_counter()
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    eng.synchronize()
    res[name] = {"encrypt_tensor_s": time.perf_counter() - t0, "cells": spec.input.positions(), "images": p.n // 2}
    if name == "c4":
        y = hb.forward_encrypted(eng.model(spec), x, eng, seed=13)
        eng.synchronize()
        t2 = time.perf_counter()
        eng.decrypt_tensor(y, p.n // 2)
        res[name]["decrypt_tensor_s"] = time.perf_counter() - t2
    del x
    eng.close()
print(json.dumps(res))
