#!/usr/bin/env python
"""Client-side timing (one GPU): encrypt_tensor of the C4 input set (4096
images x 3072 positions, net-n8192-d8) and decrypt_tensor of the logits.
Encode runs on the host (long-double FFT, bit-identical to the reference's
encode_real, all host threads); encryption runs on the device."""
import time, numpy as np, sys
sys.path.insert(0, '/root/repo')
import bench, paper_1911_11377_b200 as hb
p = hb.preset_params("net-n8192-d8")
spec = bench.c4_spec(hb)
eng = hb.CkksEngine(p).keygen(1)
data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
x = eng.encrypt_tensor(data, seed=11, shape=spec.input); eng.synchronize()
t0 = time.perf_counter(); x = eng.encrypt_tensor(data, seed=11, shape=spec.input); eng.synchronize(); t1 = time.perf_counter()
m = eng.model(spec); y = hb.forward_encrypted(m, x, eng, seed=13); eng.synchronize()
t2 = time.perf_counter(); out = eng.decrypt_tensor(y, p.n // 2); t3 = time.perf_counter()
print({"encrypt_tensor_s": t1 - t0, "cells": spec.input.positions(), "decrypt_tensor_s": t3 - t2})
