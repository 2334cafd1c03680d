#!/usr/bin/env python
"""Benchmark of the encrypted-CNN hot path (BASELINE.json north_star).

Default workload (N=1): SURVEY §8(d) C4 -- the CIFAR-10-shaped CNN with the
degree-2 polynomial ReLU on encrypted synthetic 32x32x3 images, preset
net-n8192-d8 (4096 images packed in the slots of one ciphertext set). C5
(AlexNet-like COWC at 64x64x3) needs ~266 GiB of layer rings even when
row-streamed, more than one B200 holds, so C4 is the largest
BASELINE config that fits one GPU and is the headline. The same line reports,
measured: C5's AlexNet stack (alexnet32_preset, large-n16384-d24) on one full
8192-image set at 32x32x3 (row-streamed), with its 64x64 time extrapolated
from those per-layer times; C3 (CryptoNets-style) on a full set with its
output words checked against the reference; C2's NTT and HE-mul ops/s.

A step = forward_encrypted over one set (4096 images) with the input
ciphertexts resident in HBM (`value`); `e2e` repeats it through the public
API from pinned host buffers: H2D of the input ciphertexts, forward, D2H of
the output ciphertexts. Under torchrun each rank evaluates its own set (batch
sharding, weak scaling) and the output ciphertexts are gathered to rank 0 with
one NCCL all_gather -- the only collective.

--impl reference times the reference's own CPU path (oracle/_ref, compiled
from the unmodified reference headers) on the host cores: the same C4 stack
on an 8x8 crop of the images, extrapolated to the full 32x32 set layer by
layer from the reference's own per-layer timings and exact op-count ratios.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted images/sec (AlexNet-like COWC) at 1/2/4/8 B200; NTT & HE-mul ops/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")


def c4_spec(hb, image=32):
    spec = hb.ModelSpec(hb.Shape.spatial(image, image, 3))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.conv2d(16, 3, 3), hb.LayerSpec.activation("relu-poly2"), hb.LayerSpec.avg_pool2d(2),
                   hb.LayerSpec.conv2d(32, 3, 3), hb.LayerSpec.activation("relu-poly2"), hb.LayerSpec.dense(10)]
    return hb.glorot_weights(spec, 4)


def c3_spec(hb):
    spec = hb.ModelSpec(hb.Shape.spatial(28, 28, 1))
    spec.activations["square"] = hb.PolyActivation([0.0, 0.0, 1.0], 1.0, "square")
    spec.layers = [hb.LayerSpec.zero_pad2d(1), hb.LayerSpec.conv2d(5, 5, 5, stride=2, valid=True),
                   hb.LayerSpec.activation("square"), hb.LayerSpec.dense(100), hb.LayerSpec.activation("square"),
                   hb.LayerSpec.dense(10)]
    spec = hb.glorot_weights(spec, 4)
    for i in (1, 3, 5):
        spec.weights[i] = spec.weights[i] * 0.5
    return spec


def layer_work(hb, spec):
    """Per-layer work counts used to extrapolate layer times between input
    sizes of the same stack: conv = sum over output pixels of valid taps x
    filters (layers.hpp:174-211 skips clipped taps), activation / pool =
    output cells, zero-pad = fresh border encryptions, dense = inputs x units."""
    out, cur = [], spec.input
    shapes = spec.shapes()
    for l, shp in zip(spec.layers, shapes):
        if l.kind == hb.CONV2D:
            def taps(n_in, n_out, k, s):
                if l.valid:
                    return [k] * n_out
                need = (n_out - 1) * s + k
                pad = (need - n_in) // 2 if need > n_in else 0
                return [sum(1 for kk in range(k) if 0 <= o * s + kk - pad < n_in) for o in range(n_out)]
            ty = taps(cur.h, shp.h, l.kernel_h, l.stride)
            tx = taps(cur.w, shp.w, l.kernel_w, l.stride)
            out.append(sum(ty) * sum(tx) * cur.c * l.filters)
        elif l.kind in (hb.ACTIVATION, hb.AVG_POOL2D):
            out.append(shp.positions())
        elif l.kind == hb.ZERO_PAD2D:
            out.append(shp.positions() - cur.positions())
        elif l.kind == hb.DENSE:
            out.append(cur.positions() * l.units)
        else:
            out.append(0)
        cur = shp
    return out


def c3_cryptonets(hb, device, with_reference, stream=None, steps=20, warmup=5):
    """the CryptoNets-style stack (pad -> conv 5x5/2 -> square
    -> dense 100 -> square -> dense 10) on 4096 encrypted synthetic 28x28x1
    images per set (net-n8192-d8), device-timed; with the reference, the same
    set through oracle/_ref on all host threads, and the output ciphertext
    words compared (full-config parity)."""
    import torch
    p = hb.preset_params("net-n8192-d8")
    spec = c3_spec(hb)
    eng = hb.CkksEngine(p, device=device).keygen(1)
    if stream is not None:
        eng.set_stream(stream)
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    model = eng.model(spec)
    # enough warm passes that the clocks are back up after the host-only legs before it
    for _ in range(warmup):
        y = hb.forward_encrypted(model, x, eng, seed=13)
    eng.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        y = hb.forward_encrypted(model, x, eng, seed=13)
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) / 1e3 / steps
    res = {"preset": "net-n8192-d8", "images_per_set": p.n // 2, "ms_per_set": sec * 1e3,
           "images_per_s": (p.n // 2) / sec}
    if with_reference:
        from oracle import ref
        if ref.available():
            threads = os.cpu_count() or 1
            r = ref.RefEngine.from_params(p).keygen(1)
            rx = r.encrypt_tensor(data, spec.input, seed=11, threads=threads)
            t0 = time.perf_counter()
            ry, _ = r.forward_encrypted(spec, rx, seed=13, threads=threads)
            wall = time.perf_counter() - t0
            res["reference"] = {"seconds_per_set": wall, "images_per_s": (p.n // 2) / wall, "threads": threads,
                                "kind": "reference", "sample": "the full C3 set (no extrapolation)"}
            res["output_words_equal_reference"] = bool(np.array_equal(y.words(), ry.words()))
    eng.close()
    return res


def crop_extrapolation_check(hb, eng, full_ms, crop=16):
    """Validates C5's 32x32 -> 64x64 extrapolation on C4, where both sizes
    run: the C4 stack on a crop x crop x 3 input, each layer's CUDA-event time
    scaled by the same layer_work ratios, against the measured 32x32 step."""
    spec = c4_spec(hb, crop)
    model = eng.model(spec)
    x = eng.encrypt_tensor(np.random.default_rng(3).uniform(0, 1, size=(eng.params.n // 2, spec.input.positions())),
                           seed=11, shape=spec.input)
    hb.forward_encrypted(model, x, eng, seed=13)
    secs = []
    hb.forward_encrypted(model, x, eng, seed=13, layer_seconds=secs)
    wc, wf = layer_work(hb, spec), layer_work(hb, c4_spec(hb, 32))
    est = sum(s * (a / b if b else 1.0) for s, a, b in zip(secs, wf, wc))
    return {"crop": f"{crop}x{crop}x3", "extrapolated_ms": est * 1e3, "measured_ms": full_ms,
            "ratio": est * 1e3 / full_ms}


def layer_levels(hb, spec, top):
    """Input level of every layer (depth_cost ledger, model.hpp:169-182)."""
    out, lv = [], top
    for l in spec.layers:
        out.append(lv)
        if l.kind in (hb.CONV2D, hb.AVG_POOL2D, hb.DENSE):
            lv -= 1
        elif l.kind == hb.ACTIVATION:
            lv -= 2  # degree-2 surrogates: ceil(log2 2) + 1
    return out


def reference_per_op_estimate(hb, spec, p, threads, r=None, cache=None):
    """The reference's own forward_encrypted time for one set of `spec`,
    estimated per op (C5 cannot run on the CPU): each layer's op
    count x the reference's measured per-op throughput at that layer's level
    on all host threads through its parallel_for (oracle/_ref
    ref_time_layer_op): conv / dense = outputs x (zero + bias + rescale) +
    scalar MACs (layer_work); activation = cells x eval_encrypted;
    avg_pool = outputs x (4 MAC-equivalents + rescale); zero_pad = border cells
    x encrypt + mod_switch."""
    from oracle import ref
    if r is None:
        r = ref.RefEngine.from_params(p).keygen(1)
    levels, shapes, work = layer_levels(hb, spec, len(p.primes) - 1), spec.shapes(), layer_work(hb, spec)
    cache = {} if cache is None else cache

    def rate(op, lv, inner):
        key = (op, lv, inner)
        if key not in cache:
            count = threads if op == 0 else 2 * threads
            # twice: the first pass pays the allocator's first-touch page faults
            t = min(r.time_layer_op(op, lv, count, inner, threads) for _ in range(2))
            cache[key] = count / t  # items per second
        return cache[key]

    per_layer, t_ops = [], time.perf_counter()
    for l, lv, shp, w in zip(spec.layers, levels, shapes, work):
        if l.kind in (hb.CONV2D, hb.DENSE):
            outs = shp.positions()
            base, full = 1.0 / rate(1, lv, 0), 1.0 / rate(1, lv, 64)
            per_layer.append(outs * base + w * (full - base) / 64)
        elif l.kind == hb.ACTIVATION:
            per_layer.append(shp.positions() / rate(0, lv, 0))
        elif l.kind == hb.AVG_POOL2D:
            per_layer.append(shp.positions() / rate(1, lv, 4))
        elif l.kind == hb.ZERO_PAD2D:
            per_layer.append(w / rate(2, lv, 0) if w else 0.0)
        else:
            per_layer.append(0.0)
    return {"seconds_per_set": float(sum(per_layer)), "layer_s": [round(v, 3) for v in per_layer],
            "threads": threads, "probe_wall_s": time.perf_counter() - t_ops}


def c5_measured(hb, device, stream=None, image=32, check=8, with_reference=True):
    """C5 (AlexNet-like COWC: alexnet32_preset layers, large-n16384-d24, 8192
    images per ciphertext set) on one FULL set of encrypted synthetic
    image x image x 3 inputs, device-timed with CUDA events. The layer tensors
    (conv1's output alone is 576 GiB at 32x32) run row-streamed (stream.cpp):
    rings of rows and column tiles sized to the free HBM. The 64x64 COWC
    patches need ~266 GiB of rings even streamed, more than one
    B200 holds, so that size is extrapolated from this measured run's
    per-layer times by exact work ratios (method checked on C4, 16x16 ->
    32x32, where both run)."""
    import torch
    p = hb.preset_params("large-n16384-d24")
    t0 = time.perf_counter()
    eng = hb.CkksEngine(p, device=device).keygen(1)
    if stream is not None:
        eng.set_stream(stream)
    spec = hb.glorot_weights(hb.alexnet32_preset(image=image), 1)
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    x = eng.encrypt_tensor(data, seed=11, shape=spec.input)
    eng.synchronize()
    setup = time.perf_counter() - t0
    model = eng.model(spec)
    secs = []
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    y = hb.forward_encrypted(model, x, eng, seed=13, layer_seconds=secs)
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) / 1e3
    res = {"preset": "large-n16384-d24", "images_per_set": p.n // 2, "input": f"{image}x{image}x3",
           "seconds_per_set": sec, "images_per_s": (p.n // 2) / sec, "out_level": y.level,
           "layer_s": [round(v, 4) for v in secs], "client_encrypt_s": setup,
           "execution": "one full set, row-streamed spatial layers (rings of rows + column tiles), first run "
                        "(weight caches and stream plans built inside the timed region)"}
    if check:
        from oracle import ref
        if ref.available():
            plain = ref.forward_plain(spec, data[:check])
            dec = 1.0 / (1.0 + np.exp(-eng.decrypt_tensor(y, p.n // 2)[:check]))
            res["max_abs_err_vs_plain"] = float(np.max(np.abs(dec - plain)))
    w32, w64 = layer_work(hb, spec), layer_work(hb, hb.alexnet32_preset(image=64))
    t64 = sum(v * (b / a if a else 1.0) for v, a, b in zip(secs, w32, w64))
    res["64x64_extrapolated"] = {"seconds_per_set": t64, "images_per_s": (p.n // 2) / t64,
                                 "method": "measured 32x32 per-layer times x exact per-layer work ratios"}
    del y, x, model
    if image == 32:
        # the same method one size down, on the same stack: a measured 16x16 set
        # extrapolated to 32x32 against the measured 32x32 set above (warm weight
        # caches excluded: the 16x16 pass builds its own)
        spec16 = hb.glorot_weights(hb.alexnet32_preset(image=16), 1)
        d16 = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec16.input.positions()))
        x16 = eng.encrypt_tensor(d16, seed=11, shape=spec16.input)
        m16 = eng.model(spec16)
        s16 = []
        hb.forward_encrypted(m16, x16, eng, seed=13)  # caches and plans
        s.record()
        hb.forward_encrypted(m16, x16, eng, seed=13, layer_seconds=s16)
        e.record()
        torch.cuda.synchronize()
        w16 = layer_work(hb, spec16)
        t32 = sum(v * (b / a if a else 1.0) for v, a, b in zip(s16, w16, w32))
        res["method_check_on_c5"] = {"from": "16x16 (measured, warm)", "to": "32x32", "extrapolated_s": t32,
                                     "measured_s": sec, "ratio": t32 / sec, "measured_16x16_s": s.elapsed_time(e) / 1e3}
        del x16, m16
    eng.close()
    if with_reference:
        from oracle import ref
        if ref.available():
            threads = os.cpu_count() or 1
            rl, cache = ref.RefEngine.from_params(p).keygen(1), {}
            est = reference_per_op_estimate(hb, spec, p, threads, rl, cache)
            spec64 = hb.glorot_weights(hb.alexnet32_preset(image=64), 1)
            est64 = reference_per_op_estimate(hb, spec64, p, threads, rl, cache)
            # method check: the same estimator on C3, whose full set the reference runs
            pc = hb.preset_params("net-n8192-d8")
            c3 = c3_spec(hb)
            rc = ref.RefEngine.from_params(pc).keygen(1)
            c3_est = reference_per_op_estimate(hb, c3, pc, threads, rc)
            data3 = np.random.default_rng(3).uniform(0, 1, size=(pc.n // 2, c3.input.positions()))
            rx = rc.encrypt_tensor(data3, c3.input, seed=11, threads=threads)
            t0 = time.perf_counter()
            rc.forward_encrypted(c3, rx, seed=13, threads=threads)
            c3_wall = time.perf_counter() - t0
            res["reference_estimate"] = {
                "kind": "reference", "cores": threads,
                "sample": "per-op throughputs of the reference's layer ops (oracle/_ref) at every layer level on all "
                          "host threads x the stack's op counts (SURVEY 8(d): C5 does not run on the CPU)",
                "32x32": {"seconds_per_set": est["seconds_per_set"],
                          "images_per_s": (p.n // 2) / est["seconds_per_set"], "layer_s": est["layer_s"]},
                "64x64": {"seconds_per_set": est64["seconds_per_set"],
                          "images_per_s": (p.n // 2) / est64["seconds_per_set"]},
                "method_check_on_c3": {"estimated_s": c3_est["seconds_per_set"], "measured_s": c3_wall,
                                       "ratio": c3_est["seconds_per_set"] / c3_wall},
                "probe_wall_s": est["probe_wall_s"] + est64["probe_wall_s"]}
    return res


# ---------------------------------------------------------------- helpers

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self._stop = threading.Event()
        self._proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self._proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                           "--format=csv,noheader,nounits", "-lms", "200"],
                                          stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self._proc = None
        return self

    def _read(self):
        for line in self._proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self._proc:
            self._proc.terminate()
            try:
                self._proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self._proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4) if s[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def measured_traffic(kernel):
    """DRAM bytes per launch for `kernel` from the newest committed ncu
    capture (profiles/r02_traffic.json, else r01), or None when that kernel
    was not captured."""
    for name in ("r02_traffic.json", "r01_traffic.json"):
        try:
            with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", name)) as f:
                t = json.load(f).get(kernel)
            if t:
                return t["dram_bytes_per_launch"]
        except (OSError, ValueError, KeyError):
            continue
    return None


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "_fallback": True}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


def max_over_ranks(seconds, device):
    """Max of a per-rank device time over all ranks (the job's time)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([seconds], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_outputs(words):
    """The only collective of the sharded path: every rank's output ciphertext
    words gathered to all ranks (NCCL all_gather on GPUs, gloo in the CPU tests)."""
    import torch
    import torch.distributed as dist
    gathered = [torch.empty_like(words) for _ in range(dist.get_world_size())]
    dist.all_gather(gathered, words)
    return gathered


# ---------------------------------------------------------------- reference (CPU) path

def reference_c4_images_per_s(threads):
    """The reference's forward_encrypted on an 8x8 crop of the C4 images,
    extrapolated per layer to the full 32x32 set by exact op-count ratios
    (conv: output cells x valid taps; activation/pool: cells; dense: inputs)."""
    import paper_1911_11377_b200 as hb
    from oracle import ref

    p = hb.preset_params("net-n8192-d8")
    crop, full = 8, 32
    spec = c4_spec(hb, crop)
    r = ref.RefEngine.from_params(p).keygen(1)
    rng = np.random.default_rng(3)
    data = rng.uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    x = r.encrypt_tensor(data, spec.input, seed=11, threads=threads)
    t0 = time.perf_counter()
    _, secs = r.forward_encrypted(spec, x, seed=13, threads=threads)
    wall = time.perf_counter() - t0

    def taps(side):  # valid 3x3 same-conv taps summed over output pixels of a side x side map
        per = [min(3, i + 2, side - i + 1, side) for i in range(side)]
        return sum(per) ** 2

    ratios = [16.0 * taps(full) / (16.0 * taps(crop)) * 1.0,   # conv1 (cells x taps, c_out same)
              (full * full) / (crop * crop),                 # act1
              (full * full) / (crop * crop),                 # pool1
              taps(full // 2) / taps(crop // 2),             # conv2
              (full * full) / (crop * crop),                 # act2
              (full * full) / (crop * crop)]                 # dense: in_f ratio
    est = float(sum(s * k for s, k in zip(secs, ratios)))
    return p.n // 2 / est, est, wall, [float(s) for s in secs]


def c4_config(world):
    """The `config` object of both arms' lines (the driver compares them)."""
    in_gib = 32 * 32 * 3 * 2 * 9 * 8192 * 8 / 2 ** 30  # input set: 3072 cells x 2 polys x 9 limbs x N words
    return {"workload": "C4 CIFAR-10-shaped CNN + poly ReLU (conv16-act-pool-conv32-act-dense10), "
                        "net-n8192-d8, 4096 encrypted images per set per GPU",
            "preset": "net-n8192-d8", "images_per_set": 4096, "sets_per_gpu_per_step": 1,
            "parallelism": f"dp{world} (batch sharding; NCCL all_gather of output ciphertexts only)",
            "l2": f"inputs larger than L2 ({in_gib:.2f} GiB of input ciphertexts)",
            "profiling": "per-kernel CUDA events on the launching stream inside the timed region"}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        v, est, wall, secs = reference_c4_images_per_s(threads)
        if i >= args.warmup:
            vals.append((v, est, wall))
    value = float(np.median([v for v, _, _ in vals]))
    ms = float(np.median([e for _, e, _ in vals])) * 1e3
    sample = "C4 stack on an 8x8 crop (1/16 of the cells), per-layer op-count extrapolation to 32x32; 4096 images/set"
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "config": c4_config(world),
            "execution": f"reference forward_encrypted on {threads} host threads (its parallel_for), rank 0 only",
            "cpu_baseline": {"value": value, "unit": "images/s", "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our path

def microbench(hb, eng_dev, n=16384, count=256):
    """C2: NTT/INTT and HE-mul (tensor + relinearize + rescale) throughput at
    chain [60, 40 x 8], uniform-random residues as synthetic ciphertexts."""
    import torch
    p = hb.CkksParams(n, hb.find_chain(n, [60] + [40] * 8), 2.0 ** 40)
    eng = hb.CkksEngine(p, device=eng_dev).keygen(1)
    eng.set_stream(torch.cuda.current_stream().cuda_stream)
    L = p.top_level
    rng = np.random.default_rng(5)
    words = np.empty((count, 2, L + 1, n), dtype=np.uint64)
    for i, q in enumerate(p.primes):
        words[:, :, i, :] = rng.integers(0, q, size=(count, 2, n), dtype=np.uint64)
    x = eng.tensor_from_words(words, L, p.scale)
    y = eng.tensor_from_words(words[::-1].copy(), L, p.scale)
    dptr = x.device_ptr()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import ctypes
    polys = 2 * count
    for _ in range(2):
        hb._check(hb.lib().hecnn_ntt_forward(eng.ctx, ctypes.c_void_p(dptr), ctypes.c_size_t(L), ctypes.c_size_t(polys)))
        hb._check(hb.lib().hecnn_ntt_inverse(eng.ctx, ctypes.c_void_p(dptr), ctypes.c_size_t(L), ctypes.c_size_t(polys)))
    torch.cuda.synchronize()
    reps = 5
    s.record()
    for _ in range(reps):
        hb._check(hb.lib().hecnn_ntt_forward(eng.ctx, ctypes.c_void_p(dptr), ctypes.c_size_t(L), ctypes.c_size_t(polys)))
        hb._check(hb.lib().hecnn_ntt_inverse(eng.ctx, ctypes.c_void_p(dptr), ctypes.c_size_t(L), ctypes.c_size_t(polys)))
    e.record()
    torch.cuda.synchronize()
    ntt_s = s.elapsed_time(e) / 1e3
    ntt_ops = reps * 2 * polys * (L + 1) / ntt_s
    eng.mul(x, y)
    torch.cuda.synchronize()
    s.record()
    for _ in range(2):
        z = eng.mul(x, y)
    e.record()
    torch.cuda.synchronize()
    mul_s = s.elapsed_time(e) / 1e3
    del z
    res = {"n": n, "chain": "[60,40x8]", "level": L, "ciphertexts": count,
           "ntt_ops_per_s": ntt_ops, "he_mul_ops_per_s": 2 * count / mul_s}
    eng.close()
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1911_11377_b200 as hb

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.current_stream()

    p = hb.preset_params("net-n8192-d8")
    batch = p.n // 2
    spec = c4_spec(hb)
    eng = hb.CkksEngine(p, device=local).keygen(1)
    eng.set_stream(stream.cuda_stream)
    model = eng.model(spec)
    rng = np.random.default_rng(3 + rank)
    data = rng.uniform(0, 1, size=(batch, spec.input.positions()))
    x = eng.encrypt_tensor(data, seed=11 + rank, shape=spec.input)     # client side, untimed
    in_words = x.words()
    assert batch == c4_config(world)["images_per_set"] and in_words.nbytes == 32 * 32 * 3 * 2 * 9 * 8192 * 8
    host_in = torch.from_numpy(in_words.reshape(-1).view(np.int64)).pin_memory()
    h2d_bytes = in_words.nbytes

    for _ in range(args.warmup):
        y = hb.forward_encrypted(model, x, eng, seed=13)
    torch.cuda.synchronize()
    out_cells, out_level = y.cells, y.level
    out_words_n = y.words().size
    host_out = torch.empty(out_words_n, dtype=torch.int64).pin_memory()

    # ---- device-resident timed region
    launches0 = eng.launches()
    eng.profile_reset()
    eng.profile(True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        s.record(stream)
        for _ in range(args.steps):
            y = hb.forward_encrypted(model, x, eng, seed=13)
        e.record(stream)
        torch.cuda.synchronize()
    eng.profile(False)
    prof = eng.profile_read()
    launches = eng.launches() - launches0
    dev_s = s.elapsed_time(e) / 1e3
    gather_words = torch.empty(out_words_n, dtype=torch.int64, device=f"cuda:{local}")
    eng.copy_to_device(y, gather_words.data_ptr())
    if world > 1:
        dev_s = max_over_ranks(dev_s, f"cuda:{local}")
        gathered = gather_outputs(gather_words)
        torch.cuda.synchronize()
        assert all(g.numel() == gather_words.numel() for g in gathered)

    # ---- end to end through the public API from pinned host memory
    xe = eng.empty_tensor(x.cells, x.level, x.scale)
    xe.set_shape(spec.input, batch)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    # Serving pipeline: two input buffers; the H2D of set k+1 runs on a copy
    # stream under set k's compute (events order buffer reuse); every step
    # still moves its whole input H2D and its logits D2H inside the region.
    xe2 = [xe, eng.empty_tensor(x.cells, x.level, x.scale)]
    xe2[1].set_shape(spec.input, batch)
    copy = torch.cuda.Stream(device=f"cuda:{local}")
    landed = [torch.cuda.Event(), torch.cuda.Event()]
    consumed = [torch.cuda.Event(), torch.cuda.Event()]
    t0 = time.perf_counter()
    s.record(stream)
    copy.wait_stream(stream)
    eng.upload_async(xe2[0], host_in.data_ptr(), copy.cuda_stream)
    landed[0].record(copy)
    for k in range(args.steps):
        b = k % 2
        stream.wait_event(landed[b])
        if k + 1 < args.steps:
            nb = 1 - b
            if k >= 1:
                copy.wait_event(consumed[nb])  # set k-1 is done reading that buffer
            eng.upload_async(xe2[nb], host_in.data_ptr(), copy.cuda_stream)
            landed[nb].record(copy)
        ye = hb.forward_encrypted(model, xe2[b], eng, seed=13)
        consumed[b].record(stream)
        eng.download_async(ye, host_out.data_ptr(), stream.cuda_stream)
    e.record(stream)
    torch.cuda.synchronize()
    e2e_s = s.elapsed_time(e) / 1e3
    if world > 1:
        e2e_s = max_over_ranks(e2e_s, f"cuda:{local}")
    assert np.array_equal(host_out.numpy().view(np.uint64), y.words().reshape(-1)), "e2e output differs"

    images = world * batch * args.steps
    line = None
    if rank == 0:
        # dominant kernel and its roofline
        pk = peaks()
        int_only_peak = eng.modmul_peak()
        # The modmul roofline is the faster of the two pipes the kernels use:
        # exact FP64 modmuls (primes < 2^42, all but the 60-bit chain prime)
        # run ~2.7x faster than 64-bit Shoup on the integer pipes.
        int_peak = max(eng.fp64_modmul_peak(), int_only_peak)
        top = max(prof.items(), key=lambda kv: kv[1]["ms"])
        name, st = top
        kernel_avg_ms = st["ms"] / max(st["launches"], 1)
        # the key switch finishes limb 0 in its k_ks_aux_* kernels (keyswitch.cu
        # "aux"): their time is charged to the key switch's launches
        helpers = {k: v for k, v in prof.items() if k.startswith("k_ks_aux")} if name == "k_keyswitch" else {}
        avg_ms = (st["ms"] + sum(v["ms"] for v in helpers.values())) / max(st["launches"], 1)
        ops_per_launch = st["ops"] / max(st["launches"], 1)
        bytes_per_launch = st["bytes"] / max(st["launches"], 1)
        achieved_ops = ops_per_launch / (avg_ms / 1e3)
        achieved_gbs = bytes_per_launch / (avg_ms / 1e3) / 1e9
        int_bound = achieved_ops / int_peak >= achieved_gbs / pk["hbm_gbs"]
        roofline = {
            "kernel": name, "bound": "int" if int_bound else "hbm",
            "achieved": achieved_ops / 1e9 if int_bound else achieved_gbs,
            "peak": int_peak / 1e9 if int_bound else pk["hbm_gbs"],
            "unit": "Gmodmul/s" if int_bound else "GB/s",
            "frac": (achieved_ops / int_peak) if int_bound else achieved_gbs / pk["hbm_gbs"],
            "traffic": measured_traffic(name),
            "ops_per_launch": ops_per_launch, "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
            "includes": [name] + sorted(helpers),
            "kernel_only": {"avg_launch_ms": kernel_avg_ms,
                            "frac": ops_per_launch / (kernel_avg_ms / 1e3) / int_peak if int_bound else
                            bytes_per_launch / (kernel_avg_ms / 1e3) / 1e9 / pk["hbm_gbs"]},
            "share_of_step": avg_ms * st["launches"] / 1e3 / dev_s,
            "peak_source": "int: live probe of chained exact FP64 modmuls (hecnn_fp64_modmul_peak, the faster "
                           "pipe; integer 64-bit Shoup probe reported as int_shoup_peak); hbm: MEASURED_PEAKS.json",
            "int_shoup_peak": int_only_peak / 1e9,
            "hbm_view": {"achieved_gbs": achieved_gbs, "peak_gbs": pk["hbm_gbs"], "frac": achieved_gbs / pk["hbm_gbs"]},
        }
        # the standalone NTT kernels (north star: >= 50% of roofline on NTT and key
        # switch); an N = 2^13 limb-NTT is balanced between the FP64 pipe and HBM,
        # so its roofline time is the larger of the two
        ntt_roof = {}
        for kname in ("k_ntt_fwd_block", "k_ntt_inv_block", "k_ntt_inv_rescale"):
            v = prof.get(kname)
            if v and v["ms"] > 0:
                ops_s, gbs = v["ops"] / (v["ms"] / 1e3), v["bytes"] / (v["ms"] / 1e3) / 1e9
                ntt_roof[kname] = {"achieved_gmodmul_s": ops_s / 1e9, "achieved_gbs": gbs,
                                   "frac": max(ops_s / int_peak, gbs / pk["hbm_gbs"]),
                                   "ms_per_step": v["ms"] / args.steps}
        roofline["ntt_kernels"] = ntt_roof
        kernels = {k: {"ms_per_step": v["ms"] / args.steps, "launches_per_step": v["launches"] / args.steps,
                       "gmodmul_s": (v["ops"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else 0.0,
                       "gb_s": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] > 0 else 0.0}
                   for k, v in sorted(prof.items(), key=lambda kv: -kv[1]["ms"])}
        del x, y, xe, ye
        xcheck = (crop_extrapolation_check(hb, eng, dev_s / args.steps * 1e3, crop=16)
                  if world == 1 and not args.no_c5 else None)
        eng.trim()  # hand C4's cached arena back before the larger C2/C5 runs
        # single-GPU reference figures: at N > 1 the other ranks would idle at the final barrier
        mb = microbench(hb, local) if world == 1 and not args.no_micro else None
        # C3 while the GPU is still busy-clocked (after C5's host-only reference legs its
        # short timed region caught the clock ramp)
        c3 = (c3_cryptonets(hb, local, with_reference=not args.no_cpu_baseline, stream=stream.cuda_stream)
              if world == 1 and not args.no_c5 else None)
        c5 = (c5_measured(hb, local, stream=stream.cuda_stream, with_reference=not args.no_cpu_baseline)
              if world == 1 and not args.no_c5 else None)
        if c5 is not None:
            c5["method_check_on_c4"] = xcheck
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            from oracle import ref
            if ref.available():
                v, est, wall, _ = reference_c4_images_per_s(os.cpu_count() or 1)
                cpu = {"value": v, "unit": "images/s", "cores": os.cpu_count() or 1, "kind": "reference",
                       "sample": f"reference forward_encrypted on an 8x8 crop of C4 ({wall:.1f}s wall), per-layer "
                                 "op-count extrapolation to the 32x32 set"}
        line = {"metric": METRIC, "value": images / dev_s, "unit": "images/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": dev_s / args.steps * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
                "data": "synthetic (uniform [0,1] 32x32x3 images, numpy Glorot weights)",
                "config": c4_config(world),
                "clocks": clk.summary(),
                "e2e": {"value": images / e2e_s, "unit": "images/s", "h2d_bytes_per_step": h2d_bytes,
                        "d2h_bytes_per_step": out_words_n * 8},
                "gpu_launches": launches, "roofline": roofline, "cpu_baseline": cpu,
                "output": {"cells": out_cells, "level": out_level},
                "microbench_c2": mb, "c3_cryptonets": c3, "c5_alexnet_cowc": c5, "kernels": kernels}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-micro", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (AlexNet-COWC) full-set run and C3")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
