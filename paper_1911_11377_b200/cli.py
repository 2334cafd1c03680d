"""Command-line front end over the B200 engine for the reference's file
formats: the reference's `hecnn keygen / infer / bench`
subcommands (proj/tools/hecnn_cli.cpp:96-290) on its key blobs
(ckks_serialize.hpp), model files (model_io.hpp: JSON manifest + f64 weight
blob) and HDTS datasets (synthetic.hpp:88-114), so a directory prepared with
the reference CLI runs here unchanged:

    python -m paper_1911_11377_b200.cli keygen --preset net-n8192-d8 --out keys/
    python -m paper_1911_11377_b200.cli infer --keys keys/ --model m --data d.bin \\
        --mode encrypted --batch 4096 --out preds.csv

Same options, defaults, seeds (encrypt with derive_seed(seed, begin), forward
with derive_seed(seed, 0xf000 + begin)), CSV `id,logit,label,ms` and exit
codes (0 ok, 2 validation error, 3 runtime failure). Encrypted inference runs
on the device (the reference's `--threads` is accepted and ignored); `plain`
mode is a numpy restatement of forward_plain (layers.hpp:65-168), host-only
and not on the hot path."""
import argparse
import json
import math
import os
import struct
import sys
import time

import numpy as np

from . import (ACTIVATION, AVG_POOL2D, CONV2D, DENSE, SIGMOID, ZERO_PAD2D, CkksEngine, LayerSpec, ModelSpec,
               PolyActivation, Shape, derive_seed, forward_encrypted, load_evaluation_key, load_public_key,
               load_secret_key, blob_params, preset_params, save_evaluation_key, save_public_key, save_secret_key)

_KIND_NAMES = {CONV2D: "conv2d", AVG_POOL2D: "avg_pool2d", ZERO_PAD2D: "zero_pad2d", DENSE: "dense",
               ACTIVATION: "activation", SIGMOID: "sigmoid"}


# ---------------------------------------------------------------- file formats

def load_model(base: str):
    """load_model (model_io.hpp:105-181): manifest `base.json` + `base.weights.bin`,
    strict index checks with the reference's messages. Returns (ModelSpec,
    channel_scale)."""
    with open(base + ".json") as f:
        j = json.load(f)
    if j["format_version"] != 1:
        raise RuntimeError("load_model: unsupported model format version")
    m = ModelSpec(Shape.spatial(int(j["input"]["h"]), int(j["input"]["w"]), int(j["input"]["c"])))
    scale = list(j.get("preprocessing", {}).get("channel_scale", []))
    for lj in j["layers"]:
        kind = lj["kind"]
        if kind == "conv2d":
            pad = lj.get("padding", "same")
            if pad not in ("same", "valid"):
                raise ValueError("model manifest: bad padding mode")
            k = lj["kernel"]
            m.layers.append(LayerSpec.conv2d(int(lj["filters"]), int(k[0]), int(k[1]), int(lj.get("stride", 1)),
                                             pad == "valid"))
        elif kind == "avg_pool2d":
            m.layers.append(LayerSpec.avg_pool2d(int(lj["pool"])))
        elif kind == "zero_pad2d":
            m.layers.append(LayerSpec.zero_pad2d(int(lj["pad"])))
        elif kind == "dense":
            m.layers.append(LayerSpec.dense(int(lj["units"])))
        elif kind == "activation":
            m.layers.append(LayerSpec.activation(lj["surrogate"]))
        elif kind == "sigmoid":
            m.layers.append(LayerSpec.sigmoid())
        else:
            raise ValueError("model manifest: unknown layer kind '" + kind + "'")
    for name, aj in j.get("activations", {}).items():
        m.activations[name] = PolyActivation([float(c) for c in aj["coefficients"]], float(aj["interval"]),
                                             aj["name"])
    m.ensure_param_slots()
    with open(base + ".weights.bin", "rb") as f:
        raw = f.read()
    if len(raw) % 8:
        raise RuntimeError("load_model: weight blob length not a multiple of 8")
    blob = np.frombuffer(raw, dtype="<f8")
    expected, cur = [], m.input
    for i, l in enumerate(m.layers):
        layer_in = Shape.flattened(cur.positions()) if (l.kind == DENSE and not cur.flat) else cur
        if l.kind == CONV2D:
            expected.append((i, l.kernel_h * l.kernel_w * layer_in.c * l.filters, l.filters))
        elif l.kind == DENSE:
            expected.append((i, layer_in.positions() * l.units, l.units))
        cur = _shape_after(l, layer_in)
    index = j["weights_index"]
    if len(index) != 2 * len(expected):
        raise RuntimeError("load_model: weight index entry count disagrees with architecture")
    expect_off, last_off, first = 0, 0, True
    for e, (layer, wc, bc) in enumerate(expected):
        for part in range(2):
            entry = index[2 * e + part]
            off, cnt = int(entry["offset"]), int(entry["count"])
            if int(entry["layer"]) != layer or cnt != (wc if part == 0 else bc):
                raise RuntimeError("load_model: weight index disagrees with layer shapes")
            if not first and off <= last_off:
                raise RuntimeError("load_model: weight offsets not increasing")
            if off != expect_off:
                raise RuntimeError("load_model: weight offsets not contiguous")
            if off + cnt > blob.size:
                raise RuntimeError("load_model: weight blob truncated (shape disagreement)")
            (m.weights if part == 0 else m.biases)[layer] = np.array(blob[off:off + cnt])
            last_off, first, expect_off = off, False, off + cnt
    if expect_off != blob.size:
        raise RuntimeError("load_model: weight blob length disagrees with architecture")
    return m, scale


def _shape_after(l, cur):
    if l.kind == CONV2D:
        if l.valid:
            return Shape.spatial((cur.h - l.kernel_h) // l.stride + 1, (cur.w - l.kernel_w) // l.stride + 1, l.filters)
        return Shape.spatial((cur.h + l.stride - 1) // l.stride, (cur.w + l.stride - 1) // l.stride, l.filters)
    if l.kind == AVG_POOL2D:
        return Shape.spatial(cur.h // l.pool, cur.w // l.pool, cur.c)
    if l.kind == ZERO_PAD2D:
        return Shape.spatial(cur.h + 2 * l.pad, cur.w + 2 * l.pad, cur.c)
    if l.kind == DENSE:
        return Shape.flattened(l.units)
    return cur


def load_dataset(path: str):
    """load_dataset (synthetic.hpp:102-114): "HDTS" | u16 version | u32 count |
    u16 h, w, c | u8 labels[count] | f64 samples (batch-major). Returns
    (images [count][h*w*c], labels, Shape)."""
    with open(path, "rb") as f:
        raw = f.read()
    if raw[:4] != b"HDTS":
        raise RuntimeError("dataset: bad magic")
    if len(raw) < 16:
        raise RuntimeError("io: unexpected end of file")
    version, count, h, w, c = struct.unpack_from("<HIHHH", raw, 4)
    if version != 1:
        raise RuntimeError("dataset: unsupported version")
    labels = np.frombuffer(raw, dtype=np.uint8, count=count, offset=16)
    need = 16 + count + count * h * w * c * 8
    if len(raw) < need:
        raise RuntimeError("io: unexpected end of file")
    images = np.frombuffer(raw, dtype="<f8", count=count * h * w * c, offset=16 + count).reshape(count, h * w * c)
    return np.array(images), np.array(labels), Shape.spatial(h, w, c)


def apply_channel_scale(x: np.ndarray, shape: Shape, scale):
    """apply_channel_scale (hecnn_cli.cpp:65-72): NHWC positions, channel = p % c."""
    if not scale or shape.flat:
        return x
    s = np.array([scale[c % len(scale)] for c in range(shape.c)])
    return x * np.tile(s, shape.h * shape.w)[None, :]


# ---------------------------------------------------------------- plain mode

def forward_plain(m: ModelSpec, x: np.ndarray, layer_seconds=None) -> np.ndarray:
    """forward_plain (layers.hpp:65-168) in numpy on [batch][positions] NHWC:
    conv (same / valid, stride, clipped taps), avg_pool, zero_pad, dense,
    polynomial activation, sigmoid. Host-only; the encrypted path never uses it."""
    cur, shp = np.asarray(x, dtype=np.float64), m.input
    b = cur.shape[0]
    for i, l in enumerate(m.layers):
        t0 = time.perf_counter()
        if l.kind == CONV2D:
            out = _shape_after(l, shp)
            img = cur.reshape(b, shp.h, shp.w, shp.c)
            need_h, need_w = (out.h - 1) * l.stride + l.kernel_h, (out.w - 1) * l.stride + l.kernel_w
            pt = 0 if l.valid else max(0, (need_h - shp.h) // 2)
            pl = 0 if l.valid else max(0, (need_w - shp.w) // 2)
            padded = np.zeros((b, shp.h + need_h, shp.w + need_w, shp.c))
            padded[:, pt:pt + shp.h, pl:pl + shp.w, :] = img
            wt = m.weights[i].reshape(l.kernel_h, l.kernel_w, shp.c, l.filters)
            acc = np.zeros((b, out.h, out.w, l.filters))
            for ky in range(l.kernel_h):
                for kx in range(l.kernel_w):
                    patch = padded[:, ky:ky + (out.h - 1) * l.stride + 1:l.stride,
                                   kx:kx + (out.w - 1) * l.stride + 1:l.stride, :]
                    acc += np.einsum("byxc,co->byxo", patch, wt[ky, kx])
            cur, shp = (acc + m.biases[i]).reshape(b, -1), out
        elif l.kind == AVG_POOL2D:
            out = _shape_after(l, shp)
            img = cur.reshape(b, shp.h, shp.w, shp.c)[:, :out.h * l.pool, :out.w * l.pool, :]
            cur = img.reshape(b, out.h, l.pool, out.w, l.pool, shp.c).mean(axis=(2, 4)).reshape(b, -1)
            shp = out
        elif l.kind == ZERO_PAD2D:
            out = _shape_after(l, shp)
            img = np.zeros((b, out.h, out.w, shp.c))
            img[:, l.pad:l.pad + shp.h, l.pad:l.pad + shp.w, :] = cur.reshape(b, shp.h, shp.w, shp.c)
            cur, shp = img.reshape(b, -1), out
        elif l.kind == DENSE:
            w = m.weights[i].reshape(cur.shape[1], l.units)
            cur, shp = cur @ w + m.biases[i], Shape.flattened(l.units)
        elif l.kind == ACTIVATION:
            coeffs = m.activations[l.surrogate].coefficients
            y = np.zeros_like(cur)
            for c in reversed(coeffs):
                y = y * cur + c
            cur = y
        elif l.kind == SIGMOID:
            cur = 1.0 / (1.0 + np.exp(-cur))
        if layer_seconds is not None:
            layer_seconds.append(time.perf_counter() - t0)
    return cur


# ---------------------------------------------------------------- subcommands

def _key_paths(d):
    return os.path.join(d, "sk.bin"), os.path.join(d, "pk.bin"), os.path.join(d, "evk.bin")


def cmd_keygen(a):
    """cmd_keygen (hecnn_cli.cpp:96-122): keys written as the reference's blobs."""
    p = preset_params(a.preset, a.presets_file or "", a.degenerate)
    os.makedirs(a.out, exist_ok=True)
    paths = _key_paths(a.out)
    for path in paths:
        if os.path.exists(path) and not a.force:
            raise ValueError("refusing to overwrite existing key file " + path + " (use --force)")
    eng = CkksEngine(p).keygen(a.seed)
    for path, blob in zip(paths, (save_secret_key(eng), save_public_key(eng), save_evaluation_key(eng))):
        with open(path, "wb") as f:
            f.write(blob)
    print(f"wrote keys for preset {a.preset} to {a.out}")
    return 0


def load_keys(d: str):
    """load_keys (hecnn_cli.cpp:39-51): an engine holding the three keys."""
    blobs = []
    for path in _key_paths(d):
        with open(path, "rb") as f:
            blobs.append(f.read())
    params = [blob_params(b)[1] for b in blobs]
    if any(q.primes != params[0].primes or q.n != params[0].n or q.scale != params[0].scale for q in params[1:]):
        raise RuntimeError("key files disagree on parameters")
    eng = CkksEngine(params[0])
    load_secret_key(eng, blobs[0])
    load_public_key(eng, blobs[1])
    load_evaluation_key(eng, blobs[2])
    return eng


def _logits_model(m: ModelSpec) -> ModelSpec:
    """model_without_trailing_sigmoid (hecnn_cli.cpp:53-56)"""
    if m.layers and m.layers[-1].kind == SIGMOID:
        return ModelSpec(m.input, m.layers[:-1], m.activations, m.weights[:-1], m.biases[:-1])
    return m


def _depth_cost(m: ModelSpec) -> int:
    cost = 0
    for l in m.layers:
        if l.kind in (CONV2D, AVG_POOL2D, DENSE):
            cost += 1
        elif l.kind == ACTIVATION:
            cost += m.activations[l.surrogate].encrypted_depth()
    return cost


def _print_layer_timings(m, secs, label, out=sys.stdout):
    """print_layer_timings (hecnn_cli.cpp:74-88)"""
    out.write(f"# per-layer timings ({label})\n")
    total = 0.0
    for i, s in enumerate(secs):
        out.write(f"  layer {i:2d}  {_KIND_NAMES[m.layers[i].kind]:<12}{s * 1000:.3f} ms\n")
        total += s
    out.write(f"  total {total * 1000:.3f} ms\n")


def _data_path(p: str) -> str:
    d = os.environ.get("HECNN_DATA_DIR")
    return os.path.join(d, p) if d and p and "/" not in p else p


def cmd_infer(a):
    """cmd_infer (hecnn_cli.cpp:173-234)"""
    model, chscale = load_model(a.model)
    logits_model = _logits_model(model)
    images, labels, shape = load_dataset(_data_path(a.data))
    count = min(a.limit, images.shape[0])
    if a.batch == 0:
        raise ValueError("infer: batch must be >= 1")
    encrypted = a.mode in ("encrypted", "degenerate")
    eng = None
    if encrypted:
        eng = load_keys(a.keys)
        if a.preset:
            want = preset_params(a.preset, a.presets_file or "", a.mode == "degenerate")
            if want.primes != eng.params.primes or want.n != eng.params.n or want.scale != eng.params.scale:
                raise ValueError("infer: key files do not match preset " + a.preset)
        if (a.mode == "degenerate") != bool(eng.params.degenerate_noise):
            raise ValueError("infer: mode '" + a.mode + "' needs keys generated " +
                             ("with --degenerate" if a.mode == "degenerate" else "without --degenerate"))
        if a.batch > eng.n // 2:
            raise ValueError("infer: batch exceeds slot count")
        budget = len(eng.params.primes) - 1
        if _depth_cost(logits_model) > budget:
            raise ValueError(f"infer: model depth cost {_depth_cost(logits_model)} exceeds preset depth budget {budget}")
    elif a.mode != "plain":
        raise ValueError("infer: unknown mode '" + a.mode + "'")
    dev_model = eng.model(logits_model) if encrypted else None
    secs = []
    with open(a.out, "w") as out:
        out.write("id,logit,label,ms\n")
        for begin in range(0, count, a.batch):
            bsz = min(a.batch, count - begin)
            x = apply_channel_scale(images[begin:begin + bsz], shape, chscale)
            t0 = time.perf_counter()
            secs = []
            if encrypted:
                xe = eng.encrypt_tensor(x, seed=derive_seed(a.seed, begin), shape=logits_model.input)
                ye = forward_encrypted(dev_model, xe, eng, seed=derive_seed(a.seed, 0xF000 + begin), layer_seconds=secs)
                logits = eng.decrypt_tensor(ye, bsz)
            else:
                logits = forward_plain(logits_model, x, secs)
            ms = (time.perf_counter() - t0) * 1000.0 / bsz
            for i in range(bsz):
                lg = float(logits[i, 0])
                out.write(f"{begin + i},{lg:.17g},{1 if lg > 0 else 0},{ms:.3f}\n")
    if count > 0:
        _print_layer_timings(logits_model, secs, a.mode)
    print(f"wrote predictions for {count} images to {a.out}")
    return 0


def cmd_bench(a):
    """cmd_bench (hecnn_cli.cpp:236-290): plain vs encrypted per-layer table."""
    model, chscale = load_model(a.model)
    logits_model = _logits_model(model)
    images, labels, shape = load_dataset(_data_path(a.data))
    count = min(a.limit, images.shape[0], a.batch)
    if count == 0:
        raise ValueError("bench: no images")
    eng = load_keys(a.keys)
    if _depth_cost(logits_model) > len(eng.params.primes) - 1:
        raise ValueError("bench: model depth cost exceeds preset depth budget")
    x = apply_channel_scale(images[:count], shape, chscale)
    plain_secs, enc_secs = [], []
    t0 = time.perf_counter()
    ref = forward_plain(logits_model, x, plain_secs)
    plain_total = time.perf_counter() - t0
    t0 = time.perf_counter()
    xe = eng.encrypt_tensor(x, seed=a.seed, shape=logits_model.input)
    ye = forward_encrypted(eng.model(logits_model), xe, eng, seed=derive_seed(a.seed, 0xBE), layer_seconds=enc_secs)
    dec = eng.decrypt_tensor(ye, count)
    enc_total = time.perf_counter() - t0
    max_delta = float(np.max(np.abs(dec[:, 0] - ref[:, 0])))
    lines = [f"# bench: batch {count}, model {a.model}",
             f"{'layer':<6}{'kind':<13}{'plain_ms':>12}{'encrypted_ms':>14}{'ratio':>10}"]
    for i, l in enumerate(logits_model.layers):
        pm, em = plain_secs[i] * 1000, enc_secs[i] * 1000
        lines.append(f"{i:<6}{_KIND_NAMES[l.kind]:<13}{pm:>12.3f}{em:>14.3f}{(em / pm if pm > 0 else 0.0):>10.1f}")
    lines.append(f"{'total':<19}{plain_total * 1000:>12.3f}{enc_total * 1000:>14.3f}{enc_total / plain_total:>10.1f}")
    lines.append(f"# max |encrypted - plain| logit delta: {max_delta:.6g}")
    table = "\n".join(lines) + "\n"
    sys.stdout.write(table)
    if a.out:
        with open(a.out, "w") as f:
            f.write(table)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="hecnn-b200", description="leveled CKKS encrypted CNN inference on a B200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    kg = sub.add_parser("keygen", help="generate secret/public/evaluation keys")
    kg.add_argument("--preset", default="test-n4096-d4")
    kg.add_argument("--presets-file", default="")
    kg.add_argument("--out", required=True)
    kg.add_argument("--seed", type=int, default=1)
    kg.add_argument("--force", action="store_true")
    kg.add_argument("--degenerate", action="store_true")
    for name in ("infer", "bench"):
        p = sub.add_parser(name)
        if name == "infer":
            p.add_argument("--preset", default="")
            p.add_argument("--presets-file", default="")
            p.add_argument("--keys", default="")
            p.add_argument("--mode", default="plain")
            p.add_argument("--out", required=True)
        else:
            p.add_argument("--keys", required=True)
            p.add_argument("--out", default="")
        p.add_argument("--model", required=True)
        p.add_argument("--data", required=True)
        p.add_argument("--batch", type=int, default=8)
        p.add_argument("--threads", type=int, default=1)  # accepted; the GPU grid replaces parallel_for
        p.add_argument("--seed", type=int, default=1)
        p.add_argument("--limit", type=int, default=sys.maxsize)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:  # argparse: usage errors exit 2 like CLI11 parse errors
        return int(e.code or 0)
    try:
        return {"keygen": cmd_keygen, "infer": cmd_infer, "bench": cmd_bench}[a.cmd](a)
    except (ValueError, KeyError) as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except Exception as e:  # noqa: BLE001 -- the reference maps every other exception to 3
        sys.stderr.write(f"error: {e}\n")
        return 3


if __name__ == "__main__":
    sys.exit(main())
