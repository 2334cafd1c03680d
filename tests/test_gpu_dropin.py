"""GPU: the reference's own sample flow (samples/encrypted_inference.cpp,
samples/roundtrip.cpp) compiled as C++ against the drop-in header
include/hecnn_b200/hecnn.hpp + libhecnn_b200.so, and its encrypted logits
compared word-for-word with the reference run on the same keys, seeds and
inputs."""
import os
import subprocess

import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_dropin_matches_reference(ref, tmp_path):
    exe = tmp_path / "dropin"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/dropin_inference.cpp",
                    f"-L{ROOT}/paper_1911_11377_b200/lib", "-lhecnn_b200", f"-Wl,-rpath,{ROOT}/paper_1911_11377_b200/lib",
                    "-o", str(exe)], check=True)
    spec = hb.tiny_preset()
    ref.init_random_weights(spec, 3)
    imgs, _ = ref.gen_synthetic(4, 8, 3, 5)
    blob = b""
    for arr in (spec.weights[0], spec.biases[0], spec.weights[3], spec.biases[3], imgs.reshape(-1)):
        blob += np.uint64(arr.size).tobytes() + np.ascontiguousarray(arr, np.float64).tobytes()
    (tmp_path / "in.bin").write_bytes(blob)
    out = subprocess.run([str(exe), str(tmp_path / "in.bin"), str(tmp_path / "out.bin"), str(tmp_path / "blobs.bin")], check=True,
                         capture_output=True, text=True).stdout
    assert "image 3 logit" in out
    raw = (tmp_path / "out.bin").read_bytes()
    level = int(np.frombuffer(raw[:4], np.uint32)[0])
    scale = float(np.frombuffer(raw[4:12], np.float64)[0])
    n = 4096
    words = np.frombuffer(raw[12:12 + 2 * (level + 1) * n * 8], np.uint64).reshape(2, level + 1, n)
    logits = np.frombuffer(raw[12 + 2 * (level + 1) * n * 8:], np.float64)

    p = hb.preset_params("nn-n4096-d8")
    r = ref.RefEngine.from_params(p).keygen(7)
    x = r.encrypt_tensor(imgs, spec.input, seed=11)
    y, _ = r.forward_encrypted(spec, x, seed=13)
    assert y.info()[1] == level and y.info()[2] == scale
    assert np.array_equal(y.words()[0], words)
    assert np.array_equal(r.decrypt_tensor(y, 4)[:, 0], logits)
    plain = ref.forward_plain(spec, imgs)[:, 0]
    assert np.max(np.abs(logits - plain)) < 1e-2
    # ckks_serialize.hpp through the drop-in: byte-identical to the reference's blobs
    blobs = (tmp_path / "blobs.bin").read_bytes()
    ct_blob = r.save_ciphertext(y.words()[0], level, scale)
    assert blobs == ct_blob + r.save_key(3)


def test_cpp_scalar_fast_path_matches_reference(ref, tmp_path):
    """tests/cpp/dropin_scalar.cpp: a layer kernel written against the drop-in
    header with the reference's scalar fast path (make_zero_ciphertext,
    make_scalar_plain, mul_scalar_mac, add_scalar_inplace, rescale, mul_plain,
    add_plain, add_inplace) -- the same chain on the reference, word for word."""
    exe = tmp_path / "dropin_scalar"
    subprocess.run(["g++", "-std=c++20", "-O2", f"-I{ROOT}/include", f"{ROOT}/tests/cpp/dropin_scalar.cpp",
                    f"-L{ROOT}/paper_1911_11377_b200/lib", "-lhecnn_b200", f"-Wl,-rpath,{ROOT}/paper_1911_11377_b200/lib",
                    "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), str(tmp_path / "s.bin")], check=True, capture_output=True, text=True).stdout
    for line in out.splitlines():
        got, want = float(line.split()[2]), float(line.split()[4].rstrip(")"))
        assert abs(got - want) < 1e-5, line
    raw = (tmp_path / "s.bin").read_bytes()
    level = int(np.frombuffer(raw[:4], np.uint32)[0])
    scale = float(np.frombuffer(raw[4:12], np.float64)[0])
    n = 4096
    words = np.frombuffer(raw[12:], np.uint64).reshape(2, level + 1, n)

    p = hb.preset_params("nn-n4096-d8")
    r = ref.RefEngine.from_params(p).keygen(1)
    top = p.top_level
    v, u = [0.5, -0.25, 0.125, 1.0], [-0.75, 0.5, 0.25, -0.125]
    x, y = r.encrypt(v, seed=21), r.encrypt(u, seed=22)
    acc_scale = p.scale * p.scale
    acc = r.scalar_mac(np.zeros_like(x), x, top, acc_scale, p.scale, 0.3, p.scale)
    acc = r.scalar_mac(acc, y, top, acc_scale, p.scale, -1.25, p.scale, b=0.0625)
    z, zs = r.rescale(acc, top, acc_scale)
    w, wl, ws = r.plain_op(2, z, top - 1, zs, [0.5], p.scale, True)
    s, sl, ss = r.plain_op(0, w, wl, ws, v, ws, False)
    q = np.asarray(p.primes[: sl + 1], dtype=np.uint64)[None, :, None]
    doubled = (s + s) % q  # add_inplace(s, s); residues < 2^61, no overflow
    assert (level, scale) == (sl, ss)
    assert np.array_equal(words, doubled)
