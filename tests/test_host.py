"""CPU: host logic of the product -- chain search, presets, model specs,
encoder/decoder and samplers (which must stay bit-identical to the
reference's libm / long-double / mt19937_64 behaviour), the C-ABI symbol
table, and loud failure without a GPU."""
import json
import os
import re

import numpy as np
import pytest

import paper_1911_11377_b200 as hb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.mark.parametrize("preset", [p.name for p in hb.builtin_presets()])
def test_chain_matches_reference_golden(preset):
    d = hb.find_preset(preset)
    assert hb.find_chain(d.n, d.prime_bits) == [int(v) for v in G[f"chain_{preset}"]]


def test_chain_errors():
    with pytest.raises(ValueError, match="bit_size out of range"):
        hb.find_chain(16, [61])
    with pytest.raises(ValueError, match="power of two"):
        hb.find_chain(12, [40])


def test_presets_json_shadowing(tmp_path):
    f = tmp_path / "p.json"
    f.write_text(json.dumps({"presets": [{"name": "toy-n16", "n": 32, "prime_bits": [40, 30], "log2_scale": 25}]}))
    d = hb.find_preset("toy-n16", str(f))
    assert d.n == 32 and d.prime_bits == [40, 30] and d.sigma == 3.2
    assert hb.find_preset("net-n8192-d8", str(f)).n == 8192
    with pytest.raises(ValueError, match="unknown parameter preset"):
        hb.find_preset("nope")


def test_alexnet_shapes_and_depth():
    """test_nn.cpp:34-48 and :77-85"""
    m = hb.alexnet32_preset()
    s = m.shapes()
    assert len(s) == 21
    assert s[0] == hb.Shape.spatial(32, 32, 96) and s[2] == hb.Shape.spatial(16, 16, 96)
    assert s[5] == hb.Shape.spatial(8, 8, 256) and s[6] == hb.Shape.spatial(10, 10, 256)
    assert s[9] == hb.Shape.spatial(5, 5, 384) and s[14] == hb.Shape.spatial(4, 4, 384)
    assert s[15] == hb.Shape.flattened(4096) and s[19] == hb.Shape.flattened(1)
    assert m.depth_cost() == 23


def test_encode_decode_match_reference_golden():
    p = hb.CkksParams(256, [int(v) for v in G["r256_primes"]], 2.0 ** 40)
    enc = hb.host_encode_real(p, G["r256_vals"], 3)
    assert np.array_equal(enc, G["r256_encode"])
    dec = hb.host_decode_real(p, G["r256_encode"], 3, p.scale)
    assert np.array_equal(dec, G["r256_decode"])


def test_encryption_randomness_matches_reference_golden():
    p = hb.CkksParams(256, [int(v) for v in G["r256_primes"]], 2.0 ** 40)
    r, e0, e1 = hb.host_encryption_randomness(p, 123)
    assert np.array_equal(r, G["r256_rand_r"]) and np.array_equal(e0, G["r256_rand_e0"])
    assert np.array_equal(e1, G["r256_rand_e1"])
    assert set(np.unique(r)) <= {-1, 0, 1} and np.abs(e0).max() <= 19


def test_encode_errors():
    p = hb.CkksParams(256, [int(v) for v in G["r256_primes"]], 2.0 ** 40)
    with pytest.raises(ValueError, match="vector longer than slot count"):
        hb.host_encode_real(p, np.zeros(129), 3)
    with pytest.raises(ValueError, match="overflow the active modulus"):
        hb.host_encode_real(p, np.ones(4), 0, scale=2.0 ** 58)


def test_host_numerics_against_live_reference(ref):
    rng = np.random.default_rng(9)
    for preset in ("test-n4096-d4", "net-n8192-d8"):
        p = hb.preset_params(preset)
        r = ref.RefEngine.from_params(p)
        v = rng.uniform(-2, 2, p.n // 2)
        for level in (p.top_level, 1):
            e = hb.host_encode_real(p, v, level)
            assert np.array_equal(e, r.encode(v, level))
            assert np.array_equal(hb.host_decode_real(p, e, level, p.scale), r.decode(e, level, p.scale))
        for seed in (1, 2 ** 63 + 5):
            assert all(np.array_equal(a, b) for a, b in zip(hb.host_encryption_randomness(p, seed),
                                                             r.encryption_randomness(seed)))


def test_capi_exports_every_declared_symbol():
    """The C-ABI library loads and exports exactly the symbols include/hecnn_b200.h declares."""
    hdr = open(os.path.join(ROOT, "include", "hecnn_b200.h")).read()
    declared = set(re.findall(r"\b(?:int|const char\*)\s+(hecnn_\w+)\s*\(", hdr))
    assert declared == set(hb.EXPORTED_SYMBOLS)
    L = hb.lib()
    for name in declared:
        assert hasattr(L, name), name
    import subprocess
    nm = subprocess.run(["nm", "-D", "--defined-only", hb.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in nm.splitlines() if " T " in ln}
    assert exported == declared


def test_no_silent_cpu_fallback():
    """Without a usable GPU the engine refuses loudly instead of computing on the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="CUDA"):
        hb.CkksEngine(hb.preset_params("toy-n16"))


def test_dropin_header_compiles():
    """The C++ drop-in header (include/hecnn_b200/hecnn.hpp) and both sample
    programs written against it compile (syntax only: no GPU, no link)."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for src in ("dropin_inference.cpp", "dropin_scalar.cpp"):
        subprocess.run(["g++", "-std=c++20", "-fsyntax-only", f"-I{root}/include", f"{root}/tests/cpp/{src}"], check=True)
