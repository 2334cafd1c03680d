"""CPU: the command-line front end's readers of the reference's file formats
(paper_1911_11377_b200/cli.py) against files the reference itself writes --
model manifests + weight blobs (model_io.hpp), HDTS datasets (synthetic.hpp)
-- the numpy plain forward against the reference's forward_plain, the seed
derivation against splitmix64, and the reference's rejection texts for
malformed model files. The encrypted `infer` path is in test_gpu_cli.py."""
import json
import os

import numpy as np
import pytest

import paper_1911_11377_b200 as hb
from paper_1911_11377_b200 import cli


def tiny_model(ref, seed=5):
    spec = hb.ModelSpec(hb.Shape.spatial(8, 8, 3))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.zero_pad2d(1), hb.LayerSpec.conv2d(4, 3, 3, stride=2, valid=True),
                   hb.LayerSpec.activation("relu-poly2"), hb.LayerSpec.avg_pool2d(2), hb.LayerSpec.conv2d(3, 3, 3),
                   hb.LayerSpec.dense(2), hb.LayerSpec.dense(1), hb.LayerSpec.sigmoid()]
    return ref.init_random_weights(spec, seed)


def test_reads_reference_model_and_dataset(ref, tmp_path):
    spec = tiny_model(ref)
    base = str(tmp_path / "m")
    ref.save_model(spec, base)
    ref.save_dataset(16, 8, 3, 7, str(tmp_path / "d.bin"))
    m, scale = cli.load_model(base)
    assert [l.kind for l in m.layers] == [l.kind for l in spec.layers]
    for a, b in zip(m.weights, spec.weights):
        assert (a is None and b is None) or np.array_equal(a, b)
    assert scale == [1.0, 1.0, 1.0]
    images, labels, shape = cli.load_dataset(str(tmp_path / "d.bin"))
    want, want_labels = ref.gen_synthetic(16, 8, 3, 7)
    assert (shape.h, shape.w, shape.c) == (8, 8, 3)
    assert np.array_equal(images, want) and np.array_equal(labels, want_labels)
    # the numpy plain forward is the reference's forward_plain up to summation order
    got = cli.forward_plain(m, images)
    assert np.max(np.abs(got - ref.forward_plain(spec, images))) < 1e-12


def test_model_file_rejections_match_reference(ref, tmp_path):
    spec = tiny_model(ref)
    base = str(tmp_path / "m")
    ref.save_model(spec, base)
    with open(base + ".weights.bin", "ab") as f:
        f.write(b"\0" * 8)
    for err in (RuntimeError,):
        with pytest.raises(err, match="weight blob length disagrees with architecture"):
            cli.load_model(base)
        with pytest.raises(RuntimeError, match="weight blob length disagrees with architecture"):
            ref.load_model_check(base)
    ref.save_model(spec, base)
    j = json.load(open(base + ".json"))
    j["format_version"] = 2
    json.dump(j, open(base + ".json", "w"))
    with pytest.raises(RuntimeError, match="unsupported model format version"):
        cli.load_model(base)
    with pytest.raises(RuntimeError, match="unsupported model format version"):
        ref.load_model_check(base)


def test_derive_seed_is_the_reference_splitmix():
    # splitmix64 known value (seed 0) and CkksEngine::derive_seed composition
    assert hb.splitmix64(0) == 0xE220A8397B1DCDAF
    assert hb.derive_seed(5, 0xF000) == hb.splitmix64(5 ^ hb.splitmix64(0xF000))


def test_usage_errors_exit_2(tmp_path):
    assert cli.main(["infer", "--model", "x"]) == 2  # missing required options
    base = str(tmp_path / "nope")
    assert cli.main(["infer", "--model", base, "--data", base, "--out", str(tmp_path / "o.csv")]) == 3
