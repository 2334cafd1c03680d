"""GPU: the command-line front end (paper_1911_11377_b200/cli.py) end to end
on files written by the reference: `keygen` writes key blobs byte-identical
to the reference's, and `infer --mode encrypted` on a reference model,
dataset and key directory writes the reference's CSV with logits equal (to
the last bit) to the reference's own encrypted inference with the same seeds
(hecnn_cli.cpp:173-234: encrypt with derive_seed(seed, begin), forward with
derive_seed(seed, 0xf000 + begin))."""
import csv
import os

import numpy as np
import pytest

import paper_1911_11377_b200 as hb
from paper_1911_11377_b200 import cli

pytestmark = pytest.mark.gpu


def test_keygen_writes_the_reference_blobs(ref, tmp_path):
    assert cli.main(["keygen", "--preset", "toy-n16", "--seed", "9", "--out", str(tmp_path)]) == 0
    r = ref.RefEngine.from_params(hb.preset_params("toy-n16")).keygen(9)
    for name, kind in (("sk.bin", 1), ("pk.bin", 2), ("evk.bin", 3)):
        assert open(tmp_path / name, "rb").read() == r.save_key(kind)
    assert cli.main(["keygen", "--preset", "toy-n16", "--out", str(tmp_path)]) == 2  # no --force


def test_encrypted_infer_matches_reference(ref, tmp_path):
    preset = "nn-n4096-d8"
    p = hb.preset_params(preset)
    spec = hb.ModelSpec(hb.Shape.spatial(8, 8, 3))
    spec.activations["relu-poly2"] = hb.relu_default_surrogate()
    spec.layers = [hb.LayerSpec.conv2d(4, 3, 3), hb.LayerSpec.activation("relu-poly2"), hb.LayerSpec.avg_pool2d(2),
                   hb.LayerSpec.dense(1), hb.LayerSpec.sigmoid()]
    spec = ref.init_random_weights(spec, 3)
    base, data, keys = str(tmp_path / "m"), str(tmp_path / "d.bin"), tmp_path / "keys"
    ref.save_model(spec, base)
    ref.save_dataset(12, 8, 3, 5, data)
    os.makedirs(keys)
    r = ref.RefEngine.from_params(p).keygen(4)
    for name, kind in (("sk.bin", 1), ("pk.bin", 2), ("evk.bin", 3)):
        open(keys / name, "wb").write(r.save_key(kind))
    out = str(tmp_path / "preds.csv")
    rc = cli.main(["infer", "--mode", "encrypted", "--preset", preset, "--keys", str(keys), "--model", base,
                   "--data", data, "--batch", "5", "--seed", "21", "--out", out])
    assert rc == 0
    rows = list(csv.DictReader(open(out)))
    assert [int(x["id"]) for x in rows] == list(range(12))
    # the reference's own path with the same seeds, batch by batch
    images, labels, shape = cli.load_dataset(data)
    logits_spec = hb.ModelSpec(spec.input, spec.layers[:-1], spec.activations, spec.weights[:-1], spec.biases[:-1])
    want = []
    for begin in range(0, 12, 5):
        x = images[begin:begin + 5]
        rx = r.encrypt_tensor(x, spec.input, seed=hb.derive_seed(21, begin))
        ry, _ = r.forward_encrypted(logits_spec, rx, seed=hb.derive_seed(21, 0xF000 + begin))
        want.extend(r.decrypt_tensor(ry, x.shape[0])[:, 0])
    got = [float(x["logit"]) for x in rows]
    assert got == [float(f"{v:.17g}") for v in want]
    assert [int(x["label"]) for x in rows] == [1 if v > 0 else 0 for v in want]
