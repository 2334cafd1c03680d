"""GPU: whole BASELINE configs word for word against the reference (SURVEY
§8(d)): C3 (CryptoNets-style, 28x28x1) and C4 (CIFAR-shaped with the degree-2
ReLU surrogate, 32x32x3), each on a full set of 4096 encrypted synthetic
images at net-n8192-d8 -- the same inputs, keys and seeds on both sides, the
reference running on every host core. C4's reference pass takes about a
minute on a 16-core host."""
import os

import numpy as np
import pytest

import bench
import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config", ["c3", "c4"])
def test_full_config_matches_reference(ref, config):
    p = hb.preset_params("net-n8192-d8")
    spec = bench.c3_spec(hb) if config == "c3" else bench.c4_spec(hb)
    threads = os.cpu_count() or 1
    data = np.random.default_rng(3).uniform(0, 1, size=(p.n // 2, spec.input.positions()))
    eng = hb.CkksEngine(p).keygen(1)
    y = hb.forward_encrypted(spec, eng.encrypt_tensor(data, seed=11, shape=spec.input), eng, seed=13)
    r = ref.RefEngine.from_params(p).keygen(1)
    ry, _ = r.forward_encrypted(spec, r.encrypt_tensor(data, spec.input, seed=11, threads=threads), seed=13,
                                threads=threads)
    assert (y.level, y.scale) == ry.info()[1:]
    assert np.array_equal(y.words(), ry.words())
    # and the decrypted logits agree with the plain model within the reference's tolerance
    plain = ref.forward_plain(spec, data[:64])
    dec = eng.decrypt_tensor(y, p.n // 2)[:64]
    assert np.max(np.abs(dec - plain)) < 1e-2
