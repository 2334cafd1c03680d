"""Wire format (CKKS blob v1, ckks_serialize.hpp): the native codec's header
reader against blobs written by the reference itself, and the reference's
error texts for rejected blobs (test_ckks.cpp:489-495). Host-only: no GPU.
The device-side round trips are in test_gpu_blob.py."""
import numpy as np
import pytest

import paper_1911_11377_b200 as hb


@pytest.mark.parametrize("preset", ["toy-n16", "nn-n4096-d8"])
def test_header_of_reference_blobs(ref, preset):
    p = hb.preset_params(preset)
    r = ref.RefEngine.from_params(p).keygen(123)
    blobs = {hb.BLOB_SECRET_KEY: r.save_key(1), hb.BLOB_PUBLIC_KEY: r.save_key(2), hb.BLOB_EVAL_KEY: r.save_key(3),
             hb.BLOB_CIPHERTEXT: r.save_ciphertext(r.encrypt(np.linspace(-1, 1, p.n // 2), 5), p.top_level, p.scale)}
    for kind, b in blobs.items():
        k, q = hb.blob_params(b)
        assert k == kind
        assert (q.n, q.primes, q.scale, q.sigma, q.degenerate_noise) == (p.n, p.primes, p.scale, p.sigma, False)


def test_rejected_blobs_carry_the_reference_errors(ref):
    p = hb.preset_params("toy-n16")
    r = ref.RefEngine.from_params(p).keygen(1)
    good = r.save_key(1)
    cases = [b"nope", b"CKKS\x02\x00" + good[6:], good[:9]]
    for bad in cases:
        with pytest.raises(RuntimeError) as ours:
            hb.blob_params(bad)
        with pytest.raises(RuntimeError) as theirs:
            ref.RefEngine.load_key_check(bad, 1)
        assert str(ours.value) == str(theirs.value)
