"""Wire format on the device (CKKS blob v1, ckks_serialize.hpp): key and
ciphertext blobs are byte-identical to the reference's, and blobs written by
the reference load straight into device keys / tensors
(test_ckks.cpp:455-520 restated across the two implementations)."""
import numpy as np
import pytest

import paper_1911_11377_b200 as hb

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("preset", ["toy-n16", "nn-n4096-d8"])
def test_key_blobs_byte_identical_to_reference(ref, preset):
    """byte-identical serialization across engine instances (test_ckks.cpp:498-520)"""
    p = hb.preset_params(preset)
    eng = hb.CkksEngine(p).keygen(123)
    r = ref.RefEngine.from_params(p).keygen(123)
    assert hb.save_secret_key(eng) == r.save_key(1)
    assert hb.save_public_key(eng) == r.save_key(2)
    assert hb.save_evaluation_key(eng) == r.save_key(3)


def test_ciphertext_blobs_round_trip_through_both(ref):
    """Reference encrypts and saves; the device loads, squares and saves; the
    bytes equal the reference's own square -> save (scale bits included)."""
    p = hb.preset_params("nn-n4096-d8")
    r = ref.RefEngine.from_params(p).keygen(7)
    eng = hb.CkksEngine(p).keygen(7)
    cts = [r.encrypt(np.linspace(-1, 1, p.n // 2) * (k + 1) / 4, 50 + k) for k in range(3)]
    blobs = [r.save_ciphertext(c, p.top_level, p.scale) for c in cts]
    x = hb.load_ciphertexts(eng, blobs)
    assert (x.cells, x.level, x.scale) == (3, p.top_level, p.scale)
    assert np.array_equal(x.words(), np.stack(cts).reshape(x.words().shape))
    for k in range(3):
        assert hb.save_ciphertext(eng, x, k) == blobs[k]
    y = eng.square(x)
    for k in range(3):
        want, ws = r.square(cts[k], p.top_level, p.scale)
        assert hb.save_ciphertext(eng, y, k) == r.save_ciphertext(want, p.top_level - 1, ws)
        # and the reference reads our blob back word for word
        w, lv, sc = r.load_ciphertext(hb.save_ciphertext(eng, y, k))
        assert lv == p.top_level - 1 and sc == ws and np.array_equal(w.reshape(-1), want.reshape(-1))


def test_reference_keys_drive_the_device(ref):
    """A server context with only the reference's public and evaluation key
    blobs (no keygen on the device) evaluates bit-exactly."""
    p = hb.preset_params("nn-n4096-d8")
    r = ref.RefEngine.from_params(p).keygen(99)
    eng = hb.CkksEngine(p)
    hb.load_public_key(eng, r.save_key(2))
    hb.load_evaluation_key(eng, r.save_key(3))
    ct = r.encrypt(np.linspace(-0.5, 0.5, p.n // 2), 3)
    x = hb.load_ciphertext(eng, r.save_ciphertext(ct, p.top_level, p.scale))
    want, _ = r.square(ct, p.top_level, p.scale)
    assert np.array_equal(eng.square(x).words()[0], want)
    with pytest.raises(ValueError, match="no secret key"):
        hb.save_secret_key(eng)
    hb.load_secret_key(eng, r.save_key(1))
    assert hb.save_secret_key(eng) == r.save_key(1)


def test_blob_rejections(ref):
    p = hb.preset_params("toy-n16")
    r = ref.RefEngine.from_params(p).keygen(1)
    eng = hb.CkksEngine(p)
    with pytest.raises(RuntimeError, match="wrong object kind"):
        hb.load_public_key(eng, r.save_key(1))
    with pytest.raises(RuntimeError, match="bad magic"):
        hb.load_ciphertext(eng, b"nope")
    other = hb.preset_params("nn-n4096-d8")
    r2 = ref.RefEngine.from_params(other).keygen(1)
    with pytest.raises(ValueError, match="parameters differ"):
        hb.load_evaluation_key(eng, r2.save_key(3))
    ct = r.encrypt(np.linspace(-1, 1, p.n // 2), 5)
    top = r.save_ciphertext(ct, p.top_level, p.scale)
    lower, ls = r.rescale(ct, p.top_level, p.scale)
    with pytest.raises(ValueError, match="share level and scale"):
        hb.load_ciphertexts(eng, [top, r.save_ciphertext(lower, p.top_level - 1, ls)])


def test_blob_rejects_inconsistent_levels_and_unreduced_words(ref):
    """A header level below the polynomials' level must be rejected before any
    word is copied (the storage is sized by the header), and residues >= q_i
    are rejected instead of reaching the kernels unreduced."""
    p = hb.preset_params("toy-n16")
    r = ref.RefEngine.from_params(p).keygen(1)
    eng = hb.CkksEngine(p)
    ct = r.encrypt(np.linspace(-1, 1, p.n // 2), 5)
    top = bytearray(r.save_ciphertext(ct, p.top_level, p.scale))
    hdr = 4 + 2 + 2 + 4 + 2 + 8 * len(p.primes) + 8 + 8 + 1
    lvl_at = hdr + 8
    assert int.from_bytes(top[lvl_at:lvl_at + 2], "little") == p.top_level
    bad = bytearray(top)
    bad[lvl_at:lvl_at + 2] = (0).to_bytes(2, "little")
    with pytest.raises(ValueError, match="polynomial level exceeds"):
        hb.load_ciphertext(eng, bytes(bad))
    bad = bytearray(top)
    w0 = lvl_at + 2 + 2 + 1  # c0: level u16, rep u8, then the first residue of limb 0
    bad[w0:w0 + 8] = (p.primes[0]).to_bytes(8, "little")
    with pytest.raises(ValueError, match="not reduced"):
        hb.load_ciphertext(eng, bytes(bad))
    assert np.array_equal(hb.load_ciphertext(eng, bytes(top)).words()[0], ct)
