"""TEST INFRASTRUCTURE ONLY -- parity checker, never the product.

ctypes wrapper of oracle/_ref/libhecnn_ref.so: the UNMODIFIED reference
library (hecnn, /root/reference/proj/include) compiled by oracle/Makefile
behind oracle/ref_driver.cpp. Only tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg, --impl reference) may import this module.
"""
from __future__ import annotations

import ctypes
import os
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_LIB = os.path.join(HERE, "_ref", "libhecnn_ref.so")

_lib = None
_u64p = ctypes.POINTER(ctypes.c_uint64)
_dblp = ctypes.POINTER(ctypes.c_double)


def available() -> bool:
    return os.path.exists(REF_LIB)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {REF_LIB} (make -C oracle ref)")
        _lib = ctypes.CDLL(REF_LIB)
        _lib.ref_last_error.restype = ctypes.c_char_p
        _lib.ref_eval_key_digits.restype = ctypes.c_size_t
    return _lib


def _check(st: int):
    if st == 0:
        return
    msg = lib().ref_last_error().decode()
    if st == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def _p(a, t=ctypes.c_uint64):
    return a.ctypes.data_as(ctypes.POINTER(t))


def find_chain(n: int, bits: Sequence[int]) -> List[int]:
    b = (ctypes.c_int * len(bits))(*bits)
    out = np.zeros(len(bits), dtype=np.uint64)
    _check(lib().ref_find_chain(ctypes.c_size_t(n), b, ctypes.c_size_t(len(bits)), _p(out)))
    return [int(v) for v in out]


class RefEngine:
    """CkksEngine of the reference (ckks.hpp:77)."""

    def __init__(self, n: int, primes: Sequence[int], scale: float, sigma: float = 3.2, degenerate: bool = False):
        self.n = n
        self.primes = [int(p) for p in primes]
        self.scale = scale
        pr = np.asarray(self.primes, dtype=np.uint64)
        h = ctypes.c_void_p()
        _check(lib().ref_engine_create(ctypes.c_size_t(n), _p(pr), ctypes.c_size_t(len(pr)), ctypes.c_double(scale),
                                       ctypes.c_double(sigma), int(degenerate), ctypes.byref(h)))
        self.h = h
        self.keys = None

    @staticmethod
    def from_params(p) -> "RefEngine":
        return RefEngine(p.n, p.primes, p.scale, p.sigma, p.degenerate_noise)

    def __del__(self):
        if getattr(self, "keys", None) is not None and _lib is not None:
            _lib.ref_keys_destroy(self.keys)
            self.keys = None
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_engine_destroy(self.h)
            self.h = None

    @property
    def top(self) -> int:
        return len(self.primes) - 1

    def relin_digits(self, level: int) -> int:
        d = ctypes.c_size_t()
        _check(lib().ref_relin_digits(self.h, ctypes.c_size_t(level), ctypes.byref(d)))
        return d.value

    def ntt_forward(self, limb: int, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        _check(lib().ref_ntt_forward(self.h, ctypes.c_size_t(limb), _p(a)))
        return a

    def ntt_inverse(self, limb: int, a: np.ndarray) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        _check(lib().ref_ntt_inverse(self.h, ctypes.c_size_t(limb), _p(a)))
        return a

    def sample_uniform(self, level: int, seed: int) -> np.ndarray:
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        _check(lib().ref_sample_uniform(self.h, ctypes.c_size_t(level), ctypes.c_uint64(seed), _p(out)))
        return out

    def rescale_poly(self, poly: np.ndarray, level: int) -> np.ndarray:
        poly = np.ascontiguousarray(poly, dtype=np.uint64)
        out = np.empty((level, self.n), dtype=np.uint64)
        _check(lib().ref_rescale_poly(self.h, _p(poly), ctypes.c_size_t(level), _p(out)))
        return out

    def reconstruct(self, poly: np.ndarray, level: int, words: int) -> np.ndarray:
        poly = np.ascontiguousarray(poly, dtype=np.uint64)
        out = np.empty((self.n, words), dtype=np.uint64)
        _check(lib().ref_reconstruct(self.h, _p(poly), ctypes.c_size_t(level), ctypes.c_size_t(words), _p(out)))
        return out

    def keygen(self, seed: int) -> "RefEngine":
        h = ctypes.c_void_p()
        _check(lib().ref_keygen(self.h, ctypes.c_uint64(seed), ctypes.byref(h)))
        if self.keys is not None:
            lib().ref_keys_destroy(self.keys)
        self.keys = h
        return self

    def export_keys(self):
        L = self.top + 1
        D = lib().ref_eval_key_digits(self.keys)
        s = np.empty((L, self.n), dtype=np.uint64)
        b = np.empty((L, self.n), dtype=np.uint64)
        a = np.empty((L, self.n), dtype=np.uint64)
        evk = np.empty((D, 2, L, self.n), dtype=np.uint64)
        lib().ref_export_keys(self.keys, _p(s), _p(b), _p(a), _p(evk))
        return s, b, a, evk

    # ---- ckks_serialize.hpp (blob v1), the reference's own writer/reader
    def save_key(self, kind: int) -> bytes:
        """save_secret_key / save_public_key / save_evaluation_key (kind 1/2/3)."""
        n = ctypes.c_size_t()
        _check(lib().ref_save_key(self.h, self.keys, int(kind), None, ctypes.c_size_t(0), ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().ref_save_key(self.h, self.keys, int(kind), buf, n, ctypes.byref(n)))
        return buf.raw[:n.value]

    def save_ciphertext(self, ct: np.ndarray, level: int, scale: float) -> bytes:
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        n = ctypes.c_size_t()
        args = (self.h, _p(ct), ctypes.c_size_t(level), ctypes.c_double(scale))
        _check(lib().ref_save_ciphertext(*args, None, ctypes.c_size_t(0), ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value)
        _check(lib().ref_save_ciphertext(*args, buf, n, ctypes.byref(n)))
        return buf.raw[:n.value]

    def load_ciphertext(self, blob: bytes):
        """load_ciphertext: (words [2][level+1][n], level, scale)."""
        out = np.empty(2 * (self.top + 1) * self.n, dtype=np.uint64)
        lv, sc = ctypes.c_uint32(), ctypes.c_double()
        _check(lib().ref_load_ciphertext(blob, ctypes.c_size_t(len(blob)), _p(out), ctypes.c_size_t(out.size),
                                         ctypes.byref(lv), ctypes.byref(sc)))
        return out[:2 * (lv.value + 1) * self.n].reshape(2, lv.value + 1, self.n), lv.value, sc.value

    @staticmethod
    def load_key_check(blob: bytes, kind: int):
        """Runs the reference's load_*_key; raises its error for a rejected blob."""
        _check(lib().ref_load_key_check(blob, ctypes.c_size_t(len(blob)), int(kind)))

    def encrypt(self, slots, seed: int, scale: Optional[float] = None) -> np.ndarray:
        v = np.ascontiguousarray(slots, dtype=np.float64)
        out = np.empty((2, self.top + 1, self.n), dtype=np.uint64)
        _check(lib().ref_encrypt(self.h, self.keys, _p(v, ctypes.c_double), ctypes.c_size_t(v.size),
                                 ctypes.c_double(scale or self.scale), ctypes.c_uint64(seed), _p(out)))
        return out

    def encode(self, slots, level: int, scale: Optional[float] = None) -> np.ndarray:
        v = np.ascontiguousarray(slots, dtype=np.float64)
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        _check(lib().ref_encode(self.h, _p(v, ctypes.c_double), ctypes.c_size_t(v.size),
                                ctypes.c_double(scale or self.scale), ctypes.c_size_t(level), _p(out)))
        return out

    def decode(self, poly: np.ndarray, level: int, scale: float) -> np.ndarray:
        poly = np.ascontiguousarray(poly, dtype=np.uint64)
        out = np.empty(self.n // 2, dtype=np.float64)
        _check(lib().ref_decode(self.h, _p(poly), ctypes.c_size_t(level), ctypes.c_double(scale),
                                _p(out, ctypes.c_double)))
        return out

    def encryption_randomness(self, seed: int):
        r, e0, e1 = (np.empty(self.n, dtype=np.int64) for _ in range(3))
        _check(lib().ref_encryption_randomness(self.h, ctypes.c_uint64(seed), _p(r, ctypes.c_int64),
                                               _p(e0, ctypes.c_int64), _p(e1, ctypes.c_int64)))
        return r, e0, e1

    def decrypt(self, ct: np.ndarray, level: int, scale: float) -> np.ndarray:
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.empty(self.n // 2, dtype=np.float64)
        _check(lib().ref_decrypt(self.h, self.keys, _p(ct), ctypes.c_size_t(level), ctypes.c_double(scale),
                                 _p(out, ctypes.c_double)))
        return out

    def decrypt_raw(self, ct: np.ndarray, level: int, scale: float) -> np.ndarray:
        ct = np.ascontiguousarray(ct, dtype=np.uint64)
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        _check(lib().ref_decrypt_raw(self.h, self.keys, _p(ct), ctypes.c_size_t(level), ctypes.c_double(scale),
                                     _p(out)))
        return out

    def mul(self, x, y, level: int, sx: float, sy: float):
        x, y = (np.ascontiguousarray(v, dtype=np.uint64) for v in (x, y))
        out = np.empty((2, level, self.n), dtype=np.uint64)
        s = ctypes.c_double()
        _check(lib().ref_mul(self.h, self.keys, _p(x), _p(y), ctypes.c_size_t(level), ctypes.c_double(sx),
                             ctypes.c_double(sy), _p(out), ctypes.byref(s)))
        return out, s.value

    def square(self, x, level: int, sx: float):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty((2, level, self.n), dtype=np.uint64)
        s = ctypes.c_double()
        _check(lib().ref_square(self.h, self.keys, _p(x), ctypes.c_size_t(level), ctypes.c_double(sx), _p(out),
                                ctypes.byref(s)))
        return out, s.value

    def rescale(self, x, level: int, sx: float):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty((2, level, self.n), dtype=np.uint64)
        s = ctypes.c_double()
        _check(lib().ref_rescale(self.h, _p(x), ctypes.c_size_t(level), ctypes.c_double(sx), _p(out),
                                 ctypes.byref(s)))
        return out, s.value

    def mul_const(self, x, level: int, sx: float, c: float, cscale: float):
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty((2, level, self.n), dtype=np.uint64)
        s = ctypes.c_double()
        _check(lib().ref_mul_const(self.h, _p(x), ctypes.c_size_t(level), ctypes.c_double(sx), ctypes.c_double(c),
                                   ctypes.c_double(cscale), _p(out), ctypes.byref(s)))
        return out, s.value

    def scalar_plain(self, c: float, scale: float, level: int) -> np.ndarray:
        out = np.empty(level + 1, dtype=np.uint64)
        _check(lib().ref_scalar_plain(self.h, ctypes.c_double(c), ctypes.c_double(scale), ctypes.c_size_t(level),
                                      _p(out)))
        return out

    def scalar_mac(self, acc, x, level: int, acc_scale: float, sx: float, c: float, cscale: float, b=None):
        acc = np.ascontiguousarray(acc, dtype=np.uint64)
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty((2, level + 1, self.n), dtype=np.uint64)
        _check(lib().ref_scalar_mac(self.h, _p(acc), _p(x), ctypes.c_size_t(level), ctypes.c_double(acc_scale),
                                    ctypes.c_double(sx), ctypes.c_double(c), ctypes.c_double(cscale),
                                    ctypes.c_int(b is not None), ctypes.c_double(b or 0.0), _p(out)))
        return out

    def plain_op(self, op: int, x, level: int, sx: float, slots, pscale: float, constant: bool):
        """op 0 add_plain, 1 mul_plain_raw, 2 mul_plain with encode_real(slots) or encode_const(slots[0])."""
        x = np.ascontiguousarray(x, dtype=np.uint64)
        v = np.ascontiguousarray(slots, dtype=np.float64)
        out = np.empty(2 * (level + 1) * self.n, dtype=np.uint64)
        lv = ctypes.c_uint32()
        s = ctypes.c_double()
        _check(lib().ref_plain_op(self.h, ctypes.c_int(op), _p(x), ctypes.c_size_t(level), ctypes.c_double(sx),
                                  _p(v, ctypes.c_double), ctypes.c_size_t(v.size), ctypes.c_double(pscale),
                                  ctypes.c_int(constant), _p(out), ctypes.byref(lv), ctypes.byref(s)))
        k = lv.value + 1
        return out[: 2 * k * self.n].reshape(2, k, self.n).copy(), lv.value, s.value

    def eval_activation(self, coeffs, bound: float, x, level: int, sx: float):
        c = np.ascontiguousarray(coeffs, dtype=np.float64)
        x = np.ascontiguousarray(x, dtype=np.uint64)
        out = np.empty(2 * (level + 1) * self.n, dtype=np.uint64)
        lv = ctypes.c_uint32()
        s = ctypes.c_double()
        _check(lib().ref_eval_activation(self.h, self.keys, _p(c, ctypes.c_double), ctypes.c_size_t(c.size),
                                          ctypes.c_double(bound), _p(x), ctypes.c_size_t(level), ctypes.c_double(sx),
                                          _p(out), ctypes.byref(lv), ctypes.byref(s)))
        k = lv.value + 1
        return out[: 2 * k * self.n].reshape(2, k, self.n).copy(), lv.value, s.value

    # ---- tensors / network
    def encrypt_tensor(self, data: np.ndarray, shape, seed: int, threads: int = 1) -> "RefTensor":
        data = np.ascontiguousarray(data, dtype=np.float64)
        batch = data.shape[0]
        h = ctypes.c_void_p()
        _check(lib().ref_encrypt_tensor(self.h, self.keys, _p(data, ctypes.c_double), ctypes.c_size_t(batch),
                                        int(shape.flat), ctypes.c_size_t(shape.h), ctypes.c_size_t(shape.w),
                                        ctypes.c_size_t(shape.c), ctypes.c_size_t(shape.feat), ctypes.c_uint64(seed),
                                        ctypes.c_uint(threads), ctypes.byref(h)))
        return RefTensor(self, h)

    def tensor_from(self, words: np.ndarray, level: int, scale: float, shape, batch: int) -> "RefTensor":
        words = np.ascontiguousarray(words, dtype=np.uint64)
        cells = words.size // (2 * (level + 1) * self.n)
        h = ctypes.c_void_p()
        _check(lib().ref_tensor_from(self.h, _p(words), ctypes.c_size_t(cells), ctypes.c_size_t(level),
                                     ctypes.c_double(scale), int(shape.flat), ctypes.c_size_t(shape.h),
                                     ctypes.c_size_t(shape.w), ctypes.c_size_t(shape.c), ctypes.c_size_t(shape.feat),
                                     ctypes.c_size_t(batch), ctypes.byref(h)))
        return RefTensor(self, h)

    def forward_encrypted(self, model_spec, x: "RefTensor", seed: int, threads: int = 1):
        desc, keep = model_spec.to_desc()
        h = ctypes.c_void_p()
        secs = np.zeros(max(len(model_spec.layers), 1), dtype=np.float64)
        _check(lib().ref_forward_encrypted(self.h, self.keys, ctypes.byref(desc), x.h, ctypes.c_uint64(seed),
                                           ctypes.c_uint(threads), ctypes.byref(h), _p(secs, ctypes.c_double)))
        return RefTensor(self, h), secs[: len(model_spec.layers)]

    def decrypt_tensor(self, t: "RefTensor", batch: int, threads: int = 1) -> np.ndarray:
        cells, _, _ = t.info()
        out = np.empty((batch, cells), dtype=np.float64)
        _check(lib().ref_decrypt_tensor(self.h, self.keys, t.h, ctypes.c_uint(threads), _p(out, ctypes.c_double)))
        return out

    def time_ntt(self, level: int, count: int, threads: int) -> float:
        s = ctypes.c_double()
        _check(lib().ref_time_ntt(self.h, ctypes.c_size_t(level), ctypes.c_size_t(count), ctypes.c_uint(threads),
                                  ctypes.byref(s)))
        return s.value

    def time_layer_op(self, op: int, level: int, count: int, inner: int, threads: int) -> float:
        """Seconds for `count` independent items of a reference layer op over its
        parallel_for (0: relu-poly2 eval_encrypted, 1: one conv/dense output with
        `inner` scalar MACs + bias + rescale, 2: one zero-pad border encryption)."""
        s = ctypes.c_double()
        _check(lib().ref_time_layer_op(self.h, self.keys, int(op), ctypes.c_size_t(level), ctypes.c_size_t(count),
                                       ctypes.c_size_t(inner), ctypes.c_uint(threads), ctypes.byref(s)))
        return s.value

    def time_mul(self, level: int, count: int, threads: int) -> float:
        s = ctypes.c_double()
        _check(lib().ref_time_mul(self.h, self.keys, ctypes.c_size_t(level), ctypes.c_size_t(count),
                                  ctypes.c_uint(threads), ctypes.byref(s)))
        return s.value


class RefTensor:
    def __init__(self, eng: RefEngine, h):
        self.eng = eng
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_tensor_destroy(self.h)
            self.h = None

    def info(self):
        cells, level, scale = ctypes.c_size_t(), ctypes.c_uint32(), ctypes.c_double()
        lib().ref_tensor_info(self.h, ctypes.byref(cells), ctypes.byref(level), ctypes.byref(scale))
        return cells.value, level.value, scale.value

    def words(self) -> np.ndarray:
        cells, level, _ = self.info()
        out = np.empty((cells, 2, level + 1, self.eng.n), dtype=np.uint64)
        lib().ref_tensor_export(self.eng.h, self.h, _p(out))
        return out


def forward_plain(model_spec, data: np.ndarray) -> np.ndarray:
    desc, keep = model_spec.to_desc()
    data = np.ascontiguousarray(data, dtype=np.float64)
    outs = model_spec.shapes()[-1].positions() if model_spec.layers else model_spec.input.positions()
    out = np.empty((data.shape[0], outs), dtype=np.float64)
    _check(lib().ref_forward_plain(ctypes.byref(desc), _p(data, ctypes.c_double), ctypes.c_size_t(data.shape[0]),
                                   _p(out, ctypes.c_double)))
    return out


def save_model(model_spec, base: str):
    """The reference's save_model (model_io.hpp:61-103) of a model spec."""
    desc, keep = model_spec.to_desc()
    _check(lib().ref_save_model(ctypes.byref(desc), base.encode()))


def save_dataset(count: int, image: int, channels: int, seed: int, path: str):
    """The reference's gen_synthetic + save_dataset (an HDTS file)."""
    _check(lib().ref_save_dataset(ctypes.c_size_t(count), ctypes.c_size_t(image), ctypes.c_size_t(channels),
                                  ctypes.c_uint64(seed), path.encode()))


def load_model_check(base: str):
    """Runs the reference's load_model on `base`; raises its error if rejected."""
    _check(lib().ref_load_model_weights(base.encode(), None, None, ctypes.c_size_t(0)))


def rng_uniform(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.float64)
    _check(lib().ref_rng_uniform(ctypes.c_uint64(seed), ctypes.c_size_t(count), _p(out, ctypes.c_double)))
    return out


def gen_synthetic(count: int, image: int, channels: int, seed: int):
    imgs = np.empty((count, image * image * channels), dtype=np.float64)
    labels = np.empty(count, dtype=np.uint8)
    _check(lib().ref_gen_synthetic(ctypes.c_size_t(count), ctypes.c_size_t(image), ctypes.c_size_t(channels),
                                   ctypes.c_uint64(seed), _p(imgs, ctypes.c_double), _p(labels, ctypes.c_uint8)))
    return imgs, labels


def init_random_weights(model_spec, seed: int):
    """init_random_weights (model_io.hpp:183-203) into model_spec.weights/biases."""
    model_spec.ensure_param_slots()
    counts = model_spec.param_counts()
    ws, bs = [], []
    wp = (ctypes.POINTER(ctypes.c_double) * len(model_spec.layers))()
    bp = (ctypes.POINTER(ctypes.c_double) * len(model_spec.layers))()
    for i, (wc, bc) in enumerate(counts):
        w = np.zeros(wc, dtype=np.float64) if wc else None
        b = np.zeros(bc, dtype=np.float64) if bc else None
        ws.append(w)
        bs.append(b)
        # the reference sizes weights itself; the driver copies into our buffers
        model_spec.weights[i] = w
        model_spec.biases[i] = b
        wp[i] = _p(w, ctypes.c_double) if w is not None else None
        bp[i] = _p(b, ctypes.c_double) if b is not None else None
    # the desc carries zero-filled buffers of the right size (validated shapes)
    desc, keep = model_spec.to_desc()
    _check(lib().ref_init_random_weights(ctypes.byref(desc), ctypes.c_uint64(seed), wp, bp))
    return model_spec
