"""B200-native CKKS evaluation engine for the encrypted-CNN hot path of the
reference library ``hecnn`` (arXiv 1911.11377).

This module is a thin ctypes binding of the C-ABI in ``include/hecnn_b200.h``
(shared library ``lib/libhecnn_b200.so``: sm_100a kernels + C++ host engine).
Names and argument meaning follow the reference's C++ API
(``proj/include/hecnn``): ``CkksEngine`` (ckks.hpp:77), ``encrypt_tensor`` /
``decrypt_tensor`` (tensor.hpp:77-106), ``forward_encrypted``
(layers.hpp:299), ``eval_encrypted`` (activation.hpp:228), ``LayerSpec`` /
``ModelSpec`` (model.hpp:12-97) and the presets (presets.hpp:33-49).
Errors: the reference's ``std::invalid_argument`` surfaces as ``ValueError``
and ``std::runtime_error`` as ``RuntimeError``, with the reference's text.

There is no CPU fallback: importing works without a GPU, but every call that
reaches the device fails loudly when the extension or the GPU is missing.
"""
from __future__ import annotations

import ctypes
import json
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HECNN_B200_LIB") or os.path.join(_HERE, "lib", "libhecnn_b200.so")

HECNN_OK, HECNN_EINVAL, HECNN_ERUNTIME, HECNN_ECUDA = 0, 1, 2, 3

# C-ABI symbols declared in include/hecnn_b200.h (checked by tests/test_capi.py)
EXPORTED_SYMBOLS = (
    "hecnn_last_error", "hecnn_abi_version", "hecnn_find_chain", "hecnn_context_create",
    "hecnn_context_destroy", "hecnn_context_set_stream", "hecnn_context_synchronize", "hecnn_context_info",
    "hecnn_relin_digits", "hecnn_launch_count", "hecnn_keygen", "hecnn_import_keys", "hecnn_export_secret_key",
    "hecnn_export_public_key", "hecnn_eval_key_digits", "hecnn_export_eval_key", "hecnn_device_alloc",
    "hecnn_device_free", "hecnn_memcpy_h2d", "hecnn_memcpy_d2h", "hecnn_ntt_forward", "hecnn_ntt_inverse",
    "hecnn_poly_add", "hecnn_poly_sub", "hecnn_poly_neg", "hecnn_poly_pointwise_mul", "hecnn_poly_pointwise_mac",
    "hecnn_rescale_poly", "hecnn_key_switch", "hecnn_tensor_create", "hecnn_tensor_destroy", "hecnn_tensor_info",
    "hecnn_tensor_set_shape", "hecnn_tensor_shape", "hecnn_tensor_data", "hecnn_tensor_upload",
    "hecnn_tensor_download", "hecnn_tensor_upload_async", "hecnn_tensor_download_async", "hecnn_encrypt_tensor", "hecnn_encrypt_raw", "hecnn_decrypt_raw",
    "hecnn_decrypt_tensor", "hecnn_ct_add", "hecnn_ct_sub", "hecnn_ct_mul", "hecnn_ct_square", "hecnn_ct_rescale",
    "hecnn_ct_mod_switch", "hecnn_ct_mul_const", "hecnn_ct_add_const", "hecnn_eval_activation",
    "hecnn_model_create", "hecnn_model_destroy", "hecnn_model_depth_cost", "hecnn_forward_encrypted",
    "hecnn_model_set_streaming",
    "hecnn_profile_enable", "hecnn_profile_reset", "hecnn_profile_read", "hecnn_modmul_peak",
    "hecnn_tensor_copy_to_device", "hecnn_host_encode_real", "hecnn_host_decode_real",
    "hecnn_host_encryption_randomness", "hecnn_fp64_modmul_peak", "hecnn_context_trim",
    "hecnn_blob_params", "hecnn_blob_save_key", "hecnn_blob_load_key", "hecnn_blob_save_ciphertext",
    "hecnn_blob_load_ciphertexts", "hecnn_make_scalar_plain", "hecnn_ct_zero", "hecnn_ct_add_inplace",
    "hecnn_ct_scalar_mac", "hecnn_ct_add_scalar", "hecnn_ct_add_plain", "hecnn_ct_mul_plain",
)

_lib = None

_V, _SZ, _U32, _U64, _D, _I = (ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_double,
                                ctypes.c_int)
_PV = ctypes.POINTER(ctypes.c_void_p)
_PSZ = ctypes.POINTER(ctypes.c_size_t)
_PU64 = ctypes.POINTER(ctypes.c_uint64)
_PD = ctypes.POINTER(ctypes.c_double)
_PI64 = ctypes.POINTER(ctypes.c_int64)
# argument types of every C-ABI entry (include/hecnn_b200.h); pointers to
# opaque handles and device memory travel as void*
_SIGNATURES = {
    "hecnn_abi_version": [],
    "hecnn_host_encode_real": [_SZ, _PU64, _SZ, _PD, _SZ, _D, _SZ, _PU64],
    "hecnn_host_decode_real": [_SZ, _PU64, _SZ, _PU64, _SZ, _D, _PD, _SZ],
    "hecnn_host_encryption_randomness": [_SZ, _D, _I, _U64, _PI64, _PI64, _PI64],
    "hecnn_find_chain": [_SZ, ctypes.POINTER(ctypes.c_int), _SZ, _PU64],
    "hecnn_context_create": [_SZ, _PU64, _SZ, _D, _D, _I, _I, _PV],
    "hecnn_context_destroy": [_V],
    "hecnn_context_set_stream": [_V, _V],
    "hecnn_context_synchronize": [_V],
    "hecnn_context_trim": [_V, _PSZ],
    "hecnn_context_info": [_V, _PSZ, _PSZ, _PD],
    "hecnn_relin_digits": [_V, _SZ, _PSZ],
    "hecnn_launch_count": [_V, _PU64],
    "hecnn_profile_enable": [_V, _I],
    "hecnn_profile_reset": [_V],
    "hecnn_profile_read": [_V, ctypes.c_char_p, _SZ],
    "hecnn_modmul_peak": [_V, _PD],
    "hecnn_fp64_modmul_peak": [_V, _PD],
    "hecnn_keygen": [_V, _U64],
    "hecnn_import_keys": [_V, _PU64, _PU64, _PU64, _PU64, _SZ],
    "hecnn_export_secret_key": [_V, _PU64],
    "hecnn_export_public_key": [_V, _PU64, _PU64],
    "hecnn_eval_key_digits": [_V, _PSZ],
    "hecnn_export_eval_key": [_V, _PU64],
    "hecnn_device_alloc": [_V, _SZ, _PV],
    "hecnn_device_free": [_V, _V],
    "hecnn_memcpy_h2d": [_V, _V, _V, _SZ],
    "hecnn_memcpy_d2h": [_V, _V, _V, _SZ],
    "hecnn_ntt_forward": [_V, _V, _SZ, _SZ],
    "hecnn_ntt_inverse": [_V, _V, _SZ, _SZ],
    "hecnn_poly_add": [_V, _V, _V, _V, _SZ, _SZ],
    "hecnn_poly_sub": [_V, _V, _V, _V, _SZ, _SZ],
    "hecnn_poly_neg": [_V, _V, _V, _SZ, _SZ],
    "hecnn_poly_pointwise_mul": [_V, _V, _V, _V, _SZ, _SZ],
    "hecnn_poly_pointwise_mac": [_V, _V, _V, _V, _SZ, _SZ],
    "hecnn_rescale_poly": [_V, _V, _V, _SZ, _SZ],
    "hecnn_key_switch": [_V, _V, _V, _SZ, _SZ],
    "hecnn_tensor_create": [_V, _SZ, _U32, _D, _PV],
    "hecnn_tensor_destroy": [_V],
    "hecnn_tensor_info": [_V, _PSZ, ctypes.POINTER(ctypes.c_uint32), _PD],
    "hecnn_tensor_set_shape": [_V, _I, _SZ, _SZ, _SZ, _SZ],
    "hecnn_tensor_shape": [_V, ctypes.POINTER(ctypes.c_int), _PSZ, _PSZ, _PSZ, _PSZ],
    "hecnn_tensor_data": [_V, ctypes.POINTER(_PU64)],
    "hecnn_tensor_upload": [_V, _V, _PU64],
    "hecnn_tensor_download": [_V, _V, _PU64],
    "hecnn_tensor_upload_async": [_V, _V, _PU64, _V],
    "hecnn_tensor_download_async": [_V, _V, _PU64, _V],
    "hecnn_tensor_copy_to_device": [_V, _V, _V],
    "hecnn_encrypt_tensor": [_V, _PD, _SZ, _SZ, _U64, _PV],
    "hecnn_encrypt_raw": [_V, _PU64, _PI64, _PI64, _PI64, _SZ, _D, _PV],
    "hecnn_decrypt_raw": [_V, _V, _PU64],
    "hecnn_decrypt_tensor": [_V, _V, _SZ, _PD],
    "hecnn_ct_add": [_V, _V, _V, _PV],
    "hecnn_ct_sub": [_V, _V, _V, _PV],
    "hecnn_ct_mul": [_V, _V, _V, _PV],
    "hecnn_ct_square": [_V, _V, _PV],
    "hecnn_ct_rescale": [_V, _V, _PV],
    "hecnn_ct_mod_switch": [_V, _V, _U32, _PV],
    "hecnn_ct_mul_const": [_V, _V, _D, _D, _PV],
    "hecnn_ct_add_const": [_V, _V, _D, _PV],
    "hecnn_eval_activation": [_V, _PD, _SZ, _D, _V, _PV],
    "hecnn_make_scalar_plain": [_V, _D, _D, _SZ, _PU64],
    "hecnn_ct_zero": [_V, _SZ, _U32, _D, _PV],
    "hecnn_ct_add_inplace": [_V, _V, _V],
    "hecnn_ct_scalar_mac": [_V, _V, _V, _PU64, _SZ, _D, _U32],
    "hecnn_ct_add_scalar": [_V, _V, _D],
    "hecnn_ct_add_plain": [_V, _V, _PU64, _U32, _D, _PV],
    "hecnn_ct_mul_plain": [_V, _V, _PU64, _U32, _D, _I, _I, _PV],
    "hecnn_model_create": [_V, _V, _PV],
    "hecnn_model_destroy": [_V],
    "hecnn_model_depth_cost": [_V, _PSZ],
    "hecnn_model_set_streaming": [_V, _I, _SZ, _SZ],
    "hecnn_forward_encrypted": [_V, _V, _V, _U64, _PV, _PD],
    "hecnn_blob_params": [_V, _SZ, ctypes.POINTER(ctypes.c_int), _PSZ, _V, _PSZ, _PD, _PD, ctypes.POINTER(ctypes.c_int)],
    "hecnn_blob_save_key": [_V, _I, _V, _SZ, _PSZ],
    "hecnn_blob_load_key": [_V, _I, _V, _SZ],
    "hecnn_blob_save_ciphertext": [_V, _V, _SZ, _V, _SZ, _PSZ],
    "hecnn_blob_load_ciphertexts": [_V, _PV, _PSZ, _SZ, _PV],
}


def lib() -> ctypes.CDLL:
    """Load the in-tree extension; raise if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"hecnn_b200 CUDA extension not built: {LIB_PATH} (run __graft_entry__.build())")
        L = ctypes.CDLL(LIB_PATH)
        L.hecnn_last_error.restype = ctypes.c_char_p
        L.hecnn_last_error.argtypes = []
        for name, args in _SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = ctypes.c_int
            fn.argtypes = args
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status == HECNN_OK:
        return
    msg = lib().hecnn_last_error().decode()
    if status == HECNN_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


_u64p = ctypes.POINTER(ctypes.c_uint64)
_dblp = ctypes.POINTER(ctypes.c_double)


def _ptr(a: np.ndarray, ctype=ctypes.c_uint64):
    return a.ctypes.data_as(ctypes.POINTER(ctype))


# ---------------------------------------------------------------- params

KRELIN_BASE_BITS = 20            # ckks.hpp:75
KSCALE_REL_TOL = 2.0 ** -30      # ckks.hpp:74
RELU_QUAD_COEFF = 0.000469841857369822  # activation.hpp:21


def find_chain(n: int, prime_bits: Sequence[int]) -> List[int]:
    """RingParams::create (ring.hpp:20-30)."""
    bits = (ctypes.c_int * len(prime_bits))(*prime_bits)
    out = np.zeros(len(prime_bits), dtype=np.uint64)
    _check(lib().hecnn_find_chain(ctypes.c_size_t(n), bits, ctypes.c_size_t(len(prime_bits)), _ptr(out)))
    return [int(v) for v in out]


def host_encode_real(params: "CkksParams", values, level: int, scale: Optional[float] = None) -> np.ndarray:
    """encode_real (ckks.hpp:105-129) on the host: residues [(level+1)][n]."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    pr = np.asarray(params.primes, dtype=np.uint64)
    out = np.empty((level + 1, params.n), dtype=np.uint64)
    _check(lib().hecnn_host_encode_real(params.n, _ptr(pr), len(pr), _ptr(v, ctypes.c_double), v.size,
                                        scale or params.scale, level, _ptr(out)))
    return out


def host_decode_real(params: "CkksParams", poly: np.ndarray, level: int, scale: float, count: Optional[int] = None):
    """decode (ckks.hpp:142-154) on the host: real parts of the slots."""
    poly = np.ascontiguousarray(poly, dtype=np.uint64)
    pr = np.asarray(params.primes, dtype=np.uint64)
    count = count or params.n // 2
    out = np.empty(count, dtype=np.float64)
    _check(lib().hecnn_host_decode_real(params.n, _ptr(pr), len(pr), _ptr(poly), level, scale,
                                        _ptr(out, ctypes.c_double), count))
    return out


def host_encryption_randomness(params: "CkksParams", seed: int):
    """make_encryption_randomness (ckks.hpp:238-244): (r, e0, e1) signed coefficients."""
    r, e0, e1 = (np.empty(params.n, dtype=np.int64) for _ in range(3))
    _check(lib().hecnn_host_encryption_randomness(params.n, params.sigma, int(params.degenerate_noise), seed,
                                                  _ptr(r, ctypes.c_int64), _ptr(e0, ctypes.c_int64),
                                                  _ptr(e1, ctypes.c_int64)))
    return r, e0, e1


@dataclass
class PresetDef:
    """presets.hpp:17-31"""
    name: str
    n: int
    prime_bits: List[int]
    log2_scale: int
    sigma: float = 3.2


def builtin_presets() -> List[PresetDef]:
    """presets.hpp:33-49"""
    return [
        PresetDef("toy-n16", 16, [40, 21, 21, 21], 20, 3.2),
        PresetDef("test-n4096-d4", 4096, [60, 40, 40, 40, 40], 40, 3.2),
        PresetDef("nn-n4096-d8", 4096, [60] + [40] * 8, 40, 3.2),
        PresetDef("net-n8192-d8", 8192, [60] + [40] * 8, 40, 3.2),
        PresetDef("large-n16384-d24", 16384, [60] + [40] * 24, 40, 3.2),
    ]


def find_preset(name: str, config_path: str = "") -> PresetDef:
    """find_preset (presets.hpp:67-76): a JSON file shadows built-ins."""
    if config_path:
        with open(config_path) as f:
            for e in json.load(f)["presets"]:
                if e["name"] == name:
                    return PresetDef(e["name"], int(e["n"]), list(e["prime_bits"]), int(e["log2_scale"]),
                                     float(e.get("sigma", 3.2)))
    for d in builtin_presets():
        if d.name == name:
            return d
    raise ValueError(f"unknown parameter preset: {name}")


@dataclass
class CkksParams:
    """CkksParams (ckks.hpp:21-34); ring = (n, primes)."""
    n: int
    primes: List[int]
    scale: float
    sigma: float = 3.2
    degenerate_noise: bool = False

    @staticmethod
    def from_preset(p: PresetDef, degenerate_noise: bool = False) -> "CkksParams":
        return CkksParams(p.n, find_chain(p.n, p.prime_bits), math.ldexp(1.0, p.log2_scale), p.sigma,
                          degenerate_noise)

    @property
    def top_level(self) -> int:
        return len(self.primes) - 1

    @property
    def slot_count(self) -> int:
        return self.n // 2


def preset_params(name: str, config_path: str = "", degenerate_noise: bool = False) -> CkksParams:
    """preset_params (presets.hpp:78-83)"""
    return CkksParams.from_preset(find_preset(name, config_path), degenerate_noise)


# ---------------------------------------------------------------- tensors

class EncryptedTensor:
    """A device batch of ciphertexts sharing (scale, level): TensorEncrypted
    (tensor.hpp:61-75), or one Ciphertext (ckks.hpp:68-72) when cells == 1.
    Words are [cells][2][level+1][n] u64, coefficient domain."""

    def __init__(self, engine: "CkksEngine", handle: ctypes.c_void_p):
        self._engine = engine
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hecnn_tensor_destroy(self._h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _info(self):
        cells, level, scale = ctypes.c_size_t(), ctypes.c_uint32(), ctypes.c_double()
        _check(lib().hecnn_tensor_info(self._h, ctypes.byref(cells), ctypes.byref(level), ctypes.byref(scale)))
        return cells.value, level.value, scale.value

    @property
    def cells(self) -> int:
        return self._info()[0]

    @property
    def level(self) -> int:
        return self._info()[1]

    @property
    def scale(self) -> float:
        return self._info()[2]

    def shape(self):
        flat, h, w, c, b = ctypes.c_int(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().hecnn_tensor_shape(self._h, ctypes.byref(flat), ctypes.byref(h), ctypes.byref(w),
                                        ctypes.byref(c), ctypes.byref(b)))
        return (bool(flat.value), h.value, w.value, c.value, b.value)

    def set_shape(self, shape: "Shape", batch: int) -> "EncryptedTensor":
        _check(lib().hecnn_tensor_set_shape(self._h, int(shape.flat), shape.h if not shape.flat else shape.feat,
                                            shape.w, shape.c, batch))
        return self

    def device_ptr(self) -> int:
        p = _u64p()
        _check(lib().hecnn_tensor_data(self._h, ctypes.byref(p)))
        return ctypes.cast(p, ctypes.c_void_p).value or 0

    def words(self) -> np.ndarray:
        cells, level, _ = self._info()
        out = np.empty((cells, 2, level + 1, self._engine.n), dtype=np.uint64)
        _check(lib().hecnn_tensor_download(self._engine.ctx, self._h, _ptr(out)))
        return out


# ---------------------------------------------------------------- model

@dataclass
class Shape:
    """Shape (tensor.hpp:16-39)"""
    flat: bool = False
    h: int = 0
    w: int = 0
    c: int = 0
    feat: int = 0

    @staticmethod
    def spatial(h: int, w: int, c: int) -> "Shape":
        return Shape(False, h, w, c, 0)

    @staticmethod
    def flattened(f: int) -> "Shape":
        return Shape(True, 0, 0, 0, f)

    def positions(self) -> int:
        return self.feat if self.flat else self.h * self.w * self.c


CONV2D, AVG_POOL2D, ZERO_PAD2D, DENSE, ACTIVATION, SIGMOID = range(6)

_M64 = (1 << 64) - 1


def splitmix64(x: int) -> int:
    """splitmix64 (common.hpp:164-169)"""
    x = (x + 0x9E3779B97F4A7C15) & _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def derive_seed(seed: int, domain: int) -> int:
    """CkksEngine::derive_seed (ckks.hpp:507): splitmix64(seed ^ splitmix64(domain))"""
    return splitmix64((seed & _M64) ^ splitmix64(domain & _M64))


@dataclass
class LayerSpec:
    """LayerSpec (model.hpp:12-76)"""
    kind: int
    filters: int = 0
    kernel_h: int = 0
    kernel_w: int = 0
    stride: int = 1
    valid: bool = False
    pool: int = 0
    pad: int = 0
    units: int = 0
    surrogate: str = ""

    @staticmethod
    def conv2d(filters, kh, kw, stride=1, valid=False):
        return LayerSpec(CONV2D, filters=filters, kernel_h=kh, kernel_w=kw, stride=stride, valid=valid)

    @staticmethod
    def avg_pool2d(pool):
        return LayerSpec(AVG_POOL2D, pool=pool)

    @staticmethod
    def zero_pad2d(pad):
        return LayerSpec(ZERO_PAD2D, pad=pad)

    @staticmethod
    def dense(units):
        return LayerSpec(DENSE, units=units)

    @staticmethod
    def activation(name):
        return LayerSpec(ACTIVATION, surrogate=name)

    @staticmethod
    def sigmoid():
        return LayerSpec(SIGMOID)


@dataclass
class PolyActivation:
    """PolyActivation (activation.hpp:24-45)"""
    coefficients: List[float]
    interval_bound: float = 3.0 / (8.0 * RELU_QUAD_COEFF)
    source: str = "relu"

    def degree(self) -> int:
        return max(len(self.coefficients) - 1, 0)

    def encrypted_depth(self) -> int:
        d, lg = self.degree(), 0
        while (1 << lg) < d:
            lg += 1
        return lg + 1


def relu_default_surrogate() -> PolyActivation:
    """activation.hpp:47-49"""
    return PolyActivation([0.0, 0.5, RELU_QUAD_COEFF])


class _LayerDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("filters", ctypes.c_int32), ("kernel_h", ctypes.c_int32),
                ("kernel_w", ctypes.c_int32), ("stride", ctypes.c_int32), ("padding_valid", ctypes.c_int32),
                ("pool", ctypes.c_int32), ("pad", ctypes.c_int32), ("units", ctypes.c_int32),
                ("activation", ctypes.c_int32), ("weights", _dblp), ("n_weights", ctypes.c_size_t),
                ("biases", _dblp), ("n_biases", ctypes.c_size_t)]


class _ActDesc(ctypes.Structure):
    _fields_ = [("coefficients", _dblp), ("n_coefficients", ctypes.c_size_t), ("interval_bound", ctypes.c_double)]


class _ModelDesc(ctypes.Structure):
    _fields_ = [("input_flat", ctypes.c_int32), ("input_h", ctypes.c_size_t), ("input_w", ctypes.c_size_t),
                ("input_c", ctypes.c_size_t), ("input_features", ctypes.c_size_t),
                ("layers", ctypes.POINTER(_LayerDesc)), ("n_layers", ctypes.c_size_t),
                ("activations", ctypes.POINTER(_ActDesc)), ("n_activations", ctypes.c_size_t)]


@dataclass
class ModelSpec:
    """ModelSpec (model.hpp:78-97); weights/biases parallel to layers."""
    input: Shape
    layers: List[LayerSpec] = field(default_factory=list)
    activations: Dict[str, PolyActivation] = field(default_factory=dict)
    weights: List[Optional[np.ndarray]] = field(default_factory=list)
    biases: List[Optional[np.ndarray]] = field(default_factory=list)

    def ensure_param_slots(self):
        while len(self.weights) < len(self.layers):
            self.weights.append(None)
        while len(self.biases) < len(self.layers):
            self.biases.append(None)

    def shapes(self) -> List[Shape]:
        """shape_infer (model.hpp:145-157), without validation (the engine validates)."""
        out, cur = [], self.input
        for l in self.layers:
            if l.kind == DENSE and not cur.flat:
                cur = Shape.flattened(cur.positions())
            if l.kind == CONV2D:
                def dim(i, k):
                    return (i + l.stride - 1) // l.stride if not l.valid else (i - k) // l.stride + 1
                cur = Shape.spatial(dim(cur.h, l.kernel_h), dim(cur.w, l.kernel_w), l.filters)
            elif l.kind == AVG_POOL2D:
                cur = Shape.spatial(cur.h // l.pool, cur.w // l.pool, cur.c)
            elif l.kind == ZERO_PAD2D:
                cur = Shape.spatial(cur.h + 2 * l.pad, cur.w + 2 * l.pad, cur.c)
            elif l.kind == DENSE:
                cur = Shape.flattened(l.units)
            out.append(cur)
        return out

    def param_counts(self) -> List[tuple]:
        """param_counts (model.hpp:160-164) per layer."""
        res, cur = [], self.input
        shapes = self.shapes()
        for i, l in enumerate(self.layers):
            inp = Shape.flattened(cur.positions()) if (l.kind == DENSE and not cur.flat) else cur
            if l.kind == CONV2D:
                res.append((l.kernel_h * l.kernel_w * inp.c * l.filters, l.filters))
            elif l.kind == DENSE:
                res.append((inp.positions() * l.units, l.units))
            else:
                res.append((0, 0))
            cur = shapes[i]
        return res

    def depth_cost(self) -> int:
        """depth_cost (model.hpp:169-182)"""
        c = 0
        for l in self.layers:
            if l.kind in (CONV2D, AVG_POOL2D, DENSE):
                c += 1
            elif l.kind == ACTIVATION:
                c += self.activations[l.surrogate].encrypted_depth()
        return c

    def to_desc(self):
        """Build the hecnn_model_desc; returns (desc, keepalive)."""
        self.ensure_param_slots()
        names = list(self.activations.keys())
        keep = []
        acts = (_ActDesc * max(len(names), 1))()
        for i, nm in enumerate(names):
            c = np.ascontiguousarray(self.activations[nm].coefficients, dtype=np.float64)
            keep.append(c)
            acts[i] = _ActDesc(_ptr(c, ctypes.c_double), c.size, self.activations[nm].interval_bound)
        layers = (_LayerDesc * max(len(self.layers), 1))()
        for i, l in enumerate(self.layers):
            w = self.weights[i]
            b = self.biases[i]
            wp, nw, bp, nb = None, 0, None, 0
            if w is not None:
                w = np.ascontiguousarray(w, dtype=np.float64)
                keep.append(w)
                wp, nw = _ptr(w, ctypes.c_double), w.size
            if b is not None:
                b = np.ascontiguousarray(b, dtype=np.float64)
                keep.append(b)
                bp, nb = _ptr(b, ctypes.c_double), b.size
            act = -1
            if l.kind == ACTIVATION:
                act = names.index(l.surrogate) if l.surrogate in names else len(names) + 1000
            layers[i] = _LayerDesc(l.kind, l.filters, l.kernel_h, l.kernel_w, l.stride, int(l.valid), l.pool, l.pad,
                                   l.units, act, wp, nw, bp, nb)
        desc = _ModelDesc(int(self.input.flat), self.input.h, self.input.w, self.input.c, self.input.feat,
                          layers, len(self.layers), acts, len(names))
        keep += [acts, layers]
        return desc, keep


def tiny_preset() -> ModelSpec:
    """tiny_preset (model.hpp:223-235)"""
    m = ModelSpec(Shape.spatial(8, 8, 3))
    m.activations["relu-poly2"] = relu_default_surrogate()
    m.layers = [LayerSpec.conv2d(4, 3, 3), LayerSpec.activation("relu-poly2"), LayerSpec.avg_pool2d(2),
                LayerSpec.dense(1)]
    m.ensure_param_slots()
    return m


def alexnet32_preset(image: int = 32) -> ModelSpec:
    """alexnet32_preset (model.hpp:189-219); `image` = 64 gives the COWC 64x64x3 variant."""
    m = ModelSpec(Shape.spatial(image, image, 3))
    m.activations["relu-poly2"] = relu_default_surrogate()
    act = lambda: LayerSpec.activation("relu-poly2")  # noqa: E731
    m.layers = [LayerSpec.conv2d(96, 11, 11), act(), LayerSpec.avg_pool2d(2), LayerSpec.conv2d(256, 5, 5), act(),
                LayerSpec.avg_pool2d(2), LayerSpec.zero_pad2d(1), LayerSpec.conv2d(384, 3, 3), act(),
                LayerSpec.avg_pool2d(2), LayerSpec.zero_pad2d(1), LayerSpec.conv2d(384, 3, 3), act(),
                LayerSpec.zero_pad2d(1), LayerSpec.avg_pool2d(2), LayerSpec.dense(4096), act(),
                LayerSpec.dense(4096), act(), LayerSpec.dense(1), LayerSpec.sigmoid()]
    m.ensure_param_slots()
    return m


def glorot_weights(model: ModelSpec, seed: int) -> ModelSpec:
    """Synthetic Glorot-uniform weights in the layout of init_random_weights
    (model_io.hpp:183-203), drawn from numpy (the values are synthetic inputs,
    not a parity target; parity tests pass identical arrays to both sides)."""
    rng = np.random.default_rng(seed)
    model.ensure_param_slots()
    cur = model.input
    shapes = model.shapes()
    for i, (l, (wc, bc)) in enumerate(zip(model.layers, model.param_counts())):
        if wc:
            inp = Shape.flattened(cur.positions()) if (l.kind == DENSE and not cur.flat) else cur
            fan_in = l.kernel_h * l.kernel_w * inp.c if l.kind == CONV2D else inp.positions()
            fan_out = l.filters if l.kind == CONV2D else l.units
            lim = math.sqrt(6.0 / (fan_in + fan_out))
            model.weights[i] = (rng.random(wc) * 2 - 1) * lim
            model.biases[i] = (rng.random(bc) * 2 - 1) * 0.05
        cur = shapes[i]
    return model


class Model:
    """A ModelSpec registered with an engine (hecnn_model)."""

    def __init__(self, engine: "CkksEngine", spec: ModelSpec):
        self._engine = engine
        self.spec = spec
        desc, keep = spec.to_desc()
        h = ctypes.c_void_p()
        _check(lib().hecnn_model_create(engine.ctx, ctypes.byref(desc), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.hecnn_model_destroy(self._h)
            self._h = None

    def depth_cost(self) -> int:
        c = ctypes.c_size_t()
        _check(lib().hecnn_model_depth_cost(self._h, ctypes.byref(c)))
        return c.value

    STREAM_AUTO, STREAM_ALWAYS, STREAM_NEVER = 0, 1, 2

    def set_streaming(self, mode: int = 0, tile: int = 0, mem_budget: int = 0) -> "Model":
        """Row-streamed execution of the spatial layers (hecnn_model_set_streaming):
        mode 0 streams only what does not fit in device memory, 1 always, 2 never;
        tile = stage-output columns per tile (0: from the budget); mem_budget =
        device bytes to plan with (0: free memory). Output words do not depend on it."""
        _check(lib().hecnn_model_set_streaming(self._h, int(mode), ctypes.c_size_t(tile), ctypes.c_size_t(mem_budget)))
        return self


# ---------------------------------------------------------------- engine

@dataclass
class ScalarPlain:
    """CkksEngine::ScalarPlain (ckks.hpp:400-405): residues per active prime."""
    residues: np.ndarray
    scale: float
    level: int


@dataclass
class EncodedPlaintext:
    """EncodedPlaintext (ckks.hpp:21-72): coefficient-domain residues [level+1][n]."""
    poly: np.ndarray
    scale: float
    level: int
    is_constant: bool = False


class CkksEngine:
    """CkksEngine (ckks.hpp:77-636) on one B200. Keys live on the device."""

    def __init__(self, params: CkksParams, device: int = 0):
        self.params = params
        self.n = params.n
        primes = np.asarray(params.primes, dtype=np.uint64)
        h = ctypes.c_void_p()
        _check(lib().hecnn_context_create(ctypes.c_size_t(params.n), _ptr(primes), ctypes.c_size_t(len(primes)),
                                          ctypes.c_double(params.scale), ctypes.c_double(params.sigma),
                                          int(params.degenerate_noise), int(device), ctypes.byref(h)))
        self.ctx = h
        self._children = []

    def close(self):
        if getattr(self, "ctx", None) and _lib is not None:
            _lib.hecnn_context_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        self.close()

    @property
    def top_level(self) -> int:
        return len(self.params.primes) - 1

    @property
    def slot_count(self) -> int:
        return self.n // 2

    def depth_budget(self) -> int:
        return self.top_level

    def relin_digits(self, level: int) -> int:
        d = ctypes.c_size_t()
        _check(lib().hecnn_relin_digits(self.ctx, ctypes.c_size_t(level), ctypes.byref(d)))
        return d.value

    def launches(self) -> int:
        v = ctypes.c_uint64()
        _check(lib().hecnn_launch_count(self.ctx, ctypes.byref(v)))
        return v.value

    def synchronize(self):
        _check(lib().hecnn_context_synchronize(self.ctx))

    def trim(self) -> int:
        """Return wholly free device-arena segments to the driver."""
        f = ctypes.c_size_t()
        _check(lib().hecnn_context_trim(self.ctx, ctypes.byref(f)))
        return f.value

    def set_stream(self, stream_ptr: int):
        _check(lib().hecnn_context_set_stream(self.ctx, ctypes.c_void_p(stream_ptr)))

    # ---- measurement
    def profile(self, on: bool):
        _check(lib().hecnn_profile_enable(self.ctx, int(on)))

    def profile_reset(self):
        _check(lib().hecnn_profile_reset(self.ctx))

    def profile_read(self) -> dict:
        buf = ctypes.create_string_buffer(1 << 16)
        _check(lib().hecnn_profile_read(self.ctx, buf, ctypes.c_size_t(len(buf))))
        return json.loads(buf.value.decode())

    def modmul_peak(self) -> float:
        v = ctypes.c_double()
        _check(lib().hecnn_modmul_peak(self.ctx, ctypes.byref(v)))
        return v.value

    def fp64_modmul_peak(self) -> float:
        v = ctypes.c_double()
        _check(lib().hecnn_fp64_modmul_peak(self.ctx, ctypes.byref(v)))
        return v.value

    def copy_to_device(self, t: "EncryptedTensor", dst_ptr: int):
        _check(lib().hecnn_tensor_copy_to_device(self.ctx, t.handle, ctypes.c_void_p(dst_ptr)))

    def upload_into(self, t: "EncryptedTensor", host_ptr: int):
        """H2D of a [cells][2][level+1][n] host buffer (pinned for full speed)."""
        _check(lib().hecnn_tensor_upload(self.ctx, t.handle, ctypes.cast(host_ptr, _u64p)))

    def download_into(self, t: "EncryptedTensor", host_ptr: int):
        _check(lib().hecnn_tensor_download(self.ctx, t.handle, ctypes.cast(host_ptr, _u64p)))

    def upload_async(self, t: "EncryptedTensor", host_ptr: int, stream: int = 0):
        """Enqueue the H2D on `stream` (cudaStream_t as int; 0 = the context's stream) and
        return; host_ptr must be pinned and outlive the copy."""
        _check(lib().hecnn_tensor_upload_async(self.ctx, t.handle, ctypes.cast(host_ptr, _u64p),
                                               ctypes.c_void_p(stream or None)))

    def download_async(self, t: "EncryptedTensor", host_ptr: int, stream: int = 0):
        _check(lib().hecnn_tensor_download_async(self.ctx, t.handle, ctypes.cast(host_ptr, _u64p),
                                                 ctypes.c_void_p(stream or None)))

    def empty_tensor(self, cells: int, level: int, scale: float) -> "EncryptedTensor":
        h = ctypes.c_void_p()
        _check(lib().hecnn_tensor_create(self.ctx, ctypes.c_size_t(cells), ctypes.c_uint32(level),
                                         ctypes.c_double(scale), ctypes.byref(h)))
        return self._wrap(h)

    # ---- keys
    def keygen(self, seed: int) -> "CkksEngine":
        _check(lib().hecnn_keygen(self.ctx, ctypes.c_uint64(seed)))
        return self

    def import_keys(self, secret=None, pk_b=None, pk_a=None, evk=None):
        def p(a):
            return None if a is None else _ptr(np.ascontiguousarray(a, dtype=np.uint64))
        arrs = [None if a is None else np.ascontiguousarray(a, dtype=np.uint64) for a in (secret, pk_b, pk_a, evk)]
        digits = 0 if evk is None else arrs[3].shape[0]
        _check(lib().hecnn_import_keys(self.ctx, *(None if a is None else _ptr(a) for a in arrs),
                                       ctypes.c_size_t(digits)))

    def export_secret_key(self) -> np.ndarray:
        out = np.empty((self.top_level + 1, self.n), dtype=np.uint64)
        _check(lib().hecnn_export_secret_key(self.ctx, _ptr(out)))
        return out

    def export_public_key(self):
        b = np.empty((self.top_level + 1, self.n), dtype=np.uint64)
        a = np.empty_like(b)
        _check(lib().hecnn_export_public_key(self.ctx, _ptr(b), _ptr(a)))
        return b, a

    def export_eval_key(self) -> np.ndarray:
        d = ctypes.c_size_t()
        _check(lib().hecnn_eval_key_digits(self.ctx, ctypes.byref(d)))
        out = np.empty((d.value, 2, self.top_level + 1, self.n), dtype=np.uint64)
        _check(lib().hecnn_export_eval_key(self.ctx, _ptr(out)))
        return out

    # ---- raw device memory for the ring tier
    def to_device(self, a: np.ndarray) -> int:
        a = np.ascontiguousarray(a, dtype=np.uint64)
        p = ctypes.c_void_p()
        _check(lib().hecnn_device_alloc(self.ctx, ctypes.c_size_t(a.nbytes), ctypes.byref(p)))
        _check(lib().hecnn_memcpy_h2d(self.ctx, p, a.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(a.nbytes)))
        return p.value

    def from_device(self, dptr: int, shape, free: bool = True) -> np.ndarray:
        out = np.empty(shape, dtype=np.uint64)
        _check(lib().hecnn_memcpy_d2h(self.ctx, out.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(dptr),
                                      ctypes.c_size_t(out.nbytes)))
        if free:
            _check(lib().hecnn_device_free(self.ctx, ctypes.c_void_p(dptr)))
        return out

    def free(self, dptr: int):
        _check(lib().hecnn_device_free(self.ctx, ctypes.c_void_p(dptr)))

    def _ring_call(self, fn, polys: np.ndarray, level: int, *extra):
        polys = np.ascontiguousarray(polys, dtype=np.uint64)
        count = polys.size // ((level + 1) * self.n)
        d = self.to_device(polys)
        _check(fn(self.ctx, ctypes.c_void_p(d), ctypes.c_size_t(level), ctypes.c_size_t(count), *extra))
        return self.from_device(d, polys.shape)

    def ntt_forward(self, polys: np.ndarray, level: int) -> np.ndarray:
        """ntt_transform Forward (ring.hpp:326-342) on [count][level+1][n]."""
        return self._ring_call(lib().hecnn_ntt_forward, polys, level)

    def ntt_inverse(self, polys: np.ndarray, level: int) -> np.ndarray:
        return self._ring_call(lib().hecnn_ntt_inverse, polys, level)

    def _binary(self, fn, a, b, level, mac=False):
        a = np.ascontiguousarray(a, dtype=np.uint64)
        b = np.ascontiguousarray(b, dtype=np.uint64)
        count = a.size // ((level + 1) * self.n)
        da, db = self.to_device(a), self.to_device(b)
        if mac:
            _check(fn(self.ctx, ctypes.c_void_p(da), ctypes.c_void_p(db), ctypes.c_void_p(db),
                      ctypes.c_size_t(level), ctypes.c_size_t(count)))
            self.free(db)
            return self.from_device(da, a.shape)
        _check(fn(self.ctx, ctypes.c_void_p(da), ctypes.c_void_p(db), ctypes.c_void_p(da), ctypes.c_size_t(level),
                  ctypes.c_size_t(count)))
        self.free(db)
        return self.from_device(da, a.shape)

    def poly_add(self, a, b, level):
        return self._binary(lib().hecnn_poly_add, a, b, level)

    def poly_sub(self, a, b, level):
        return self._binary(lib().hecnn_poly_sub, a, b, level)

    def poly_pointwise_mul(self, a, b, level):
        return self._binary(lib().hecnn_poly_pointwise_mul, a, b, level)

    def rescale_poly(self, polys: np.ndarray, level: int) -> np.ndarray:
        """rescale_poly (ring.hpp:419-442): [count][level+1][n] -> [count][level][n]"""
        polys = np.ascontiguousarray(polys, dtype=np.uint64)
        count = polys.size // ((level + 1) * self.n)
        din = self.to_device(polys)
        dout = self.to_device(np.zeros((count, max(level, 1), self.n), dtype=np.uint64))
        st = lib().hecnn_rescale_poly(self.ctx, ctypes.c_void_p(din), ctypes.c_void_p(dout), ctypes.c_size_t(level),
                                      ctypes.c_size_t(count))
        self.free(din)
        if st != HECNN_OK:
            self.free(dout)
            _check(st)
        return self.from_device(dout, (count, level, self.n))

    def key_switch(self, d2: np.ndarray, level: int) -> np.ndarray:
        """key_switch (ckks.hpp:601-630): [count][level+1][n] -> [count][2][level+1][n] NTT domain"""
        d2 = np.ascontiguousarray(d2, dtype=np.uint64)
        count = d2.size // ((level + 1) * self.n)
        din = self.to_device(d2)
        dout = self.to_device(np.zeros((count, 2, level + 1, self.n), dtype=np.uint64))
        st = lib().hecnn_key_switch(self.ctx, ctypes.c_void_p(din), ctypes.c_void_p(dout), ctypes.c_size_t(level),
                                    ctypes.c_size_t(count))
        self.free(din)
        if st != HECNN_OK:
            self.free(dout)
            _check(st)
        return self.from_device(dout, (count, 2, level + 1, self.n))

    # ---- tensors
    def _wrap(self, h) -> EncryptedTensor:
        return EncryptedTensor(self, h)

    def tensor_from_words(self, words: np.ndarray, level: int, scale: float) -> EncryptedTensor:
        words = np.ascontiguousarray(words, dtype=np.uint64)
        cells = words.size // (2 * (level + 1) * self.n)
        h = ctypes.c_void_p()
        _check(lib().hecnn_tensor_create(self.ctx, ctypes.c_size_t(cells), ctypes.c_uint32(level),
                                         ctypes.c_double(scale), ctypes.byref(h)))
        t = self._wrap(h)
        _check(lib().hecnn_tensor_upload(self.ctx, h, _ptr(words)))
        return t

    def encrypt_tensor(self, data: np.ndarray, seed: int, shape: Optional[Shape] = None) -> EncryptedTensor:
        """encrypt_tensor (tensor.hpp:77-94): data [batch][positions]."""
        data = np.ascontiguousarray(data, dtype=np.float64)
        batch, positions = data.shape
        h = ctypes.c_void_p()
        _check(lib().hecnn_encrypt_tensor(self.ctx, _ptr(data, ctypes.c_double), ctypes.c_size_t(batch),
                                          ctypes.c_size_t(positions), ctypes.c_uint64(seed), ctypes.byref(h)))
        t = self._wrap(h)
        if shape is not None:
            t.set_shape(shape, batch)
        else:
            t.set_shape(Shape.flattened(positions), batch)
        return t

    def encrypt_raw(self, m: np.ndarray, r, e0, e1, scale: float) -> EncryptedTensor:
        """encrypt with explicit randomness (ckks.hpp:249-266)."""
        m = np.ascontiguousarray(m, dtype=np.uint64)
        r, e0, e1 = (np.ascontiguousarray(v, dtype=np.int64) for v in (r, e0, e1))
        count = r.size // self.n
        h = ctypes.c_void_p()
        _check(lib().hecnn_encrypt_raw(self.ctx, _ptr(m), _ptr(r, ctypes.c_int64), _ptr(e0, ctypes.c_int64),
                                       _ptr(e1, ctypes.c_int64), ctypes.c_size_t(count), ctypes.c_double(scale),
                                       ctypes.byref(h)))
        return self._wrap(h)

    def decrypt_raw(self, t: EncryptedTensor) -> np.ndarray:
        cells, level, _ = t._info()
        out = np.empty((cells, level + 1, self.n), dtype=np.uint64)
        _check(lib().hecnn_decrypt_raw(self.ctx, t.handle, _ptr(out)))
        return out

    def decrypt_tensor(self, t: EncryptedTensor, batch: int) -> np.ndarray:
        """decrypt_tensor (tensor.hpp:96-106): [batch][positions]"""
        out = np.empty((batch, t.cells), dtype=np.float64)
        _check(lib().hecnn_decrypt_tensor(self.ctx, t.handle, ctypes.c_size_t(batch), _ptr(out, ctypes.c_double)))
        return out

    def _unary(self, fn, *args) -> EncryptedTensor:
        h = ctypes.c_void_p()
        _check(fn(self.ctx, *args, ctypes.byref(h)))
        return self._wrap(h)

    def add(self, x, y):
        return self._unary(lib().hecnn_ct_add, x.handle, y.handle)

    def sub(self, x, y):
        return self._unary(lib().hecnn_ct_sub, x.handle, y.handle)

    def mul(self, x, y):
        return self._unary(lib().hecnn_ct_mul, x.handle, y.handle)

    def square(self, x):
        return self._unary(lib().hecnn_ct_square, x.handle)

    def rescale(self, x):
        return self._unary(lib().hecnn_ct_rescale, x.handle)

    def mod_switch(self, x, level):
        return self._unary(lib().hecnn_ct_mod_switch, x.handle, ctypes.c_uint32(level))

    def mul_const(self, x, c, scale):
        """mul_plain(x, encode_const(c, scale, x.level))"""
        return self._unary(lib().hecnn_ct_mul_const, x.handle, ctypes.c_double(c), ctypes.c_double(scale))

    def add_const(self, x, c):
        """add_plain(x, encode_const(c, x.scale, x.level))"""
        return self._unary(lib().hecnn_ct_add_const, x.handle, ctypes.c_double(c))

    # ---- the scalar fast path and plaintext operands (ckks.hpp:283-311, 372-472),
    # applied to every cell of a tensor

    def make_scalar_plain(self, c: float, scale: float, level: int) -> "ScalarPlain":
        """make_scalar_plain (ckks.hpp:407-423): round(c * scale) mod q_i, i <= level."""
        r = np.empty(level + 1, dtype=np.uint64)
        _check(lib().hecnn_make_scalar_plain(self.ctx, ctypes.c_double(c), ctypes.c_double(scale),
                                             ctypes.c_size_t(level), _ptr(r)))
        return ScalarPlain(r, scale, level)

    def make_zero_ciphertext(self, level: int, scale: float, cells: int = 1) -> EncryptedTensor:
        """make_zero_ciphertext (ckks.hpp:431-438), `cells` of them."""
        return self._unary(lib().hecnn_ct_zero, ctypes.c_size_t(cells), ctypes.c_uint32(level), ctypes.c_double(scale))

    def add_inplace(self, acc: EncryptedTensor, x: EncryptedTensor) -> None:
        """add_inplace (ckks.hpp:440-445)."""
        _check(lib().hecnn_ct_add_inplace(self.ctx, acc.handle, x.handle))

    def mul_scalar_mac(self, acc: EncryptedTensor, x: EncryptedTensor, sp) -> None:
        """mul_scalar_mac (ckks.hpp:448-465): acc += x * sp. `sp` is one
        ScalarPlain for every cell or a sequence of them, one per cell (same
        scale and level)."""
        sps = [sp] if isinstance(sp, ScalarPlain) else list(sp)
        if not sps:
            raise ValueError("mul_scalar_mac: no scalar")
        if any(q.scale != sps[0].scale or q.level != sps[0].level for q in sps):
            raise ValueError("mul_scalar_mac: per-cell scalars must share one scale and level")
        r = np.ascontiguousarray(np.stack([q.residues for q in sps]), dtype=np.uint64)
        _check(lib().hecnn_ct_scalar_mac(self.ctx, acc.handle, x.handle, _ptr(r), ctypes.c_size_t(len(sps)),
                                         ctypes.c_double(sps[0].scale), ctypes.c_uint32(sps[0].level)))

    def add_scalar_inplace(self, ct: EncryptedTensor, c: float) -> None:
        """add_scalar_inplace (ckks.hpp:468-472): c encoded at ct's own scale."""
        _check(lib().hecnn_ct_add_scalar(self.ctx, ct.handle, ctypes.c_double(c)))

    def encode_const(self, c: float, scale: float, level: int) -> "EncodedPlaintext":
        """encode_const (ckks.hpp:132-140): the constant polynomial round(c * scale)."""
        sp = self.make_scalar_plain(c, scale, level)
        poly = np.zeros((level + 1, self.params.n), dtype=np.uint64)
        poly[:, 0] = sp.residues
        return EncodedPlaintext(poly, scale, level, True)

    def encode_real(self, values, scale: float, level: int) -> "EncodedPlaintext":
        """encode_real (ckks.hpp:124-129) on the host."""
        return EncodedPlaintext(host_encode_real(self.params, values, level, scale), scale, level, False)

    def add_plain(self, x: EncryptedTensor, m: "EncodedPlaintext") -> EncryptedTensor:
        """add_plain (ckks.hpp:305-311) of one plaintext to every cell."""
        poly = np.ascontiguousarray(m.poly, dtype=np.uint64)
        return self._unary(lib().hecnn_ct_add_plain, x.handle, _ptr(poly), ctypes.c_uint32(m.level),
                           ctypes.c_double(m.scale))

    def mul_plain_raw(self, x: EncryptedTensor, m: "EncodedPlaintext") -> EncryptedTensor:
        """mul_plain_raw (ckks.hpp:372-393): scale multiplies, level unchanged."""
        return self._mul_plain(x, m, 0)

    def mul_plain(self, x: EncryptedTensor, m: "EncodedPlaintext") -> EncryptedTensor:
        """mul_plain (ckks.hpp:395-398): mul_plain_raw then rescale."""
        return self._mul_plain(x, m, 1)

    def _mul_plain(self, x, m, rescale):
        poly = np.ascontiguousarray(m.poly, dtype=np.uint64)
        return self._unary(lib().hecnn_ct_mul_plain, x.handle, _ptr(poly), ctypes.c_uint32(m.level),
                           ctypes.c_double(m.scale), ctypes.c_int(1 if m.is_constant else 0), ctypes.c_int(rescale))

    def eval_activation(self, act: PolyActivation, x: EncryptedTensor) -> EncryptedTensor:
        c = np.ascontiguousarray(act.coefficients, dtype=np.float64)
        return self._unary(lib().hecnn_eval_activation, _ptr(c, ctypes.c_double), ctypes.c_size_t(c.size),
                           ctypes.c_double(act.interval_bound), x.handle)

    def model(self, spec: ModelSpec) -> Model:
        return Model(self, spec)


def encrypt_tensor(eng: CkksEngine, x: np.ndarray, seed: int, shape: Optional[Shape] = None) -> EncryptedTensor:
    return eng.encrypt_tensor(x, seed, shape)


def decrypt_tensor(eng: CkksEngine, x: EncryptedTensor, batch: int) -> np.ndarray:
    return eng.decrypt_tensor(x, batch)


def eval_encrypted(act: PolyActivation, x: EncryptedTensor, eng: CkksEngine) -> EncryptedTensor:
    return eng.eval_activation(act, x)


def forward_encrypted(model, x: EncryptedTensor, eng: CkksEngine, seed: int = 1,
                      layer_seconds: Optional[list] = None) -> EncryptedTensor:
    """forward_encrypted (layers.hpp:299-368). `model` is a ModelSpec or Model."""
    m = model if isinstance(model, Model) else Model(eng, model)
    nl = len(m.spec.layers)
    secs = np.zeros(max(nl, 1), dtype=np.float64)
    h = ctypes.c_void_p()
    _check(lib().hecnn_forward_encrypted(eng.ctx, m._h, x.handle, ctypes.c_uint64(seed), ctypes.byref(h),
                                         _ptr(secs, ctypes.c_double) if layer_seconds is not None else None))
    if layer_seconds is not None:
        layer_seconds[:] = list(secs[:nl])
    return EncryptedTensor(eng, h)


# ---------------------------------------------------------------- wire format
# CKKS blob v1 (ckks_serialize.hpp): byte-identical to the reference's
# save_* output; the native codec decodes straight into device tensors/keys.

BLOB_SECRET_KEY, BLOB_PUBLIC_KEY, BLOB_EVAL_KEY, BLOB_CIPHERTEXT = 1, 2, 3, 4


def _blob_call(fn, *args) -> bytes:
    size = ctypes.c_size_t()
    _check(fn(*args, None, ctypes.c_size_t(0), ctypes.byref(size)))
    buf = ctypes.create_string_buffer(size.value)
    _check(fn(*args, buf, ctypes.c_size_t(size.value), ctypes.byref(size)))
    return buf.raw[:size.value]


def blob_params(blob: bytes):
    """read_header (ckks_serialize.hpp:41-58): (kind, CkksParams) of a blob."""
    kind, n, cnt = ctypes.c_int(), ctypes.c_size_t(), ctypes.c_size_t(0)
    scale, sigma, deg = ctypes.c_double(), ctypes.c_double(), ctypes.c_int()
    _check(lib().hecnn_blob_params(blob, len(blob), ctypes.byref(kind), ctypes.byref(n), None, ctypes.byref(cnt),
                                   ctypes.byref(scale), ctypes.byref(sigma), ctypes.byref(deg)))
    primes = np.empty(cnt.value, dtype=np.uint64)
    _check(lib().hecnn_blob_params(blob, len(blob), None, None, _ptr(primes), ctypes.byref(cnt), None, None, None))
    return kind.value, CkksParams(n.value, [int(q) for q in primes], scale.value, sigma.value, bool(deg.value))


def save_secret_key(eng: "CkksEngine") -> bytes:
    """save_secret_key (ckks_serialize.hpp:79-82) of the engine's secret key."""
    return _blob_call(lib().hecnn_blob_save_key, eng.ctx, BLOB_SECRET_KEY)


def save_public_key(eng: "CkksEngine") -> bytes:
    """save_public_key (ckks_serialize.hpp:90-94)."""
    return _blob_call(lib().hecnn_blob_save_key, eng.ctx, BLOB_PUBLIC_KEY)


def save_evaluation_key(eng: "CkksEngine") -> bytes:
    """save_evaluation_key (ckks_serialize.hpp:104-112)."""
    return _blob_call(lib().hecnn_blob_save_key, eng.ctx, BLOB_EVAL_KEY)


def load_key(eng: "CkksEngine", kind: int, blob: bytes) -> "CkksEngine":
    """load_secret_key / load_public_key / load_evaluation_key into the engine
    (the blob's parameters must equal the engine's)."""
    _check(lib().hecnn_blob_load_key(eng.ctx, int(kind), blob, len(blob)))
    return eng


def load_secret_key(eng: "CkksEngine", blob: bytes) -> "CkksEngine":
    return load_key(eng, BLOB_SECRET_KEY, blob)


def load_public_key(eng: "CkksEngine", blob: bytes) -> "CkksEngine":
    return load_key(eng, BLOB_PUBLIC_KEY, blob)


def load_evaluation_key(eng: "CkksEngine", blob: bytes) -> "CkksEngine":
    return load_key(eng, BLOB_EVAL_KEY, blob)


def save_ciphertext(eng: "CkksEngine", t: EncryptedTensor, cell: int = 0) -> bytes:
    """save_ciphertext (ckks_serialize.hpp:124-130) of one cell of a tensor."""
    return _blob_call(lib().hecnn_blob_save_ciphertext, eng.ctx, t.handle, ctypes.c_size_t(cell))


def load_ciphertexts(eng: "CkksEngine", blobs) -> EncryptedTensor:
    """load_ciphertext (ckks_serialize.hpp:133-141) of each blob, as the cells
    of one device tensor (shared level and scale, tensor.hpp:52-62)."""
    blobs = [bytes(b) for b in blobs]
    ptrs = (ctypes.c_void_p * len(blobs))(*[ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p) for b in blobs])
    lens = (ctypes.c_size_t * len(blobs))(*[len(b) for b in blobs])
    h = ctypes.c_void_p()
    _check(lib().hecnn_blob_load_ciphertexts(eng.ctx, ptrs, lens, ctypes.c_size_t(len(blobs)), ctypes.byref(h)))
    return eng._wrap(h)


def load_ciphertext(eng: "CkksEngine", blob: bytes) -> EncryptedTensor:
    return load_ciphertexts(eng, [blob])
