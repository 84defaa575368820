"""Python (ctypes) front-end of the CPU oracle -- TEST INFRASTRUCTURE.

Wraps oracle/liboracle.so (the restatement, oracle.c) and, when present,
oracle/_ref/libtrainc_ref.so (the reference's own exec_base compiled from
/root/reference).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
import this module; the product path never does.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from paper_2303_04759_b200.abi import (BF16, F16, F32, I32, U8, Tensor, make_attrs,
                                       make_tensor)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libtrainc_ref.so")

_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.orc_exec.restype = ctypes.c_int
        _lib.orc_last_error.restype = ctypes.c_char_p
        _lib.orc_quantize_f16.restype = ctypes.c_float
        _lib.orc_quantize_f16.argtypes = [ctypes.c_float]
        _lib.orc_quantize_bf16.restype = ctypes.c_float
        _lib.orc_quantize_bf16.argtypes = [ctypes.c_float]
        _lib.orc_float_to_half_bits.restype = ctypes.c_uint16
        _lib.orc_float_to_half_bits.argtypes = [ctypes.c_float]
        _lib.orc_half_bits_to_float.restype = ctypes.c_float
        _lib.orc_half_bits_to_float.argtypes = [ctypes.c_uint16]
        _lib.orc_rng_new.restype = ctypes.c_void_p
        _lib.orc_rng_new.argtypes = [ctypes.c_uint64]
        _lib.orc_rng_free.argtypes = [ctypes.c_void_p]
        _lib.orc_rng_fill_uniform.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_float, ctypes.c_float]
        _lib.orc_rng_fill_below.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_uint32]
        _lib.orc_dropout_keep_step.restype = ctypes.c_int
        _lib.orc_dropout_keep_step.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                               ctypes.c_float, ctypes.c_uint32]
        _lib.orc_dropout_keep.restype = ctypes.c_int
        _lib.orc_dropout_keep.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_float]
    return _lib


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        if not ref_available():
            raise RuntimeError("oracle/_ref not built (reference tree absent)")
        _ref = ctypes.CDLL(REF_PATH)
        _ref.ref_exec.restype = ctypes.c_int
        _ref.ref_last_error.restype = ctypes.c_char_p
        _ref.ref_float_to_half_bits.restype = ctypes.c_uint16
        _ref.ref_float_to_half_bits.argtypes = [ctypes.c_float]
        _ref.ref_half_bits_to_float.restype = ctypes.c_float
        _ref.ref_half_bits_to_float.argtypes = [ctypes.c_uint16]
        _ref.ref_rng_fill_uniform.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int64,
                                              ctypes.c_float, ctypes.c_float]
        _ref.ref_rng_fill_below.argtypes = [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int64,
                                            ctypes.c_uint32]
        _ref.ref_exec_opt.restype = ctypes.c_int
        _ref.ref_infer.restype = ctypes.c_int
    return _ref


def _np_for(dtype):
    if dtype == I32:
        return np.int32
    if dtype == U8:
        return np.uint8
    return np.float32


class HostTensor:
    """A host array plus its declared dtype (half types are f32 storage on the
    half grid, as in trainc::Tensor, tensor.hpp:22-30)."""

    def __init__(self, arr: np.ndarray, dtype: int = F32):
        self.dtype = dtype
        self.arr = np.ascontiguousarray(arr, dtype=_np_for(dtype))

    def desc(self) -> Tensor:
        return make_tensor(self.arr.ctypes.data, self.dtype, self.arr.shape)


def _as_host(x, dtype=None):
    if isinstance(x, HostTensor):
        return x
    x = np.asarray(x)
    if dtype is None:
        dtype = I32 if x.dtype == np.int32 else F32
    return HostTensor(x, dtype)


def run(op: str, inputs, out_specs, attrs=None, impl: str = "oracle"):
    """Execute `op` on host arrays.  out_specs = [(shape, dtype), ...].
    impl = "oracle" (oracle.c) or "ref" (the reference's exec_base)."""
    ins = [_as_host(x) for x in inputs]
    outs = [HostTensor(np.zeros(s, dtype=_np_for(d)), d) for s, d in out_specs]
    in_arr = (Tensor * max(1, len(ins)))(*[t.desc() for t in ins])
    out_arr = (Tensor * max(1, len(outs)))(*[t.desc() for t in outs])
    a, na, keep = make_attrs(attrs)
    if impl == "oracle":
        L = lib()
        rc = L.orc_exec(op.encode(), in_arr, len(ins), out_arr, len(outs), a, na)
        err = L.orc_last_error
    else:
        L = ref()
        rc = L.ref_exec(op.encode(), in_arr, len(ins), out_arr, len(outs), a, na)
        err = L.ref_last_error
    if rc != 0:
        raise RuntimeError(f"{impl}.{op}: {err().decode()}")
    del keep
    return [o.arr for o in outs]


def ref_opt_matmul(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """The reference's opt dialect matmul (matmul_blocked, backends.hpp:280-304)."""
    A, B = HostTensor(a), HostTensor(b)
    C = HostTensor(np.zeros((a.shape[0], b.shape[1]), np.float32))
    if ref().ref_exec_opt(ctypes.byref(A.desc()), ctypes.byref(B.desc()), None, 0, ctypes.byref(C.desc())) != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return C.arr


def rng_uniform(seed: int, n: int, lo=-1.0, hi=1.0, impl="oracle") -> np.ndarray:
    out = np.empty(n, dtype=np.float32)
    if impl == "oracle":
        r = lib().orc_rng_new(seed)
        lib().orc_rng_fill_uniform(r, out.ctypes.data, n, lo, hi)
        lib().orc_rng_free(r)
    else:
        ref().ref_rng_fill_uniform(seed, out.ctypes.data, n, lo, hi)
    return out


def rng_below(seed: int, n: int, bound: int, impl="oracle") -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    if impl == "oracle":
        r = lib().orc_rng_new(seed)
        lib().orc_rng_fill_below(r, out.ctypes.data, n, bound)
        lib().orc_rng_free(r)
    else:
        ref().ref_rng_fill_below(seed, out.ctypes.data, n, bound)
    return out


def dropout_keep_mask(seed: int, salt: int, n: int, p: float, step: int = 0) -> np.ndarray:
    """keep bits of elements 0..n-1 of a dropout site (step: the Philox
    counter's rng_step word)"""
    L = lib()
    return np.array([L.orc_dropout_keep_step(seed, salt, i, p, step) for i in range(n)], dtype=np.uint8)


__all__ = ["run", "HostTensor", "rng_uniform", "rng_below", "ref_available", "lib", "ref",
           "F32", "F16", "BF16", "I32", "U8", "dropout_keep_mask"]


# --- TNSR format restatement (tensor.hpp:76-139), numpy ------------------------
# "TNSR", u8 code, u8 rank, u64 LE dims, raw LE data.  Codes 0 f32 / 1 f16 are
# the reference's (save_tensor tensor.hpp:80-99, load_tensor :108-133); 2 bf16
# (uint16 bits) and 3 i32 are the backend's extension.
TNSR_NP = {0: "<f4", 1: "<f2", 2: "<u2", 3: "<i4"}


def tnsr_bytes(arr: np.ndarray, code: int) -> bytes:
    a = np.require(arr, TNSR_NP[code], "C")
    head = b"TNSR" + bytes([code, a.ndim]) + np.asarray(a.shape, "<u8").tobytes()
    return head + a.tobytes()


def tnsr_parse(buf: bytes) -> tuple[np.ndarray, int]:
    if buf[:4] != b"TNSR":
        raise ValueError("bad tensor file magic")
    code, rank = buf[4], buf[5]
    if code not in TNSR_NP:
        raise ValueError("bad tensor file header")
    shape = tuple(int(d) for d in np.frombuffer(buf, "<u8", rank, 6))
    off = 6 + 8 * rank
    n = int(np.prod(shape, dtype=np.int64))
    dt = np.dtype(TNSR_NP[code])
    if len(buf) < off + n * dt.itemsize:
        raise ValueError("truncated tensor file")
    return np.frombuffer(buf, dt, n, off).reshape(shape).copy(), code


def ref_tnsr_save(path: str, data: np.ndarray, code: int):
    """The reference's own save_tensor (oracle/_ref) on float data."""
    r = ref()
    a = np.require(data, np.float32, "C")
    shape = (ctypes.c_int64 * max(a.ndim, 1))(*a.shape)
    rc = r.ref_tnsr_save(os.fsencode(path), ctypes.c_void_p(a.ctypes.data), code, a.ndim, shape)
    if rc != 0:
        raise RuntimeError(r.ref_last_error().decode())


def ref_tnsr_load(path: str, cap: int) -> tuple[np.ndarray, int]:
    """The reference's own load_tensor (oracle/_ref): values widened to float."""
    r = ref()
    out = np.empty(cap, np.float32)
    code, rank = ctypes.c_int(), ctypes.c_int()
    shape = (ctypes.c_int64 * 8)()
    rc = r.ref_tnsr_load(os.fsencode(path), ctypes.c_void_p(out.ctypes.data), ctypes.c_int64(cap),
                         ctypes.byref(code), ctypes.byref(rank), shape)
    if rc != 0:
        raise RuntimeError(r.ref_last_error().decode())
    shp = tuple(shape[:rank.value])
    return out[:int(np.prod(shp, dtype=np.int64))].reshape(shp), code.value
