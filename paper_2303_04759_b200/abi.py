"""ctypes mirror of include/tcb200.h (the C ABI of libtcb200.so).

Only plain structs and dtype helpers live here; the loader is in
``paper_2303_04759_b200.runtime``.
"""
from __future__ import annotations

import ctypes

import numpy as np

F32, F16, BF16, I32, U8 = 0, 1, 2, 3, 4
DTYPE_NAMES = {F32: "f32", F16: "f16", BF16: "bf16", I32: "i32", U8: "u8"}
DTYPE_CODES = {v: k for k, v in DTYPE_NAMES.items()}
DTYPE_BYTES = {F32: 4, F16: 2, BF16: 2, I32: 4, U8: 1}

ATTR_INT, ATTR_FLOAT, ATTR_STR = 0, 1, 2


class Tensor(ctypes.Structure):
    """tcb_tensor / orc_tensor (identical layouts)."""

    _fields_ = [
        ("ptr", ctypes.c_void_p),
        ("dtype", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("shape", ctypes.c_int64 * 8),
        ("stride", ctypes.c_int64 * 8),
    ]


class Attr(ctypes.Structure):
    """tcb_attr / orc_attr: mirrors ir::AttrValue (ir.hpp:29-30)."""

    _fields_ = [
        ("key", ctypes.c_char_p),
        ("kind", ctypes.c_int32),
        ("i", ctypes.c_int64),
        ("d", ctypes.c_double),
        ("s", ctypes.c_char_p),
    ]


def make_tensor(ptr: int, dtype: int, shape) -> Tensor:
    t = Tensor()
    t.ptr = ptr
    t.dtype = dtype
    t.rank = len(shape)
    for i, d in enumerate(shape):
        t.shape[i] = int(d)
    return t


def make_attrs(attrs: dict | None):
    """dict -> (Attr array, keepalive list).  bool/int -> int, float -> float,
    str -> str, exactly the AttrValue variant."""
    attrs = attrs or {}
    arr = (Attr * max(1, len(attrs)))()
    keep = []
    for i, (k, v) in enumerate(attrs.items()):
        kb = k.encode()
        keep.append(kb)
        arr[i].key = kb
        if isinstance(v, bool) or isinstance(v, (int, np.integer)):
            arr[i].kind = ATTR_INT
            arr[i].i = int(v)
        elif isinstance(v, (float, np.floating)):
            arr[i].kind = ATTR_FLOAT
            arr[i].d = float(v)
        else:
            vb = str(v).encode()
            keep.append(vb)
            arr[i].kind = ATTR_STR
            arr[i].s = vb
    return arr, len(attrs), keep


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest-even bf16 value, returned as float32 (same contract as
    oracle.c orc_quantize_bf16 and __float2bfloat16_rn)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF
    r = np.where(nan, ((u >> 16) | 0x40) & 0xFFFF, r)
    return (r.astype(np.uint32) << 16).view(np.float32).reshape(x.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 (already on the bf16 grid or not) -> uint16 bf16 bits (RNE)."""
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)


def bf16_from_bits(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)
