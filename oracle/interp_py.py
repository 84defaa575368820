"""ctypes front-end of oracle/liboracle_interp.so -- the CPU ANF interpreter
over the oracle kernels (TEST INFRASTRUCTURE; see interp.cpp)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle_interp.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"{LIB} not built (make -C oracle)")
        L = ctypes.CDLL(LIB)
        L.orc_interp_create.restype = ctypes.c_void_p
        L.orc_interp_create.argtypes = [ctypes.c_char_p]
        L.orc_interp_destroy.argtypes = [ctypes.c_void_p]
        L.orc_interp_step.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                      ctypes.POINTER(ctypes.c_float)]
        L.orc_interp_read.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64]
        L.orc_interp_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


class Interp:
    def __init__(self, cfg_string: str):
        h = lib().orc_interp_create(cfg_string.encode())
        if not h:
            raise RuntimeError(lib().orc_interp_last_error().decode())
        self.h = h

    def step(self, ids: np.ndarray, labels: np.ndarray) -> float:
        ids = np.ascontiguousarray(ids, np.int32)
        labels = np.ascontiguousarray(labels, np.int32)
        out = ctypes.c_float()
        if lib().orc_interp_step(self.h, ids.ctypes.data, labels.ctypes.data, ctypes.byref(out)):
            raise RuntimeError(lib().orc_interp_last_error().decode())
        return float(out.value)

    def read(self, name: str, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        if lib().orc_interp_read(self.h, name.encode(), out.ctypes.data, n):
            raise RuntimeError(lib().orc_interp_last_error().decode())
        return out

    def __del__(self):
        try:
            lib().orc_interp_destroy(self.h)
        except Exception:
            pass
