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
        L.orc_interp_create_rank.restype = ctypes.c_void_p
        L.orc_interp_create_rank.argtypes = [ctypes.c_char_p, ctypes.c_int]
        L.orc_interp_step_coll.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.POINTER(ctypes.c_float), COLL_FN, ctypes.c_int]
        L.orc_interp_write.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64]
        L.orc_interp_read_grad.restype = ctypes.c_int64
        L.orc_interp_read_grad.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        L.orc_world_create.restype = ctypes.c_void_p
        L.orc_world_create.argtypes = [ctypes.c_char_p, ctypes.c_int]
        L.orc_world_destroy.argtypes = [ctypes.c_void_p]
        L.orc_world_step.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.orc_world_rank.restype = ctypes.c_void_p
        L.orc_world_rank.argtypes = [ctypes.c_void_p, ctypes.c_int]
        _lib = L
    return _lib


# int coll(kind, const float* in, int64 in_n, float* out, int64 out_n, int world, int rank)
COLL_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float), ctypes.c_int64,
                           ctypes.POINTER(ctypes.c_float), ctypes.c_int64, ctypes.c_int, ctypes.c_int)


class World:
    """N ranks of the ZeRO step in lockstep on the deterministic in-process bus
    (SPEC.md:549-556)."""

    def __init__(self, cfg_string: str, n: int):
        h = lib().orc_world_create(cfg_string.encode(), n)
        if not h:
            raise RuntimeError(lib().orc_interp_last_error().decode())
        self.h, self.n = h, n

    def step(self, ids: np.ndarray, labels: np.ndarray) -> np.ndarray:
        """ids/labels: [n, T] per-rank batches"""
        ids = np.ascontiguousarray(ids, np.int32)
        labels = np.ascontiguousarray(labels, np.int32)
        out = np.zeros(self.n, np.float32)
        if lib().orc_world_step(self.h, ids.ctypes.data, labels.ctypes.data, out.ctypes.data):
            raise RuntimeError(lib().orc_interp_last_error().decode())
        return out

    def read(self, rank: int, name: str, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        if lib().orc_interp_read(lib().orc_world_rank(self.h, rank), name.encode(), out.ctypes.data, n):
            raise RuntimeError(lib().orc_interp_last_error().decode())
        return out

    def __del__(self):
        try:
            lib().orc_world_destroy(self.h)
        except Exception:
            pass


class Interp:
    def __init__(self, cfg_string: str, rank: int = 0):
        h = lib().orc_interp_create_rank(cfg_string.encode(), rank)
        if not h:
            raise RuntimeError(lib().orc_interp_last_error().decode())
        self.h = h
        self.rank = rank

    def step(self, ids: np.ndarray, labels: np.ndarray, coll=None) -> float:
        """coll: optional python collective (kind, in[np], out[np], world, rank)
        used for world > 1 collectives (e.g. torch.distributed gloo)."""
        ids = np.ascontiguousarray(ids, np.int32)
        labels = np.ascontiguousarray(labels, np.int32)
        out = ctypes.c_float()
        if coll is None:
            cb = ctypes.cast(None, COLL_FN)
        else:
            def _cb(kind, inp, in_n, outp, out_n, world, rank):
                try:
                    coll(kind, np.ctypeslib.as_array(inp, (in_n,)), np.ctypeslib.as_array(outp, (out_n,)),
                         world, rank)
                    return 0
                except Exception as e:  # noqa: BLE001 - reported through the C status
                    print("collective callback failed:", e)
                    return 1
            cb = COLL_FN(_cb)
        if lib().orc_interp_step_coll(self.h, ids.ctypes.data, labels.ctypes.data, ctypes.byref(out), cb,
                                      self.rank):
            raise RuntimeError(lib().orc_interp_last_error().decode())
        return float(out.value)

    def read(self, name: str, n: int) -> np.ndarray:
        out = np.empty(n, np.float32)
        if lib().orc_interp_read(self.h, name.encode(), out.ctypes.data, n):
            raise RuntimeError(lib().orc_interp_last_error().decode())
        return out

    def write(self, name: str, arr: np.ndarray):
        arr = np.ascontiguousarray(arr)
        assert arr.itemsize == 4
        if lib().orc_interp_write(self.h, name.encode(), arr.ctypes.data, arr.size):
            raise RuntimeError(lib().orc_interp_last_error().decode())

    def grad(self) -> np.ndarray:
        """The flat f32 gradient the optimizer consumed in the last step."""
        n = lib().orc_interp_read_grad(self.h, None, 0)
        out = np.empty(n, np.float32)
        lib().orc_interp_read_grad(self.h, out.ctypes.data, n)
        return out

    def __del__(self):
        try:
            lib().orc_interp_destroy(self.h)
        except Exception:
            pass
