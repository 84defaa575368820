"""ctypes loader for libtcb200.so plus a thin op-level helper.

The product path is native (C ABI -> sm_100a kernels); this module only binds
it.  If the library is missing or the device is not sm_100 every call raises --
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

from .abi import (BF16, F16, F32, I32, U8, Attr, Tensor, make_attrs, make_tensor)

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "lib", "libtcb200.so")

_lib = None


class TcbError(RuntimeError):
    """Non-zero status from libtcb200; .code is the TCB_ERR_* value."""

    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class UnimplementedOp(TcbError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libtcb200.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.tcb_last_error.restype = ctypes.c_char_p
        L.tcb_plan_key.restype = ctypes.c_char_p
        L.tcb_supported_ops.restype = ctypes.c_char_p
        L.tcb_plan_create.argtypes = [ctypes.c_char_p, ctypes.POINTER(Tensor), ctypes.c_int,
                                      ctypes.POINTER(Tensor), ctypes.c_int, ctypes.POINTER(Attr),
                                      ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p)]
        L.tcb_launch.argtypes = [ctypes.c_void_p, ctypes.POINTER(Tensor), ctypes.c_int,
                                 ctypes.POINTER(Tensor), ctypes.c_int, ctypes.c_void_p]
        L.tcb_plan_destroy.argtypes = [ctypes.c_void_p]
        L.tcb_plan_num_kernels.argtypes = [ctypes.c_void_p]
        L.tcb_plan_key.argtypes = [ctypes.c_void_p]
        L.tcb_init.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
        _lib = L
    return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().tcb_last_error().decode()
        if rc == 1:
            raise UnimplementedOp(rc, msg)
        raise TcbError(rc, msg)


def supported_ops() -> list[str]:
    return lib().tcb_supported_ops().decode().split()


def _torch_dtype_code(t) -> int:
    import torch
    return {torch.float32: F32, torch.float16: F16, torch.bfloat16: BF16, torch.int32: I32,
            torch.uint8: U8}[t.dtype]


def _torch_dtype(code: int):
    import torch
    return {F32: torch.float32, F16: torch.float16, BF16: torch.bfloat16, I32: torch.int32,
            U8: torch.uint8}[code]


class Plan:
    """A tcb_plan: one shape-specialised b200 kernel launch plan."""

    def __init__(self, op: str, in_specs, out_specs, attrs=None, closure_hash=None):
        L = lib()
        self.op = op if "." in op else "b200." + op
        self.in_specs = [(tuple(s), d) for s, d in in_specs]
        self.out_specs = [(tuple(s), d) for s, d in out_specs]
        ins = (Tensor * max(1, len(in_specs)))(*[make_tensor(0, d, s) for s, d in in_specs])
        outs = (Tensor * max(1, len(out_specs)))(*[make_tensor(0, d, s) for s, d in out_specs])
        a, na, keep = make_attrs(attrs)
        h = ctypes.c_void_p()
        check(L.tcb_plan_create(self.op.encode(), ins, len(in_specs), outs, len(out_specs), a, na,
                                closure_hash.encode() if closure_hash else None, ctypes.byref(h)))
        del keep
        self.h = h

    @property
    def key(self) -> str:
        return lib().tcb_plan_key(self.h).decode()

    @property
    def num_kernels(self) -> int:
        return lib().tcb_plan_num_kernels(self.h)

    def launch(self, in_ptrs, out_ptrs, stream=None):
        ins = (Tensor * max(1, len(in_ptrs)))(
            *[make_tensor(p, d, s) for p, (s, d) in zip(in_ptrs, self.in_specs)])
        outs = (Tensor * max(1, len(out_ptrs)))(
            *[make_tensor(p, d, s) for p, (s, d) in zip(out_ptrs, self.out_specs)])
        check(lib().tcb_launch(self.h, ins, len(in_ptrs), outs, len(out_ptrs), stream))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().tcb_plan_destroy(self.h)
        except Exception:
            pass


def run_op(op: str, inputs, out_specs, attrs=None, outs=None):
    """Run one b200 op on CUDA torch tensors (test/bench helper).
    out_specs: [(shape, dtype_code)]; returns freshly allocated outputs."""
    import torch
    in_specs = [(tuple(t.shape), _torch_dtype_code(t)) for t in inputs]
    for t in inputs:
        assert t.is_cuda and t.is_contiguous()
    plan = Plan(op, in_specs, out_specs, attrs)
    if outs is None:
        outs = [torch.empty(s, dtype=_torch_dtype(d), device=inputs[0].device) for s, d in out_specs]
    stream = torch.cuda.current_stream().cuda_stream
    plan.launch([t.data_ptr() for t in inputs], [o.data_ptr() for o in outs], stream)
    return outs
