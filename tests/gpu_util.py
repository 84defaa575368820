"""Shared helpers for the GPU parity tests: run one op through libtcb200 (the
product, on cuda:0) and through the CPU oracle on identical inputs."""
from __future__ import annotations

import numpy as np

from oracle import oracle_py as O
from paper_2303_04759_b200.abi import BF16, F16, F32, I32, U8, bf16_round

_NP_HALF = {F16: np.float16}


def quantize(x: np.ndarray, dtype: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    if dtype == BF16:
        return bf16_round(x)
    if dtype == F16:
        return x.astype(np.float16).astype(np.float32)
    return x


def to_torch(x: np.ndarray, dtype: int):
    import torch
    if dtype == I32:
        return torch.from_numpy(np.ascontiguousarray(x, dtype=np.int32)).cuda()
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    return t.to({F32: torch.float32, F16: torch.float16, BF16: torch.bfloat16}[dtype]).contiguous()


def from_torch(t) -> np.ndarray:
    import torch
    if t.dtype in (torch.int32, torch.uint8):
        return t.cpu().numpy()
    return t.float().cpu().numpy()


def run_both(op, inputs, out_specs, attrs=None):
    """inputs: list of (np array, dtype).  Returns (gpu_outs, oracle_outs) as
    float32/int32 numpy arrays."""
    from paper_2303_04759_b200.runtime import run_op
    qin = [(quantize(x, d) if d not in (I32, U8) else np.asarray(x), d) for x, d in inputs]
    g = run_op(op, [to_torch(x, d) for x, d in qin], out_specs, attrs)
    import torch
    torch.cuda.synchronize()
    o = O.run(op, [O.HostTensor(x, d) for x, d in qin], out_specs, attrs)
    return [from_torch(t) for t in g], o


def bits_equal(a: np.ndarray, b: np.ndarray) -> bool:
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    if a.dtype == np.float32:
        return np.array_equal(a.view(np.uint32), b.view(np.uint32)) or np.array_equal(a, b)
    return np.array_equal(a, b)


def rel_err(a: np.ndarray, b: np.ndarray) -> float:
    """Norm-wise relative error (max_rel_error's 1e-9
    floor makes elementwise relative error meaningless near zero)."""
    a = a.astype(np.float64).ravel()
    b = b.astype(np.float64).ravel()
    d = np.linalg.norm(a - b)
    n = max(np.linalg.norm(b), 1e-30)
    return float(d / n)


def max_ulp_bf16(a: np.ndarray, b: np.ndarray) -> int:
    """max distance in bf16 ulps between two arrays of bf16-grid values"""
    ai = (np.ascontiguousarray(a, np.float32).view(np.int32) >> 16).astype(np.int64)
    bi = (np.ascontiguousarray(b, np.float32).view(np.int32) >> 16).astype(np.int64)
    # map sign-magnitude to a monotone integer line
    ai = np.where(ai < 0, -(ai & 0x7FFF), ai)
    bi = np.where(bi < 0, -(bi & 0x7FFF), bi)
    return int(np.max(np.abs(ai - bi))) if a.size else 0
