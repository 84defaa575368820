"""Builds the native parts in-tree (the .so files travel to the GPU box with
the repo snapshot; nothing is JIT-compiled or pip-installed).

  paper_2303_04759_b200/lib/libtcb200.so   -- sm_100a kernels + C ABI (nvcc)
  oracle/liboracle.so, oracle/_ref/...     -- CPU checker (make -C oracle)
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "lib")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
BASE = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
        "-Xptxas", "-warn-spills"]
# kernels whose results must be bit-identical to the CPU oracle are compiled
# without FMA contraction
EXACT = {"k_elementwise.cu", "k_reduce.cu", "k_optim.cu", "k_gemm_exact.cu", "fold.cu", "k_closure.cu"}
SOURCES = ["abi.cu", "k_elementwise.cu", "k_reduce.cu", "k_optim.cu", "k_gemm_exact.cu",
           "k_gemm_ops.cu", "k_gemm_tc.cu", "k_attention.cu", "k_flash.cu", "k_closure.cu", "k_transformer.cu",
           "k_layernorm.cu", "k_layernorm_dx.cu", "comm.cu", "fold.cu"]


def _newer(src_list, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in src_list)


def _compile(src, verbose=False):
    srcp = os.path.join(CSRC, src)
    obj = os.path.join(OBJ, src.replace(".cu", ".o"))
    deps = [srcp] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith(".cuh")]
    deps.append(os.path.join(ROOT, "include", "tcb200.h"))
    if not _newer(deps, obj):
        return obj
    cmd = [NVCC, *ARCH, *BASE, "-c", srcp, "-o", obj]
    if src in EXACT:
        cmd.insert(1, "-fmad=false")
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build_tcb(verbose=False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(LIB, exist_ok=True)
    with ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), SOURCES))
    out = os.path.join(LIB, "libtcb200.so")
    if _newer(objs, out):
        cmd = [NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return out


def build_oracle() -> None:
    r = subprocess.run(["make", "-C", os.path.join(ROOT, "oracle")], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


def build_all(verbose=False) -> None:
    build_oracle()
    build_tcb(verbose)
    from . import host_build  # C++ host runtime (needs the reference headers at build time)
    host_build.build_host()


if __name__ == "__main__":
    build_oracle()
    print(build_tcb(verbose="-v" in sys.argv))
