"""Build the C++ host runtime libtrainc_b200.so (capi.cpp + headers in host/).

It is compiled against the reference's public headers
(/root/reference/proj/include: IR, registry, KernelCache) -- the b200 backend
plugs into that API -- and links libtcb200.so.  The .so is built in-tree and
travels with the repo snapshot; on a box without the reference tree the
prebuilt library is used as is.
"""
from __future__ import annotations

import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
REF_INC = os.environ.get("TRAINC_REF_INC", "/root/reference/proj/include")
OUT = os.path.join(PKG, "lib", "libtrainc_b200.so")
CXXFLAGS = ["-std=c++20", "-O2", "-fPIC", "-Wall", "-Wno-unused-variable", "-Wno-unused-function"]


def _sources():
    hs = [os.path.join(PKG, "host", f) for f in os.listdir(os.path.join(PKG, "host"))]
    return hs + [os.path.join(ROOT, "include", h) for h in ("tcb200.h", "trainc_b200.h")]


def build_host(force: bool = False) -> str:
    if not os.path.isdir(os.path.join(REF_INC, "trainc")):
        if os.path.exists(OUT):
            return OUT  # prebuilt (GPU box: the reference tree is not present)
        raise RuntimeError(f"reference headers not found at {REF_INC} and no prebuilt {OUT}")
    if not force and os.path.exists(OUT):
        t = os.path.getmtime(OUT)
        if all(os.path.getmtime(s) <= t for s in _sources()):
            return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = ["g++", *CXXFLAGS, f"-I{REF_INC}", f"-I{os.path.join(ROOT, 'include')}",
           "-shared", "-o", OUT, os.path.join(PKG, "host", "capi.cpp"),
           f"-L{os.path.join(PKG, 'lib')}", "-ltcb200", "-Wl,-rpath,$ORIGIN"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"host build failed:\n{r.stderr[-8000:]}")
    return OUT


if __name__ == "__main__":
    print(build_host(force=True))
