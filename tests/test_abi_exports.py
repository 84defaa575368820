"""The drop-in boundary loads on a CPU-only host and exports every function its
header declares: include/tcb200.h -> libtcb200.so, include/trainc_b200.h ->
libtrainc_b200.so (no compute calls; those need the GPU)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2303_04759_b200", "lib")

DECL = re.compile(r"^[A-Za-z_][\w\s\*]*?\b(tc?b_\w+)\s*\(", re.M)


def declared(header):
    with open(os.path.join(ROOT, "include", header)) as f:
        src = re.sub(r"/\*.*?\*/", "", f.read(), flags=re.S)
    return sorted(set(DECL.findall(src)))


@pytest.mark.parametrize("header,lib", [("tcb200.h", "libtcb200.so"), ("trainc_b200.h", "libtrainc_b200.so")])
def test_library_exports_every_declared_symbol(header, lib):
    names = declared(header)
    assert len(names) > 10, names
    path = os.path.join(LIB, lib)
    if not os.path.exists(path):
        pytest.skip(f"{lib} not built")
    ctypes.CDLL(os.path.join(LIB, "libtcb200.so"), mode=ctypes.RTLD_GLOBAL)
    L = ctypes.CDLL(path)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_headers_compile_as_c():
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "t.c")
        with open(src, "w") as f:
            f.write('#include "tcb200.h"\n#include "trainc_b200.h"\nint main(void){return 0;}\n')
        r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-c", src,
                            "-o", os.path.join(d, "t.o")], capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
