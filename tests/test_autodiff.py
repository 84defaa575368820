"""Autodiff pass (host/graph.hpp).

tests/cpp/autodiff_test.cpp checks dependency_report's known answers (tanh ->
{y}, matmul -> both inputs, add -> {}), the fan-out accumulation chain, the
NeedsY-vs-NeedsBoth liveness property and determinism on hand-built graphs.
Gradient VALUES are pinned by tests/test_step_independent.py (torch f64 and
finite differences) and per op by tests/test_oracle_torch.py.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = os.environ.get("TRAINC_REF_INC", "/root/reference/proj/include")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_INC, "trainc")), reason="reference headers absent")
def test_autodiff_spec_examples_cpp(tmp_path):
    exe = str(tmp_path / "autodiff_test")
    r = subprocess.run(["g++", "-std=c++20", "-O1", f"-I{REF_INC}", f"-I{ROOT}/paper_2303_04759_b200/host",
                        f"-I{ROOT}/include", "-o", exe, f"{ROOT}/tests/cpp/autodiff_test.cpp"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
