"""Text IR (text.hpp) for b200 step graphs through host/text_ext.hpp.

The reference printer labels every non-f32 dtype "f16" and its lexer reads
`%t.0` as one identifier, so neither a bf16 step nor a tuple field survives its
own round trip.  The extension spells bf16/i32 parameter tokens and prints
tuple fields as `%t .0`.  Checks: print -> parse -> print is byte-identical,
types re-infer to the builder's, and parse errors surface.
"""
import os
import subprocess

import pytest

from paper_2303_04759_b200.session import ModelConfig, graph_text, text_reprint

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = os.environ.get("TRAINC_REF_INC", "/root/reference/proj/include")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_INC, "trainc")), reason="reference headers absent")
def test_text_roundtrip_cpp(tmp_path):
    exe = str(tmp_path / "text_rt")
    r = subprocess.run(["g++", "-std=c++20", "-O1", f"-I{REF_INC}", f"-I{ROOT}/paper_2303_04759_b200/host",
                        f"-I{ROOT}/include", "-o", exe, f"{ROOT}/tests/cpp/text_roundtrip_test.cpp"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr


@pytest.mark.parametrize("cfg", [ModelConfig.tiny(), ModelConfig.tiny(dtype="bf16", opt="adam"),
                                 ModelConfig.bert_base(B=2)])
def test_dispatched_step_text_roundtrip(cfg):
    t = graph_text(cfg, "text")
    head = t.splitlines()[0]
    assert "%ids: i32[" in head
    if cfg.dtype == "bf16":
        assert "%p16: bf16[" in head
    assert "b200." in t  # the dispatched dialect ops
    assert text_reprint(t) == t


def test_parse_errors_surface():
    with pytest.raises(RuntimeError, match="unknown dtype|dtype"):
        text_reprint("fn main(%x: q8[2]) {\n  %x\n}\n")
    with pytest.raises(RuntimeError):
        text_reprint("fn main(%x: f32[2]) {\n  let %y = add(%x, %nope);\n  %y\n}\n")
