"""Declarative b200 fusion patterns:
names, priorities, root ops, `disable_patterns`, and the spec's priority
monotonicity -- switching a pattern off drops its matches to zero and leaves
every other pattern's matches unchanged -- plus value equivalence of the
graphs with a pattern off (CPU interpreter)."""
import numpy as np
import pytest

from oracle.interp_py import Interp
from paper_2303_04759_b200.session import ModelConfig, graph_text, synthetic_batch


def census(cfg):
    out = {}
    for line in graph_text(cfg, "fusion").splitlines():
        name, prio, root, n = line.split()
        out[name] = (int(prio), root, int(n))
    return out


def test_pattern_table_priorities_unique_and_descending_roots():
    c = census(ModelConfig.tiny())
    prios = [p for n, (p, r, k) in c.items() if n.startswith("b200.")]
    assert len(set(prios)) == len(prios)
    assert {r for n, (p, r, k) in c.items() if n.startswith("b200.")} >= {"gelu_dx", "layer_norm_dx", "colsum"}


@pytest.mark.parametrize("which", ["b200.dgrad_saved_deriv_epilogue", "b200.ln_dx_residual_dy2",
                                   "b200.ln_dx_bias_grad", "b200.ce_masked_colsum", "b200.tied_embedding_base",
                                   "b200.dgrad_wgrad_pair", "b200.ln_post_dropout", "b200.ln_dx_in_dropout"])
def test_disabling_a_pattern_zeroes_it_and_leaves_others(which):
    base = ModelConfig.bert_base(B=2)
    full = census(base)
    assert full[which][2] > 0
    off = census(ModelConfig.bert_base(B=2, disable_patterns=which))
    assert off[which][2] == 0
    for name, (p, r, k) in full.items():
        if name != which and name.startswith("b200."):
            assert off[name][2] == k, (which, name, k, off[name][2])


def test_unknown_pattern_name_is_an_error():
    with pytest.raises(RuntimeError, match="no fusion pattern"):
        graph_text(ModelConfig.tiny(disable_patterns="b200.nonexistent"), "fusion")


@pytest.mark.parametrize("which", ["b200.dgrad_gelu_epilogue", "b200.ln_dx_residual_dy2", "b200.ln_dx_bias_grad",
                                   "b200.ce_masked_colsum", "b200.tied_embedding_base"])
def test_pattern_off_is_value_equivalent(which):
    """f32 steps (save_deriv=0 so the GELU' epilogue pattern fires): the
    interpreter with the pattern off equals the fused one within 1e-6."""
    kw = dict(kind="bert", L=1, H=64, A=2, F=128, V=128, S=16, B=2, dtype="f32", opt="sgd", lr=0.0)
    c1 = ModelConfig(**kw)
    c0 = ModelConfig(**kw, disable_patterns=which)
    ids, labels = synthetic_batch(c1)
    k1 = c1.cfg_string(model_only=True) + ";save_deriv=0"
    k0 = c0.cfg_string(model_only=True) + ";save_deriv=0"
    o1, o0 = Interp(k1), Interp(k0)
    l1, l0 = o1.step(ids, labels), o0.step(ids, labels)
    assert abs(l1 - l0) <= 1e-6 * abs(l0)
    g1, g0 = o1.grad().astype(np.float64), o0.grad().astype(np.float64)
    assert np.linalg.norm(g1 - g0) <= 1e-6 * np.linalg.norm(g0)


def test_pattern_fusion_strictly_cuts_instructions():
    """kernel invocations after fusion < before (the IR's call
    lets: every one is a launch or an alias)."""
    def calls(c):
        return sum(1 for l in graph_text(c, "ir").splitlines() if "= b200." in l and ".view(" not in l)
    assert calls(ModelConfig.bert_base(B=2)) < calls(ModelConfig.bert_base(B=2, fuse=0))


def test_attention_saved_mask_on_the_autocast_graph():
    """b200.attention_saved_mask: the AutoCast'd all-f32 BERT step gets the
    hand-built graph's stored attention keep bits (every attention stores them,
    every attention_dx reads them), and the interpreter of that graph equals
    the one with the pattern off bit for bit (same Philox bits)."""
    kw = dict(kind="bert", L=2, H=128, A=2, F=256, V=128, S=16, B=2, dtype="f32", opt="adam", lr=1e-3, p=0.1)
    c1 = ModelConfig(**kw)
    c1.extra["autocast"] = "b200+fold+fuse"
    ir = graph_text(c1, "ir")
    att = [l for l in ir.splitlines() if "= b200.attention(" in l]
    dx = [l for l in ir.splitlines() if "= b200.attention_dx(" in l]
    assert att and all("save_mask=1" in l for l in att) and all("save_mask=1" in l for l in dx)
    c0 = ModelConfig(**kw, disable_patterns="b200.attention_saved_mask")
    c0.extra["autocast"] = "b200+fold+fuse"
    assert "save_mask=1" not in "".join(l for l in graph_text(c0, "ir").splitlines() if "attention" in l)
    ids, labels = synthetic_batch(c1)
    o1 = Interp(c1.cfg_string(model_only=True) + ";autocast=b200+fold+fuse")
    o0 = Interp(c0.cfg_string(model_only=True) + ";autocast=b200+fold+fuse")
    for _ in range(2):
        l1, l0 = o1.step(ids, labels), o0.step(ids, labels)
        assert np.float32(l1).tobytes() == np.float32(l0).tobytes()
    assert o1.grad().tobytes() == o0.grad().tobytes()


def test_embedding_sum_pattern_on_the_autocast_graph():
    """b200.embedding_sum: under the b200 policy the AutoCast'd BERT front is
    the hand-built one (one embedding_sum gather-and-add over the bf16 tables,
    LayerNorm with its output dropout); the interpreter equals the graph with
    the pattern off bit for bit (the kernel rounds each add like the chain)."""
    kw = dict(kind="bert", L=1, H=128, A=2, F=256, V=128, S=16, B=2, dtype="f32", opt="adam", lr=1e-3, p=0.1)
    c1 = ModelConfig(**kw)
    c1.extra["autocast"] = "b200+fold+fuse"
    ir = graph_text(c1, "ir")
    assert ir.count("= b200.embedding_sum(") == 1 and "= b200.embedding(" not in ir
    c0 = ModelConfig(**kw, disable_patterns="b200.embedding_sum")
    c0.extra["autocast"] = "b200+fold+fuse"
    assert graph_text(c0, "ir").count("= b200.embedding(") == 3
    ids, labels = synthetic_batch(c1)
    o1 = Interp(c1.cfg_string(model_only=True) + ";autocast=b200+fold+fuse")
    o0 = Interp(c0.cfg_string(model_only=True) + ";autocast=b200+fold+fuse")
    for _ in range(2):
        l1, l0 = o1.step(ids, labels), o0.step(ids, labels)
        assert np.float32(l1).tobytes() == np.float32(l0).tobytes()
    assert o1.grad().tobytes() == o0.grad().tobytes()
