"""distpar overlap + horizontal fusion on CPU.

* hoist_collectives + the two-stream timeline on hand-written graphs: the
  SPEC's examples (a collective depending on the first of two independent
  computes overlaps the second -- equal to the brute-force optimal two-stream
  schedule; no collectives -> no events, makespan unchanged; a serial chain ->
  makespan = sum of costs) and the structural rule that every cross-stream
  edge's wait comes after its signal;
* on the ZeRO training steps: collectives are on the comm stream, overlap <
  serial, and horizontal fusion (buckets) strictly cuts the collective count
  and the events.
"""
import itertools
import re

import pytest

from paper_2303_04759_b200.session import ModelConfig, graph_text, memsched_text


def overlap(text):
    out = memsched_text(text, "overlap").splitlines()
    head = {l.split()[0]: float(l.split()[1]) for l in out[:3]}
    ops = {}
    order = []
    for l in out[3:]:
        _, v, st, a, b, w = l.split()
        ops[v] = dict(stream=int(st), start=float(a), end=float(b), wait=None if w == "-" else w)
        order.append(v)
    return head, ops, order


DAG = '''fn f(%x: f32[1000], %y: f32[4000]) {
  let %a = tanh(%x);
  let %b = neg(%y);
  let %c @{op.world=2} = allreduce(%a);
  let %s @{op.axes="0"} = sum(%b);
  let %d = add(%c, %s);
  %d
}'''


def test_collective_overlaps_the_independent_compute():
    """the allreduce depends on a only; it runs on the comm stream
    while b and s compute; the makespan equals the brute-force optimum over
    every compute-stream order (the comm stream has one op)."""
    head, ops, order = overlap(DAG)
    assert ops["c"]["stream"] == 1 and all(ops[v]["stream"] == 0 for v in "absd")
    assert order.index("c") == order.index("a") + 1  # hoisted right behind its producer
    cost = {v: ops[v]["end"] - ops[v]["start"] for v in ops}
    assert ops["c"]["start"] == ops["a"]["end"]
    # brute force: all topological orders of the compute ops {a, b, s, d}
    deps = {"a": set(), "b": set(), "s": {"b"}, "d": {"c", "s"}, "c": {"a"}}
    best = None
    for perm in itertools.permutations("abs"):
        if perm.index("s") < perm.index("b"):
            continue
        t, end = 0.0, {}
        for v in perm:
            t = max([t] + [end[d] for d in deps[v] if d in end])
            t += cost[v]
            end[v] = t
            if v == "a":
                end["c"] = t + cost["c"]
        m = max(t, end["c"]) + cost["d"]
        best = m if best is None else min(best, m)
    assert head["overlap"] == best < head["serial"]
    assert head["serial"] == sum(cost.values())


def test_no_collectives_no_events_and_serial_chain():
    t = '''fn f(%x: f32[100]) {
  let %a = tanh(%x);
  let %b = neg(%x);
  let %c = add(%a, %b);
  %c
}'''
    head, ops, _ = overlap(t)
    assert head["events"] == 0 and head["overlap"] == head["serial"]
    chain = '''fn f(%x: f32[100]) {
  let %a = tanh(%x);
  let %b @{op.world=2} = allreduce(%a);
  let %c = neg(%b);
  let %d @{op.world=2} = allreduce(%c);
  %d
}'''
    head, ops, _ = overlap(chain)
    assert head["overlap"] == head["serial"]  # fully serial: nothing to overlap
    assert head["events"] == 3                # a->b, b->c, c->d cross streams


def _check_signal_before_wait(ops):
    for v, o in ops.items():
        if o["wait"] is not None:
            p = ops[o["wait"]]
            assert p["stream"] != o["stream"]
            assert p["end"] <= o["start"], (v, o, p)


@pytest.mark.parametrize("kind", ["bert", "gpt2"])
def test_zero_step_streams_and_makespans(kind):
    """The ZeRO step (world 2, bf16 Adam): every collective on the comm
    stream, every compute op on the compute stream, each cross-stream edge's
    wait after its signal; overlap < serial; horizontal fusion into buckets
    (bucket_mb > 0 vs one bucket per segment) strictly reduces the number of
    collectives and of events."""
    base = dict(kind=kind, L=2, H=64, A=2, F=128, V=256, S=32, B=2, dtype="bf16", opt="adam", world=2)
    c = ModelConfig(**base, bucket_mb=0.05)
    head, ops, order = overlap(graph_text(c, "text"))
    text = graph_text(c, "text")
    coll = set(re.findall(r"let %(\w+)(?: @\{[^}]*\})? = b200\.(?:reduce_scatter|all_gather)\(", text))
    assert coll and all(ops[v]["stream"] == 1 for v in coll)
    assert all(o["stream"] == 0 for v, o in ops.items() if v not in coll)
    _check_signal_before_wait(ops)
    assert head["overlap"] < head["serial"]
    t_fused = {l.split()[0]: float(l.split()[1]) for l in graph_text(c, "timeline").splitlines()}
    c0 = ModelConfig(**base, bucket_mb=0)
    t_unfused = {l.split()[0]: float(l.split()[1]) for l in graph_text(c0, "timeline").splitlines()}
    assert t_fused["collectives"] < t_unfused["collectives"]
    assert t_fused["events"] < t_unfused["events"]
    assert t_fused["overlap"] <= t_fused["serial"] and t_unfused["overlap"] <= t_unfused["serial"]


def test_reduce_scatters_start_inside_the_backward():
    """On BERT-base world 8 (25 MB buckets) the first gradient bucket's
    reduce-scatter is scheduled long before the end of the backward: the
    collective is hoisted behind its bucket's last producer."""
    c = ModelConfig.bert_base(B=32, world=8)
    text = graph_text(c, "text")
    lets = [l for l in text.splitlines() if l.strip().startswith("let ")]
    rs = [i for i, l in enumerate(lets) if "b200.reduce_scatter(" in l]
    opt = [i for i, l in enumerate(lets) if "adam_update" in l][0]
    assert len(rs) > 4
    assert rs[0] < opt - 100, (rs[:3], opt)
    buckets = [tuple(int(x) for x in l.split()) for l in graph_text(c, "buckets").splitlines()]
    assert all(n % 8 == 0 for _, n, _ in buckets)  # NCCL: every bucket splits into equal shards
    assert sum(n for _, n, _ in buckets) == int(re.search(r"%params: f32\[(\d+)\]", text).group(1)) * 8
