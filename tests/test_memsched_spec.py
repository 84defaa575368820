"""memsched against the SPEC's own oracles (VERDICT r1
"missing" item 3), on hand-written text-IR graphs and on the training steps,
through tb_memsched_text / graph_text (CPU only).

Independent checkers written here, not shared with the C++ planner:
  * `Trace`: a dynamic reference-counting trace of a let sequence (allocate a
    let's outputs when it runs, drop a storage root when its remaining-use
    count reaches zero) -- SPEC.md:450 "oracle = runtime refcount trace";
  * `enumerate_orders`: every topological order of a small DAG evaluated with
    the same accounting -- SPEC.md:464 "oracle = exhaustive topological-order
    enumeration (n <= 10)".

Accounting models.  SPEC.md:431 says params live over the whole function (the
device VM: inputs are persistent buffers) -- `transient=False`.  The SPEC's
worked examples (:454-458, "chain of 3 ... predecessor freed after each step")
only add up when a function input is freed after its last use --
`transient=True`.  Both are tested.  The diamond example's "4800 vs 5200"
(:457, :464) is not reproducible under either model as written (both orders
of x->{a,b}->c(a,b) have equal peaks); the
enumeration oracle pins what each order really costs, and a curated graph
where order matters checks that schedule() reaches the optimum.
"""
import itertools
import re

import numpy as np
import pytest

from paper_2303_04759_b200.session import ModelConfig, graph_info, graph_text, memsched_text

ALIAS = {"view", "reshape"}


def base(op):
    return op.split(".")[-1]


# ------------------------------------------------------------------ parsing
LET = re.compile(r"let %([\w.]+)(?: @\{.*?\})? = (?:([\w.]+)\((.*?)\)|%([\w.]+) \.(\d+));$")


def parse(text):
    """-> params [(id, bytes)], lets [(id, op|None, [arg ids], tuple_src, field)], ret ids"""
    head = text.splitlines()[0]
    params = []
    for pid, dt, shape in re.findall(r"%([\w.]+): (\w+)\[([\d, ]*)\]", head):
        n = int(np.prod([int(d) for d in shape.split(",") if d.strip()] or [1]))
        params.append((pid, n * (2 if dt in ("bf16", "f16") else 4)))
    lets = []
    ret = []
    for line in text.splitlines()[1:]:
        line = line.strip()
        m = LET.match(line)
        if m:
            vid, op, args, src, fld = m.groups()
            if op:
                lets.append((vid, op, re.findall(r"%([\w.]+)", args), None, None))
            else:
                lets.append((vid, None, [src], src, int(fld)))
        elif line.startswith("%") or line.startswith("("):
            ret = re.findall(r"%([\w.]+)", line)
    return params, lets, ret


def sizes_from_liveness(text, transient):
    """(var, field) -> bytes, from the planner's type inference (the types are
    not what is under test; the timing of frees is)."""
    out = {}
    for line in memsched_text(text, "liveness", 0, transient).splitlines():
        v, k, _u, _d, _l, b = line.split()
        out[(v, int(k))] = int(b)
    return out


# ---------------------------------------------------------------- the trace
class Trace:
    """Dynamic refcount execution of a let sequence (no def/last intervals).
    Storage roots: one per field of every non-alias Call; view/reshape and
    tuple_get alias their source.  Uses by alias lets count as uses."""

    def __init__(self, params, lets, ret, size, transient):
        self.root = {}      # (var, field) -> root id
        self.bytes = {}     # root -> bytes
        self.pinned = set()
        for pid, b in params:
            self.root[(pid, 0)] = pid
            self.bytes[pid] = b
            if not transient:
                self.pinned.add(pid)
        nfields = {}
        for vid, op, args, src, fld in lets:
            nfields[vid] = max(nfields.get(vid, 0), 1)
            if src is not None:
                nfields[src] = max(nfields.get(src, 1), fld + 1)
        self.lets, self.ret, self.size, self.nfields = lets, ret, size, nfields

    def run(self):
        remaining = {}

        def roots_of(v):
            return [self.root[(v, k)] for k in range(self.nfields.get(v, 1)) if (v, k) in self.root]

        # count uses per root (requires the alias structure: resolve lazily)
        alias_of = {}
        for vid, op, args, src, fld in self.lets:
            if src is not None:
                alias_of[vid] = ("get", src, fld)
            elif base(op) in ALIAS:
                alias_of[vid] = ("alias", args[0], 0)

        def resolve(v, k=0):
            while v in alias_of:
                kind, s, f = alias_of[v]
                v, k = s, (f if kind == "get" else k)
            return v, k

        for vid, op, args, src, fld in self.lets:
            for a in args:
                n = self.nfields.get(a, 1) if resolve(a)[0] == a and a not in alias_of else 1
                if a in alias_of:
                    r = resolve(a)
                    remaining[r] = remaining.get(r, 0) + 1
                else:
                    for k in range(n):
                        remaining[(a, k)] = remaining.get((a, k), 0) + 1
        keep = set()
        for r in self.ret:
            if r in alias_of:
                keep.add(resolve(r))
            else:
                for k in range(self.nfields.get(r, 1)):
                    keep.add((r, k))
        live = {}
        for pid, b in self.bytes.items():
            live[(pid, 0)] = b
        curve, first, last = [], {}, {}
        for i, (vid, op, args, src, fld) in enumerate(self.lets):
            if src is None and base(op) not in ALIAS:
                for k in range(self.nfields.get(vid, 1)):
                    live[(vid, k)] = self.size[(vid, k)]
                    first[(vid, k)] = i
            curve.append(sum(live.values()))
            used = []
            for a in args:
                if a in alias_of:
                    used.append(resolve(a))
                else:
                    used += [(a, k) for k in range(self.nfields.get(a, 1))]
            for r in used:
                last[r] = i
                remaining[r] -= 1
                if remaining[r] == 0 and r not in keep and r[0] not in self.pinned and r in live:
                    del live[r]
            # an output nobody ever reads dies right after its def
            if src is None and base(op) not in ALIAS:
                for k in range(self.nfields.get(vid, 1)):
                    r = (vid, k)
                    if remaining.get(r, 0) == 0 and r not in keep and r in live:
                        del live[r]
                        last.setdefault(r, i)
        return curve, first, last


def trace_text(text, transient):
    params, lets, ret = parse(text)
    size = sizes_from_liveness(text, transient)
    return Trace(params, lets, ret, size, transient).run()


def curve_of(text, transient):
    out = memsched_text(text, "curve", 0, transient).splitlines()
    peak = int(out[0].split()[1])
    return peak, [int(l.split()[1]) for l in out[1:]]


def fn(params, body, ret):
    hdr = ", ".join(f"%{p}: f32[{n}]" for p, n in params)
    return "fn f(" + hdr + ") {\n" + "".join(f"  let %{v} = {e};\n" for v, e in body) + f"  {ret}\n}}\n"


# ------------------------------------------------------- known answers
@pytest.mark.parametrize("transient", [True, False])
def test_single_op_peak_800(transient):
    """one op, 400 B in, 400 B out -> peak 800 B (both models)."""
    t = fn([("x", 100)], [("y", "tanh(%x)")], "%y")
    assert curve_of(t, transient)[0] == 800


def test_chain_of_three_peak():
    """a chain of 3 same-size elementwise ops -> 800 B when the
    predecessor is freed after each step (transient inputs); 1200 B when the
    input x is a persistent param."""
    t = fn([("x", 100)], [("a", "tanh(%x)"), ("b", "neg(%a)"), ("c", "tanh(%b)")], "%c")
    assert curve_of(t, True)[0] == 800
    assert curve_of(t, False)[0] == 1200


def test_liveness_examples():
    """a = f(x); b = g(a); return b -> a live on [0,1], b on
    [1,end]; an unused binding is live only at its def."""
    t = fn([("x", 100)], [("a", "tanh(%x)"), ("u", "neg(%x)"), ("b", "neg(%a)")], "%b")
    rows = {l.split()[0]: l.split() for l in memsched_text(t, "liveness", 0, False).splitlines()}
    assert (int(rows["a"][3]), int(rows["a"][4])) == (0, 2)  # a's last use is b at let 2
    assert (int(rows["u"][3]), int(rows["u"][4])) == (1, 1)  # unused: only its def
    assert int(rows["b"][4]) == 3                            # returned: to the end (n = 3)
    t2 = fn([("x", 100)], [("a", "tanh(%x)"), ("b", "neg(%a)")], "%b")
    rows = {l.split()[0]: l.split() for l in memsched_text(t2, "liveness", 0, False).splitlines()}
    assert (int(rows["a"][3]), int(rows["a"][4])) == (0, 1)
    assert int(rows["b"][3]) == 1


def diamond(order):
    body = {"a": "bcast(%x)", "b": "neg(%x)", "c": "add(%a, %b)"}
    return ("fn f(%x: f32[100]) {\n" + "".join(
        f"  let %{v} @{{op.shape=\"10,100\"}} = {body[v]};\n" if v == "a" else f"  let %{v} = {body[v]};\n"
        for v in order) + "  %c\n}\n")


@pytest.mark.parametrize("transient", [True, False])
def test_diamond_orders_match_enumeration_oracle(transient):
    """diamond x(400) -> {a(4000), b(400)} -> c(a, b): the peak of
    each order equals the refcount trace's (the exhaustive-evaluation oracle).
    Here c = add(a, b) broadcasts to a's 4000 B; under either model both
    orders cost the same: at c, a + b + c (+ x when persistent) are live ->
    8400 transient, 8800 persistent."""
    peaks = {}
    for order in (("a", "b", "c"), ("b", "a", "c")):
        t = diamond(order)
        peak, curve = curve_of(t, transient)
        tc, _, _ = trace_text(t, transient)
        assert curve == tc, (order, curve, tc)
        peaks[order] = peak
    assert set(peaks.values()) == ({8400} if transient else {8800})


def test_scheduler_moves_freeing_op_early():
    """an op that frees more than it produces (sum: 4000 B in,
    4 B out, last use) is scheduled as early as its dependencies allow; the
    p-c schedule reaches the enumeration optimum where the written order does
    not."""
    t = ("fn f(%x: f32[100]) {\n"
         "  let %a @{op.shape=\"10,100\"} = bcast(%x);\n"
         "  let %b @{op.shape=\"10,100\"} = bcast(%x);\n"
         "  let %c = neg(%b);\n"
         "  let %s @{op.axes=\"0,1\"} = sum(%a);\n"
         "  let %d = add(%c, %s);\n"
         "  %d\n}\n")
    out = memsched_text(t, "schedule", 0, True).splitlines()
    before, after = int(out[0].split()[1]), int(out[1].split()[1])
    order = out[2].split()[1:]
    assert order.index("s") == order.index("a") + 1  # sum right after its producer
    best = enumeration_optimum(t, True)
    assert after == best < before, (before, after, best)


# ------------------------------------------------------ enumeration oracle
def topo_orders(lets):
    ids = [v for v, *_ in lets]
    deps = {v: {a for a in args if a in ids} for v, _, args, _, _ in lets}
    out = []

    def rec(done, seq):
        if len(seq) == len(ids):
            out.append(list(seq))
            return
        for v in ids:
            if v not in done and deps[v] <= done:
                done.add(v)
                seq.append(v)
                rec(done, seq)
                seq.pop()
                done.remove(v)
    rec(set(), [])
    return out


def reorder(text, order):
    lines = text.splitlines()
    lets = {re.match(r"\s*let %([\w.]+)", l).group(1): l for l in lines if l.strip().startswith("let ")}
    tail = [l for l in lines[1:] if not l.strip().startswith("let ")]
    return "\n".join([lines[0]] + [lets[v] for v in order] + tail) + "\n"


def enumeration_optimum(text, transient):
    params, lets, ret = parse(text)
    size = sizes_from_liveness(text, transient)
    best = None
    for order in topo_orders(lets):
        by = {v: (v, o, a, s, f) for v, o, a, s, f in lets}
        c, _, _ = Trace(params, [by[v] for v in order], ret, size, transient).run()
        best = max(c) if best is None else min(best, max(c))
    return best


def random_dag(rng, n):
    """x: [4] (16 B) and big tensors [25,4] (400 B): unary ops keep the
    shape, add broadcasts small into big, bcast grows, sum shrinks."""
    shape = {"x": "s"}
    body = []
    for i in range(n):
        v = f"v{i}"
        prev = list(shape)
        a = prev[rng.integers(len(prev))]
        r = rng.random()
        if r < 0.25:
            e, sh = (f"bcast(%{a})", "b") if shape[a] == "s" else (f"sum(%{a})", "s")
            attr = '@{op.shape="25,4"} ' if shape[a] == "s" else '@{op.axes="0"} '
        elif r < 0.6:
            b = prev[rng.integers(len(prev))]
            if shape[a] == "s" and shape[b] == "b":
                a, b = b, a
            e, sh, attr = f"add(%{a}, %{b})", "b" if "b" in (shape[a], shape[b]) else "s", ""
        else:
            e, sh, attr = f"{['tanh', 'neg'][rng.integers(2)]}(%{a})", shape[a], ""
        shape[v] = sh
        body.append((v, attr, e))
    used = {a for _, _, e in body for a in re.findall(r"%(\w+)", e)}
    outs = [v for v, _, _ in body if v not in used]
    ret = "(" + ", ".join(f"%{v}" for v in outs) + ")"
    return ("fn f(%x: f32[4]) {\n" + "".join(f"  let %{v} {attr}= {e};\n" for v, attr, e in body)
            + f"  {ret}\n}}\n")


@pytest.mark.parametrize("seed", range(12))
def test_random_dags_vs_refcount_trace_and_enumeration(seed):
    """Random DAGs of 8 lets: (1) the planner's curve equals the refcount
    trace for the written order and for several other topological orders;
    (2) schedule() returns a topological order whose planner peak equals the
    trace's for that order; (3) its gap to the enumeration optimum is
    reported (logged, not asserted, outside curated cases)."""
    rng = np.random.default_rng(seed)
    t = random_dag(rng, 8)
    for transient in (True, False):
        params, lets, ret = parse(t)
        orders = topo_orders(lets)
        for order in [orders[0], orders[-1], orders[len(orders) // 2]]:
            tt = reorder(t, order)
            peak, curve = curve_of(tt, transient)
            tc, _, _ = trace_text(tt, transient)
            assert curve == tc, (seed, order, curve, tc)
        out = memsched_text(t, "schedule", 0, transient).splitlines()
        sched = out[2].split()[1:]
        assert sched in orders
        ts = reorder(t, sched)
        assert int(out[1].split()[1]) == max(trace_text(ts, transient)[0])
        best = enumeration_optimum(t, transient)
        print(f"seed {seed} transient={transient}: written {int(out[0].split()[1])} "
              f"scheduled {int(out[1].split()[1])} optimum {best}")
        assert int(out[1].split()[1]) >= best


# ------------------------------------------------- the training-step graphs
@pytest.mark.parametrize("kind", ["bert", "gpt2"])
def test_training_graph_liveness_equals_refcount_trace(kind):
    """the planner's liveness table on a real training step (MLP
    in the spec; here the tiny BERT / GPT-2 step with autodiff, fusion and
    the optimizer) equals the dynamic refcount trace: every storage root's
    def/last and the live-bytes curve.  The concat of the flat gradient and
    the in-place optimizer outputs are the planner's aliasing rules, so the
    text is taken with fuse=0 and compared root by root where no rule
    applies."""
    cfg = ModelConfig(kind=kind, L=2, H=64, A=2, F=128, V=64, S=8, B=2, dtype="f32", opt="sgd")
    text = graph_text(cfg, "text")
    params, lets, ret = parse(text)
    size = sizes_from_liveness(text, False)
    curve_t, first, last = Trace(params, lets, ret, size, False).run()
    rows = [l.split() for l in memsched_text(text, "liveness", 0, False).splitlines()]
    aliasing = {v for v, op, *_ in lets if op and base(op) in ("concat", "sgd_update", "cross_entropy",
                                                                "embedding_dx", "add_scalar")}
    # storage units the planner shares between vars through an in-place rule
    # (CE logits -> dlogits, SGD params, concat elision) are excluded
    unit_vars = {}
    for v, k, u, d, l, b in rows:
        unit_vars.setdefault(u, set()).add(v)
    shared = {u for u, vs in unit_vars.items() if vs & aliasing}
    checked = 0
    for v, k, u, d, l, b in rows:
        key = (v, int(k))
        if key not in first or u in shared:
            continue
        n = len(lets)
        lt = last.get(key, first[key])
        if v in ret:
            lt = n
        assert (int(d), int(l)) == (first[key], lt), (v, k, d, l, first[key], lt)
        checked += 1
    assert checked > 50, checked


def test_remat_chain_example():
    """chain a->b->c->d where a is also consumed by the last op;
    a budget that forces a's eviction -> the plan evicts a while the chain's
    big intermediates are live and replays its producer right before the last
    op; the new peak (re-run on the transformed text by the refcount trace)
    fits the budget."""
    t = ("fn f(%x: f32[100]) {\n"
         "  let %a @{op.shape=\"10,100\"} = bcast(%x);\n"
         "  let %b @{op.shape=\"4,10,100\"} = bcast(%a);\n"
         "  let %c = neg(%b);\n"
         "  let %d @{op.axes=\"0\"} = sum(%c);\n"
         "  let %e = add(%d, %a);\n"
         "  %e\n}\n")
    peak0 = curve_of(t, False)[0]
    assert peak0 == 36400  # at c: x + a + b + c
    budget = peak0 - 4000
    out = memsched_text(t, "remat", budget, False)
    lines = out.splitlines()
    assert lines[0] == "replays 1"
    splits = [l.split() for l in lines if l.startswith("split")]
    assert splits[0][1] == "a"
    new = out[out.index("fn f"):]
    assert "bcast(%x)" in new.split("let %e")[0].split("let %d")[1]  # replay between d and e
    assert max(trace_text(new, False)[0]) <= budget
    # budget >= peak: identity, empty plan
    assert memsched_text(t, "remat", peak0, False).splitlines()[0] == "replays 0"
    # below the floor (params + the largest single op's working set): BudgetInfeasible
    with pytest.raises(RuntimeError, match="exceeds budget|no evictable"):
        memsched_text(t, "remat", 20000, False)


@pytest.mark.parametrize("kind,dtype,S,B,L,frac", [("bert", "f32", 64, 8, 2, 0.6), ("bert", "bf16", 64, 8, 2, 0.6),
                                                  ("gpt2", "f32", 128, 8, 4, 0.6), ("gpt2", "bf16", 128, 8, 4, 0.5)])
def test_remat_60pct_bit_identical_in_interpreter(kind, dtype, S, B, L, frac):
    """the training graph under a budget of state + 60% of its
    unremat activation peak fits and the rematerialised step is BIT-IDENTICAL
    to the original in the CPU interpreter: loss, gradient and updated
    parameters over 2 steps.  GPT-2 (pre-LN) needs the depth-2 chains through
    tuple producers (a linear's input is a LayerNorm output field: the
    LayerNorm is replayed whole through a twin get-let)."""
    from oracle.interp_py import Interp
    from paper_2303_04759_b200.session import synthetic_batch
    cfg = ModelConfig(kind=kind, L=L, H=64, A=2, F=256, V=512, S=S, B=B, dtype=dtype,
                      opt="adam" if dtype == "bf16" else "sgd", lr=1e-3)
    gi = graph_info(cfg)
    act = gi["planner_peak"] - gi["state_bytes"]
    budget = gi["state_bytes"] + int(frac * act)
    cfg.extra["budget"] = budget
    gr = graph_info(cfg)
    assert gr["remat_replays"] > 0 and gr["peak_after_remat"] <= budget
    key = cfg.cfg_string(model_only=True)
    o0, o1 = Interp(key), Interp(key + f";budget={budget}")
    for k in range(2):
        ids, labels = synthetic_batch(cfg, seed=cfg.seed_d + k)
        l0, l1 = o0.step(ids, labels), o1.step(ids, labels)
        assert np.float32(l0).tobytes() == np.float32(l1).tobytes()
        assert o0.grad().tobytes() == o1.grad().tobytes()
    P = gi["P_pad"]
    assert o0.read("params", P).tobytes() == o1.read("params", P).tobytes()


def test_replay_count_monotone_over_budget_sweep():
    """shrinking the budget never decreases the replay count
    (5-point sweep on the BERT-base step at B=256)."""
    cfg = ModelConfig.bert_base(B=256)
    gi = graph_info(cfg)
    act = gi["planner_peak"] - gi["state_bytes"]
    counts = []
    for f in (1.0, 0.9, 0.8, 0.7, 0.6):
        c = ModelConfig.bert_base(B=256)
        c.extra["budget"] = gi["state_bytes"] + int(f * act)
        try:
            counts.append(graph_info(c)["remat_replays"])
        except RuntimeError:
            break
    assert len(counts) >= 4, counts
    assert counts == sorted(counts), counts
    assert counts[0] == 0 and counts[-1] > 0


def test_bert_base_remat_plan_golden():
    """The BERT-base (B=4096) remat plan under a 120 GB budget -- the split
    list (victim, evict index, replay-before index) -- is pinned by the
    committed fixture tests/golden/bert_base_remat_B4096_120GB.txt (made by
    tools/gen_golden_remat.py): any change to the planner's choices shows."""
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "golden", "bert_base_remat_B4096_120GB.txt")) as f:
        gold = f.read()
    cfg = ModelConfig.bert_base(B=4096)
    cfg.extra["budget"] = 120_000_000_000
    assert graph_text(cfg, "remat") == gold
    assert int(gold.splitlines()[2].split()[1]) <= 120_000_000_000
