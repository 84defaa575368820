"""Rule-based fusion: elementwise runs become one
multi-output `ew_closure` (host/graph.hpp rule_fuse, csrc/k_closure.cu).

* the closure program on the oracle equals running its ops one by one
  through exec_base's restatement, bit for bit, on 50 random programs
  ("elementwise-only closure via ref dialect -> error = 0");
* the same programs on the device (GPU) against the oracle: f32/bf16 exact
  ops bit-identical, tanh/gelu within device-libm ulps (<= 1e-6 relative);
* on the AutoCast'd step graphs the pass finds its runs, the rules=0 and
  rules=1 interpreters agree bit for bit, and the device launches fewer kernels.
"""
import numpy as np
import pytest

from oracle import oracle_py as O
from paper_2303_04759_b200.abi import BF16, F32
from paper_2303_04759_b200.session import ModelConfig, graph_text

BIN = ["add", "sub", "mul", "div", "tanh_dx", "gelu_dx"]
UN = ["neg", "tanh", "relu", "gtz", "gelu", "copy", "add_scalar"]
ORACLE_OP = {"copy": "convert"}


def random_program(rng, nin, nins):
    """(prog string, per-instruction (op, a, b, dtype, imm), output registers)"""
    ins, prog = [], []
    for k in range(nins):
        reg = nin + k
        op = rng.choice(BIN + UN)
        a = int(rng.integers(reg))
        b = int(rng.integers(reg)) if op in BIN else a
        dt = int(rng.choice([F32, BF16]))
        imm = float(np.float32(rng.uniform(-1, 1))) if op == "add_scalar" else 0.0
        if op == "div":  # keep denominators away from zero: divide by (1 + |x|)-like register values
            b = a
        ins.append((op, a, b, dt, imm))
        prog.append(f"{op} {reg} {a} {b} {dt} {imm!r}")
    nout = int(rng.integers(1, min(4, nins) + 1))
    outs = sorted(rng.choice(np.arange(nin, nin + nins), nout, replace=False).tolist())
    return ";".join(prog) + ";", ins, outs


def op_by_op(inputs, in_dts, ins, outs):
    regs = [O.HostTensor(x, d) for x, d in zip(inputs, in_dts)]
    for op, a, b, dt, imm in ins:
        n = regs[a].arr.size
        if op in BIN:
            r = O.run(op, [regs[a], regs[b]], [((n,), dt)])[0]
        elif op == "copy":
            r = O.run("convert", [regs[a]], [((n,), dt)], {"to": "bf16" if dt == BF16 else "f32"})[0]
        elif op == "add_scalar":
            r = O.run("add_scalar", [regs[a]], [((n,), dt)], {"value": imm})[0]
        else:
            r = O.run(op, [regs[a]], [((n,), dt)])[0]
        regs.append(O.HostTensor(r, dt))
    return [regs[o].arr for o in outs], [regs[o].dtype for o in outs]


def closure_case(seed):
    rng = np.random.default_rng(seed)
    nin = int(rng.integers(1, 5))
    n = 1000
    in_dts = [int(rng.choice([F32, BF16])) for _ in range(nin)]
    inputs = []
    for d in in_dts:
        x = rng.uniform(-2, 2, n).astype(np.float32)
        inputs.append(O.HostTensor(x, d).arr if d == F32 else np.asarray(x))
    from gpu_util import quantize
    inputs = [quantize(x, d) for x, d in zip(inputs, in_dts)]
    prog, ins, outs = random_program(rng, nin, int(rng.integers(2, 9)))
    return inputs, in_dts, prog, ins, outs


def attrs_for(prog, outs, out_dts, n):
    ot = ";".join(("bf16" if d == BF16 else "f32") + f":{n}" for d in out_dts)
    return {"prog": prog, "outs": ",".join(str(o) for o in outs), "otypes": ot}


@pytest.mark.parametrize("seed", range(50))
def test_closure_equals_op_by_op_on_oracle(seed):
    inputs, in_dts, prog, ins, outs = closure_case(seed)
    ref, out_dts = op_by_op(inputs, in_dts, ins, outs)
    n = inputs[0].size
    got = O.run("ew_closure", [O.HostTensor(x, d) for x, d in zip(inputs, in_dts)],
                [((n,), d) for d in out_dts], attrs_for(prog, outs, out_dts, n))
    for g, r in zip(got, ref):
        assert np.array_equal(g.view(np.uint32), r.view(np.uint32)) or np.array_equal(g, r, equal_nan=True)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(50))
def test_closure_kernel_vs_oracle_on_device(seed):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from gpu_util import run_both
    inputs, in_dts, prog, ins, outs = closure_case(seed)
    ref, out_dts = op_by_op(inputs, in_dts, ins, outs)
    n = inputs[0].size
    g, o = run_both("ew_closure", list(zip(inputs, in_dts)), [((n,), d) for d in out_dts],
                    attrs_for(prog, outs, out_dts, n))
    transcendental = any(op in ("tanh", "gelu", "gelu_dx") for op, *_ in ins)
    for gi, oi, ri in zip(g, o, ref):
        assert np.array_equal(oi, ri, equal_nan=True)
        if transcendental:
            d = np.abs(gi.astype(np.float64) - oi) / np.maximum(np.abs(oi), 1e-6)
            assert np.nanmax(d) <= 1e-2, np.nanmax(d)  # an ulp of bf16 after libm ulps
        else:
            assert np.array_equal(gi, oi, equal_nan=True)


def test_autocast_graph_rule_fusion_and_interpreter_equality():
    """The AutoCast'd step under the default policy has elementwise runs (the
    f32 embedding adds feeding their bf16 cast); rule fusion makes them
    closures with every externally used value an output, and the interpreter
    of rules=1 equals rules=0 bit for bit.  (Under the b200 policy the
    embedding front becomes one embedding_sum and no run is left.)"""
    from oracle.interp_py import Interp
    from paper_2303_04759_b200.session import synthetic_batch
    for key in ("b200", "default"):
        c1 = ModelConfig.tiny(opt="adam", lr=1e-3)
        c1.extra["autocast"] = key
        ir = graph_text(c1, "ir")
        assert ir.count("= b200.ew_closure(") >= (1 if key == "default" else 0)
        c0 = ModelConfig.tiny(opt="adam", lr=1e-3, rules=0)
        c0.extra["autocast"] = key
        assert graph_text(c0, "ir").count("ew_closure") == 0
        ids, labels = synthetic_batch(c1)
        o1 = Interp(c1.cfg_string(model_only=True) + f";autocast={key}")
        o0 = Interp(c0.cfg_string(model_only=True) + f";autocast={key}")
        for _ in range(2):
            l1, l0 = o1.step(ids, labels), o0.step(ids, labels)
            assert np.float32(l1).tobytes() == np.float32(l0).tobytes()
        assert o1.grad().tobytes() == o0.grad().tobytes()


@pytest.mark.gpu
def test_rule_fusion_cuts_launches_and_keeps_results():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2303_04759_b200.session import Session, synthetic_batch

    def run(rules):
        c = ModelConfig.tiny(opt="adam", lr=1e-3, rules=rules)
        c.extra["autocast"] = "default"
        s = Session(c)
        s.init_params()
        ids, labels = synthetic_batch(c)
        losses = []
        for _ in range(2):
            s.set_batch(ids, labels)
            s.step()
            losses.append(s.loss())
        out = np.array(losses, np.float32), s.read("params"), s.info()["kernels_per_step"]
        s.close()
        return out

    l1, p1, k1 = run(1)
    l0, p0, k0 = run(0)
    assert k1 < k0, (k0, k1)
    assert l1.tobytes() == l0.tobytes() and p1.tobytes() == p0.tobytes()
