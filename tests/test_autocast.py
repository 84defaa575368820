"""AutoCast pass (host/autocast.hpp, §3.1.2 Fig. 3).

tests/cpp/autocast_test.cpp checks the spec's examples on hand-built graphs
(single matmul -> 2 casts; all-F32 policy -> identity; softmax after a bf16
matmul gets a cast-up; Fig. 3: two fusable consumers -> 2 exclusive casts and 0
standalone after the fusion rules, vs >= 1 with shared placement; a policy
missing an op is an error; bf16 cast round trip) and the whole f32 BERT
training step.  The Python tests read the same census through the C-ABI.
"""
import os
import subprocess

import pytest

from paper_2303_04759_b200.session import ModelConfig, autocast_info

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = os.environ.get("TRAINC_REF_INC", "/root/reference/proj/include")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF_INC, "trainc")), reason="reference headers absent")
def test_autocast_spec_examples_cpp(tmp_path):
    exe = str(tmp_path / "autocast_test")
    r = subprocess.run(["g++", "-std=c++20", "-O1", f"-I{REF_INC}", f"-I{ROOT}/paper_2303_04759_b200/host",
                        f"-I{ROOT}/include", "-o", exe, f"{ROOT}/tests/cpp/autocast_test.cpp"],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr


def test_all_f32_policy_is_identity():
    a = autocast_info(ModelConfig.tiny(), "f32")
    assert a["casts"] == 0 and a["sites"] == 0 and a["low_ops"] == 0


@pytest.mark.parametrize("opt", ["sgd", "adam"])
def test_default_policy_invariants(opt):
    a = autocast_info(ModelConfig.tiny(opt=opt), "default")
    assert a["f32_violations"] == 0
    assert a["low_ops"] > 0 and a["casts"] > 0
    # no two casts of one (producer, dtype) feed one consumer: casts <= sites
    assert a["casts"] <= a["sites"]
    s = autocast_info(ModelConfig.tiny(opt=opt), "default", "shared")
    # cast minimality bound: exclusive placement never leaves more
    # standalone casts than shared placement
    assert a["standalone_casts"] <= s["standalone_casts"]
    assert s["exclusive"] == 0


def test_b200_policy_bert_base_no_standalone_casts():
    """On the BERT-base f32 step the b200 policy leaves no standalone cast: every
    cast is either a parameter's bf16 compute copy (written by the fused Adam
    update on the device path) or inside a kernel that widens on load."""
    a = autocast_info(ModelConfig.bert_base(dtype="f32"), "b200")
    d = autocast_info(ModelConfig.bert_base(dtype="f32"), "default")
    assert a["f32_violations"] == 0 and d["f32_violations"] == 0
    assert a["standalone_casts"] == 0, a
    assert a["casts"] < d["casts"]
    # every contraction runs in bf16 under both; the b200 policy also gathers
    # the three embedding tables from their bf16 compute copy
    assert a["low_ops"] == d["low_ops"] + 3


def test_rejects_non_f32_step():
    with pytest.raises(RuntimeError, match="all-f32"):
        autocast_info(ModelConfig.tiny(dtype="bf16"), "b200")


@pytest.mark.gpu
def test_amp_verify_autocast_step_on_device():
    """amp_verify: the AutoCast'd f32 step runs on the b200
    device VM and its loss trajectory stays within 5e-2 of the f32 step's over
    50 Adam steps on identical data and init (SPEC.md:788 threshold)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import numpy as np
    from paper_2303_04759_b200.session import Session, synthetic_batch

    def losses(extra):
        cfg = ModelConfig.tiny(opt="adam", lr=1e-3)
        cfg.extra.update(extra)
        s = Session(cfg)
        s.init_params()
        ids, labels = synthetic_batch(cfg)
        out = []
        for _ in range(50):
            s.set_batch(ids, labels)
            s.step()
            out.append(s.loss())
        s.close()
        return np.array(out)

    f32 = losses({})
    amp = losses({"autocast": "b200"})
    assert np.all(np.isfinite(amp))
    assert amp[-1] < amp[0]  # it trains
    dmax = float(np.max(np.abs(amp - f32)))
    print(f"amp_verify: 50 steps, max |dloss| = {dmax:.4g}; loss {f32[0]:.4f} -> {f32[-1]:.4f} (f32), "
          f"{amp[-1]:.4f} (autocast)")
    assert dmax <= 5e-2, (f32, amp)


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["b200", "default"])
def test_autocast_step_matches_oracle_interpreter(policy):
    """The device run of the AutoCast'd step against the CPU oracle interpreter
    of the same graph, for the b200 and the SPEC default policy: first loss
    within 1e-5 relative, and every parameter segment's SGD update (lr * grad)
    within 2e-2 relative (bf16 GEMM accumulation order)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import numpy as np
    from oracle.interp_py import Interp
    from paper_2303_04759_b200.session import Session, synthetic_batch
    # SGD: the update is lr * grad, so this compares the gradients themselves
    # (Adam's first step is ~lr * sign(g), ill-conditioned for |g| ~ eps)
    cfg = ModelConfig.tiny(opt="sgd", lr=0.1)
    cfg.extra["autocast"] = policy
    ids, labels = synthetic_batch(cfg)
    s = Session(cfg)
    s.init_params()
    p0 = s.read("params")
    s.set_batch(ids, labels)
    s.step(graph=False)
    ld = s.loss()
    pd = s.read("params")
    o = Interp(cfg.cfg_string(model_only=True) + ";autocast=" + policy)
    lo = o.step(ids, labels)
    po = o.read("params", pd.size)
    assert abs(ld - lo) <= 1e-5 * abs(lo)
    for name, off, n in s.segments():
        d = pd[off:off + n] - p0[off:off + n]
        r = po[off:off + n] - p0[off:off + n]
        err = np.linalg.norm(d - r) / max(np.linalg.norm(r), 1e-30)
        assert err <= 2e-2, (name, err)
    s.close()


@pytest.mark.gpu
def test_fold_param_casts_bit_identical():
    """fold_param_casts: the AutoCast'd step with its parameter converts folded
    into the optimizer's bf16 compute copy is bit-identical to the unfolded
    one (loss and master weights over 3 Adam steps) and launches fewer kernels."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import numpy as np
    from paper_2303_04759_b200.session import Session, synthetic_batch

    def run(key):
        cfg = ModelConfig.tiny(opt="adam", lr=1e-3)
        cfg.extra["autocast"] = key
        s = Session(cfg)
        s.init_params()
        losses = []
        for k in range(3):
            s.set_batch(*synthetic_batch(cfg, seed=cfg.seed_d + k))
            s.step()
            losses.append(s.loss())
        out = (np.array(losses, np.float32), s.read("params"), s.info()["kernels_per_step"])
        s.close()
        return out

    l0, p0, k0 = run("b200")
    l1, p1, k1 = run("b200+fold")
    assert l0.tobytes() == l1.tobytes()
    assert p0.tobytes() == p1.tobytes()
    assert k1 < k0, (k0, k1)
    # + fusion re-run on the bf16 graph: dgrad+wgrad pair launches with
    # K-sliced wgrad (another f32 summation order) -> tolerance, fewer kernels
    l2, p2, k2 = run("b200+fold+fuse")
    assert np.max(np.abs(l2 - l1) / np.abs(l1)) <= 1e-3, (l1, l2)
    assert k2 < k1, (k1, k2)
