#!/usr/bin/env python3
"""Time the b200 GEMM (linear / matmul_t) at the BERT-base shapes with CUDA
events; used for ncu captures (`ncu -k regex:k_gemm_tc ... python
tools/probe_gemm.py --only N`)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2303_04759_b200.abi import BF16, F32  # noqa: E402
from paper_2303_04759_b200.runtime import Plan  # noqa: E402

T = 4096
# (name, op, M, K, N, ta, tb, out)
SHAPES = [
    ("qkv_fwd", "matmul_t", T, 768, 2304, 0, 0, BF16),
    ("proj_fwd", "matmul_t", T, 768, 768, 0, 0, BF16),
    ("ffn1_fwd", "matmul_t", T, 768, 3072, 0, 0, BF16),
    ("ffn2_fwd", "matmul_t", T, 3072, 768, 0, 0, BF16),
    ("ffn1_dgrad", "matmul_t", T, 3072, 768, 0, 1, BF16),
    ("ffn1_wgrad", "matmul_t", 768, T, 3072, 1, 0, F32),
    ("decoder_fwd", "matmul_t", T, 768, 30528, 0, 1, BF16),
    ("big_sq", "matmul_t", 8192, 8192, 8192, 0, 1, BF16),
]


def run(name, op, M, K, N, ta, tb, out, iters, tile=None, cublas=True):
    a = torch.randn(K, M, device="cuda") if ta else torch.randn(M, K, device="cuda")
    b = torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda")
    a, b = a.to(torch.bfloat16).contiguous(), b.to(torch.bfloat16).contiguous()
    c = torch.empty(M, N, device="cuda", dtype=torch.float32 if out == F32 else torch.bfloat16)
    at = {"ta": ta, "tb": tb}
    if tile:
        at.update({"tc_bn": tile[0], "tc_cg": tile[1]})
    plan = Plan(op, [(tuple(a.shape), BF16), (tuple(b.shape), BF16)], [((M, N), out)], at)
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        plan.launch([a.data_ptr(), b.data_ptr()], [c.data_ptr()], s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        plan.launch([a.data_ptr(), b.data_ptr()], [c.data_ptr()], s)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1000 / iters
    tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
    if not cublas:
        return {"name": name, "tile": tile, "us": round(us, 2), "tflops": round(tf, 1)}
    # cuBLAS yardstick (out-of-band only): same operands, bf16 out
    at = a.t() if ta else a
    bt = b.t() if tb else b
    for _ in range(3):
        torch.matmul(at, bt)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        torch.matmul(at, bt)
    e1.record()
    torch.cuda.synchronize()
    ucb = e0.elapsed_time(e1) * 1000 / iters
    return {"name": name, "M": M, "K": K, "N": N, "ta": ta, "tb": tb, "us": round(us, 2), "tflops": round(tf, 1),
            "cublas_us": round(ucb, 2), "cublas_tflops": round(2.0 * M * N * K / (ucb * 1e-6) / 1e12, 1)}


def trace(iters, only=None):
    """Per-CTA timeline of one launch (globaltimer ns, 16 slots per CTA):
    entry, setup done, first operand stage landed (MMA), last MMA commit,
    accumulator ready / chunks done for tiles 0-2 (epilogue warp 0), MMA
    commit of tiles 0-2, epilogue drained."""
    cases = [("ffn1_fwd", "matmul_t", 4096, 768, 3072, 0, 0, BF16, {}),
             ("ffn1_fwd_gelu_grad", "linear", 4096, 768, 3072, 0, 0, BF16, {"act": "gelu", "save_preact": 1, "save": "grad"}),
             ("ffn1_fwd_gelu_grad_notma", "linear", 4096, 768, 3072, 0, 0, BF16,
              {"act": "gelu", "save_preact": 1, "save": "grad", "tc_notma": 1}),
             ("ffn1_fwd_bias", "linear", 4096, 768, 3072, 0, 0, BF16, {}),
             ("ffn1_fwd_preact", "linear", 4096, 768, 3072, 0, 0, BF16, {"act": "gelu", "save_preact": 1}),
             ("ffn1_fwd_gelu_only", "linear", 4096, 768, 3072, 0, 0, BF16, {"act": "gelu"}),
             ("ffn2_dgrad_deriv", "matmul_dact", 4096, 768, 3072, 0, 1, BF16, {"act": "deriv"}),
             ("proj_fwd", "matmul_t", 4096, 768, 768, 0, 0, BF16, {}),
             ("qkv_fwd", "matmul_t", 4096, 768, 2304, 0, 0, BF16, {}),
             ("ffn2_fwd", "matmul_t", 4096, 3072, 768, 0, 0, BF16, {}),
             ("proj_wgrad", "matmul_t", 768, 4096, 768, 1, 0, F32, {}),
             ("ffn1_wgrad", "matmul_t", 768, 4096, 3072, 1, 0, F32, {}),
             ("decoder_fwd", "matmul_t", 4096, 768, 30528, 0, 1, BF16, {})]
    import numpy as np
    for name, op, M, K, N, ta, tb, out, extra in cases:
        if only and name not in only:
            continue
        a = torch.randn(K, M, device="cuda") if ta else torch.randn(M, K, device="cuda")
        b = torch.randn(N, K, device="cuda") if tb else torch.randn(K, N, device="cuda")
        a, b = a.to(torch.bfloat16).contiguous(), (0.05 * b).to(torch.bfloat16).contiguous()
        c = torch.empty(M, N, device="cuda", dtype=torch.float32 if out == F32 else torch.bfloat16)
        tr = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
        at = {"ta": ta, "tb": tb, "tc_trace": tr.data_ptr(), **extra}
        ins, ptrs, outs, optrs = [(tuple(a.shape), BF16), (tuple(b.shape), BF16)], [a.data_ptr(), b.data_ptr()], \
            [((M, N), out)], [c.data_ptr()]
        keep = []
        if op == "linear":
            bias = torch.zeros(N, device="cuda")
            u = torch.empty_like(c)
            keep += [bias, u]
            ins.append(((N,), F32))
            ptrs.append(bias.data_ptr())
            if extra.get("save_preact"):
                outs.append(((M, N), out))
                optrs.append(u.data_ptr())
            at.pop("ta"), at.pop("tb")
        elif op == "matmul_dact":
            aux = torch.randn(M, N, device="cuda").to(torch.bfloat16)
            keep.append(aux)
            ins.append(((M, N), BF16))
            ptrs.append(aux.data_ptr())
            at.pop("ta")
        plan = Plan(op, ins, outs, at)
        s = torch.cuda.current_stream().cuda_stream
        for _ in range(3):
            plan.launch(ptrs, optrs, s)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            plan.launch(ptrs, optrs, s)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        tr.zero_()
        plan.launch(ptrs, optrs, s)  # the traced launch runs alone
        torch.cuda.synchronize()
        t = tr.view(148, 16).cpu().numpy().astype("float64")
        t = t[t[:, 0] > 0]
        base = t[:, 0].min()
        rel = (t[:, :16] - base) / 1000.0
        rel[t[:, :16] == 0] = float("nan")
        q = lambda col: [round(float(np.nanpercentile(rel[:, col], p)), 2) if np.isfinite(rel[:, col]).any() else None
                         for p in (0, 50, 100)]
        print(json.dumps({"name": name, "us": round(us, 2), "ctas": len(t), "entry": q(0), "setup": q(1),
                          "first_stage": q(2), "commit_t0": q(12), "acc_t0": q(4), "chunks_t0": q(6),
                          "released_t0": q(7), "commit_t1": q(13), "acc_t1": q(8), "chunks_t1": q(9),
                          "commit_t2": q(14), "acc_t2": q(10), "chunks_t2": q(11), "last_commit": q(3),
                          "epi_done": q(5)}), flush=True)


def pairs(iters):
    """BERT-base backward GEMM pairs (dgrad [+act'] and wgrad sharing dY): one
    grouped launch vs the two separate launches."""
    T = 4096
    cases = [("qkv", 768, 2304, 0), ("proj", 768, 768, 0), ("ffn1", 768, 3072, 0), ("ffn2_dact", 3072, 768, 1)]
    for name, Hin, Hout, dact in cases:
        # linear y = x W (x [T, Hin], W [Hin, Hout]); dY [T, Hout]
        x = torch.randn(T, Hin, device="cuda").to(torch.bfloat16)
        w = (0.02 * torch.randn(Hin, Hout, device="cuda")).to(torch.bfloat16)
        dy = torch.randn(T, Hout, device="cuda").to(torch.bfloat16)
        u = torch.randn(T, Hin, device="cuda").to(torch.bfloat16)
        dx = torch.empty(T, Hin, device="cuda", dtype=torch.bfloat16)
        dw = torch.empty(Hin, Hout, device="cuda")
        ins0 = [((T, Hout), BF16), ((Hin, Hout), BF16)] + ([((T, Hin), BF16)] if dact else [])
        p0 = Plan("matmul_dact" if dact else "matmul_t", ins0, [((T, Hin), BF16)],
                  {"tb": 1, **({"act": "gelu"} if dact else {})})
        p1 = Plan("matmul_t", [((T, Hin), BF16), ((T, Hout), BF16)], [((Hin, Hout), F32)], {"ta": 1, "out": "f32"})
        a0 = [dy.data_ptr(), w.data_ptr()] + ([u.data_ptr()] if dact else [])
        t0 = time_plan(p0, a0, [dx.data_ptr()], iters)
        t1 = time_plan(p1, [x.data_ptr(), dy.data_ptr()], [dw.data_ptr()], iters)
        at = {"n0": 3 if dact else 2, "ta0": 0, "tb0": 1, "ta1": 1, "tb1": 0, "out1": "f32"}
        if dact:
            at["act0"] = "gelu"
        pp = Plan("matmul_pair", ins0 + [((T, Hin), BF16), ((T, Hout), BF16)], [((T, Hin), BF16), ((Hin, Hout), F32)], at)
        tp = time_plan(pp, a0 + [x.data_ptr(), dy.data_ptr()], [dx.data_ptr(), dw.data_ptr()], iters)
        pr = Plan("matmul_pair", ins0 + [((T, Hin), BF16), ((T, Hout), BF16)], [((T, Hin), BF16), ((Hin, Hout), F32)],
                  {**at, "static_rr": 1})
        trr = time_plan(pr, a0 + [x.data_ptr(), dy.data_ptr()], [dx.data_ptr(), dw.data_ptr()], iters)
        print(json.dumps({"name": name, "dgrad_us": round(t0, 2), "wgrad_us": round(t1, 2), "sum_us": round(t0 + t1, 2),
                          "pair_lpt_us": round(tp, 2), "pair_round_robin_us": round(trr, 2)}), flush=True)


def pair_trace(iters):
    """The step's four backward pairs (FFN2 with the saved-derivative act'):
    time and per-CTA end spread for the planner's K-slice choice and for
    forced wsplit 1 / 2 / 4 (tuning data for gemm_pair_wsplit)."""
    import numpy as np
    T = 4096
    cases = [("qkv", 768, 2304, 0), ("proj", 768, 768, 0), ("ffn1", 768, 3072, 0), ("ffn2_deriv", 3072, 768, 1)]
    for name, Hin, Hout, dact in cases:
        x = torch.randn(T, Hin, device="cuda").to(torch.bfloat16)
        w = (0.02 * torch.randn(Hin, Hout, device="cuda")).to(torch.bfloat16)
        dy = torch.randn(T, Hout, device="cuda").to(torch.bfloat16)
        u = torch.randn(T, Hin, device="cuda").to(torch.bfloat16)
        dx = torch.empty(T, Hin, device="cuda", dtype=torch.bfloat16)
        dw = torch.empty(Hin, Hout, device="cuda")
        ins0 = [((T, Hout), BF16), ((Hin, Hout), BF16)] + ([((T, Hin), BF16)] if dact else [])
        a0 = [dy.data_ptr(), w.data_ptr()] + ([u.data_ptr()] if dact else [])
        for bn, ws in [tuple(int(v) for v in c.split(':')) for c in os.environ.get('PAIR_CFGS', '256:0,256:1,256:2,192:0,192:1,192:2,128:0,128:1,128:2').split(',')]:
            tr = torch.zeros(148 * 16, dtype=torch.int64, device="cuda")
            at = {"n0": 3 if dact else 2, "ta0": 0, "tb0": 1, "ta1": 1, "tb1": 0, "out1": "f32", "tc_trace": tr.data_ptr(),
                  "tc_bn": bn, "tc_cg": 2}
            if dact:
                at["act0"] = "deriv"
            if ws:
                at["wsplit"] = ws
            pp = Plan("matmul_pair", ins0 + [((T, Hin), BF16), ((T, Hout), BF16)],
                      [((T, Hin), BF16), ((Hin, Hout), F32)], at)
            args = (a0 + [x.data_ptr(), dy.data_ptr()], [dx.data_ptr(), dw.data_ptr()])
            us = time_plan(pp, *args, iters)
            tr.zero_()
            pp.launch(*args, torch.cuda.current_stream().cuda_stream)
            torch.cuda.synchronize()
            t = tr.view(148, 16).cpu().numpy().astype("float64")
            t = t[t[:, 0] > 0]
            rel = (t[:, 5] - t[:, 0].min()) / 1000.0
            print(json.dumps({"pair": name, "bn": bn, "wsplit": ws or "planner", "us": round(us, 2), "ctas": len(t),
                              "epi_done_min_med_max": [round(float(np.percentile(rel, p)), 2) for p in (0, 50, 100)]}),
                  flush=True)


def sweep(iters):
    """Every tile configuration on every BERT-base shape (cost-model calibration)."""
    for sh in SHAPES[:-1]:
        for tile in [(256, 2), (192, 2), (128, 2), (256, 1), (192, 1), (128, 1)]:
            print(json.dumps(run(*sh, iters=iters, tile=tile, cublas=False)), flush=True)


def linear_gelu(iters, M=4096, K=768, N=3072):
    """FFN1 forward as the step runs it: bias + GeLU + saved pre-activation."""
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (0.02 * torch.randn(K, N, device="cuda")).to(torch.bfloat16)
    b = torch.zeros(N, device="cuda")
    y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    u = torch.empty_like(y)
    res = []
    for act, save, what in (("gelu", 1, "preact"), ("gelu", 1, "grad"), ("none", 0, "")):
        outs = [((M, N), BF16), ((M, N), BF16)] if save else [((M, N), BF16)]
        at = {"act": act, "save_preact": save, **({"save": what} if save else {})}
        plan = Plan("linear", [((M, K), BF16), ((K, N), BF16), ((N,), F32)], outs, at)
        us = time_plan(plan, [x.data_ptr(), w.data_ptr(), b.data_ptr()],
                       [y.data_ptr(), u.data_ptr()][:len(outs)], iters)
        res.append({"name": f"linear_{act}{'_' + what if save else ''}_{M}x{K}x{N}", "us": round(us, 2),
                    "tflops": round(2.0 * M * N * K / us / 1e6, 1)})
    # the FFN2 backward data gradient with the fused GELU' epilogue vs plain
    dy = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w2 = (0.02 * torch.randn(N, K, device="cuda")).to(torch.bfloat16)
    plan = Plan("matmul_dact", [((M, K), BF16), ((N, K), BF16), ((M, N), BF16)], [((M, N), BF16)],
                {"tb": 1, "act": "gelu"})
    us = time_plan(plan, [dy.data_ptr(), w2.data_ptr(), u.data_ptr()], [y.data_ptr()], iters)
    res.append({"name": f"matmul_dact_gelu_{M}x{K}x{N}", "us": round(us, 2), "tflops": round(2.0 * M * N * K / us / 1e6, 1)})
    plan = Plan("matmul_dact", [((M, K), BF16), ((N, K), BF16), ((M, N), BF16)], [((M, N), BF16)],
                {"tb": 1, "act": "deriv"})
    us = time_plan(plan, [dy.data_ptr(), w2.data_ptr(), u.data_ptr()], [y.data_ptr()], iters)
    res.append({"name": f"matmul_dact_deriv_{M}x{K}x{N}", "us": round(us, 2), "tflops": round(2.0 * M * N * K / us / 1e6, 1)})
    plan = Plan("matmul_t", [((M, K), BF16), ((N, K), BF16)], [((M, N), BF16)], {"tb": 1})
    us = time_plan(plan, [dy.data_ptr(), w2.data_ptr()], [y.data_ptr()], iters)
    res.append({"name": f"matmul_t_tb_{M}x{K}x{N}", "us": round(us, 2), "tflops": round(2.0 * M * N * K / us / 1e6, 1)})
    return res


def cublas_epilogue(iters, M=4096, K=768, N=3072):
    """Vendor yardstick for the roofline kernel: cuBLASLt with its fused
    bias+GELU epilogue (torch._addmm_activation, tanh-GELU, one output) and
    cuBLAS + a separate torch GELU, on FFN1's shape."""
    x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (0.02 * torch.randn(K, N, device="cuda")).to(torch.bfloat16)
    b = torch.zeros(N, device="cuda", dtype=torch.bfloat16)

    def t(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) * 1000 / iters
    res = []
    for name, fn in (("cublaslt_bias_gelu_epilogue", lambda: torch._addmm_activation(b, x, w, use_gelu=True)),
                     ("cublas_matmul_plus_torch_gelu", lambda: torch.nn.functional.gelu(torch.addmm(b, x, w))),
                     ("cublas_matmul_plain", lambda: torch.matmul(x, w))):
        us = t(fn)
        res.append({"name": f"{name}_{M}x{K}x{N}", "us": round(us, 2), "tflops": round(2.0 * M * N * K / us / 1e6, 1)})
    return res


def time_plan(plan, ins, outs, iters):
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(3):
        plan.launch(ins, outs, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        plan.launch(ins, outs, s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1000 / iters


def attention(iters, p=0.1):
    """BERT-base attention closures (B=32, S=128, A=12, dh=64)."""
    B, S, A, H = 32, 128, 12, 768
    T = B * S
    qkv = torch.randn(T, 3 * H, device="cuda").to(torch.bfloat16)
    ctx = torch.empty(T, H, device="cuda", dtype=torch.bfloat16)
    probs = torch.empty(B * A * S, S, device="cuda", dtype=torch.bfloat16)
    dq = torch.empty_like(qkv)
    at = {"heads": A, "seq": S, "p": p, "seed": 7, "salt": 1}
    f = Plan("attention", [((T, 3 * H), BF16)], [((T, H), BF16), ((B * A * S, S), BF16)], at)
    b = Plan("attention_dx", [((T, 3 * H), BF16), ((B * A * S, S), BF16), ((T, H), BF16)], [((T, 3 * H), BF16)], at)
    uf = time_plan(f, [qkv.data_ptr()], [ctx.data_ptr(), probs.data_ptr()], iters)
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    ft = Plan("attention", [((T, 3 * H), BF16)], [((T, H), BF16), ((B * A * S, S), BF16)], {**at, "tc_trace": tr.data_ptr()})
    ft.launch([qkv.data_ptr()], [ctx.data_ptr(), probs.data_ptr()], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    import numpy as np
    t = tr.view(148, 8).cpu().numpy().astype("float64")
    t = t[t[:, 0] > 0]
    d = np.diff(t[:, :6], axis=1) / 1000.0
    print(json.dumps({"attn_fwd_phase_us(head 2): load_wait, qk_mma, softmax, store+pd+pv, epilogue":
                      [round(float(np.median(d[:, k])), 2) for k in range(5)]}), flush=True)
    ub = time_plan(b, [qkv.data_ptr(), probs.data_ptr(), ctx.data_ptr()], [dq.data_ptr()], iters)
    fl = 4.0 * B * A * S * S * 64
    return [{"name": "attention_fwd", "us": round(uf, 2), "tflops": round(fl / uf / 1e6, 1)},
            {"name": "attention_bwd", "us": round(ub, 2), "tflops": round(2 * fl / ub / 1e6, 1)}]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", type=int, default=-1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--attention", action="store_true")
    ap.add_argument("--linear", action="store_true")
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--pairs", action="store_true")
    ap.add_argument("--pair-trace", action="store_true")
    ap.add_argument("--cublas-epi", action="store_true")
    args = ap.parse_args()
    if args.cublas_epi:
        for r in cublas_epilogue(args.iters):
            print(json.dumps(r), flush=True)
        return
    if args.pairs:
        pairs(args.iters)
        return
    if args.pair_trace:
        pair_trace(args.iters)
        return
    if args.trace:
        trace(args.iters, os.environ.get("TRACE_ONLY", "").split(",") if os.environ.get("TRACE_ONLY") else None)
        return
    if args.sweep:
        sweep(args.iters)
        return
    if args.linear:
        for r in linear_gelu(args.iters):
            print(json.dumps(r), flush=True)
        return
    if args.attention:
        for r in attention(args.iters):
            print(json.dumps(r), flush=True)
        return
    shapes = SHAPES if args.only < 0 else [SHAPES[args.only]]
    for sh in shapes:
        print(json.dumps(run(*sh, iters=args.iters)), flush=True)


if __name__ == "__main__":
    main()
