"""Per-GEMM in-step timing of the BERT-base step (vm.profile, eager, events
around every instruction): shapes, us, TF/s and fraction of the dense bf16
peak, grouped by GEMM class.  Writes JSON lines to stdout."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_04759_b200.session import ModelConfig, Session, synthetic_batch  # noqa: E402


def prod(t):
    return int(np.prod(t))


def gemm_flops(r):
    op = r["op"].split(".")[-1]
    ins, outs = r["in"], r["out"]
    if op in ("linear", "matmul_t", "matmul_dact"):
        M, N = outs[0][0], prod(outs[0]) // outs[0][0]
        return 2 * M * N * (prod(ins[0]) // M)
    if op == "matmul_pair":
        n0 = 3 if len(ins) == 5 else 2  # (a0, b0 [, aux0], a1, b1)
        f = 0
        for p, a in ((0, 0), (1, n0)):
            M = outs[p][0]
            f += 2 * prod(outs[p]) * (prod(ins[a]) // M)
        return f
    return 0


def main():
    cfg = ModelConfig.bert_base(B=int(os.environ.get("B", "32")))
    s = Session(cfg)
    s.init_params()
    s.set_batch(*synthetic_batch(cfg))
    for _ in range(3):
        s.step(graph=True)
    rows = s.profile(7)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("bf16_tflops", 1600)
    tot = {}
    for r in rows:
        f = gemm_flops(r)
        if not f:
            continue
        tf = f / (r["us"] * 1e-6) / 1e12
        key = r["op"].split(".")[-1] + " " + "|".join("x".join(map(str, t)) for t in r["in"][:2]) + " -> " + \
            "|".join("x".join(map(str, t)) for t in r["out"])
        e = tot.setdefault(key, {"n": 0, "us": 0.0, "flops": 0})
        e["n"] += 1
        e["us"] += r["us"]
        e["flops"] += f
    for k, e in sorted(tot.items(), key=lambda kv: -kv[1]["us"]):
        tf = e["flops"] / (e["us"] * 1e-6) / 1e12
        print(json.dumps({"gemm": k, "launches": e["n"], "us_each": round(e["us"] / e["n"], 2),
                          "us_total": round(e["us"], 1), "tflops": round(tf, 1), "frac_peak": round(tf / peak, 3)}))
    s.close()


if __name__ == "__main__":
    main()
