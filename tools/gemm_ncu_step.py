"""Eager BERT-base steps for an ncu capture of the step's tcgen05 GEMMs:

  ncu --metrics <list> -k regex:k_gemm_tc -s <skip> -c <count> python tools/gemm_ncu_step.py

Writes gpurun_out/gemm_order.json: the k_gemm_tc launch order of ONE step
(one launch per linear / matmul_t / matmul_dact / matmul_pair let, in let
order) with a class name per launch, so the ncu rows can be labelled."""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_04759_b200.session import ModelConfig, Session, synthetic_batch  # noqa: E402

STEPS = int(os.environ.get("STEPS", "3"))


def classify(op, out_type):
    if op == "linear":
        n = out_type.split("[")[1].split(",")[1].rstrip("];) ")
        return {"2304": "qkv_fwd", "768": "proj_or_ffn2_fwd", "3072": "ffn1_fwd(gelu)", "30528": "decoder_fwd"}.get(
            n, "linear")
    return op


def main():
    cfg = ModelConfig.bert_base(B=32)
    s = Session(cfg)
    ir = s.text("ir")
    order = []
    for line in ir.splitlines():
        m = re.search(r"= b200\.(linear|matmul_t|matmul_dact|matmul_pair)\(.*: (.*);$", line.strip())
        if m:
            order.append({"op": m.group(1), "type": m.group(2)[:120]})
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "gemm_order.json"), "w") as f:
        json.dump(order, f)
    s.init_params()
    s.set_batch(*synthetic_batch(cfg))
    for _ in range(STEPS):
        s.step(graph=False)
    s.sync()
    print("gemm launches per step", len(order))
    s.close()


if __name__ == "__main__":
    main()
