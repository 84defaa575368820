"""compute-sanitizer target: the r02 kernels (radix-sorted embedding_dx at
1-3 passes and both sort paths, the specialised GEMM epilogues) plus one
BERT-base B=2 training step through the VM."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_2303_04759_b200.abi import BF16, F32, I32
from paper_2303_04759_b200.runtime import run_op
from paper_2303_04759_b200.session import ModelConfig, Session, synthetic_batch

H = 64
for T, V in ((3000, 30000), (9000, 70000), (4100, 2)):
    ids = torch.randint(0, V, (T,), dtype=torch.int32, device="cuda")
    dy = torch.randn(T, H, device="cuda")
    run_op("embedding_dx", [ids, dy], [((V, H), F32)], {"rows": V})
x = torch.randn(300, 256, device="cuda").to(torch.bfloat16)
w = torch.randn(256, 200, device="cuda").to(torch.bfloat16)
b = torch.randn(200, device="cuda")
run_op("linear", [x, w, b], [((300, 200), BF16)] * 2, {"act": "gelu", "save_preact": 1, "save": "grad"})
run_op("linear", [x, w, b], [((300, 200), BF16)], {})
u = torch.randn(300, 256, device="cuda").to(torch.bfloat16)
dyy = torch.randn(300, 200, device="cuda").to(torch.bfloat16)
run_op("matmul_dact", [dyy, w, u], [((300, 256), BF16)], {"tb": 1, "act": "deriv"})
torch.cuda.synchronize()
cfg = ModelConfig.bert_base(B=2)
s = Session(cfg)
s.init_params()
s.set_batch(*synthetic_batch(cfg))
s.step(graph=False)
s.sync()
print("SANITIZE TARGET OK loss", s.loss())
