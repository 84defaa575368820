#!/usr/bin/env python3
"""Two launches each of the FFN1 forward (bias+GELU, save=grad) and the FFN2
backward dgrad with act=deriv -- a fixed launch order for ncu -s/-c captures."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2303_04759_b200.abi import BF16, F32  # noqa: E402
from paper_2303_04759_b200.runtime import Plan  # noqa: E402

M, K, N = 4096, 768, 3072
x = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (0.02 * torch.randn(K, N, device="cuda")).to(torch.bfloat16)
b = torch.zeros(N, device="cuda")
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
u = torch.empty_like(y)
s = torch.cuda.current_stream().cuda_stream
p = Plan("linear", [((M, K), BF16), ((K, N), BF16), ((N,), F32)], [((M, N), BF16)] * 2,
         {"act": "gelu", "save_preact": 1, "save": "grad"})
for _ in range(2):
    p.launch([x.data_ptr(), w.data_ptr(), b.data_ptr()], [y.data_ptr(), u.data_ptr()], s)
dy = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w2 = (0.02 * torch.randn(N, K, device="cuda")).to(torch.bfloat16)
q = Plan("matmul_dact", [((M, K), BF16), ((N, K), BF16), ((M, N), BF16)], [((M, N), BF16)], {"tb": 1, "act": "deriv"})
for _ in range(2):
    q.launch([dy.data_ptr(), w2.data_ptr(), u.data_ptr()], [y.data_ptr()], s)
r = Plan("matmul_t", [((M, K), BF16), ((N, K), BF16)], [((M, N), BF16)], {"tb": 1})
for _ in range(2):
    r.launch([dy.data_ptr(), w2.data_ptr()], [y.data_ptr()], s)
torch.cuda.synchronize()
