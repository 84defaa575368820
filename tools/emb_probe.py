import sys, json, torch
sys.path.insert(0, ".")
from paper_2303_04759_b200.abi import BF16, F32, I32
from paper_2303_04759_b200.runtime import Plan
def t(plan, ins, outs, it=3):
    s = torch.cuda.current_stream().cuda_stream
    plan.launch(ins, outs, s); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): plan.launch(ins, outs, s)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
H = 768
for T in (4096, 65536, 1115392):
    for V, kind in ((30528, "word"), (512, "pos"), (2, "type")):
        if kind == "word": ids = torch.randint(0, 30522, (T,), dtype=torch.int32, device="cuda")
        elif kind == "pos": ids = (torch.arange(T, device="cuda") % 128).to(torch.int32)
        else: ids = torch.zeros(T, dtype=torch.int32, device="cuda")
        dy = torch.randn(T, H, device="cuda").to(torch.bfloat16)
        out = torch.zeros(V, H, device="cuda")
        p = Plan("embedding_dx", [((T,), I32), ((T, H), BF16)], [((V, H), F32)], {"rows": V})
        ms = t(p, [ids.data_ptr(), dy.data_ptr()], [out.data_ptr()], 3 if T > 100000 else 20)
        print(json.dumps({"T": T, "table": kind, "ms": round(ms, 3)}), flush=True)
