"""A/B BERT-base B=32 step variants given as ModelConfig keyword overrides
(CUDA-graph replay, CUDA events), alternating sessions:
  python tools/ab_cfg.py flash=2 ...   (each arg one variant; 'base' = defaults)"""
import ctypes
import json
import sys

sys.path.insert(0, ".")
from paper_2303_04759_b200 import runtime as R  # noqa: E402
from paper_2303_04759_b200.session import ModelConfig, Session, synthetic_batch  # noqa: E402


def run(kw):
    cfg = ModelConfig.bert_base(B=32, **kw)
    s = Session(cfg)
    s.init_params()
    s.set_batch(*synthetic_batch(cfg))
    for _ in range(5):
        s.step(graph=True)
    s.sync()
    L = R.lib()
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    R.check(L.tcb_event_create(ctypes.byref(e0)))
    R.check(L.tcb_event_create(ctypes.byref(e1)))
    best = []
    for _ in range(5):
        R.check(L.tcb_event_record(e0, ctypes.c_void_p(s.stream)))
        for _ in range(30):
            s.step(graph=True)
        R.check(L.tcb_event_record(e1, ctypes.c_void_p(s.stream)))
        s.sync()
        ms = ctypes.c_float()
        R.check(L.tcb_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
        best.append(ms.value / 30)
    k = s.info()["kernels_per_step"]
    s.close()
    return round(sorted(best)[len(best) // 2], 4), k


if __name__ == "__main__":
    variants = [dict(kv.split("=", 1) for kv in a.split(",")) if a != "base" else {} for a in sys.argv[1:]]
    variants = [{k: int(v) for k, v in d.items()} for d in variants]
    for rnd in range(2):
        for v in variants:
            ms, k = run(v)
            print(json.dumps({"variant": v or "base", "ms": ms, "kernels": k}), flush=True)
