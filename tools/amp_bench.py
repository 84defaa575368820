"""BERT-base seq128 B=32 Adam step rate: the hand-built bf16 graph vs the
AutoCast'd f32 graph (b200 policy), CUDA-graph replay, CUDA events."""
import ctypes
import json

from paper_2303_04759_b200 import runtime as R
from paper_2303_04759_b200.session import ModelConfig, Session, synthetic_batch


def rate(cfg, steps=20, warm=5):
    s = Session(cfg)
    s.init_params()
    ids, labels = synthetic_batch(cfg)
    s.set_batch(ids, labels)
    for _ in range(warm):
        s.step()
    s.sync()
    L = R.lib()
    e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
    R.check(L.tcb_event_create(ctypes.byref(e0)))
    R.check(L.tcb_event_create(ctypes.byref(e1)))
    R.check(L.tcb_event_record(e0, ctypes.c_void_p(s.stream)))
    for _ in range(steps):
        s.step()
    R.check(L.tcb_event_record(e1, ctypes.c_void_p(s.stream)))
    s.sync()
    ms = ctypes.c_float()
    R.check(L.tcb_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
    info = s.info()
    loss = s.loss()
    s.close()
    return {"ms_per_step": round(ms.value / steps, 4), "samples_per_s": round(cfg.B * steps / (ms.value * 1e-3), 1),
            "kernels_per_step": info["kernels_per_step"], "loss": round(loss, 4)}


import sys

keys = sys.argv[1:] or ["direct", "b200", "b200+fold", "b200+fold+fuse"]
out = {}
for k in keys:
    if k == "direct":
        out["direct_bf16"] = rate(ModelConfig.bert_base())
    else:
        c = ModelConfig.bert_base(dtype="f32")
        c.extra["autocast"] = k
        out["autocast_" + k] = rate(c)
print(json.dumps(out))
