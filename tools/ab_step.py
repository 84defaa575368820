"""A/B the BERT-base step (CUDA-graph replay, CUDA events) between two
environment settings, alternating sessions: python tools/ab_step.py VAR=val"""
import os
import subprocess
import sys

CODE = r'''
import os, sys, json, ctypes
sys.path.insert(0, ".")
from paper_2303_04759_b200.session import ModelConfig, Session, synthetic_batch
from paper_2303_04759_b200 import runtime as R
cfg = ModelConfig.bert_base(B=32)
s = Session(cfg); s.init_params(); s.set_batch(*synthetic_batch(cfg))
for _ in range(5): s.step(graph=True)
s.sync()
L = R.lib(); e0, e1 = ctypes.c_void_p(), ctypes.c_void_p()
R.check(L.tcb_event_create(ctypes.byref(e0))); R.check(L.tcb_event_create(ctypes.byref(e1)))
best = []
for rep in range(5):
    R.check(L.tcb_event_record(e0, ctypes.c_void_p(s.stream)))
    for _ in range(30): s.step(graph=True)
    R.check(L.tcb_event_record(e1, ctypes.c_void_p(s.stream)))
    s.sync()
    ms = ctypes.c_float(); R.check(L.tcb_event_elapsed_ms(e0, e1, ctypes.byref(ms)))
    best.append(ms.value / 30)
print(json.dumps({"ms": sorted(best)[len(best)//2], "all": best, "kernels": s.info()["kernels_per_step"]}))
'''


def run(env_extra):
    env = dict(os.environ)
    env.update(env_extra)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    return out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]


if __name__ == "__main__":
    kv = dict(a.split("=", 1) for a in sys.argv[1:])
    for i in range(3):
        print("A (default):", run({}))
        print("B", kv, ":", run(kv))
