"""Which parameter segments does the device AutoCast step update differently
from the oracle interpreter of the same graph (one Adam step)?"""
import numpy as np
from oracle.interp_py import Interp
from paper_2303_04759_b200.session import ModelConfig, Session, synthetic_batch

cfg = ModelConfig.tiny(opt="adam", lr=1e-3)
cfg.extra["autocast"] = "b200"
ids, labels = synthetic_batch(cfg)
s = Session(cfg)
s.init_params()
p0 = s.read("params")
s.set_batch(ids, labels)
s.step(graph=False)
print("device loss", s.loss())
pd = s.read("params")
o = Interp(cfg.cfg_string(model_only=True) + ";autocast=b200")
print("oracle loss", o.step(ids, labels))
po = o.read("params", pd.size)
for name, off, n in s.segments():
    d = pd[off:off + n] - p0[off:off + n]
    r = po[off:off + n] - p0[off:off + n]
    err = np.linalg.norm(d - r) / max(np.linalg.norm(r), 1e-30)
    print(f"{name:24s} n={n:8d} upd_dev={np.linalg.norm(d):.4e} upd_orc={np.linalg.norm(r):.4e} rel={err:.3e}")
