"""Diagnose the default-config C1 step (dev tool)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle import core
from paper_2602_02016_b200 import shampoo, roots
from paper_2602_02016_b200.linalg import PrecisionMode

rng = np.random.default_rng(0)
w = rng.standard_normal((1024, 1024)); g = rng.standard_normal((1024, 1024))
cfg = shampoo.ShampooConfig()
orig = roots.ndb_split
log = []
def spy(*a, **k):
    y, z, rep = orig(*a, **k)
    log.append(rep.to_list())
    return y, z, rep
shampoo.ndb_split = spy
st = shampoo.init_state([w], cfg)
out, st = shampoo.step(st, [w], [g], cfg, seed=0)
ost = core.init_state([w], core.OracleConfig())
oout, ost, orep = core.step(ost, [w], [g], core.OracleConfig(), seed=0)
for c, lst in enumerate(log):
    print("chain", c, [(r.iterations, f"{r.residual:.1e}", int(r.converged)) for r in lst])
print("oracle chains", [[(r.iterations, int(r.converged)) for r in ch] for ch in orep[0]])
R = st.groups[0].roots.cpu().numpy(); Ro = ost["groups"][0]["roots"]
print("per-block roots relF", [f"{np.linalg.norm(R[i]-Ro[i])/np.linalg.norm(Ro[i]):.1e}" for i in range(R.shape[0])])
ema = st.groups[0].ema.double().cpu().numpy(); emao = ost["groups"][0]["ema"]
print("ema relF", np.linalg.norm(ema-emao)/np.linalg.norm(emao))
from paper_2602_02016_b200.eigensolver import inverse_root_f64
fb = inverse_root_f64(st.groups[0].ema, 1e-10, 4).double().cpu().numpy()
print("fallback-all relF per block", [f"{np.linalg.norm(fb[i]-Ro[i])/np.linalg.norm(Ro[i]):.1e}" for i in range(4)])
lam = np.linalg.eigvalsh(emao[:4] + 1e-10*np.eye(256)); print("cond", lam[:, -1]/lam[:, 0])
print("update relF", np.linalg.norm((out[0]-w)-(oout[0]-w))/np.linalg.norm(oout[0]-w))
