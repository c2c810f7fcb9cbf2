"""Diagnose config 1's fixed-10 step against the oracle, stage by stage (dev tool): EMA, scales, roots, update."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle import core  # noqa: E402
from paper_2602_02016_b200 import shampoo  # noqa: E402
from paper_2602_02016_b200.linalg import PrecisionMode  # noqa: E402

prec = {"f64": PrecisionMode.FULL64, "f32": PrecisionMode.EMULATED32}[os.environ.get("PREC", "f64")]
rng = np.random.default_rng(0)
w = rng.standard_normal((1024, 1024))
g = rng.standard_normal((1024, 1024))
cfg = shampoo.ShampooConfig(block_size=256, solver=shampoo.SolverConfig(method="ndb", tolerance=0.0, max_iters=10,
                                                                        precision=prec))
st = shampoo.init_state([w], cfg)
out, st = shampoo.step(st, [w], [g], cfg, seed=0)
ocfg = core.OracleConfig(block_size=256, method="ndb", tolerance=0.0, max_iters=10)
ost = core.init_state([w], ocfg)
oout, ost, _ = core.step(ost, [w], [g], ocfg, seed=0)


def relf(x, y):
    return float(np.linalg.norm(x - y) / np.linalg.norm(y))


for gi, (grp, og) in enumerate(zip(st.groups, ost["groups"])):
    ema, emao = grp.ema.double().cpu().numpy(), og["ema"]
    R, Ro = grp.roots.double().cpu().numpy(), og["roots"]
    n, p = og["dim"], og["p"]
    a = ema + ocfg.epsilon * np.eye(n)
    sco = core.group_scales(emao + ocfg.epsilon * np.eye(n), ocfg.scaling, ocfg.pool, ocfg.pi_iters,
                            core.block_seed(core.block_seed(0, 0), gi))
    ours = st.runtime.scratch.tensor("scale", (len(grp.members),)).double().cpu().numpy()
    print(f"  scales: ours vs oracle relmax {np.abs(ours / sco - 1).max():.2e}  ({ours[:3]} vs {sco[:3]})")
    sc = sco
    ahat = a / sc[:, None, None]
    if p == 2:
        _, Rf, _ = core.batched_newton_db(ahat, 0.0, 10)
    else:
        y1, _, _ = core.batched_newton_db(ahat, 0.0, 10)
        _, Rf, _ = core.batched_newton_db(y1, 0.0, 10)
    Rf = Rf * np.power(sc, -1.0 / p)[:, None, None]
    # the same float64 solve on our ema rounded to fp32 (the input's own resolution) and on the oracle ema
    print(f"group {gi} dim {n} p {p}: ema relF {relf(ema, emao):.2e}  roots relF {relf(R, Ro):.2e}  "
          f"(float64 solve of our ema vs oracle: {relf(Rf, Ro):.2e}; ours vs float64 solve of our ema: {relf(R, Rf):.2e})")
    print("  per-block roots relF", " ".join(f"{relf(R[i], Ro[i]):.1e}" for i in range(min(8, R.shape[0]))))
print("update relF", relf(out[0] - w, oout[0] - w))
