"""Debug: ShardedDash world 1, exchange chunks 1 vs 2 vs the 1-GPU step, per layer and step."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2602_02016_b200.shampoo import GraftConfig, ShampooConfig, SolverConfig, init_state, step  # noqa
from paper_2602_02016_b200.sharded import ShardedDash  # noqa

os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
dist.init_process_group("gloo", rank=0, world_size=1)
rng = np.random.default_rng(0)
shapes = [(96, 64), (64,), (40, 72), (130, 33)]
params = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
grads = [[torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes] for _ in range(3)]
cfg = ShampooConfig(block_size=32, solver=SolverConfig(tolerance=0.0, max_iters=10))
st = init_state(params, cfg)
cur = [p.clone() for p in params]
ref = []
for gs in grads:
    cur, st = step(st, cur, gs, cfg, seed=5)
    ref.append([c.clone() for c in cur])
for nx in (1, 2):
    ps = [p.clone() for p in params]
    opt = ShardedDash(ps, cfg, rank=0, world=1, exchange_chunks=nx)
    print("nx", nx, "bounds", opt.bounds, "overlap", opt._overlappable())
    for k, gs in enumerate(grads):
        opt.step(ps, gs, seed=5)
        print("  step", k, [float((a - b).abs().max()) for a, b in zip(ps, ref[k])])
