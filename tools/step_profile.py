"""Per-launch GEMM timing of one 953M DASH step (development tool): groups launches by (tiles, flops)."""
from __future__ import annotations

import collections
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import workload_shapes  # noqa: E402
from paper_2602_02016_b200 import _lib  # noqa: E402
from paper_2602_02016_b200.linalg import PrecisionMode  # noqa: E402
from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig, init_state, step  # noqa: E402

method = sys.argv[1] if len(sys.argv) > 1 else "ndb"
prec = PrecisionMode.F16 if len(sys.argv) > 2 and sys.argv[2] == "f16" else PrecisionMode.EMULATED32
shapes, bsz = workload_shapes("llama953m")
cfg = ShampooConfig(block_size=bsz, solver=SolverConfig(method=method, tolerance=0.0, max_iters=10, precision=prec))
g = torch.Generator(device="cuda").manual_seed(1234)
params = [torch.randn(s, device="cuda", generator=g) * 0.02 for s in shapes]
grads = [torch.randn(s, device="cuda", generator=g) * 1e-3 for s in shapes]
state = init_state(params, cfg)
for _ in range(3):
    step(state, params, grads, cfg, inplace=True)
torch.cuda.synchronize()
_lib.gemm_timing(True)
ev = {}
step(state, params, grads, cfg, inplace=True, events=ev)
torch.cuda.synchronize()
lst = _lib.gemm_timing_list()
_lib.gemm_timing(False)
agg = collections.OrderedDict()
for ms, fl, iss, tiles in lst:
    a = agg.setdefault((tiles, fl), [0, 0.0, iss])
    a[0] += 1
    a[1] += ms
for (tiles, fl), (n, ms, iss) in agg.items():
    print(f"tiles={tiles:7d} alg={fl / 1e12:7.3f} TF x{n:3d}: {ms:8.2f} ms  alg {fl * n / ms / 1e9:6.1f} TF/s  "
          f"issued {iss * n / ms / 1e9:6.1f} TF/s")
print("gemm total ms", sum(x[0] for x in lst))
for a, b in (("start", "accumulated"), ("accumulated", "refreshed"), ("refreshed", "applied")):
    print(a, "->", b, f"{ev[a][0].elapsed_time(ev[b][0]):.2f} ms")
