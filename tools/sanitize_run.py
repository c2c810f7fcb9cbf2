"""Small-shape run of every DASH kernel family for compute-sanitizer (development tool).

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_run.py

Covers: split / unsplit, the tcgen05 grouped GEMM (split 3-pass and fp16 modes; 128- and 256-wide pair tiles),
Newton-DB (upper pair-block storage + fill), coupled Newton, Clenshaw, the tensor-core and fp32 power
iterations (incl. the collapsed-pool retry), the Jacobi eigensolver and one optimizer step (prep, statistics
EMA, symmetrize, apply, update kernels).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import core  # noqa: E402  (input generator only)
from paper_2602_02016_b200 import chebyshev, eigensolver, linalg, roots, shampoo, spectral  # noqa: E402
from paper_2602_02016_b200.linalg import PrecisionMode, SplitStack  # noqa: E402


def main() -> None:
    torch.manual_seed(0)
    a = torch.randn(2, 256, 256, device="cuda")
    b = torch.randn(2, 256, 256, device="cuda")
    for mode in (PrecisionMode.EMULATED32, PrecisionMode.F16):
        linalg.bmm(a, b, mode)
    spd = np.stack([core.random_spd(256, c, seed=i, scale=0.5) for i, c in enumerate([10.0, 1e2])])
    st = torch.as_tensor(spd, dtype=torch.float32, device="cuda")
    for mode in (PrecisionMode.EMULATED32, PrecisionMode.F16):  # fp16 symmetric launches use 256-wide tiles
        sa = SplitStack.from_float(st)
        _, z, _ = roots.ndb_split(sa, None, 0.0, 3, mode, complete=False)
        roots.fill_lower(z)
        y, _, _ = roots.ndb_split(sa, None, 0.0, 3, mode, complete=False, outputs="y")  # last iteration: Y only
        roots.fill_lower(y)
        c2 = chebyshev.fit_inverse_root(4, degree=6)  # Clenshaw on the split stack (fused full-piece epilogue)
        ones = torch.ones(2, device="cuda")
        chebyshev.clenshaw_split(sa, c2, ones, ones, None, SplitStack(2, 256, 256), mode)
        roots.batched_coupled_newton(st, roots.CnConfig(p=4, tolerance=0.0, max_iters=2), mode)
    chebyshev.batched_clenshaw_matrix(st, chebyshev.fit_inverse_root(4, degree=6), np.ones(2))
    n = 3
    ema = torch.as_tensor(np.stack([core.random_spd(128, 10.0, seed=i) for i in range(n)] + [np.zeros((128, 128))]),
                          dtype=torch.float32, device="cuda")
    sc, inv = torch.zeros(n + 1, device="cuda"), torch.zeros(n + 1, device="cuda")
    status = torch.zeros(n + 1, dtype=torch.int32, device="cuda")
    spectral.power_iteration_scales(ema, 0.0, 16, 3, 7, sc, inv, status, a_split=SplitStack.from_float(ema))
    spectral.batched_multi_power_iteration(spd[:, :96, :96], 16, 3, 1)
    eigensolver.jacobi(torch.as_tensor(spd[:, :48, :48], device="cuda"))
    rng = np.random.default_rng(0)
    shapes = [(96, 64), (64,), (40, 72)]
    params = [rng.standard_normal(s) for s in shapes]
    cfg = shampoo.ShampooConfig(block_size=32, solver=shampoo.SolverConfig(tolerance=0.0, max_iters=3))
    state = shampoo.init_state(params, cfg)
    for _ in range(2):
        params, state = shampoo.step(state, params, [rng.standard_normal(s) for s in shapes], cfg)
    torch.cuda.synchronize()
    print("sanitize run complete")


if __name__ == "__main__":
    main()
