"""End-to-end (pinned host buffers) step time of the 953M bench workload vs the pipeline chunk count (dev tool).

    python tools/e2e_probe.py --chunks 1 2 4 8
"""
from __future__ import annotations

import argparse
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from bench import workload_shapes  # noqa: E402
from paper_2602_02016_b200.linalg import PrecisionMode  # noqa: E402
from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig, init_state, step  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    shapes, bsz = workload_shapes("llama953m")
    cfg = ShampooConfig(block_size=bsz, solver=SolverConfig(method="ndb", tolerance=0.0, max_iters=10,
                                                            precision=PrecisionMode.EMULATED32))
    g = torch.Generator().manual_seed(0)
    hp = [(torch.randn(s, generator=g) * 0.02).pin_memory() for s in shapes]
    hg = [(torch.randn(s, generator=g) * 1e-3).pin_memory() for s in shapes]
    for k in args.chunks:
        os.environ["DASH_HOST_CHUNKS"] = str(k)
        st = init_state(hp, cfg)
        for _ in range(2):
            out, st = step(st, hp, hg, cfg)
            del out
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            out, st = step(st, hp, hg, cfg)
            del out
        torch.cuda.synchronize()
        print(f"chunks={k}: e2e {(time.perf_counter() - t0) / args.steps * 1e3:.1f} ms/step", flush=True)
        del st
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
