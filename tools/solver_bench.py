"""GEMM / solver micro-benchmark on one B200 (development tool, not part of the product path).

    python tools/solver_bench.py --n 256 --b 1024 --iters 10 [--mode f32|f16] [--solver ndb|cheb]

Times (CUDA events, per tcgen05 launch) a standalone batched product and a fixed-iteration Newton-DB
solve on a seeded SPD stack, and prints per-launch-kind ms and algorithmic TFLOP/s (2 B^3 per product).
"""
from __future__ import annotations

import argparse
import collections
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_02016_b200 import _lib  # noqa: E402
from paper_2602_02016_b200.linalg import PrecisionMode, SplitStack, bmm_split  # noqa: E402
from paper_2602_02016_b200.roots import ndb_split  # noqa: E402


def spd_stack(n: int, b: int, seed: int = 0) -> torch.Tensor:
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(n, b, b, device="cuda", generator=g)
    a = x @ x.transpose(1, 2) / b + 0.05 * torch.eye(b, device="cuda")
    lam = torch.linalg.matrix_norm(a, ord=2)
    return a / (2 * lam[:, None, None])


def report(tag: str, lst) -> None:
    agg = collections.OrderedDict()
    for ms, fl, _iss, tiles in lst:
        k = (tiles, fl)
        t = agg.setdefault(k, [0, 0.0])
        t[0] += 1
        t[1] += ms
    tot_ms = sum(v[1] for v in agg.values())
    tot_fl = sum(k[1] * v[0] for k, v in agg.items())
    for (tiles, fl), (cnt, ms) in agg.items():
        print(f"  {tag}: tiles={tiles:7d} launches={cnt:4d} {ms / cnt:8.3f} ms/launch "
              f"{fl * cnt / (ms * 1e-3) / 1e12:7.1f} TFLOP/s")
    print(f"  {tag}: total {tot_ms:.2f} ms, {tot_fl / 1e12:.2f} TF -> {tot_fl / (tot_ms * 1e-3) / 1e12:.1f} TFLOP/s")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--mode", default="f32", choices=["f64", "f32", "f16"])
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--solver", default="ndb", choices=["ndb", "cheb"])
    ap.add_argument("--degree", type=int, default=60)
    args = ap.parse_args()
    mode = {"f64": PrecisionMode.FULL64, "f32": PrecisionMode.EMULATED32, "f16": PrecisionMode.F16}[args.mode]
    a = spd_stack(args.n, args.b)
    sa = SplitStack.from_float(a)
    c = SplitStack(args.n, args.b, args.b)
    for _ in range(2):
        bmm_split(sa, sa, out=c, mode=mode)
    torch.cuda.synchronize()
    _lib.gemm_timing(True)
    for _ in range(args.reps):
        bmm_split(sa, sa, out=c, mode=mode)
    torch.cuda.synchronize()
    report("bmm", _lib.gemm_timing_list())
    _lib.gemm_timing(False)
    if args.solver == "cheb":
        from paper_2602_02016_b200.chebyshev import clenshaw_split, fit_inverse_root

        coef = fit_inverse_root(4, degree=args.degree, num_points=1000, interval=(1e-10, 1.0 + 1e-10))
        one = torch.ones(args.n, device="cuda")
        out = SplitStack(args.n, args.b, args.b)
        clenshaw_split(sa, coef, one, one, None, out, mode)
        torch.cuda.synchronize()
        _lib.gemm_timing(True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps):
            clenshaw_split(sa, coef, one, one, None, out, mode)
        e1.record()
        torch.cuda.synchronize()
        report("cheb", _lib.gemm_timing_list())
        _lib.gemm_timing(False)
        print(f"  cheb wall (events) {e0.elapsed_time(e1) / args.reps:.2f} ms per evaluation")
        return
    ndb_split(sa, None, 0.0, args.iters, mode)
    torch.cuda.synchronize()
    _lib.gemm_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.reps):
        ndb_split(sa, None, 0.0, args.iters, mode)
    e1.record()
    torch.cuda.synchronize()
    report("ndb", _lib.gemm_timing_list())
    _lib.gemm_timing(False)
    print(f"  ndb wall (events) {e0.elapsed_time(e1) / args.reps:.2f} ms per solve")


if __name__ == "__main__":
    main()
