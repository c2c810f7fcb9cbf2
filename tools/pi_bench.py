"""Power-iteration micro-benchmark (development tool): times dash_power_iteration on a seeded SPD stack."""
from __future__ import annotations

import argparse
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_02016_b200.spectral import power_iteration_scales  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1820)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--iters", type=int, nargs="+", default=[1, 10, 30])
    ap.add_argument("--tc", action="store_true", help="tensor-core kernel on the split stack")
    args = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.empty(args.n, args.b, args.b, device="cuda")
    for i in range(0, args.n, 64):  # chunked: x x^T / b keeps the peak memory bounded
        x = torch.randn(min(64, args.n - i), args.b, args.b, device="cuda", generator=g)
        a[i:i + 64] = x @ x.transpose(1, 2) / args.b
    from paper_2602_02016_b200.linalg import SplitStack

    a_split = SplitStack.from_float(a + 1e-10 * torch.eye(args.b, device="cuda"))
    sc = torch.zeros(args.n, device="cuda")
    inv = torch.zeros(args.n, device="cuda")
    stt = torch.zeros(args.n, dtype=torch.int32, device="cuda")
    for it in args.iters:
        power_iteration_scales(a, 1e-10, 16, it, 0, sc, inv, stt, a_split=a_split if args.tc else None)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        power_iteration_scales(a, 1e-10, 16, it, 0, sc, inv, stt, a_split=a_split if args.tc else None)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        flops = 2.0 * args.n * args.b * args.b * 16 * (it + 1)
        if os.environ.get("DASH_PI_EXP", "0") != "0":
            print("section cycles (wait MMA, TMEM ld, reduce, normalise, publish):", stt[1:6].tolist())
        print(f"iters={it:3d}: {ms:8.2f} ms  {flops / ms / 1e9:7.1f} TFLOP/s (fp32 FMA)  scale[0]={float(sc[0]):.6g}")


if __name__ == "__main__":
    main()
