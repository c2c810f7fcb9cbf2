"""Residual floor / accuracy probe of the device Newton-DB solver (development tool, not product).

    python tools/floor_probe.py [--kmax 40]

For SPD stacks of several sizes and condition numbers (random_spd, spectrum top 0.5) and the literal
config-1 statistics (one EMA step of Gaussian gradients, PI-like 2 lambda_max scaling) it runs the
batched Newton-DB in fixed-iteration mode for k = 2..kmax and prints, per k, the largest per-block
residual max|E - I| and the relF of Z against the float64 eigh inverse square root.
"""
from __future__ import annotations

import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import core  # noqa: E402  (checker only)
from paper_2602_02016_b200 import roots  # noqa: E402
from paper_2602_02016_b200.linalg import PrecisionMode  # noqa: E402


def inv_sqrt(a):
    w, q = np.linalg.eigh(a)
    return (q / np.sqrt(w)[..., None, :]) @ np.swapaxes(q, -1, -2)


def c1_stack(b=256):
    rng = np.random.default_rng(0)
    rng.standard_normal((1024, 1024))
    g = rng.standard_normal((1024, 1024))
    blocks = [g[i:i + b, j:j + b] for i in range(0, 1024, b) for j in range(0, 1024, b)]
    a = np.stack([0.05 * x @ x.T + 1e-10 * np.eye(b) for x in blocks][:8])
    lam = np.linalg.eigvalsh(a)[:, -1]
    return a / (2 * lam[:, None, None])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kmax", type=int, default=30)
    ap.add_argument("--mode", default="f32", choices=["f64", "f32", "f16"])
    args = ap.parse_args()
    mode = {"f64": PrecisionMode.FULL64, "f32": PrecisionMode.EMULATED32, "f16": PrecisionMode.F16}[args.mode]
    cases = []
    for b, n in ((256, 8), (1024, 4)):
        for cond in (1e1, 1e2, 1e3, 1e4):
            cases.append((f"B={b} cond={cond:g}", np.stack([core.random_spd(b, cond, seed=i, scale=0.5) for i in range(n)])))
    cases.append(("C1 literal (cond~1e6)", c1_stack()))
    for name, a in cases:
        ref = inv_sqrt(a)
        at = torch.from_numpy(a).float().cuda()
        row = []
        for k in range(2, args.kmax + 1):
            _, z, rep = roots.batched_newton_db(at, roots.NdbConfig(tolerance=0.0, max_iters=k), mode)
            zz = z.double().cpu().numpy()
            err = np.linalg.norm(zz - ref) / np.linalg.norm(ref)
            r = max(x.residual for x in rep)
            it = min(x.iterations for x in rep)
            row.append(f"k={k}:r={r:.1e}/z={err:.1e}" + ("" if it == k else f"(frz{it})"))
        print(name)
        for i in range(0, len(row), 6):
            print("   " + "  ".join(row[i:i + 6]))
        sys.stdout.flush()


if __name__ == "__main__":
    main()
