"""Summarise an ncu launch list (gpu__time_duration.sum CSV) per kernel name (development tool).

    python tools/launch_summary.py gpurun_out/launches.csv --steps 4 [--title "..."]
"""
from __future__ import annotations

import argparse
import collections
import csv


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--steps", type=float, default=1.0, help="optimizer steps covered by the list")
    ap.add_argument("--title", default="")
    args = ap.parse_args()
    lines = [ln for ln in open(args.csv) if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"])
        v = v / 1e6 if r["Metric Unit"] == "ns" else v / 1e3 if r["Metric Unit"] in ("us", "usecond") else v
        tot[r["Kernel Name"]] += v
        cnt[r["Kernel Name"]] += 1
    total = sum(tot.values())
    if args.title:
        print(f"# {args.title}")
    print(f"# {len(rows)} launches, {total / args.steps:.2f} ms/step over {args.steps:g} steps")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:20]:
        print(f"{v / args.steps:9.2f} ms/step {100 * v / total:5.1f}%  launches/step={cnt[k] / args.steps:6.1f}  {k[:110]}")


if __name__ == "__main__":
    main()
