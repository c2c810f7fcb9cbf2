"""Benchmark: DASH optimizer step (B200) on the Llama-style ~1B parameter set.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl dash|reference] [--workload llama953m]

One "step" = one full DASH optimizer step (shampoo.step): Adam/graft prep, statistics EMA for every
L/R block, per-group symmetrize + power-iteration scaling + batched Newton-DB inverse 4th / square roots
(fixed 10 iterations per chain, SolverConfig(tolerance=0, max_iters=10)), root rescale, and the
grafted update L^(-1/4) G R^(-1/4) -- refresh every step (update_freq = 1), block size 1024.
Synthetic data: params N(0, 0.02^2), grads N(0, 1e-3^2), seeded.

`value` = ms per step, device-timed with CUDA events, inputs resident in HBM, max over ranks.
`e2e`   = the same step through the public API with host (pinned CPU) params/grads: H2D of grads and
          params and D2H of the new params inside the timed region.
N > 1 (`--gpus N` re-launches itself under torchrun when WORLD_SIZE is unset): gradient blocks are sharded
across ranks (greedy LPT on per-block solver cost) and the updated parameter shards are all-gathered with NCCL;
total work is fixed, so scaling is "strong".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DASH optimizer step ms at 1/2/4/8 B200; Newton-DB batched solver TFLOP/s"
SOLVER_DESC = {"ndb": "Newton-DB p=4/2 fixed {k} iters/chain", "cn": "coupled Newton p=4/2 fixed {k} iters",
               "cbshv": "Chebyshev/Clenshaw degree 60"}


def workload_shapes(name: str):
    from tests.golden.cases import C1, llama_124m, llama_953m

    return {"llama953m": (llama_953m(), 1024), "llama124m": (llama_124m(), 1024), "c1": (C1, 256)}[name]


def solver_products(method: str, exponent: int, iters: int, degree: int = 60) -> int:
    """Reference products per block: NDB 1+3(k-1) per chain (2 chains for p=4), CN 3k (p=2) /
    4k (p=4), Clenshaw d-1."""
    if method == "ndb":
        return (2 if exponent == 4 else 1) * (1 + 3 * (iters - 1))
    if method == "cn":
        return (4 if exponent == 4 else 3) * iters
    return degree - 1


def solver_flops(shapes, bsz: int, iters: int, method: str = "ndb") -> dict:
    """Algorithmic FLOPs per step: 2 r^2 c + 2 c^2 r stats/apply, 2 B^3 per solver product."""
    from paper_2602_02016_b200.shampoo import build_layout

    layers, specs = build_layout(shapes, bsz)
    ndb = 0.0
    for g in specs:
        ndb += len(g.members) * solver_products(method, g.exponent, iters) * 2.0 * g.dim ** 3
    stats = apply = 0.0
    for lay in layers:
        if lay.is_matrix:
            for (r0, r1), (c0, c1) in lay.layout.block_spans:
                r, c = r1 - r0, c1 - c0
                stats += 2.0 * r * r * c + 2.0 * c * c * r
                apply += 2.0 * r * r * c + 2.0 * r * c * c
        else:
            for s, e in lay.chunk_bounds:
                stats += 2.0 * (e - s) ** 2
                apply += 2.0 * (e - s) ** 2
    return {"ndb": ndb, "stats": stats, "apply": apply}


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    QUERY = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.path = tempfile.NamedTemporaryFile(suffix=".csv", delete=False).name
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i].lower() == "active"})
        loaded = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


# ----------------------------------------------------------------------------- CPU baseline (oracle port)
def _host_threads() -> int:
    return min(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1), 64)


def cpu_baseline(shapes, bsz, iters, method: str = "ndb", blocks_per_group: int = 1, reps: int = 3):
    """The reference algorithm (float64 oracle restatement) on the host cores, measured per component.

    * every distinct gradient-block shape (r, c) (and 1-D chunk length): one optimizer step of a layer of exactly
      that shape with the refresh skipped -- statistics EMA, Adam, the U = L^(-1/4) G R^(-1/4) apply and the grafted
      update (shampoo.py:238-278, :380-403) -- times the number of such blocks in the workload (the per-layer work
      is a sum over its blocks plus elementwise passes over its elements, so this is exact up to loop overhead);
    * every (dim, p) preconditioner group: the refresh of `blocks_per_group` blocks (a = ema + eps I, pooled
      power iteration 16 x 30, the solver at the bench's settings, the rescale; shampoo.py:312-349), times the
      group size / sample size (fixed-iteration solver cost does not depend on the values).
    BLAS runs on every host thread available (scipy-openblas caps at 64).  Each component is the median of
    `reps` timings."""
    import threadpoolctl

    from oracle import core
    from paper_2602_02016_b200.shampoo import build_layout

    threads = _host_threads()
    t_start = time.perf_counter()
    rng = np.random.default_rng(0)
    cfg = core.OracleConfig(block_size=bsz, method=method, tolerance=0.0, max_iters=iters, update_freq=2)
    layers, specs = build_layout(shapes, bsz)
    counts: dict = {}
    for lay in layers:
        if lay.is_matrix:
            for (r0, r1), (c0, c1) in lay.layout.block_spans:
                counts[(r1 - r0, c1 - c0)] = counts.get((r1 - r0, c1 - c0), 0) + 1
        else:
            for s0, e0 in lay.chunk_bounds:
                counts[(e0 - s0,)] = counts.get((e0 - s0,), 0) + 1
    parts = {}

    def timed(fn):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts)

    with threadpoolctl.threadpool_limits(threads):
        layer_ms = 0.0
        for shp, cnt in sorted(counts.items()):
            theta = rng.standard_normal(shp) * 0.02
            grad = rng.standard_normal(shp) * 1e-3

            def one_block():
                st = core.init_state([theta], cfg)
                st["step"] = 1  # 1 % update_freq(2) != 0: statistics + apply only
                core.step(st, [theta], [grad], cfg, seed=0)

            dt = timed(one_block)
            layer_ms += dt * cnt * 1e3
            parts[f"block{shp}"] = {"ms_each": round(dt * 1e3, 2), "count": cnt}
        group_ms = 0.0
        for gi, g in enumerate(specs):
            k = min(blocks_per_group, len(g.members))
            x = rng.standard_normal((k, g.dim, g.dim + 8)) * 1e-3
            ema = np.einsum("nij,nkj->nik", x, x) * 0.05

            def refresh_sample():
                a = ema + cfg.epsilon * np.eye(g.dim)
                sc = core.group_scales(a, "pi", 16, 30, core.block_seed(7, gi))
                ahat = a / sc[:, None, None]
                if method == "ndb":
                    if g.exponent == 2:
                        _, roots, _ = core.batched_newton_db(ahat, 0.0, iters)
                    else:
                        y1, _, _ = core.batched_newton_db(ahat, 0.0, iters)
                        _, roots, _ = core.batched_newton_db(y1, 0.0, iters)
                elif method == "cn":
                    roots, _ = core.batched_coupled_newton(ahat, g.exponent, 0.0, iters)
                else:
                    coeffs, _ = core.cheb_coefficients(g.exponent, 60, 1000, None)
                    roots = core.batched_clenshaw(a, coeffs, sc, g.exponent)
                return roots * np.power(sc, -1.0 / g.exponent)[:, None, None]

            dt = timed(refresh_sample)
            group_ms += dt / k * len(g.members) * 1e3
            parts[f"group{g.dim}/p{g.exponent}"] = {"ms_per_block": round(dt / k * 1e3, 1), "blocks": len(g.members),
                                                    "sampled": k}
    wall = time.perf_counter() - t_start
    return {
        "value": round(layer_ms + group_ms, 1),
        "unit": "ms",
        "cores": threads,
        "nproc": os.cpu_count(),
        "blas_threads": threads,
        "kind": "port",
        "sample": (f"float64 oracle of the reference step, timed per component on this host ({threads} BLAS threads): "
                   f"statistics + apply + graft of one block of every distinct block shape x its count, and the "
                   f"refresh (PI 16x30 + {SOLVER_DESC[method].format(k=iters)}) of {blocks_per_group} block(s) per "
                   f"(dim, p) group x group size; measured in {wall:.1f} s (not extrapolated by FLOPs)"),
        "components_ms": {"stats_apply": round(layer_ms, 1), "refresh": round(group_ms, 1)},
        "parts": parts,
    }


def c1_pair(iters: int, with_gpu: bool = True) -> dict:
    """Config 1 (one 1024x1024 layer, B = 256, NDB fixed `iters`, PI) end to end on both sides: the reference
    algorithm (float64 oracle, all host threads) runs it in full, so this ratio is same-config and unextrapolated."""
    import threadpoolctl

    from oracle import core

    rng = np.random.default_rng(0)
    w = rng.standard_normal((1024, 1024))
    g = rng.standard_normal((1024, 1024))
    ocfg = core.OracleConfig(block_size=256, method="ndb", tolerance=0.0, max_iters=iters)
    with threadpoolctl.threadpool_limits(_host_threads()):
        times = []
        for _ in range(3):
            ost = core.init_state([w], ocfg)
            t0 = time.perf_counter()
            oout, _, _ = core.step(ost, [w], [g], ocfg, seed=0)
            times.append(time.perf_counter() - t0)
    res = {"workload": f"c1: one (1024,1024) layer, B=256, NDB fixed {iters} iters/chain, PI 16x30, one step",
           "reference_ms": round(statistics.median(times) * 1e3, 1), "reference_threads": _host_threads()}
    if with_gpu:
        import torch

        from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig, init_state, step

        cfg = ShampooConfig(block_size=256, solver=SolverConfig(method="ndb", tolerance=0.0, max_iters=iters))
        hw = torch.from_numpy(w.astype(np.float32)).pin_memory()
        hg = torch.from_numpy(g.astype(np.float32)).pin_memory()
        st = init_state([hw], cfg)
        for _ in range(3):
            st = init_state([hw], cfg)
            step(st, [hw], [hg], cfg, seed=0)
        torch.cuda.synchronize()
        e2e = []
        for _ in range(5):
            st = init_state([hw], cfg)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out, _ = step(st, [hw], [hg], cfg, seed=0)
            torch.cuda.synchronize()
            e2e.append(time.perf_counter() - t0)
        d = (out[0].double().numpy() - w)
        ref = oout[0] - w
        res["dash_e2e_ms"] = round(statistics.median(e2e) * 1e3, 3)
        res["ratio_reference_over_dash_e2e"] = round(res["reference_ms"] / res["dash_e2e_ms"], 1)
        res["parity_update_relF"] = float(np.linalg.norm(d - ref) / np.linalg.norm(ref))
    return res


def bench_parity(iters: int, method: str = "ndb", precision: str = "f32") -> dict:
    """The benchmarked configuration's numerics against the float64 oracle, in the same run: B = 1024, PI 16 x 30,
    the bench's solver and precision, refresh every step, on a layer set with the bench's (1024, p=4) and
    (1024, p=2) groups; three steps (the statistics become full rank), last step compared."""
    import torch

    from oracle import core
    from paper_2602_02016_b200.linalg import PrecisionMode
    from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig, init_state, step

    shapes = [(2048, 1024), (1024,)]
    rng = np.random.default_rng(7)
    params = [rng.standard_normal(s) * 0.02 for s in shapes]
    grads = [[rng.standard_normal(s) * 1e-3 for s in shapes] for _ in range(3)]
    prec = {"f32": PrecisionMode.EMULATED32, "f16": PrecisionMode.F16}[precision]
    cfg = ShampooConfig(block_size=1024, solver=SolverConfig(method=method, tolerance=0.0, max_iters=iters,
                                                             precision=prec))
    ocfg = core.OracleConfig(block_size=1024, method=method, tolerance=0.0, max_iters=iters)
    st, ost = init_state(params, cfg), core.init_state(params, ocfg)
    cur, ocur = params, params
    for gs in grads:
        prev, oprev = cur, ocur
        cur, st = step(st, cur, gs, cfg, seed=5)
        ocur, ost, _ = core.step(ost, ocur, gs, ocfg, seed=5)
    torch.cuda.synchronize()

    def relf(x, y):
        return float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300))

    upd = max(relf(c - p, oc - op) for c, p, oc, op in zip(cur, prev, ocur, oprev))
    rts = max(relf(g.roots.double().cpu().numpy(), og["roots"]) for g, og in zip(st.groups, ost["groups"]))
    tol = {"f32": (5e-4, 1e-4), "f16": (3e-2, 5e-2)}[precision]
    return {"case": f"layers {shapes}, B=1024, groups 1024/p4 x4 + 1024/p2 x1, 3 steps, last compared",
            "relF_update": upd, "relF_roots": rts, "tol": {"update": tol[0], "roots": tol[1]},
            "pass": bool(upd < tol[0] and rts < tol[1])}


# ----------------------------------------------------------------------------- DASH arm
def run_dash(args):
    import torch
    import torch.distributed as dist

    from paper_2602_02016_b200 import _lib
    from paper_2602_02016_b200.linalg import PrecisionMode
    from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig, init_state, step

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DASH_DIST_BACKEND=gloo: ranks may share a GPU (exchange staged through the host) -- a functional check of
    # the sharded path on a one-GPU box; the measured multi-GPU runs use NCCL, one rank per GPU
    backend = os.environ.get("DASH_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    shapes, bsz = workload_shapes(args.workload)
    prec = {"f32": PrecisionMode.EMULATED32, "f16": PrecisionMode.F16}[args.precision]
    cfg = ShampooConfig(block_size=bsz, solver=SolverConfig(method=args.solver, tolerance=0.0,
                                                            max_iters=args.iters, precision=prec))
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234)
    params = [torch.randn(s, device="cuda", generator=gen) * 0.02 for s in shapes]
    grads = [torch.randn(s, device="cuda", generator=gen) * 1e-3 for s in shapes]
    events: dict = {}
    if world > 1:
        from paper_2602_02016_b200.sharded import ShardedDash

        opt = ShardedDash(params, cfg, rank=rank, world=world)
        shard_units, shard_ag_bytes = opt.units, opt.allgather_bytes
        do_step = lambda ev=None: opt.step(params, grads, events=ev)  # noqa: E731
    else:
        state = init_state(params, cfg)
        do_step = lambda ev=None: step(state, params, grads, cfg, inplace=True, events=ev)  # noqa: E731

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        do_step()
    barrier()
    launches0 = _lib.launch_count()
    _lib.gemm_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier()
        ev0.record()
        for _ in range(args.steps):
            do_step(events)
        ev1.record()
        barrier()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    phases = {}
    if events.get("start"):
        for a, b, name in (("start", "accumulated", "accumulate"), ("accumulated", "refreshed", "refresh"),
                           ("refreshed", "applied", "apply")):
            phases[name] = round(sum(x.elapsed_time(y) for x, y in zip(events[a], events[b])) / args.steps, 3)
        if events.get("exchanged"):  # sharded: pack + all-gather + unpack
            phases["exchange"] = round(sum(x.elapsed_time(y) for x, y in zip(events["applied"], events["exchanged"]))
                                       / args.steps, 3)
    n_gemm, gemm_ms, gemm_flops = _lib.gemm_timing_read()
    per_launch = _lib.gemm_timing_list()
    _lib.gemm_timing(False)
    gemm_issued = sum(x[2] for x in per_launch)
    launches = _lib.launch_count() - launches0  # every library kernel launched in the timed region (K steps)
    ms = ms_local
    if world > 1:
        t = torch.tensor([ms_local], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- end-to-end through the public API with host buffers (pinned), H2D + D2H inside the region
    e2e = None
    dev_peak = 0
    if not args.no_e2e:
        hp = [p.cpu().pin_memory() for p in params]
        hg = [g.cpu().pin_memory() for g in grads]
        # release the device-resident run first: two optimizer states at 953M would need ~170 GB of HBM
        dev_peak = torch.cuda.max_memory_allocated()
        if world > 1:
            del opt
        else:
            del state
        del do_step
        params.clear()
        grads.clear()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        h2d = sum(t.numel() * 4 for t in hp) + sum(t.numel() * 4 for t in hg)
        d2h = sum(t.numel() * 4 for t in hp)
        if world == 1:
            state_e = init_state(hp, cfg)

            def e2e_step():
                nonlocal state_e
                out, state_e = step(state_e, hp, hg, cfg)
                del out  # the caller keeps what it needs; the pinned block returns to the host cache
        else:  # every rank: H2D of its (replicated, DDP-style) gradients and parameters, sharded step, D2H
            from paper_2602_02016_b200.sharded import ShardedDash

            dp = [p.cuda() for p in hp]
            dg = [g.cuda() for g in hg]
            opt_e = ShardedDash(dp, cfg, rank=rank, world=world)
            outs = [torch.empty_like(p).pin_memory() for p in hp]

            def e2e_step():
                for d, h in zip(dp, hp):
                    d.copy_(h, non_blocking=True)
                for d, h in zip(dg, hg):
                    d.copy_(h, non_blocking=True)
                opt_e.step(dp, dg)
                for o, d in zip(outs, dp):
                    o.copy_(d, non_blocking=True)
                torch.cuda.current_stream().synchronize()
        for _ in range(max(args.warmup, 2)):  # warm the host path (pinned output buffers cycle through the cache)
            e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_local = (time.perf_counter() - t0) / args.steps * 1e3
        if world > 1:  # max over ranks
            t = torch.tensor([e2e_local], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_local = float(t.item())
        e2e = {"value": e2e_local, "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    fl = solver_flops(shapes, bsz, args.iters, args.solver)
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    peak = peaks.get("bf16_tflops_sustained", 1420.2)
    # aggregate over every GEMM launch (the small groups' launches run on a second stream, concurrently with the
    # big group's, so their event durations overlap and this understates the rate) ...
    all_achieved = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else 0.0
    # ... and the dominant launch class (the launch shape with the most event time: the Newton-DB Y*E / E*Z
    # launch over the largest group), per launch: its algorithmic flops / its mean duration
    classes: dict = {}
    for ms_l, fl_l, is_l, tiles_l in per_launch:
        c = classes.setdefault((int(tiles_l), round(fl_l)), [0, 0.0, 0.0, 0.0])
        c[0] += 1
        c[1] += ms_l
        c[2] += fl_l
        c[3] += is_l
    dom_key, dom = max(classes.items(), key=lambda kv: kv[1][1]) if classes else ((0, 0), [0, 0.0, 0.0, 0.0])
    achieved = dom[2] / (dom[1] * 1e-3) / 1e12 if dom[1] > 0 else 0.0
    issued_tf = dom[3] / (dom[1] * 1e-3) / 1e12 if dom[1] > 0 else 0.0
    dom_desc = {"tiles": dom_key[0], "launches": dom[0], "mean_ms": round(dom[1] / max(dom[0], 1), 3),
                "share_of_gemm_time": round(dom[1] / gemm_ms, 3) if gemm_ms > 0 else None}
    # DRAM bytes per launch of the dominant launch (the Newton-DB Y*E / E*Z launch over the 1820-block group) from
    # the committed ncu --set full capture of this build: ncu cannot run inside a timed bench (it replays kernels)
    traffic, traffic_src = None, None
    for name in ("r2_gemm_traffic.json", "r1_gemm_traffic.json"):
        tr_file = ROOT / "profiles" / name
        if tr_file.exists():
            tr = json.loads(tr_file.read_text())
            traffic, traffic_src = tr.get("bytes_per_launch"), f"profiles/{name}: {tr.get('source')}"
            break
    result = {
        "metric": METRIC,
        "value": round(ms, 3),
        "unit": "ms",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms, 3),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": ("fp16x3-split products (hi*hi + hi*lo + lo*hi), fp32 accumulate/storage" if args.precision == "f32"
                  else "fp16 products, fp32 accumulate/storage"),
        "data": "synthetic (params N(0,0.02^2), grads N(0,1e-3^2), seeded)",
        "config": {
            "workload": f"{args.workload} DASH step, B={bsz}, {SOLVER_DESC[args.solver].format(k=args.iters)}, "
                        f"PI scaling (pool 16 x 30 iters), update_freq=1, grafting beta2=0.999",
            "params": int(sum(int(np.prod(s)) for s in shapes)),
            "precond_blocks": None,
            "parallelism": (f"block-sharded x{world} ({os.environ.get('DASH_DIST_BACKEND', 'nccl')})" if world > 1
                            else "single GPU"),
            "l2": "working set (EMA/roots/iterates, GBs) >> 126 MB L2; no explicit flush",
            "solver_precision": args.precision,
        },
        "solver_tflops_per_s": None,
        "roofline": {
            "bound": "tensor",
            "kernel": (f"dash_gemm2_kernel<{3 if args.precision == 'f32' else 1}> (tcgen05 cta_group::2 grouped GEMM), "
                       "dominant launch class: the Newton-DB product launch over the largest preconditioner group"),
            "dominant_launch": dom_desc,
            "achieved": round(achieved, 1),
            "achieved_def": ("algorithmic: 2 M N K per reference product (solver blocks 2 B^3) per launch of the "
                             "dominant launch class / its mean CUDA-event duration in the timed steps"),
            "issued_tensor_tflops": round(issued_tf, 1),
            "issued_frac": round(issued_tf / peak, 4),
            "issued_def": ("fp16 tensor-core flops actually issued (tiles x 2 x 256 x 128 x padded K x passes; "
                           "symmetric solver products run only the upper-triangle tiles) / the same durations"),
            "all_gemm_achieved": round(all_achieved, 1),
            "all_gemm_def": ("the same over every GEMM launch (statistics, solvers of every group, apply); the small "
                             "groups run concurrently on a second stream, so their overlapping durations make this "
                             "an underestimate"),
            "peak": peak,
            "unit": "TFLOP/s",
            "frac": round(achieved / peak, 4),
            "traffic": traffic,
            "traffic_source": traffic_src,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step)",
            "flops_per_step": {k: round(v / 1e12, 3) for k, v in fl.items()},
            "gemm_launches_timed": n_gemm,
            "gemm_ms_per_step": round(gemm_ms / args.steps, 3),
        },
        "gpu_launches": int(launches), "gpu_launches_per_step": int(launches) // args.steps,
        "clocks": clk.summary(),
        "e2e": e2e,
    }
    from paper_2602_02016_b200.shampoo import build_layout

    _, specs = build_layout(shapes, bsz)
    result["config"]["precond_blocks"] = {f"{g.dim}x{g.dim}/p{g.exponent}": len(g.members) for g in specs}
    result["phases_ms"] = phases
    # peak device memory of the device-timed run (tensors incl. workspaces; the e2e run reuses it after a release)
    result["hbm_peak_gb"] = round((dev_peak if e2e is not None else torch.cuda.max_memory_allocated()) / 1e9, 1)
    if world > 1:  # block sharding balance (balance.block_report): solver-cost makespan vs mean, all-gather bytes
        from paper_2602_02016_b200.balance import block_balance, block_report

        rep = block_report(shard_units, block_balance(shard_units, world))
        result["balance"] = {"units": len(shard_units), "units_per_rank": list(rep.units_per_rank),
                             "imbalance": round(rep.imbalance, 4),
                             "allgather_bytes_per_rank": rep.allgather_bytes}
    if phases.get("refresh"):  # Newton-DB algorithmic FLOPs / refresh phase (includes PI, splits, rescale)
        result["solver_tflops_per_s"] = round(fl["ndb"] / world / (phases["refresh"] * 1e-3) / 1e12, 1)
    if world > 1:
        result["allgather_bytes_per_step"] = shard_ag_bytes
    if rank == 0 and not args.no_parity:
        result["parity"] = bench_parity(args.iters, args.solver, args.precision)
    if rank == 0 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(shapes, bsz, args.iters, method=args.solver)
        if args.solver == "ndb" and args.precision == "f32":
            result["c1"] = c1_pair(args.iters)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_reference(args):
    """The reference's own algorithm on the host cores: the float64 oracle restatement (the reference is pure
    Python/NumPy and /root/reference does not exist on the GPU box), every host thread for BLAS.  Each step is
    one per-component measurement of the workload (cpu_baseline); rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    shapes, bsz = workload_shapes(args.workload)
    steps = []
    for _ in range(args.warmup + args.steps):
        steps.append(cpu_baseline(shapes, bsz, args.iters, method=args.solver, reps=1))
    timed = steps[args.warmup:]
    v = statistics.median([c["value"] for c in timed])
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(v, 1),
        "unit": "ms",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(v, 1),
        "higher_is_better": False,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (seeded)",
        "config": {"workload": f"{args.workload} DASH step, B={bsz}, {SOLVER_DESC[args.solver].format(k=args.iters)}, "
                               "PI scaling (pool 16 x 30 iters), update_freq=1, grafting beta2=0.999",
                   "parallelism": "host CPU"},
        "cpu_baseline": {k: timed[-1][k] for k in ("kind", "cores", "nproc", "blas_threads", "sample")}
                        | {"value": round(v, 1), "unit": "ms"},
        "e2e": {"value": round(v, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "components_ms": timed[-1]["components_ms"],
    }
    if args.solver == "ndb" and not args.no_cpu:
        line["c1"] = c1_pair(args.iters, with_gpu=False)
    print(json.dumps(line), flush=True)


def run_train(args):
    """Config 5's full training step on one GPU: Llama-953M forward + backward (bf16 autocast, fp32 master
    weights, synthetic tokens) and the DASH step on its gradients (NDB fixed iters, PI, B = 1024)."""
    import torch

    from paper_2602_02016_b200 import _lib
    from paper_2602_02016_b200.linalg import PrecisionMode
    from paper_2602_02016_b200.llama import LlamaShape, TrainStep
    from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    shape = LlamaShape()
    prec = {"f32": PrecisionMode.EMULATED32, "f16": PrecisionMode.F16}[args.precision]
    cfg = ShampooConfig(block_size=1024, solver=SolverConfig(method=args.solver, tolerance=0.0, max_iters=args.iters,
                                                             precision=prec))
    trainer = TrainStep(shape, cfg, "cuda", seed=0)
    batch, seq = args.batch, args.seq
    g = torch.Generator().manual_seed(0)
    host_tokens = [torch.randint(0, shape.vocab, (batch, seq + 1), generator=g).pin_memory() for _ in range(2)]
    dev_tokens = [t.cuda() for t in host_tokens]
    for i in range(args.warmup):
        trainer(dev_tokens[i % 2])
    torch.cuda.synchronize()
    events: dict = {}
    launches0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for i in range(args.steps):
            loss = trainer(dev_tokens[i % 2], events=events)
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = _lib.launch_count() - launches0  # every library kernel launched in the timed region (K steps)
    fwd_bwd = statistics.mean(a.elapsed_time(b) for a, b in zip([ev0] + events["applied"][:-1], events["backward_done"]))
    opt = statistics.mean(a.elapsed_time(b) for a, b in zip(events["backward_done"], events["applied"]))
    # end to end: the caller's token batch from pinned host memory, the loss read back every step
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(args.steps):
        loss = trainer(host_tokens[i % 2].cuda(non_blocking=True))
        float(loss)
    torch.cuda.synchronize()
    e2e = (time.perf_counter() - t0) / args.steps * 1e3
    tokens = batch * seq
    print(json.dumps({
        "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "bf16 model fwd/bwd (fp32 master), fp16x3-split DASH products",
        "data": "synthetic tokens (uniform over the vocabulary), random-init Llama-953M",
        "config": {"workload": f"llama953m-train: full training step (fwd + bwd + DASH, B=1024, "
                               f"{SOLVER_DESC[args.solver].format(k=args.iters)}, PI)", "global_batch": batch,
                   "seq_len": seq, "tokens_per_step": tokens, "parallelism": "single GPU"},
        "phases_ms": {"forward_backward": round(fwd_bwd, 3), "dash_step": round(opt, 3)},
        "tokens_per_s": round(tokens / (ms * 1e-3), 1), "final_loss": float(loss), "gpu_launches": int(launches),
        "gpu_launches_per_step": int(launches) // args.steps,
        "clocks": clk.summary(),
        "e2e": {"value": round(e2e, 3), "unit": "ms", "h2d_bytes_per_step": tokens * 8 + batch * 8,
                "d2h_bytes_per_step": 4},
    }), flush=True)


def spawn_ranks(args) -> int:
    """`--gpus N` without a torchrun environment: re-launch this script under torchrun with N local ranks."""
    import torch

    if args.gpus > torch.cuda.device_count():
        print(json.dumps({"error": f"--gpus {args.gpus} but only {torch.cuda.device_count()} GPUs visible"}))
        return 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={29500 + os.getpid() % 1000}", str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["dash", "reference"], default="dash")
    ap.add_argument("--workload", default="llama953m", choices=["llama953m", "llama124m", "c1", "llama953m-train"])
    ap.add_argument("--batch", type=int, default=4, help="llama953m-train: sequences per step")
    ap.add_argument("--seq", type=int, default=1024, help="llama953m-train: tokens per sequence")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--precision", default="f32", choices=["f32", "f16"])
    ap.add_argument("--solver", default="ndb", choices=["ndb", "cn", "cbshv"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "dash":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus and int(os.environ.get("RANK", 0)) == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}; using WORLD_SIZE",
              file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "llama953m-train":
        run_train(args)
    else:
        run_dash(args)


if __name__ == "__main__":
    main()
