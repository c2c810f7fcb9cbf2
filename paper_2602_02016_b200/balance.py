"""Greedy worker assignment and sync-cost report (drop-in for the reference ``balance.py``), plus the
per-block variant that drives the B200 block sharding (``sharded.py``).

``greedy_balance`` / ``simulate_sync_cost`` keep the reference's semantics (balance.py:45-73): entries
sorted by size, largest first, each to the currently least-loaded worker; ties on load go to the lowest
worker index, ties on size to the lowest id; makespan = largest load x compute cost, broadcast volume =
total x broadcast cost.  ``block_balance`` applies the same rule to gradient blocks with the solver
cost model of SURVEY §8(e) (2 (r^3 + c^3) per 2-D block: two Newton chains; len^3 per 1-D chunk) and
``block_report`` adds what the multi-GPU step actually moves: the all-gather bytes per rank.
"""
from __future__ import annotations

import heapq
from dataclasses import dataclass, field
from typing import Sequence


@dataclass
class WorkerAssignment:
    layer_ids: list[int] = field(default_factory=list)
    load: int = 0


@dataclass
class Assignment:
    workers: list[WorkerAssignment]
    sizes: dict[int, int]

    @property
    def num_workers(self) -> int:
        return len(self.workers)


@dataclass(frozen=True)
class CostModel:
    compute_per_param: float = 1.0
    broadcast_per_param: float = 1.0


@dataclass(frozen=True)
class SyncCostReport:
    makespan: float
    broadcast_volume: float
    worker_loads: tuple[int, ...]


def _check_entries(layer_sizes: Sequence[tuple[int, int]], workers: int) -> None:
    """The reference's preconditions and messages (balance.py:47-56)."""
    if workers < 1:
        raise ValueError("need at least one worker")
    if not layer_sizes:
        raise ValueError("no layers to assign")
    seen: set[int] = set()
    bad = next(((i, n) for i, n in layer_sizes if n <= 0), None)
    if bad is not None:
        raise ValueError(f"layer {bad[0]} has non-positive parameter count {bad[1]}")
    for i, _ in layer_sizes:
        if i in seen:
            raise ValueError("duplicate layer ids")
        seen.add(i)


def greedy_balance(layer_sizes: Sequence[tuple[int, int]], workers: int) -> Assignment:
    """Longest-processing-time-first assignment (balance.py:45-64).

    A min-heap of (load, worker) pops the least-loaded worker, the lowest index among equal loads; entries are
    visited by decreasing size, the lowest id among equal sizes.  O(n log workers) instead of a linear scan
    per entry (the block sharding assigns ~2000 units)."""
    _check_entries(layer_sizes, workers)
    heap = [(0, w) for w in range(workers)]  # already a valid heap
    buckets: list[list[int]] = [[] for _ in range(workers)]
    totals = [0] * workers
    for ident, size in sorted(layer_sizes, key=lambda e: (-e[1], e[0])):
        load, w = heapq.heappop(heap)
        buckets[w].append(ident)
        totals[w] = load + size
        heapq.heappush(heap, (totals[w], w))
    return Assignment(workers=[WorkerAssignment(layer_ids=b, load=t) for b, t in zip(buckets, totals)],
                      sizes=dict(layer_sizes))


def simulate_sync_cost(assignment: Assignment, cost_model: CostModel = CostModel()) -> SyncCostReport:
    """Makespan (largest load x per-param compute cost) and broadcast volume (every parameter broadcast once
    x per-param cost) of an assignment (balance.py:67-73)."""
    per_worker = tuple(w.load for w in assignment.workers)
    return SyncCostReport(makespan=cost_model.compute_per_param * max(per_worker),
                          broadcast_volume=cost_model.broadcast_per_param * sum(per_worker),
                          worker_loads=per_worker)


# ----------------------------------------------------------------------------- block sharding
def block_cost(rows: int, cols: int, matrix: bool) -> int:
    """Solver cost of one gradient block: two Newton chains on the rows x rows and cols x cols
    preconditioners of a 2-D block (inverse 4th roots), one chain on a 1-D chunk (inverse square root)."""
    return 2 * (rows ** 3 + cols ** 3) if matrix else rows ** 3


def block_balance(units, workers: int) -> Assignment:
    """greedy_balance over gradient blocks (``units``: objects with rows / cols / matrix); ids are unit
    indices, sizes their block_cost."""
    return greedy_balance([(i, block_cost(u.rows, u.cols, u.matrix)) for i, u in enumerate(units)], workers)


@dataclass(frozen=True)
class BlockReport:
    makespan: int               # largest per-rank solver cost
    imbalance: float            # makespan / mean load (1.0 = perfect)
    worker_loads: tuple[int, ...]
    allgather_bytes: int        # bytes each rank receives per step (fp32 shards padded to the largest)
    units_per_rank: tuple[int, ...]


def block_report(units, assignment: Assignment) -> BlockReport:
    rep = simulate_sync_cost(assignment)
    loads = rep.worker_loads
    mean = sum(loads) / len(loads)
    shard = [sum(units[i].rows * units[i].cols for i in w.layer_ids) for w in assignment.workers]
    return BlockReport(makespan=max(loads), imbalance=(max(loads) / mean) if mean > 0 else 1.0,
                       worker_loads=loads, allgather_bytes=4 * max(shard) * (len(shard) - 1),
                       units_per_rank=tuple(len(w.layer_ids) for w in assignment.workers))
