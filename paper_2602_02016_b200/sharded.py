"""Block-sharded DASH step across GPUs (one process per GPU, torch.distributed over NCCL).

SURVEY.md §8(e): gradient blocks are independent (batched ops, freezing, reports and grafting are all
per block), so the sharding unit is the gradient block: its L and R preconditioners, its slice of the
Adam state and its update U live on the owner rank.  Assignment is a deterministic greedy LPT over the
per-block solver cost (r^3 + c^3 per 2-D block, len^3 per 1-D chunk, times chains), largest first,
each to the least-loaded rank with ties to the lowest rank -- the rule of the reference's simulated
balancer (balance.py:57-62) applied to blocks instead of layers.

Per step every rank runs the full DASH pipeline on its own blocks (same kernels, same per-block seeds
as the 1-GPU path, so results are identical to the unsharded step), packs its updated parameter blocks
into a block-major buffer, and one NCCL all-gather assembles every rank's shard (the B200 equivalent
of the paper's post-update parameter broadcast); an unpack kernel scatters the blocks
back into the flat parameter space.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .balance import block_balance, block_cost
from .shampoo import (GroupSpec, LayerState, PrecondGroup, ShampooConfig, ShampooState, SlotRef, _Runtime,
                      accumulate, block_rows, build_layout, check_step_status, refresh_inverse_roots)
from .spectral import block_seed


@dataclass(frozen=True)
class Unit:
    """One sharding unit: a gradient block of a 2-D layer or a chunk of a 1-D layer."""

    layer_id: int
    idx: int
    rows: int
    cols: int
    matrix: bool

    @property
    def cost(self) -> int:
        return block_cost(self.rows, self.cols, self.matrix)


def units_of(layers: list[LayerState]) -> list[Unit]:
    out = []
    for lay in layers:
        if lay.is_matrix:
            for idx, ((r0, r1), (c0, c1)) in enumerate(lay.layout.block_spans):
                out.append(Unit(lay.layer_id, idx, r1 - r0, c1 - c0, True))
        else:
            for idx, (s, e) in enumerate(lay.chunk_bounds):
                out.append(Unit(lay.layer_id, idx, e - s, 1, False))
    return out


def assign_units(units: list[Unit], world: int) -> list[list[int]]:
    """Greedy LPT (balance.block_balance): units by (-cost, index) to the least-loaded rank, ties to the
    lowest rank; returns each rank's unit indices in ascending order."""
    if world < 1:
        raise ValueError("need at least one rank")
    if not units:
        return [[] for _ in range(world)]
    return [sorted(w.layer_ids) for w in block_balance(units, world).workers]


def local_groups(specs: list[GroupSpec], owned_keys: set[tuple[int, int]]):
    """Rank-local groups: each global (dim, exponent) group restricted to the owned blocks' members,
    in global member order.  Returns (local specs, slot map (layer, side, idx) -> SlotRef, global ids)."""
    out, slot_of, gids = [], {}, []
    for gi, sp in enumerate(specs):
        mem = tuple(m for m in sp.members if (m[0], m[2]) in owned_keys)
        if not mem:
            continue
        lg = len(out)
        for slot, m in enumerate(mem):
            slot_of[m] = SlotRef(lg, slot)
        out.append(GroupSpec(sp.dim, sp.exponent, mem))
        gids.append(gi)
    return out, slot_of, gids


def packed_positions(units: list[Unit], idxs: list[int]) -> np.ndarray:
    """Block-major offsets of the given units (matrix blocks first, then chunks, like the block table)."""
    mats = [i for i in idxs if units[i].matrix]
    vecs = [i for i in idxs if not units[i].matrix]
    pos, acc = [], 0
    for i in mats + vecs:
        pos.append(acc)
        acc += units[i].rows * units[i].cols
    return np.array(pos + [acc], dtype=np.int64)


class ShardedDash:
    """DASH optimizer whose preconditioner work is sharded by gradient block across ranks.

    ``step`` runs this rank's blocks (same kernels and global per-block seeds as the 1-GPU step), agrees on
    errors with the other ranks (an all-reduce of one flag before the exchange, so a rank that raised in its
    refresh never leaves the others waiting in the all-gather), packs its updated blocks and all-gathers every
    rank's shard (NCCL; a gloo group stages the exchange through host memory).  ``state`` is rank-local: its
    groups hold only the owned blocks, and each layer's slot refs point into them (SlotRef(-1, -1) for blocks
    another rank owns), so ``save_state`` refuses it rather than writing a partial checkpoint.
    """

    def __init__(self, params, cfg: ShampooConfig, rank: int, world: int, group=None):
        import torch.distributed as dist

        self.cfg, self.rank, self.world, self.group = cfg, rank, world, group
        self.dist = dist
        shapes = [tuple(p.shape) for p in params]
        layers, specs = build_layout(shapes, cfg.block_size)
        self.units = units_of(layers)
        self.assignment = assign_units(self.units, world)
        mine = self.assignment[rank]
        owned = {(self.units[i].layer_id, self.units[i].idx) for i in mine}
        lspecs, slot_of, self.global_group_ids = local_groups(specs, owned)
        dev = torch.device("cuda", torch.cuda.current_device())
        groups = []
        for sp in lspecs:
            n = len(sp.members)
            roots = torch.zeros((n, sp.dim, sp.dim), dtype=torch.float32, device=dev)
            roots.diagonal(dim1=1, dim2=2).fill_(1.0)
            groups.append(PrecondGroup(sp.dim, sp.exponent, sp.members,
                                       torch.zeros((n, sp.dim, sp.dim), dtype=torch.float32, device=dev), roots))
        local_layers = [_local_layer(lay, slot_of) for lay in layers]
        self.state = ShampooState(step=0, layers=local_layers, groups=groups, adam=[], momentum=None)
        self.state.runtime = _Runtime(self.state, shapes, cfg.block_size, cfg.graft.beta1 > 0.0, owned=owned,
                                      slot_of=slot_of)
        rt = self.state.runtime
        rt.global_gid = self.global_group_ids
        rt.seed_index = []
        for lgi, sp in enumerate(lspecs):  # global slot of every local member (power-iteration seeds)
            gslot = {m: i for i, m in enumerate(specs[self.global_group_ids[lgi]].members)}
            rt.seed_index.append(torch.tensor([gslot[m] for m in sp.members], dtype=torch.int32, device=dev))
        self.state.adam = rt.views(rt.adam)
        self.state.momentum = rt.views(rt.mom) if rt.mom is not None else None
        # exchange layout: rank q's blocks packed block-major (matrix blocks, then chunks) in order
        sizes = [int(packed_positions(self.units, a)[-1]) for a in self.assignment]
        self.max_packed = max(sizes)
        self.allgather_bytes = 4 * self.max_packed * world
        self.send = torch.zeros(self.max_packed, dtype=torch.float32, device=dev)
        self.recv = torch.zeros(world * self.max_packed, dtype=torch.float32, device=dev)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.tables = []
        for q in range(world):
            ow = {(self.units[i].layer_id, self.units[i].idx) for i in self.assignment[q]}
            m, v = block_rows(layers, rt.offsets, ow, slot_of={k: SlotRef(0, 0) for k in _all_keys(layers)})
            rows = [r[:4] + (0, 0, -1, -1) for r in m + v]
            blocks = _to_block_tensor(rows, dev)
            pos = torch.tensor(packed_positions(self.units, self.assignment[q])[:-1] + q * self.max_packed,
                               dtype=torch.int64, device=dev)
            self.tables.append((blocks, pos, len(rows)))

    @property
    def backend(self) -> str:
        return self.dist.get_backend(self.group)

    # ------------------------------------------------------------------ step
    def step_local(self, params, grads, seed: int = 0, events: dict | None = None):
        """This rank's share of the step: stats, roots and updates of its own blocks (into theta_out)."""
        st, cfg, rt = self.state, self.cfg, self.state.runtime
        t = st.step

        def mark(name):
            if events is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                events.setdefault(name, []).append(ev)

        mark("start")
        accumulate(st, grads, cfg)
        mark("accumulated")
        refresh_inverse_roots(st, cfg, seed=block_seed(seed, t), defer_check=True)
        mark("refreshed")
        rt.load(rt.theta, params)
        # no theta_out <- theta copy: the apply writes every owned block and the unpack every other rank's, and the
        # blocks partition the parameter space
        _lib.check(_lib.lib().dash_plan_apply(rt.plan, rt.theta.data_ptr(), rt.theta_out.data_ptr(),
                                              float(cfg.lr.value(t)), _lib.stream_ptr()), "dash_plan_apply")
        mark("applied")
        check_step_status(st)
        st.step = t + 1
        return rt.theta_out

    def _all_gather(self) -> None:
        if self.backend == "nccl":
            self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
            return
        host = torch.empty(self.world * self.max_packed, dtype=torch.float32)  # gloo: stage through the host
        self.dist.all_gather_into_tensor(host, self.send.cpu(), group=self.group)
        self.recv.copy_(host)

    def step(self, params, grads, seed: int = 0, events: dict | None = None):
        """One sharded DASH step; `params` (CUDA tensors) are updated in place on every rank."""
        rt = self.state.runtime
        failure = None
        try:
            self.step_local(params, grads, seed, events)
        except Exception as exc:  # noqa: BLE001 - re-raised after the ranks agree
            failure = exc
        self.flag.fill_(1 if failure is not None else 0)
        if self.backend == "nccl":
            self.dist.all_reduce(self.flag, op=self.dist.ReduceOp.MAX, group=self.group)
            bad = int(self.flag.item())
        else:
            f = self.flag.cpu()
            self.dist.all_reduce(f, op=self.dist.ReduceOp.MAX, group=self.group)
            bad = int(f.item())
        if failure is not None:
            raise failure
        if bad:
            raise RuntimeError("DASH step failed on another rank (see its error); no parameters were exchanged")
        L = _lib.lib()
        blocks, pos, n = self.tables[self.rank]
        local_pos = pos - self.rank * self.max_packed
        _lib.check(L.dash_pack_blocks(blocks.data_ptr(), n, local_pos.data_ptr(), rt.theta_out.data_ptr(),
                                      self.send.data_ptr(), _lib.stream_ptr()), "dash_pack_blocks")
        self._all_gather()
        for q in range(self.world):
            if q == self.rank:
                continue
            b, p, nq = self.tables[q]
            _lib.check(L.dash_unpack_blocks(b.data_ptr(), nq, p.data_ptr(), self.recv.data_ptr(),
                                            rt.theta_out.data_ptr(), _lib.stream_ptr()), "dash_unpack_blocks")
        for p_, o in zip(params, rt.views(rt.theta_out)):
            p_.copy_(o)
        if events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            events.setdefault("exchanged", []).append(ev)
        return params


def _local_layer(lay: LayerState, slot_of) -> LayerState:
    """The layer with its slot refs remapped to the rank-local groups (SlotRef(-1, -1): another rank's block)."""
    def refs(side, n):
        return tuple(slot_of.get((lay.layer_id, side, i), SlotRef(-1, -1)) for i in range(n))

    n = len(lay.left_refs)
    return LayerState(lay.layer_id, lay.shape, lay.layout, lay.chunk_bounds, refs("L", n),
                      refs("R", n) if lay.right_refs is not None else None)


def _all_keys(layers):
    keys = []
    for lay in layers:
        n = len(lay.layout.block_spans) if lay.is_matrix else len(lay.chunk_bounds)
        for i in range(n):
            keys.append((lay.layer_id, "L", i))
            keys.append((lay.layer_id, "R", i))
    return keys


def _to_block_tensor(rows, dev):
    """Pack dash_block structs (C layout: int64 off + 7 int32) into a device byte tensor."""
    import ctypes

    arr = (_lib.dash_block * max(len(rows), 1))(*[_lib.dash_block(*r) for r in rows])
    raw = bytes(memoryview(arr).cast("B"))[: ctypes.sizeof(_lib.dash_block) * len(rows)] if rows else b"\0" * 64
    return torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(dev)
