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
from .shampoo import (GroupSpec, LayerState, PrecondGroup, ShampooConfig, ShampooState, SlotRef, _refresh_flags,
                      _refresh_range, _Runtime, accumulate, accumulate_chunk, block_rows, build_layout,
                      check_step_status, refresh_inverse_roots)
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

    def __init__(self, params, cfg: ShampooConfig, rank: int, world: int, group=None,
                 exchange_chunks: int | None = None):
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
        # owner-only Adam / momentum: rt.adam / rt.mom hold this rank's blocks packed (rt.sofs), no per-layer views
        self.state.adam = []
        self.state.momentum = None
        # exchange layout: per exchange chunk (a contiguous layer range), rank q's blocks of it packed block-major
        # (matrix blocks, then chunks) in order; one all-gather per chunk
        self.nx = exchange_chunks if exchange_chunks is not None else _exchange_chunks()
        self.bounds = rt.chunk_bounds(self.nx, edges=False)
        self.flag = torch.zeros(1, dtype=torch.int32, device=dev)
        any_slot = {k: SlotRef(0, 0) for k in _all_keys(layers)}
        self.xchunks = []
        for c0, c1 in zip(self.bounds[:-1], self.bounds[1:]):
            parts = [[i for i in a if c0 <= self.units[i].layer_id < c1] for a in self.assignment]
            mx = max(max(int(packed_positions(self.units, a)[-1]) for a in parts), 1)
            tables = []
            for q in range(world):
                ow = {(self.units[i].layer_id, self.units[i].idx) for i in parts[q]}
                m, v = block_rows(layers, rt.offsets, ow, slot_of=any_slot)
                rows = [r[:4] + (0, 0, -1, -1) for r in m + v]
                pos = torch.tensor(packed_positions(self.units, parts[q])[:-1] + q * mx, dtype=torch.int64,
                                   device=dev)
                tables.append((_to_block_tensor(rows, dev), pos, len(rows)))
            self.xchunks.append(_XChunk(torch.zeros(mx, dtype=torch.float32, device=dev),
                                        torch.zeros(world * mx, dtype=torch.float32, device=dev), mx, tables,
                                        tables[rank][1] - rank * mx))
        self.max_packed = sum(x.mx for x in self.xchunks)
        self.allgather_bytes = 4 * self.max_packed * world
        self.comm = torch.cuda.Stream(device=dev)

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

    def _overlappable(self) -> bool:
        """Fixed-iteration Newton / Chebyshev refreshes never raise on the host mid-step (their errors are one
        device word read at the end), so their chunks can be computed between the exchange collectives."""
        return self.nx > 1 and not self.cfg.solver.require_convergence and self.cfg.solver.method != "evd"

    def _step_chunked(self, params, grads, seed: int, mark) -> None:
        """step_local with the refresh and apply cut into the exchange chunks: chunk k's all-gather (comm
        stream) runs under chunk k+1's solves.  Per-block work is independent of the chunking, so the result is
        bit-identical to step_local's."""
        st, cfg, rt = self.state, self.cfg, self.state.runtime
        t = st.step
        mark("start")
        if len(grads) != len(st.layers):
            raise ValueError(f"expected {len(st.layers)} gradients, got {len(grads)}")
        for layer, g in zip(st.layers, grads):
            if tuple(g.shape) != layer.shape:
                raise ValueError(f"layer {layer.layer_id}: gradient shape {tuple(g.shape)} != {layer.shape}")
        chunks = rt.ensure_chunks(cfg, st.layers, self.nx, edges=False)
        rt.load(rt.grad, grads)
        rt.load(rt.theta, params)
        refresh = t % cfg.update_freq == 0
        err, oks = _refresh_flags(rt, max(1, sum(len(ch.ranges) for ch in chunks)))
        step_seed, eta, k_ok = block_seed(seed, t), float(cfg.lr.value(t)), 0
        L = _lib.lib()
        for k, ch in enumerate(chunks):
            # the chunk plans share the split-gradient / graft scratch (indexed by chunk-local block), so a
            # chunk's accumulate, refresh and apply run back to back
            accumulate_chunk(st, cfg, ch, t)
            if k == 0:
                mark("accumulated")
            if refresh:
                for gi, s0, e0 in ch.ranges:
                    _refresh_range(st, cfg, gi, s0, e0, step_seed, err, oks[k_ok:k_ok + 1])
                    k_ok += 1
            if k == len(chunks) - 1:
                mark("refreshed")
            if ch.plan is not None:
                _lib.check(L.dash_plan_apply(ch.plan, rt.theta.data_ptr(), rt.theta_out.data_ptr(), eta,
                                             _lib.stream_ptr()), "dash_plan_apply")
            yield k
        mark("applied")
        rt.stats_valid, rt.stats_eps = True, cfg.epsilon
        if refresh:
            rt.pending_err = err
        check_step_status(st)
        st.step = t + 1

    def _send(self, k: int) -> None:
        """Pack this rank's blocks of exchange chunk k (after the compute stream's work so far) and start the
        chunk's all-gather on the comm stream (NCCL) or run it host-staged (gloo)."""
        x = self.xchunks[k]
        rt = self.state.runtime
        ready = torch.cuda.Event()
        ready.record()
        self.comm.wait_event(ready)
        blocks, _, n = x.tables[self.rank]
        with torch.cuda.stream(self.comm):
            if n:
                _lib.check(_lib.lib().dash_pack_blocks(blocks.data_ptr(), n, x.local_pos.data_ptr(),
                                                       rt.theta_out.data_ptr(), x.send.data_ptr(),
                                                       _lib.stream_ptr()), "dash_pack_blocks")
            if self.backend == "nccl":
                x.work = self.dist.all_gather_into_tensor(x.recv, x.send, group=self.group, async_op=True)
            else:
                host = torch.empty(self.world * x.mx, dtype=torch.float32)
                self.dist.all_gather_into_tensor(host, x.send.cpu(), group=self.group)
                x.recv.copy_(host)
                x.work = None

    def step(self, params, grads, seed: int = 0, events: dict | None = None):
        """One sharded DASH step; `params` (CUDA tensors) are updated in place on every rank.

        Every rank issues the same collectives whatever happens locally: one all-gather per exchange chunk,
        then an all-reduce of a failure flag; a rank that raised keeps sending (its data is never unpacked) so
        no rank is left waiting, and every rank raises before touching `params` if any rank failed."""
        rt = self.state.runtime

        def mark(name):
            if events is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                events.setdefault(name, []).append(ev)

        failure = None
        sent = 0
        try:
            if self._overlappable():
                for k in self._step_chunked(params, grads, seed, mark):
                    self._send(k)
                    sent = k + 1
            else:
                self.step_local(params, grads, seed, events)
        except Exception as exc:  # noqa: BLE001 - re-raised after the ranks agree
            failure = exc
        for k in range(sent, len(self.xchunks)):
            self._send(k)
        torch.cuda.current_stream().wait_stream(self.comm)
        for x in self.xchunks:
            if x.work is not None:
                x.work.wait()
                x.work = None
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
            raise RuntimeError("DASH step failed on another rank (see its error); parameters left unchanged")
        L = _lib.lib()
        for x in self.xchunks:
            for q in range(self.world):
                b, p, nq = x.tables[q]
                if q == self.rank or not nq:
                    continue
                _lib.check(L.dash_unpack_blocks(b.data_ptr(), nq, p.data_ptr(), x.recv.data_ptr(),
                                                rt.theta_out.data_ptr(), _lib.stream_ptr()), "dash_unpack_blocks")
        for p_, o in zip(params, rt.views(rt.theta_out)):
            p_.copy_(o)
        mark("exchanged")
        return params


@dataclass
class _XChunk:
    """One exchange chunk: this rank's send buffer, the gathered buffer (world x mx), per-rank pack tables."""

    send: torch.Tensor
    recv: torch.Tensor
    mx: int
    tables: list
    local_pos: torch.Tensor  # this rank's packed positions inside `send`
    work: object = None


def _exchange_chunks() -> int:
    """Exchange chunks per step (env DASH_XCHUNKS, default 2): each chunk's all-gather hides under the next
    chunk's solves; 1 = one all-gather after the whole step."""
    import os

    try:
        return max(1, int(os.environ.get("DASH_XCHUNKS", "2")))
    except ValueError:
        return 2


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
