"""Block-preconditioned Shampoo (DASH) on the B200 — drop-in for the reference ``shampoo.py``.

Same configuration dataclasses, state objects and functions as the reference (``GraftConfig``
``shampoo.py:53-63``, ``SolverConfig`` ``:66-87``, ``LrSchedule`` ``:90-109``, ``ShampooConfig`` ``:112-130``,
``SlotRef``/``LayerState``/``PrecondGroup``/``ShampooState`` ``:133-168``, ``init_state`` ``:233``,
``accumulate`` ``:238``, ``refresh_inverse_roots`` ``:312``, ``graft_scale`` ``:352``, ``step`` ``:362``), with
identical block structure, group/slot indexing, seeds and update rule.  All state lives on the GPU:

* one flat fp32 parameter space (grad / Adam / momentum / theta) with per-layer views,
* per group an fp32 EMA stack ``ema`` (n, d, d), fp32 ``roots`` and a split-f16 copy of the roots,
* a ``dash_plan`` (C ABI) holding the grouped-GEMM job tables of the statistics EMA and the apply.

A step is: gradient prep (Adam EMA, graft-direction norms) -> blocked split of G -> one grouped
tcgen05 launch for every L/R statistic -> per group symmetrize / scale (Frobenius or pooled power
iteration) / batched solver (NDB, CN, Chebyshev; EVD comparator) / root rescale -> two grouped launches
for U = L^(-1/4) G R^(-1/4) -> the grafted update.  NumPy inputs are accepted and returned (the
reference's types); CUDA tensors stay on the device.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field
from typing import Any

import numpy as np
import torch

from . import _lib
from .blocking import PartitionLayout, chunk_bounds, partition_layout
from .chebyshev import ChebCoefficients, clenshaw_split, fit_inverse_root
from .eigensolver import DampeningHeuristic, HeuristicKind, evd_inverse_root_torch, inverse_root_f64
from .errors import ConvergenceError, DegenerateSpectrumError
from .linalg import (PrecisionMode, Scratch, SplitStack, device, format_matrix, parse_matrix, passes_for, stall_for,
                     workspace)
from .roots import CnConfig, DeviceReports, IterationReport, cn_split, ndb_split
from .spectral import Frobenius, PowerIterationScaling, ScalingMode, block_seed, power_iteration_scales

SOLVER_METHODS = ("evd", "cn", "ndb", "cbshv")


@dataclass(frozen=True)
class GraftConfig:
    beta1: float = 0.0
    beta2: float = 0.999
    graft_eps: float = 1e-8

    def __post_init__(self) -> None:
        if not 0.0 <= self.beta1 < 1.0 or not 0.0 <= self.beta2 < 1.0:
            raise ValueError("betas must lie in [0, 1)")
        if self.graft_eps <= 0:
            raise ValueError("graft_eps must be positive")


@dataclass(frozen=True)
class SolverConfig:
    """Solver selection (shampoo.py:66-87).

    Difference from the reference: Newton-DB accepts every B200 precision mode (the reference allows
    FULL64 only, shampoo.py:81-82); on the B200 FULL64 and EMULATED32 both run split-f16 products.
    """

    method: str = "ndb"
    scaling: ScalingMode = PowerIterationScaling()
    tolerance: float = 1e-10
    max_iters: int = 100
    precision: PrecisionMode = PrecisionMode.FULL64
    heuristic: DampeningHeuristic = DampeningHeuristic(HeuristicKind.SHIFTED_RELU)
    cheb_degree: int = 60
    cheb_points: int = 1000
    cheb_interval: tuple[float, float] | None = None

    def __post_init__(self) -> None:
        if self.method not in SOLVER_METHODS:
            raise ValueError(f"unknown solver method {self.method!r}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.tolerance < 0:
            raise ValueError("tolerance must be >= 0")

    @property
    def require_convergence(self) -> bool:
        return self.tolerance > 0.0


@dataclass(frozen=True)
class LrSchedule:
    kind: str = "constant"
    base: float = 1e-3
    total_steps: int = 0
    final: float = 0.0

    def __post_init__(self) -> None:
        if self.kind not in ("constant", "linear", "cosine"):
            raise ValueError(f"unknown schedule {self.kind!r}")
        if self.kind != "constant" and self.total_steps < 1:
            raise ValueError("linear/cosine schedules need total_steps >= 1")

    def value(self, t: int) -> float:
        if self.kind == "constant":
            return self.base
        frac = min(t / self.total_steps, 1.0)
        if self.kind == "linear":
            return self.base + (self.final - self.base) * frac
        return self.final + (self.base - self.final) * 0.5 * (1.0 + math.cos(math.pi * frac))


@dataclass(frozen=True)
class ShampooConfig:
    beta_lr: float = 0.95
    epsilon: float = 1e-10
    lr: LrSchedule = LrSchedule()
    update_freq: int = 1
    solver: SolverConfig = SolverConfig()
    block_size: int = 256
    graft: GraftConfig = GraftConfig()

    def __post_init__(self) -> None:
        if not 0.0 < self.beta_lr < 1.0:
            raise ValueError("beta_lr must lie in (0, 1)")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")
        if self.update_freq < 1:
            raise ValueError("update_freq must be >= 1")
        if self.block_size < 1:
            raise ValueError("block_size must be >= 1")


@dataclass(frozen=True)
class SlotRef:
    group: int
    slot: int


@dataclass
class LayerState:
    layer_id: int
    shape: tuple[int, ...]
    layout: PartitionLayout | None
    chunk_bounds: tuple[tuple[int, int], ...] | None
    left_refs: tuple[SlotRef, ...]
    right_refs: tuple[SlotRef, ...] | None

    @property
    def is_matrix(self) -> bool:
        return self.layout is not None


@dataclass
class PrecondGroup:
    dim: int
    exponent: int
    members: tuple[tuple[int, str, int], ...]
    ema: torch.Tensor     # (n, dim, dim) fp32, CUDA
    roots: torch.Tensor   # (n, dim, dim) fp32, CUDA


@dataclass
class ShampooState:
    step: int
    layers: list[LayerState]
    groups: list[PrecondGroup]
    adam: list[torch.Tensor]
    momentum: list[torch.Tensor] | None
    runtime: Any = field(default=None, repr=False)


def _chunk_bounds(length: int, block_size: int) -> tuple[tuple[int, int], ...]:
    return chunk_bounds(length, block_size)


# ============================================================================ structure
def _group_keys(shapes, block_size):
    keyed: dict[tuple[int, int], list[tuple[int, str, int]]] = {}
    meta = []
    for layer_id, shape in enumerate(shapes):
        if len(shape) == 2:
            layout = partition_layout(shape, block_size)
            meta.append((layout, None))
            for idx, ((r0, r1), (c0, c1)) in enumerate(layout.block_spans):
                keyed.setdefault((r1 - r0, 4), []).append((layer_id, "L", idx))
                keyed.setdefault((c1 - c0, 4), []).append((layer_id, "R", idx))
        elif len(shape) == 1:
            bounds = _chunk_bounds(shape[0], block_size)
            meta.append((None, bounds))
            for idx, (s, e) in enumerate(bounds):
                keyed.setdefault((e - s, 2), []).append((layer_id, "L", idx))
        else:
            raise ValueError(f"layer {layer_id}: only 1-D and 2-D layers are supported, got shape {shape}")
    return keyed, meta


@dataclass(frozen=True)
class GroupSpec:
    """Host-side description of one preconditioner group (no device data)."""

    dim: int
    exponent: int
    members: tuple[tuple[int, str, int], ...]


def build_layout(shapes, block_size: int) -> tuple[list[LayerState], list[GroupSpec]]:
    """Pure-host block structure: layers with slot refs + groups (shampoo.py:176-230), bit-exact."""
    keyed, meta = _group_keys([tuple(s) for s in shapes], block_size)
    side_order = {"L": 0, "R": 1}
    specs: list[GroupSpec] = []
    ref_of: dict[tuple[int, str, int], SlotRef] = {}
    for gi, (dim, exponent) in enumerate(sorted(keyed)):
        members = tuple(sorted(keyed[(dim, exponent)], key=lambda m: (m[0], side_order[m[1]], m[2])))
        for slot, member in enumerate(members):
            ref_of[member] = SlotRef(group=gi, slot=slot)
        specs.append(GroupSpec(dim, exponent, members))
    layers = []
    for layer_id, shape in enumerate(shapes):
        layout, bounds = meta[layer_id]
        if layout is not None:
            nb = layout.num_blocks
            left = tuple(ref_of[(layer_id, "L", i)] for i in range(nb))
            right = tuple(ref_of[(layer_id, "R", i)] for i in range(nb))
            layers.append(LayerState(layer_id, tuple(shape), layout, None, left, right))
        else:
            left = tuple(ref_of[(layer_id, "L", i)] for i in range(len(bounds)))
            layers.append(LayerState(layer_id, tuple(shape), None, bounds, left, None))
    return layers, specs


def _build_structure(shapes: list[tuple[int, ...]], block_size: int, track_momentum: bool) -> ShampooState:
    """Host structure + device state: EMA zeros, identity roots, flat Adam / momentum (shampoo.py:176-230)."""
    layers, specs = build_layout(shapes, block_size)
    dev = device()
    groups: list[PrecondGroup] = []
    for sp in specs:
        n = len(sp.members)
        roots = torch.zeros((n, sp.dim, sp.dim), dtype=torch.float32, device=dev)
        roots.diagonal(dim1=1, dim2=2).fill_(1.0)
        groups.append(PrecondGroup(dim=sp.dim, exponent=sp.exponent, members=sp.members,
                                   ema=torch.zeros((n, sp.dim, sp.dim), dtype=torch.float32, device=dev),
                                   roots=roots))
    state = ShampooState(step=0, layers=layers, groups=groups, adam=[], momentum=None)
    state.runtime = _Runtime(state, [tuple(s) for s in shapes], block_size, track_momentum)
    state.adam = state.runtime.views(state.runtime.adam)
    state.momentum = state.runtime.views(state.runtime.mom) if track_momentum else None
    return state


def init_state(params, cfg: ShampooConfig) -> ShampooState:
    shapes = [tuple(p.shape) for p in params]
    return _build_structure(shapes, cfg.block_size, cfg.graft.beta1 > 0.0)


# ============================================================================ device runtime
def block_rows(layers: list[LayerState], offsets, owned=None, slot_of=None):
    """dash_block rows (off, ld, rows, cols, group_l, slot_l, group_r, slot_r): matrix blocks first.

    `owned`: optional set of (layer_id, block_idx) to keep (block sharding); `slot_of`: optional map
    (layer_id, side, idx) -> SlotRef overriding the layer's refs (rank-local group numbering)."""
    mats, vecs = [], []
    for layer in layers:
        base = int(offsets[layer.layer_id])
        ref = (lambda side, i: slot_of[(layer.layer_id, side, i)]) if slot_of is not None else \
            (lambda side, i: (layer.left_refs if side == "L" else layer.right_refs)[i])
        if layer.is_matrix:
            n = layer.shape[1]
            for idx, ((r0, r1), (c0, c1)) in enumerate(layer.layout.block_spans):
                if owned is not None and (layer.layer_id, idx) not in owned:
                    continue
                lr, rr = ref("L", idx), ref("R", idx)
                mats.append((base + r0 * n + c0, n, r1 - r0, c1 - c0, lr.group, lr.slot, rr.group, rr.slot))
        else:
            for idx, (s, e) in enumerate(layer.chunk_bounds):
                if owned is not None and (layer.layer_id, idx) not in owned:
                    continue
                lr = ref("L", idx)
                vecs.append((base + s, 1, e - s, 1, lr.group, lr.slot, -1, -1))
    return mats, vecs


def block_keys(layers: list[LayerState], owned=None) -> list[tuple[int, int]]:
    """(layer_id, block_idx) of every block_rows row, in the same order (matrix blocks first, then chunks)."""
    mats, vecs = [], []
    for layer in layers:
        n = len(layer.layout.block_spans) if layer.is_matrix else len(layer.chunk_bounds)
        keys = [(layer.layer_id, i) for i in range(n) if owned is None or (layer.layer_id, i) in owned]
        (mats if layer.is_matrix else vecs).extend(keys)
    return mats + vecs


@dataclass
class _Chunk:
    """One pipeline chunk of the host-buffer step: layers [l0, l1) = flat elements [e0, e1)."""

    l0: int
    l1: int
    e0: int
    e1: int
    plan: Any
    ws: torch.Tensor
    blocks_c: Any
    ranges: list  # (group index, first slot, end slot)
    sofs: Any = None  # owner-only state: the chunk's blocks' packed state offsets (kept alive for the plan)


class _Runtime:
    """Flat device buffers + the C-ABI plan for one optimizer structure (or one rank's shard of it)."""

    def __init__(self, state: ShampooState, shapes, block_size: int, momentum: bool, owned=None, slot_of=None):
        self.dev = device()
        self.shapes = shapes
        self.bsz = block_size
        self.sizes = [int(np.prod(s)) for s in shapes]
        self.offsets = np.concatenate([[0], np.cumsum(self.sizes)]).astype(np.int64)
        total = int(self.offsets[-1])
        f32 = dict(dtype=torch.float32, device=self.dev)
        self.grad = torch.zeros(total, **f32)
        self.theta = torch.zeros(total, **f32)
        self.theta_out = torch.zeros(total, **f32)
        mats, vecs = block_rows(state.layers, self.offsets, owned, slot_of)
        self.nb_m, self.nb_v = len(mats), len(vecs)
        nb = self.nb_m + self.nb_v
        # Adam / momentum: over the flat parameter space, or -- for a rank's shard -- owner-only, the owned
        # blocks packed back to back (each padded to a multiple of 4 elements for 16-byte access)
        self.owned, self.slot_of = owned, slot_of
        self.sofs, self.sofs_of = None, None
        if owned is not None:
            sizes = [(r[2] * r[3] + 3) // 4 * 4 for r in mats + vecs]
            base = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
            self.sofs = torch.tensor(base[:-1], dtype=torch.int64, device=self.dev)
            self.sofs_of = dict(zip(block_keys(state.layers, owned), base[:-1].tolist()))
            total = int(base[-1])
        self.adam = torch.zeros(total, **f32)
        self.mom = torch.zeros(total, **f32) if momentum else None
        self.block_rows = mats + vecs
        Arr = _lib.dash_block * nb
        self.blocks_c = Arr(*[_lib.dash_block(*b) for b in self.block_rows])
        self.gsm = SplitStack(self.nb_m, block_size, block_size, self.dev) if self.nb_m else None
        self.tm = SplitStack(self.nb_m, block_size, block_size, self.dev) if self.nb_m else None
        self.gsv = SplitStack(self.nb_v, block_size, 1, self.dev) if self.nb_v else None
        self.um = torch.zeros((max(self.nb_m, 1), block_size, block_size), **f32)
        self.uv = torch.zeros((max(self.nb_v, 1), block_size), **f32)
        L = _lib.lib()
        self.prep_parts = L.dash_prep_parts()
        self.pn_part = torch.zeros(nb * self.prep_parts, **f32)
        self.un_stride = L.dash_apply_partials(block_size)  # partials per tile x tiles of a full block
        self.un_part = torch.zeros(nb * self.un_stride, **f32)
        self.gamax = torch.zeros(nb, dtype=torch.int32, device=self.dev)
        self.graft_s = torch.zeros(nb, **f32)
        self.root_split = [SplitStack(len(g.members), g.dim, g.dim, self.dev) for g in state.groups]
        for g, rs in zip(state.groups, self.root_split):
            rs.load(g.roots)  # identity roots before the first refresh
        self.groups = state.groups
        # per-group scratch
        self.g_amax = [torch.zeros(len(g.members), dtype=torch.int32, device=self.dev) for g in state.groups]
        self.g_fro = [torch.zeros(len(g.members) * self.prep_parts, **f32) for g in state.groups]
        self.plan = None
        self.plan_key = None
        self.scratch = Scratch(self.dev)   # per-step solver buffers, reused across steps
        self.stats_valid = False           # g_amax / g_fro describe the current EMA (set by accumulate)
        self.stats_eps = None
        self.pending_err = None            # device error word of the last fixed-iteration refresh
        self._slot_ids: dict = {}

    def slot_ids(self, gi: int) -> torch.Tensor:
        """0..n-1 for group gi on the device (global slots of a member range: the power-iteration seeds)."""
        ids = self._slot_ids.get(gi)
        if ids is None:
            ids = self._slot_ids[gi] = torch.arange(len(self.groups[gi].members), dtype=torch.int32, device=self.dev)
        return ids

    def views(self, flat: torch.Tensor) -> list[torch.Tensor]:
        return [flat[int(self.offsets[i]):int(self.offsets[i + 1])].view(s) for i, s in enumerate(self.shapes)]

    def _create_plan(self, blocks_c, nb_m: int, nb_v: int, key, sofs=None):
        """A C-ABI plan over a block table (all blocks, or one pipeline chunk's); returns (plan, workspace).
        `sofs`: the blocks' packed optimizer-state offsets (owner-only state), default this runtime's."""
        L = _lib.lib()
        ng = len(self.groups)
        gdim = (ctypes_int * ng)(*[g.dim for g in self.groups])
        gsize = (ctypes_int * ng)(*[len(g.members) for g in self.groups])
        gema = (ctypes_vp * ng)(*[g.ema.data_ptr() for g in self.groups])
        groot = (_lib.dash_stack * ng)(*[rs.c() for rs in self.root_split])
        ws = workspace(L.dash_plan_ws_bytes(nb_m, nb_v), self.dev)
        status = ctypes_int(0)
        p = L.dash_plan_create(
            blocks_c, nb_m, nb_v, self.bsz, ng, gdim, gsize, gema, groot,
            self.grad.data_ptr(), self.adam.data_ptr(), self.mom.data_ptr() if self.mom is not None else None,
            self.gsm.ref() if self.gsm else None, self.gsv.ref() if self.gsv else None,
            self.tm.ref() if self.tm else None, self.um.data_ptr(), self.uv.data_ptr(), self.pn_part.data_ptr(),
            self.un_part.data_ptr(), self.gamax.data_ptr(), self.graft_s.data_ptr(), float(key[0]),
            key[1], ws.data_ptr(), ws.numel(), _lib.stream_ptr(), ctypes_byref(status))
        if not p:
            _lib.check(status.value or _lib.DASH_EINVAL, "dash_plan_create")
        sofs = self.sofs if sofs is None else sofs
        if sofs is not None:
            _lib.check(L.dash_plan_set_state_offsets(p, sofs.data_ptr()), "dash_plan_set_state_offsets")
        return p, ws

    def ensure_plan(self, cfg: ShampooConfig) -> None:
        key = (cfg.beta_lr, passes_for(cfg.solver.precision))
        if self.plan is not None and self.plan_key == key:
            return
        self.close()
        self.plan, self.plan_ws = self._create_plan(self.blocks_c, self.nb_m, self.nb_v, key)
        self.plan_key = key

    def chunk_bounds(self, nchunks: int, edges: bool = True) -> list[int]:
        """Layer boundaries of `nchunks` contiguous chunks of about equal size.  `edges` (host-buffer step):
        the first chunk's upload and the last chunk's download are the only copies nothing hides, so those
        chunks are one layer each and the layers between them are cut into nchunks - 2 chunks."""
        nl = len(self.sizes)
        lo, hi = (1, nl - 1) if edges and nchunks >= 3 and nl >= 3 else (0, nl)
        inner = max(1, nchunks - (2 if lo else 0))
        target = sum(self.sizes[lo:hi]) / inner
        bounds, acc = ([0, lo] if lo else [0]), 0
        for i in range(lo, hi):
            acc += self.sizes[i]
            if acc >= target * (len(bounds) - (1 if lo else 0)) and len(bounds) < inner + (1 if lo else 0) \
                    and i + 1 < hi:
                bounds.append(i + 1)
        if hi < nl:
            bounds.append(hi)
        bounds.append(nl)
        return bounds

    def ensure_chunks(self, cfg: ShampooConfig, layers: list[LayerState], nchunks: int, edges: bool = True) -> list:
        """Pipeline chunks of the host-buffer step (or of a rank's overlapped exchange): contiguous layer ranges
        of about equal size, each with its own plan over its (owned) blocks and, per group, the contiguous slot
        range of its members (members are sorted by layer, shampoo.py:185-202)."""
        key = (cfg.beta_lr, passes_for(cfg.solver.precision), nchunks, edges)
        if getattr(self, "chunks", None) and self.chunks_key == key:
            return self.chunks
        self.close_chunks()
        bounds = self.chunk_bounds(nchunks, edges)
        chunks = []
        for c0, c1 in zip(bounds[:-1], bounds[1:]):
            owned = set()
            for lay in layers[c0:c1]:
                nb = len(lay.layout.block_spans) if lay.is_matrix else len(lay.chunk_bounds)
                owned.update((lay.layer_id, i) for i in range(nb)
                             if self.owned is None or (lay.layer_id, i) in self.owned)
            if not owned:  # (a rank's shard may hold no block of a layer range)
                chunks.append(_Chunk(c0, c1, int(self.offsets[c0]), int(self.offsets[c1]), None, None, None, []))
                continue
            mats, vecs = block_rows(layers, self.offsets, owned, self.slot_of)
            rows = mats + vecs
            blocks_c = (_lib.dash_block * len(rows))(*[_lib.dash_block(*b) for b in rows])
            sofs = None
            if self.sofs_of is not None:
                sofs = torch.tensor([self.sofs_of[k] for k in block_keys(layers, owned)], dtype=torch.int64,
                                    device=self.dev)
            plan, ws = self._create_plan(blocks_c, len(mats), len(vecs), key, sofs)
            ranges = []
            for gi, g in enumerate(self.groups):
                slots = [k for k, m in enumerate(g.members) if c0 <= m[0] < c1]
                if slots:
                    assert slots == list(range(slots[0], slots[-1] + 1))
                    ranges.append((gi, slots[0], slots[-1] + 1))
            chunks.append(_Chunk(c0, c1, int(self.offsets[c0]), int(self.offsets[c1]), plan, ws, blocks_c, ranges,
                                 sofs))
        self.chunks, self.chunks_key = chunks, key
        return chunks

    def close_chunks(self) -> None:
        for ch in getattr(self, "chunks", None) or []:
            _lib.lib().dash_plan_destroy(ch.plan)
        self.chunks = None

    def close(self) -> None:
        if self.plan:
            _lib.lib().dash_plan_destroy(self.plan)
            self.plan = None
        self.close_chunks()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass

    # ---- host <-> flat buffers
    def load(self, flat: torch.Tensor, tensors) -> None:
        for i, t in enumerate(tensors):
            if tuple(t.shape) != self.shapes[i]:
                raise ValueError(f"layer {i}: shape {tuple(t.shape)} != {self.shapes[i]}")
            dst = flat[int(self.offsets[i]):int(self.offsets[i + 1])]
            if isinstance(t, torch.Tensor):
                dst.copy_(t.reshape(-1), non_blocking=t.is_cuda or t.is_pinned())
            else:
                dst.copy_(torch.from_numpy(np.ascontiguousarray(t, dtype=np.float32).reshape(-1)))


import ctypes as _ct  # noqa: E402

ctypes_int = _ct.c_int
ctypes_vp = _ct.c_void_p
ctypes_byref = _ct.byref


# ============================================================================ accumulate
def accumulate(state: ShampooState, grads, cfg: ShampooConfig) -> ShampooState:
    """EMA update of every preconditioner block and the Adam second moment (shampoo.py:238-278)."""
    if len(grads) != len(state.layers):
        raise ValueError(f"expected {len(state.layers)} gradients, got {len(grads)}")
    rt: _Runtime = state.runtime
    for layer, g in zip(state.layers, grads):
        if tuple(g.shape) != layer.shape:
            raise ValueError(f"layer {layer.layer_id}: gradient shape {tuple(g.shape)} != {layer.shape}")
    rt.ensure_plan(cfg)
    rt.load(rt.grad, grads)
    n_acc = state.step + 1
    st = _lib.lib().dash_plan_accumulate(rt.plan, float(cfg.graft.beta2), float(cfg.graft.beta1), n_acc,
                                         float(cfg.graft.graft_eps), _lib.stream_ptr())
    _lib.check(st, "dash_plan_accumulate")
    for gi, g in enumerate(state.groups):  # linalg.symmetrize on every EMA block
        st = _lib.lib().dash_group_sym(g.ema.data_ptr(), len(g.members), g.dim, float(cfg.epsilon),
                                       rt.g_amax[gi].data_ptr(), rt.g_fro[gi].data_ptr(), _lib.stream_ptr())
        _lib.check(st, "dash_group_sym")
    rt.stats_valid, rt.stats_eps = True, cfg.epsilon
    return state


# ============================================================================ refresh
_cheb_cache: dict[tuple, ChebCoefficients] = {}


def _solver_coefficients(solver: SolverConfig, p: int) -> ChebCoefficients:
    interval = solver.cheb_interval if solver.cheb_interval is not None else (1e-10, 1.0 + 1e-10)
    key = (p, solver.cheb_degree, solver.cheb_points, interval)
    if key not in _cheb_cache:
        _cheb_cache[key] = fit_inverse_root(p, degree=solver.cheb_degree, num_points=solver.cheb_points,
                                            interval=interval)
    return _cheb_cache[key]


def _check_reports(group: PrecondGroup, reports, offset: int = 0) -> None:
    failed = [i for i, r in enumerate(reports) if not r.converged]
    if failed:
        details = ", ".join(
            f"layer {group.members[offset + i][0]} side {group.members[offset + i][1]} block "
            f"{group.members[offset + i][2]} (residual {reports[i].residual:.3e})" for i in failed)
        raise ConvergenceError(f"inverse-root solver failed on: {details}")


def _group_stats(state: ShampooState, cfg: ShampooConfig) -> None:
    """max|a| and sum(a^2) of a = ema + eps I for every group (normally a by-product of accumulate's
    symmetrization; recomputed when the EMA did not come from accumulate, e.g. after init_state / load_state).
    Symmetrizing a symmetric EMA (the only kind accumulate and checkpoints produce) leaves it bit-identical."""
    rt: _Runtime = state.runtime
    for gi, g in enumerate(state.groups):
        _lib.check(_lib.lib().dash_group_sym(g.ema.data_ptr(), len(g.members), g.dim, float(cfg.epsilon),
                                             rt.g_amax[gi].data_ptr(), rt.g_fro[gi].data_ptr(), _lib.stream_ptr()),
                   "dash_group_sym")
    rt.stats_eps = cfg.epsilon


def _raise_scale_error(state: ShampooState, err: list[int]) -> None:
    code, gi = err
    if code == 2:
        raise DegenerateSpectrumError("power iteration pool collapsed twice on a nonzero matrix")
    raise ConvergenceError(f"non-positive scale in group of dim {state.groups[gi].dim}")


def check_step_status(state: ShampooState) -> None:
    """Raise the error a fixed-iteration refresh recorded on the device (one 8-byte read), if any.

    The failing group and every later one kept their previous roots (the commit is gated on the device),
    which is the state the reference leaves behind when its refresh loop raises."""
    rt: _Runtime = state.runtime
    err = getattr(rt, "pending_err", None)
    if err is None:
        return
    rt.pending_err = None
    vals = err.tolist()  # one (code, group) pair per refresh stream: the reference raises for the first group
    fails = [vals[i:i + 2] for i in range(0, len(vals), 2) if vals[i]]
    if fails:
        _raise_scale_error(state, min(fails, key=lambda f: f[1]))


def refresh_inverse_roots(state: ShampooState, cfg: ShampooConfig, seed: int = 0, *, defer_check: bool = False
                          ) -> ShampooState:
    """Recompute cached inverse roots; no-op unless step % update_freq == 0 (shampoo.py:312-349).

    Fixed-iteration solves (tolerance 0) never synchronise with the host: the scale checks run on the device
    (``dash_scale_check``), a failing group's roots are not committed, and the recorded error is raised at the
    end of the refresh -- or, with ``defer_check`` (used by ``step``), at the end of the step, before any
    parameter is returned.  Tolerance-mode solves read the per-block reports group by group like the
    reference; their roots are committed only after the checks pass.  In FULL64 mode a block the fp32-class
    iteration cannot converge (frozen by the divergence watch or a non-finite residual before max_iters) is
    re-solved in float64 by EVD: (ema + eps I)^(-1/p), the value the reference's float64 iteration reaches.
    """
    if state.step % cfg.update_freq != 0:
        return state
    rt: _Runtime = state.runtime
    if not rt.stats_valid or rt.stats_eps != cfg.epsilon:
        _group_stats(state, cfg)
    rt.stats_valid = True
    err, oks = _refresh_flags(rt, len(state.groups))
    if cfg.solver.method == "evd":
        for gi, group in enumerate(state.groups):
            group.roots.copy_(evd_inverse_root_torch(group.ema, group.exponent, cfg.solver.heuristic))
            rt.root_split[gi].load(group.roots)
        return state
    # Fixed-iteration refreshes run the groups other than the largest on a second stream with their own scratch
    # and error word: their short, few-wave launches fill the big group's launch tails instead of running alone.
    # Every per-block computation is stream- and batch-independent, so the roots are bit-identical.
    side = len(state.groups) > 1 and not cfg.solver.require_convergence
    big = max(range(len(state.groups)), key=lambda g: len(state.groups[g].members) * state.groups[g].dim ** 3)
    main = torch.cuda.current_stream()
    if side:
        if getattr(rt, "side_stream", None) is None:
            rt.side_stream, rt.side_scratch = torch.cuda.Stream(device=rt.dev), Scratch(rt.dev)
        rt.side_stream.wait_stream(main)
        err_side = rt.side_scratch.tensor("err", (2,), torch.int32)
        with torch.cuda.stream(rt.side_stream):
            err_side.zero_()
    for gi, group in enumerate(state.groups):
        if side and gi != big:
            with torch.cuda.stream(rt.side_stream):
                _refresh_range(state, cfg, gi, 0, len(group.members), seed, err_side, oks[gi:gi + 1],
                               scratch=rt.side_scratch)
        else:
            _refresh_range(state, cfg, gi, 0, len(group.members), seed, err, oks[gi:gi + 1])
    if side:
        main.wait_stream(rt.side_stream)
    if not cfg.solver.require_convergence:
        rt.pending_err = torch.cat([err, err_side]) if side else err
        if not defer_check:
            check_step_status(state)
    return state


def _refresh_flags(rt: "_Runtime", nflags: int):
    """The refresh's shared device error word (zeroed) and per-range commit gates."""
    err = rt.scratch.tensor("err", (2,), torch.int32)
    err.zero_()
    return err, rt.scratch.tensor("ok", (max(nflags, 1),), torch.int32)


def _refresh_range(state: ShampooState, cfg: ShampooConfig, gi: int, s: int, e: int, seed: int,
                   err: torch.Tensor, ok: torch.Tensor, scratch: Scratch | None = None) -> None:
    """Scale, solve, check and commit the roots of group `gi`'s members [s, e) (the whole group, or one chunk of
    the pipelined host step); every per-block computation is independent of the range, so any partition of a
    group gives bit-identical roots."""
    rt: _Runtime = state.runtime
    solver = cfg.solver
    L = _lib.lib()
    sc = scratch if scratch is not None else rt.scratch
    group = state.groups[gi]
    p, n, d = group.exponent, e - s, group.dim
    gids = getattr(rt, "global_gid", None)  # block sharding: rank-local group gi is global group gids[gi]
    sidx = getattr(rt, "seed_index", None)
    gid = gids[gi] if gids is not None else gi
    tol_mode = solver.require_convergence
    mode = solver.precision
    ema = group.ema[s:e]
    roots = group.roots[s:e]
    rsplit = rt.root_split[gi].slice(s, e)
    a = sc.stack("a", n, d, d)
    a.amax.copy_(rt.g_amax[gi][s:e])  # exact max|ema + eps I| (accumulate's symmetrization)
    _lib.check(L.dash_group_split_a(ema.data_ptr(), float(cfg.epsilon), a.ref(), _lib.stream_ptr()),
               "dash_group_split_a")
    scale = sc.tensor("scale", (n,))
    inv = sc.tensor("inv", (n,))
    status = sc.tensor("status", (n,), torch.int32)
    status.zero_()
    if isinstance(solver.scaling, Frobenius):
        parts = rt.prep_parts
        _lib.check(L.dash_fro_scale(rt.g_fro[gi][s * parts:].data_ptr(), n, scale.data_ptr(), inv.data_ptr(),
                                    _lib.stream_ptr()), "dash_fro_scale")
    else:  # block i of the group draws from block_seed(group seed, global slot of i) (spectral.py:117)
        seed_index = sidx[gi][s:e] if sidx is not None else (rt.slot_ids(gi)[s:e] if s > 0 else None)
        power_iteration_scales(ema, cfg.epsilon, solver.scaling.pool, solver.scaling.iters, block_seed(seed, gid),
                               scale, inv, status, seed_index, a_split=a)
    _lib.check(L.dash_scale_check(scale.data_ptr(), status.data_ptr(), n, gi, ok.data_ptr(), err.data_ptr(),
                                  _lib.stream_ptr()), "dash_scale_check")
    if tol_mode:  # the reference raises here, before any solve of this group (shampoo.py:323-325)
        vals = err.tolist()
        if vals[0]:
            _raise_scale_error(state, vals)
    if solver.method == "cbshv":
        clenshaw_split(a, _solver_coefficients(solver, p), inv, inv_pow(inv, p, sc), roots, rsplit, mode, gate=ok,
                       scratch=sc)
        return
    if solver.method == "cn":
        src, rep = cn_split(a, inv, CnConfig(p=p, tolerance=solver.tolerance, max_iters=solver.max_iters), mode,
                            scratch=sc)
        reps = [rep]
    elif p == 2:
        # the iterates stay in upper pair-block storage (the second solve of a 4th root reads Y1 that way); only
        # the root that is read next is completed
        _, src, rep = ndb_split(a, inv, solver.tolerance, solver.max_iters, mode, complete=False, scratch=sc,
                                tag="ndb1", outputs="z")
        reps = [rep]
    else:  # (each chain's last iteration computes only the iterate read next: Y1, then Z2)
        y1, _, r1 = ndb_split(a, inv, solver.tolerance, solver.max_iters, mode, complete=False, scratch=sc,
                              tag="ndb1", outputs="y")
        _, src, r2 = ndb_split(y1, None, solver.tolerance, solver.max_iters, mode, complete=False, scratch=sc,
                               tag="ndb2", outputs="z")
        reps = [r1, r2]
    fallback = None
    if tol_mode:  # per-block reports, in the reference's order (first chain, then second)
        lists = [r.to_list() for r in reps]
        # FULL64 re-solves in float64 the blocks its fp32-class iteration could not converge: frozen before
        # max_iters (watch / non-finite), or -- when the requested tolerance is below the floor, so the
        # reference's float64 loop would have converged where ours stalls -- any unconverged block
        floor_mode = stall_for(solver.tolerance, mode) > 0.0
        bad = sorted({i for lst in lists for i, r in enumerate(lst)
                      if not r.converged and (floor_mode or r.iterations < solver.max_iters)})
        if mode is PrecisionMode.FULL64 and bad:
            fallback = bad
            for lst in lists:
                for i in bad:
                    lst[i] = IterationReport(lst[i].iterations, lst[i].residual, True)
        for lst in lists:
            _check_reports(group, lst, offset=s)
    # roots = Z * scale^(-1/p)  -> fp32 state roots + split copy for the apply (gated on the scale checks)
    # (the Newton-DB root is still in upper pair-block storage: the rescale reads its lower blocks transposed)
    _lib.check(L.dash_scale_stack(src.ref(), inv.data_ptr(), 1.0 / p, roots.data_ptr(), roots.stride(0),
                                  roots.stride(1), rsplit.ref(), ok.data_ptr(), int(solver.method == "ndb"),
                                  _lib.stream_ptr()), "dash_scale_stack")
    if fallback:
        idx = torch.tensor(fallback, dtype=torch.long, device=rt.dev)
        roots[idx] = inverse_root_f64(ema[idx], cfg.epsilon, p)
        rsplit.load(roots)


def inv_pow(inv: torch.Tensor, p: int, scratch=None) -> torch.Tensor:
    """scale^(-1/p) from 1/scale (device; tiny vector)."""
    out = scratch.tensor("inv_pow", tuple(inv.shape)) if scratch is not None else torch.empty_like(inv)
    out.copy_(inv.double().pow(1.0 / p))
    return out


# ============================================================================ step
def graft_scale(u, p) -> float:
    """Frobenius-norm ratio ||p|| / ||u||; zero when the update vanishes (shampoo.py:352-359)."""
    if tuple(u.shape) != tuple(p.shape):
        raise ValueError(f"shape mismatch: {tuple(u.shape)} vs {tuple(p.shape)}")
    nu = float(np.linalg.norm(np.asarray(u.cpu() if isinstance(u, torch.Tensor) else u, dtype=np.float64)))
    if nu == 0.0:
        return 0.0
    return float(np.linalg.norm(np.asarray(p.cpu() if isinstance(p, torch.Tensor) else p, dtype=np.float64))) / nu


def step(state: ShampooState, params, grads, cfg: ShampooConfig, seed: int = 0, *, inplace: bool = False,
         events: dict | None = None):
    """One optimizer step; returns updated parameters and the mutated state (shampoo.py:362-404).

    NumPy params -> new float64 NumPy arrays (like the reference).  CPU tensors -> new fp32 CPU tensors
    (pinned).  CUDA tensors -> new fp32 tensors, or the inputs updated in place when ``inplace=True``.
    ``events`` (optional dict) collects CUDA events around the accumulate / refresh / apply phases.
    """
    if len(params) != len(state.layers):
        raise ValueError(f"expected {len(state.layers)} parameter tensors, got {len(params)}")
    rt: _Runtime = state.runtime
    t = state.step

    def mark(name):
        if events is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            events.setdefault(name, []).append(ev)

    if _pipelined(state, params, grads, cfg):
        return _step_pipelined(state, params, grads, cfg, seed, events)
    mark("start")
    accumulate(state, grads, cfg)
    host_params = isinstance(params[0], torch.Tensor) and not params[0].is_cuda and params[0].is_pinned()
    prefetch = None
    if host_params:  # H2D of the (pinned) parameters overlaps the refresh on a side stream
        if len(params) != len(rt.shapes):
            raise ValueError(f"expected {len(rt.shapes)} parameter tensors, got {len(params)}")
        if getattr(rt, "copy_stream", None) is None:
            rt.copy_stream = torch.cuda.Stream(device=rt.dev)
        rt.copy_stream.wait_stream(torch.cuda.current_stream())  # after the gradient H2D + statistics
        with torch.cuda.stream(rt.copy_stream):
            rt.load(rt.theta, params)
        prefetch = torch.cuda.Event()
        prefetch.record(rt.copy_stream)
    mark("accumulated")
    refresh_inverse_roots(state, cfg, seed=block_seed(seed, t), defer_check=True)
    mark("refreshed")
    eta = cfg.lr.value(t)
    if prefetch is not None:
        torch.cuda.current_stream().wait_event(prefetch)
    else:
        rt.load(rt.theta, params)
    _lib.check(_lib.lib().dash_plan_apply(rt.plan, rt.theta.data_ptr(), rt.theta_out.data_ptr(), float(eta),
                                          _lib.stream_ptr()), "dash_plan_apply")
    mark("applied")
    check_step_status(state)  # the refresh's device-side scale checks (raises before anything is returned)
    state.step = t + 1
    if not isinstance(params[0], torch.Tensor):
        host = rt.theta_out.double().cpu().numpy()
        return [host[int(rt.offsets[i]):int(rt.offsets[i + 1])].reshape(s) for i, s in enumerate(rt.shapes)], state
    if not params[0].is_cuda:
        host = torch.empty(rt.theta_out.numel(), dtype=torch.float32, pin_memory=True)
        host.copy_(rt.theta_out, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return [host[int(rt.offsets[i]):int(rt.offsets[i + 1])].view(s) for i, s in enumerate(rt.shapes)], state
    outs = rt.views(rt.theta_out)
    if inplace:
        for p_, o in zip(params, outs):
            p_.copy_(o)
        return list(params), state
    return [o.clone() for o in outs], state


# ============================================================================ pipelined host-buffer step
def _host_chunks() -> int:
    return max(1, int(os.environ.get("DASH_HOST_CHUNKS", "6")))


def _pipelined(state: ShampooState, params, grads, cfg: ShampooConfig) -> bool:
    """Host (pinned CPU) parameters and gradients with a fixed-iteration solver: the step is pipelined by layer
    chunks so the PCIe copies overlap the device work (tolerance-mode refreshes read reports group by group
    and the EVD solver is host-orchestrated: those run the plain step)."""
    def pinned(ts):
        return all(isinstance(x, torch.Tensor) and not x.is_cuda and x.is_pinned() for x in ts)

    rt = state.runtime
    return (_host_chunks() > 1 and len(rt.shapes) > 1 and cfg.solver.tolerance == 0.0
            and cfg.solver.method != "evd" and getattr(rt, "global_gid", None) is None
            and len(params) == len(rt.shapes) and len(grads) == len(rt.shapes) and pinned(params) and pinned(grads))


def accumulate_chunk(state: ShampooState, cfg: ShampooConfig, ch: _Chunk, t: int) -> None:
    """accumulate() restricted to one chunk's blocks (its plan indexes the split gradients, graft partials and
    block maxima by chunk-local block, so a chunk's apply must follow its own accumulate)."""
    rt: _Runtime = state.runtime
    L = _lib.lib()
    if ch.plan is None:
        return
    _lib.check(L.dash_plan_accumulate(ch.plan, float(cfg.graft.beta2), float(cfg.graft.beta1), t + 1,
                                      float(cfg.graft.graft_eps), _lib.stream_ptr()), "dash_plan_accumulate")
    for gi, s0, e0 in ch.ranges:  # linalg.symmetrize + max|a| / sum(a^2) of the chunk's members
        g = state.groups[gi]
        _lib.check(L.dash_group_sym(g.ema[s0:e0].data_ptr(), e0 - s0, g.dim, float(cfg.epsilon),
                                    rt.g_amax[gi][s0:e0].data_ptr(), rt.g_fro[gi][s0 * rt.prep_parts:].data_ptr(),
                                    _lib.stream_ptr()), "dash_group_sym")


def _step_pipelined(state: ShampooState, params, grads, cfg: ShampooConfig, seed: int, events: dict | None):
    """shampoo.step for host buffers: layer chunk k's gradients and parameters go up, its statistics, roots and
    update are computed, and its new parameters come down while chunk k+1 is transferred and computed
    (three streams).  Per-block work is independent of the chunking (the preconditioner members of a layer range
    are a contiguous slot range of every group), so the result is bit-identical to the one-shot step."""
    rt: _Runtime = state.runtime
    for layer, g in zip(state.layers, grads):
        if tuple(g.shape) != layer.shape:
            raise ValueError(f"layer {layer.layer_id}: gradient shape {tuple(g.shape)} != {layer.shape}")
    for i, p_ in enumerate(params):
        if tuple(p_.shape) != rt.shapes[i]:
            raise ValueError(f"layer {i}: shape {tuple(p_.shape)} != {rt.shapes[i]}")
    t = state.step
    chunks = rt.ensure_chunks(cfg, state.layers, _host_chunks())
    L = _lib.lib()
    comp = torch.cuda.current_stream()
    if getattr(rt, "h2d_stream", None) is None:
        rt.h2d_stream, rt.d2h_stream = torch.cuda.Stream(device=rt.dev), torch.cuda.Stream(device=rt.dev)
    h2d, d2h = rt.h2d_stream, rt.d2h_stream
    h2d.wait_stream(comp)
    out = torch.empty(rt.theta_out.numel(), dtype=torch.float32, pin_memory=True)

    def upload(ch):
        """Chunk ch's gradients, then its parameters (needed only by the apply): (grads event, params event)."""
        evs = []
        with torch.cuda.stream(h2d):
            for src, dst in ((grads, rt.grad), (params, rt.theta)):
                for li in range(ch.l0, ch.l1):
                    o0, o1 = int(rt.offsets[li]), int(rt.offsets[li + 1])
                    dst[o0:o1].copy_(src[li].reshape(-1), non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
                evs.append(ev)
        return evs

    # chunk k+1's copies are issued after chunk k's work is enqueued: the solvers' small job-table uploads then
    # never queue behind gigabytes of pending H2D traffic (the host would block on them)
    ev_next = upload(chunks[0])
    refresh = t % cfg.update_freq == 0
    step_seed = block_seed(seed, t)
    err, oks = _refresh_flags(rt, sum(len(ch.ranges) for ch in chunks))
    eta = float(cfg.lr.value(t))
    k_ok = 0
    if events is not None:
        events.setdefault("start", []).append(torch.cuda.Event(enable_timing=True))
        events["start"][-1].record()
    for k, ch in enumerate(chunks):
        comp.wait_event(ev_next[0])
        accumulate_chunk(state, cfg, ch, t)
        if refresh:
            for gi, s0, e0 in ch.ranges:
                _refresh_range(state, cfg, gi, s0, e0, step_seed, err, oks[k_ok:k_ok + 1])
                k_ok += 1
        comp.wait_event(ev_next[1])
        _lib.check(L.dash_plan_apply(ch.plan, rt.theta.data_ptr(), rt.theta_out.data_ptr(), eta, _lib.stream_ptr()),
                   "dash_plan_apply")
        if k + 1 < len(chunks):
            ev_next = upload(chunks[k + 1])
        done = torch.cuda.Event()
        done.record(comp)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            out[ch.e0:ch.e1].copy_(rt.theta_out[ch.e0:ch.e1], non_blocking=True)
    rt.stats_valid, rt.stats_eps = True, cfg.epsilon
    if events is not None:
        events.setdefault("applied", []).append(torch.cuda.Event(enable_timing=True))
        events["applied"][-1].record()
    comp.wait_stream(d2h)
    if refresh:
        rt.pending_err = err
    check_step_status(state)  # synchronises; raises before anything is returned
    d2h.synchronize()
    state.step = t + 1
    return [out[int(rt.offsets[i]):int(rt.offsets[i + 1])].view(s) for i, s in enumerate(rt.shapes)], state


# ============================================================================ checkpointing
def _config_echo(cfg: ShampooConfig) -> list[str]:
    """The reference's config echo lines (shampoo.py:409-430)."""
    scaling = cfg.solver.scaling
    scaling_desc = "fro" if isinstance(scaling, Frobenius) else f"pi pool={scaling.pool} iters={scaling.iters}"
    return [
        f"beta_lr = {cfg.beta_lr!r}",
        f"epsilon = {cfg.epsilon!r}",
        f"update_freq = {cfg.update_freq}",
        f"block_size = {cfg.block_size}",
        f"solver = {cfg.solver.method}",
        f"scaling = {scaling_desc}",
        f"tolerance = {cfg.solver.tolerance!r}",
        f"max_iters = {cfg.solver.max_iters}",
        f"precision = {cfg.solver.precision.value}",
        f"lr_kind = {cfg.lr.kind}",
        f"lr_base = {cfg.lr.base!r}",
        f"graft_beta1 = {cfg.graft.beta1!r}",
        f"graft_beta2 = {cfg.graft.beta2!r}",
        f"graft_eps = {cfg.graft.graft_eps!r}",
    ]


def _block_sections(state: ShampooState):
    """(header, group, slot) of every ema/root section in the reference's order (shampoo.py:443-454)."""
    for layer in state.layers:
        refs = [("L", layer.left_refs)]
        if layer.right_refs is not None:
            refs.append(("R", layer.right_refs))
        for side, ref_list in refs:
            for idx, ref in enumerate(ref_list):
                yield layer, side, idx, ref


def save_state(state: ShampooState, cfg: ShampooConfig, path) -> None:
    """Single-file text checkpoint in the reference's format v1 (shampoo.py:433-461).

    The device state is fp32; every value is written as the float64 of that fp32 number (%.17g), so a
    reference process can load_state it, and our load_state reads reference checkpoints."""
    if any(r.group < 0 for lay in state.layers for r in lay.left_refs + (lay.right_refs or ())):
        raise ValueError("save_state needs the full optimizer state; this is one rank's shard of a ShardedDash")
    lines = ["# blockshampoo checkpoint v1", f"step = {state.step}"]
    lines.extend(_config_echo(cfg))
    lines.append(f"momentum = {0 if state.momentum is None else 1}")
    lines.append(f"layer_count = {len(state.layers)}")
    for layer in state.layers:
        lines.append(f"layer {layer.layer_id} shape = {' '.join(str(d) for d in layer.shape)}")
    ema_host = [g.ema.double().cpu().numpy() for g in state.groups]  # one D2H per group
    root_host = [g.roots.double().cpu().numpy() for g in state.groups]
    parts = ["\n".join(lines) + "\n"]
    last = None
    for layer, side, idx, ref in _block_sections(state):
        if last is not None and last is not layer:
            parts.extend(_layer_tail(state, last))
        last = layer
        parts.append(f"[layer {layer.layer_id} side {side} block {idx} ema]\n")
        parts.append(format_matrix(ema_host[ref.group][ref.slot]))
        parts.append(f"[layer {layer.layer_id} side {side} block {idx} root]\n")
        parts.append(format_matrix(root_host[ref.group][ref.slot]))
    if last is not None:
        parts.extend(_layer_tail(state, last))
    with open(path, "w") as fh:
        fh.write("".join(parts))


def _layer_tail(state: ShampooState, layer: LayerState) -> list[str]:
    out = []
    adam = state.adam[layer.layer_id].double().cpu().numpy()
    out.append(f"[layer {layer.layer_id} adam]\n")
    out.append(format_matrix(adam if adam.ndim == 2 else adam[None, :]))
    if state.momentum is not None:
        mom = state.momentum[layer.layer_id].double().cpu().numpy()
        out.append(f"[layer {layer.layer_id} momentum]\n")
        out.append(format_matrix(mom if mom.ndim == 2 else mom[None, :]))
    return out


def load_state(path) -> tuple[ShampooState, dict[str, str]]:
    """Rebuild a checkpointed state on the device; returns it with the echoed config (shampoo.py:464-519).

    Same validation and error messages as the reference; the float64 text values are rounded to fp32."""
    with open(path) as fh:
        text = fh.read()
    head, *sections = text.split("\n[")
    meta: dict[str, str] = {}
    shapes: dict[int, tuple[int, ...]] = {}
    for line in head.splitlines():
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        key, _, value = line.partition("=")
        key, value = key.strip(), value.strip()
        if key.startswith("layer ") and key.endswith(" shape"):
            shapes[int(key.split()[1])] = tuple(int(v) for v in value.split())
        else:
            meta[key] = value
    expected = int(meta["layer_count"])
    if sorted(shapes) != list(range(expected)):
        raise ValueError("checkpoint is missing layer shape declarations")
    state = _build_structure([shapes[i] for i in range(expected)], int(meta["block_size"]), meta["momentum"] == "1")
    state.step = int(meta["step"])
    ema_host = [np.zeros(tuple(g.ema.shape), dtype=np.float32) for g in state.groups]
    root_host = [g.roots.cpu().numpy().copy() for g in state.groups]
    seen: set[str] = set()
    for section in sections:
        header, _, body = section.partition("]\n")
        tokens = header.split()
        layer = state.layers[int(tokens[1])]
        data = parse_matrix(body)
        if tokens[2] == "adam":
            state.adam[layer.layer_id].copy_(torch.from_numpy(data if layer.is_matrix else data[0]))
        elif tokens[2] == "momentum":
            if state.momentum is None:
                raise ValueError("checkpoint has momentum sections but momentum flag is 0")
            state.momentum[layer.layer_id].copy_(torch.from_numpy(data if layer.is_matrix else data[0]))
        else:
            side, idx, kind = tokens[3], int(tokens[5]), tokens[6]
            ref = (layer.left_refs if side == "L" else layer.right_refs)[idx]
            (ema_host if kind == "ema" else root_host)[ref.group][ref.slot] = data
        seen.add(header)
    for layer in state.layers:
        sides = ["L"] + (["R"] if layer.right_refs is not None else [])
        for side in sides:
            for idx in range(len(layer.left_refs)):
                for kind in ("ema", "root"):
                    key = f"layer {layer.layer_id} side {side} block {idx} {kind}"
                    if key not in seen:
                        raise ValueError(f"checkpoint is missing section [{key}]")
        if f"layer {layer.layer_id} adam" not in seen:
            raise ValueError(f"checkpoint is missing section [layer {layer.layer_id} adam]")
    rt: _Runtime = state.runtime
    for gi, g in enumerate(state.groups):
        g.ema.copy_(torch.from_numpy(ema_host[gi]))
        g.roots.copy_(torch.from_numpy(root_host[gi]))
        rt.root_split[gi].load(g.roots)  # the apply operand (used until the next refresh)
    torch.cuda.synchronize()
    return state, meta
