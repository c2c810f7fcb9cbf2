"""Matmul-only inverse-root iterations on the B200 (drop-in for the reference ``roots.py``).

Same names, configs and report semantics as the reference (``IterationReport`` ``roots.py:32-36``,
``CnConfig`` ``:39-56``, ``NdbConfig`` ``:59-68``, ``batched_coupled_newton`` ``:216-259``,
``batched_newton_db`` ``:262-305``): one shared loop over the block stack, per-block freezing of
converged / non-finite / diverging blocks (their update factor becomes I, so their value stays put),
the 4-sample divergence watch, and a max-norm residual.  The whole loop runs on the device
(``csrc/solver.cu``): every product is a tcgen05 grouped GEMM with the Newton update fused into its
epilogue, freezing is a device kernel, and there is no host round trip per iteration.

Inputs may be NumPy arrays (returned as float64 NumPy, the reference's types) or CUDA tensors
(returned as fp32 CUDA tensors).  Differences from the reference: arithmetic is split-f16 / fp32-class
rather than float64 (see ``linalg``), and NDB accepts the reduced-precision modes.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConvergenceError, NumericalError
from .linalg import PrecisionMode, Scratch, SplitStack, batched, passes_for, stall_for, tally, workspace


@dataclass
class IterationReport:
    iterations: int
    residual: float
    converged: bool


@dataclass(frozen=True)
class CnConfig:
    p: int = 2
    c: float | None = None  # None -> (1+p)^(-1/p), so (p+1)c^p = 1
    tolerance: float = 1e-10
    max_iters: int = 100

    def __post_init__(self) -> None:
        if self.p not in (2, 4):
            raise ValueError(f"p must be 2 or 4, got {self.p}")
        if self.c is not None and self.c <= 0:
            raise ValueError("c must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")

    @property
    def resolved_c(self) -> float:
        return self.c if self.c is not None else (1.0 + self.p) ** (-1.0 / self.p)


@dataclass(frozen=True)
class NdbConfig:
    tolerance: float = 1e-10
    max_iters: int = 100

    def __post_init__(self) -> None:
        if self.tolerance < 0:
            raise ValueError("tolerance must be >= 0")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


# ----------------------------------------------------------------------------- device reports
class DeviceReports:
    """Per-block reports kept on the device until someone asks for them (one D2H copy)."""

    __slots__ = ("iters", "resid", "conv")

    def __init__(self, n: int, dev: torch.device):
        self.iters = torch.zeros(n, dtype=torch.int32, device=dev)
        self.resid = torch.zeros(n, dtype=torch.float32, device=dev)
        self.conv = torch.zeros(n, dtype=torch.int32, device=dev)

    def to_list(self) -> list[IterationReport]:
        it, rs, cv = self.iters.tolist(), self.resid.tolist(), self.conv.tolist()
        return [IterationReport(int(i), float(r), bool(c)) for i, r, c in zip(it, rs, cv)]

    def all_converged(self) -> bool:
        return bool(self.conv.all())

    def max_iters_run(self) -> int:
        return int(self.iters.max()) if self.iters.numel() else 0


def _reports(n: int, dev, scratch: Scratch | None, tag: str) -> DeviceReports:
    rep = DeviceReports.__new__(DeviceReports)
    if scratch is None:
        rep.__init__(n, dev)
        return rep
    rep.iters = scratch.tensor(tag + ".iters", (n,), torch.int32)
    rep.resid = scratch.tensor(tag + ".resid", (n,), torch.float32)
    rep.conv = scratch.tensor(tag + ".conv", (n,), torch.int32)
    return rep


def ndb_split(a: SplitStack, inv_scale: torch.Tensor | None, tol: float, max_iters: int,
              mode: PrecisionMode, complete: bool = True, *, stall: float | None = None,
              scratch: Scratch | None = None, tag: str = "ndb", outputs: str = "yz"
              ) -> tuple[SplitStack, SplitStack, DeviceReports]:
    """NDB on split stacks (device-resident fast path used by the optimizer).

    ``complete=False`` leaves Y and Z in upper pair-block storage (``dash_ndb_upper``); complete the one you
    read with :func:`fill_lower`.  ``outputs`` ("y", "z" or "yz", with ``complete=False``): the iterates the
    caller reads -- the last iteration computes only those, the other stack holds an earlier iterate.
    ``stall``: the stall cap (default: ``linalg.stall_for(tol, mode)``).  ``scratch``: reuse the output /
    workspace buffers of a previous call with the same ``tag``."""
    n, b = a.nmat, a.rows
    dev = a.data.device
    if scratch is not None:
        y, z = scratch.stack(tag + ".y", n, b, b), scratch.stack(tag + ".z", n, b, b)
    else:
        y, z = SplitStack(n, b, b, dev), SplitStack(n, b, b, dev)
    rep = _reports(n, dev, scratch, tag)
    L = _lib.lib()
    nbytes = L.dash_ndb_ws_bytes(n, b)
    ws = scratch.ws("solver", nbytes) if scratch is not None else workspace(nbytes, dev)
    need = {"y": 1, "z": 2, "yz": 3}[outputs]
    if complete and need != 3:
        raise ValueError("outputs selects iterates of the upper-stored solve (complete=False) only")
    args = [float(tol), float(stall_for(tol, mode) if stall is None else stall), int(max_iters), passes_for(mode)]
    if not complete:
        args.append(need)
    fn = L.dash_ndb if complete else L.dash_ndb_upper
    st = fn(a.ref(), inv_scale.data_ptr() if inv_scale is not None else None, y.ref(), z.ref(), *args,
            rep.iters.data_ptr(), rep.resid.data_ptr(), rep.conv.data_ptr(), ws.data_ptr(), ws.numel(),
            _lib.stream_ptr())
    _lib.check(st, "dash_ndb")
    return y, z, rep


def fill_lower(s: SplitStack) -> SplitStack:
    """Complete an upper pair-block stored stack in place (``dash_fill_lower``)."""
    _lib.check(_lib.lib().dash_fill_lower(s.ref(), _lib.stream_ptr()), "dash_fill_lower")
    return s


def cn_split(a: SplitStack, inv_scale: torch.Tensor | None, cfg: CnConfig, mode: PrecisionMode, *,
             scratch: Scratch | None = None, tag: str = "cn") -> tuple[SplitStack, DeviceReports]:
    n, b = a.nmat, a.rows
    dev = a.data.device
    x = scratch.stack(tag + ".x", n, b, b) if scratch is not None else SplitStack(n, b, b, dev)
    rep = _reports(n, dev, scratch, tag)
    L = _lib.lib()
    nbytes = L.dash_cn_ws_bytes(n, b)
    ws = scratch.ws("solver", nbytes) if scratch is not None else workspace(nbytes, dev)
    st = L.dash_cn(a.ref(), inv_scale.data_ptr() if inv_scale is not None else None, cfg.p,
                   float(cfg.resolved_c), x.ref(), float(cfg.tolerance), float(stall_for(cfg.tolerance, mode)),
                   int(cfg.max_iters), passes_for(mode),
                   rep.iters.data_ptr(), rep.resid.data_ptr(), rep.conv.data_ptr(), ws.data_ptr(), ws.numel(),
                   _lib.stream_ptr())
    _lib.check(st, "dash_cn")
    return x, rep


def _out(t: torch.Tensor, like_numpy: bool):
    return t.double().cpu().numpy() if like_numpy else t


def _ndb_products(reports: list[IterationReport]) -> int:
    k = max((r.iterations for r in reports), default=1)
    return 1 + 3 * (k - 1)  # closed-form first step costs one product (roots.py:269)


# ----------------------------------------------------------------------------- reference surface
def batched_newton_db(a, cfg: NdbConfig, mode: PrecisionMode = PrecisionMode.FULL64):
    """Denman-Beavers over a block stack with per-block freezing: (Y, Z, reports)."""
    is_np = not isinstance(a, torch.Tensor)
    at = batched(a)
    y, z, rep = ndb_split(SplitStack.from_float(at), None, cfg.tolerance, cfg.max_iters, mode)
    reports = rep.to_list()
    tally(_ndb_products(reports))
    return _out(y.to_float(), is_np), _out(z.to_float(), is_np), reports


def batched_coupled_newton(a, cfg: CnConfig, mode: PrecisionMode = PrecisionMode.FULL64):
    """Coupled Newton over a block stack with per-block freezing: (X, reports)."""
    is_np = not isinstance(a, torch.Tensor)
    at = batched(a)
    x, rep = cn_split(SplitStack.from_float(at), None, cfg, mode)
    reports = rep.to_list()
    k = max((r.iterations for r in reports), default=1)
    tally(k * (4 if cfg.p == 4 else 3))
    return _out(x.to_float(), is_np), reports


def newton_db(a, cfg: NdbConfig, mode: PrecisionMode = PrecisionMode.FULL64):
    """Unbatched NDB (roots.py:125-151): raises on divergence / non-finite like the reference."""
    y, z, rep = batched_newton_db(_as_stack1(a), cfg, mode)
    r = rep[0]
    _raise_single(r, "Denman-Beavers", cfg.max_iters)
    return y[0], z[0], r


def coupled_newton(a, cfg: CnConfig, mode: PrecisionMode = PrecisionMode.FULL64):
    """Unbatched coupled Newton (roots.py:93-122)."""
    x, rep = batched_coupled_newton(_as_stack1(a), cfg, mode)
    r = rep[0]
    _raise_single(r, "coupled Newton", cfg.max_iters)
    return x[0], r


def ndb_inverse_fourth_root(a, cfg: NdbConfig, mode: PrecisionMode = PrecisionMode.FULL64):
    """A^(-1/4) as the inverse square root of A^(1/2) (roots.py:154-163)."""
    sqrt_a, _, first = newton_db(a, cfg, mode)
    _, inv_root, second = newton_db(sqrt_a, cfg, mode)
    report = IterationReport(iterations=first.iterations + second.iterations,
                             residual=max(first.residual, second.residual),
                             converged=first.converged and second.converged)
    return inv_root, report


def _as_stack1(a):
    if isinstance(a, torch.Tensor):
        return a[None] if a.dim() == 2 else a
    a = np.asarray(a, dtype=np.float64)
    return a[None] if a.ndim == 2 else a


def _raise_single(r: IterationReport, name: str, max_iters: int) -> None:
    """The unbatched solvers raise where the reference's loop raises (roots.py:116-121, :145-150).

    In the batched report a block that stopped before ``max_iters`` without converging was frozen either
    for a non-finite residual (-> NumericalError) or by the divergence watch (-> ConvergenceError)."""
    if not np.isfinite(r.residual):
        raise NumericalError(f"{name} produced non-finite values at iteration {r.iterations}")
    if not r.converged and r.iterations < max_iters:
        raise ConvergenceError(f"{name} diverging at iteration {r.iterations} (residual {r.residual:.3e})")
