"""Largest-eigenvalue estimation and solver input scaling on the B200 (drop-in for ``spectral.py``).

``Frobenius`` / ``PowerIterationScaling`` (``spectral.py:22-41``), ``block_seed`` (``:53-55``),
``batched_multi_power_iteration`` (``:115-117``) and ``scale_factor`` (``:120-130``).  The pooled power
iteration runs one CTA per block (``csrc/step.cu: pi_kernel``) with start vectors drawn from a device
restatement of NumPy's SeedSequence + PCG64 (``csrc/rng.cuh``), so the pool is bit-identical to the
reference's ``default_rng(block_seed(seed, i)).uniform(-1, 1, (pool, n))``; the iteration itself is fp32.
"""
from __future__ import annotations

import os

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import DegenerateSpectrumError
from .linalg import batched, device


@dataclass(frozen=True)
class Frobenius:
    """Scale solver inputs by the Frobenius norm."""


@dataclass(frozen=True)
class PowerIterationScaling:
    """Scale solver inputs by twice the pooled power-iteration estimate."""

    pool: int = 16
    iters: int = 30

    def __post_init__(self) -> None:
        if self.pool < 1:
            raise ValueError("pool must be >= 1")
        if self.iters < 1:
            raise ValueError("iters must be >= 1")


ScalingMode = Frobenius | PowerIterationScaling

MAX_POOL = 16


@dataclass(frozen=True)
class SpectralEstimate:
    lam: float
    vector: np.ndarray | None = None


def block_seed(seed: int, index: int) -> int:
    """Deterministic per-block child seed (SeedSequence([seed, index]).generate_state(1, uint64)[0])."""
    return int(_lib.lib().dash_block_seed(int(seed) & (2**64 - 1), int(index) & (2**64 - 1)))


def power_iteration_scales(ema: torch.Tensor, eps: float, pool: int, iters: int, seed: int,
                           scale: torch.Tensor, inv_scale: torch.Tensor, status: torch.Tensor,
                           seed_index: torch.Tensor | None = None, a_split=None) -> None:
    """scale[i] = 2 * lambda_PI(ema[i] + eps I) with per-block seeds block_seed(seed, i) (device).

    With ``a_split`` (the solver's split stack of ema + eps I) and a block size that is a multiple of 128,
    the matvecs run on the tensor cores (dash_power_iteration_split); otherwise the fp32 kernel reads ema."""
    if pool > MAX_POOL:
        raise ValueError(f"the B200 power iteration supports pool <= {MAX_POOL}")
    n, d = ema.shape[0], ema.shape[1]
    if a_split is not None and d % 128 == 0 and d <= 1024 and not os.environ.get("DASH_PI_FP32"):
        st = _lib.lib().dash_power_iteration_split(a_split.ref(), int(pool), int(iters), int(seed) & (2**64 - 1),
                                                   scale.data_ptr(), inv_scale.data_ptr(), status.data_ptr(),
                                                   seed_index.data_ptr() if seed_index is not None else None,
                                                   _lib.stream_ptr())
        _lib.check(st, "dash_power_iteration_split")
        return
    st = _lib.lib().dash_power_iteration(ema.data_ptr(), n, d, float(eps), int(pool), int(iters),
                                         int(seed) & (2**64 - 1), scale.data_ptr(), inv_scale.data_ptr(),
                                         status.data_ptr(),
                                         seed_index.data_ptr() if seed_index is not None else None,
                                         _lib.stream_ptr())
    _lib.check(st, "dash_power_iteration")


def batched_multi_power_iteration(a, pool: int, iters: int, seed: int) -> list[SpectralEstimate]:
    """Per-block estimates; block i uses the derived seed block_seed(seed, i)."""
    at = batched(a).contiguous()
    n = at.shape[0]
    scale = torch.empty(n, dtype=torch.float32, device=at.device)
    inv = torch.empty_like(scale)
    status = torch.zeros(n, dtype=torch.int32, device=at.device)
    power_iteration_scales(at, 0.0, pool, iters, seed, scale, inv, status)
    if bool((status == 2).any()):
        raise DegenerateSpectrumError("power iteration pool collapsed twice on a nonzero matrix")
    return [SpectralEstimate(lam=0.5 * float(s)) for s in scale.tolist()]


def scale_factor(a, mode: ScalingMode, seed: int = 0) -> float:
    """Divisor that brings the spectrum into the solvers' convergence region (spectral.py:120-130)."""
    at = batched(a[None] if getattr(a, "ndim", 0) == 2 else a)
    if isinstance(mode, Frobenius):
        norm = float(torch.linalg.vector_norm(at[0].double()))
        if norm == 0.0:
            raise ValueError("cannot scale the zero matrix")
        return norm
    lam = batched_multi_power_iteration(at, mode.pool, mode.iters, seed)[0].lam
    if lam <= 0.0:
        raise ValueError("cannot scale a matrix with a zero spectral estimate")
    return 2.0 * lam


def device_uniform(seed: int, count: int) -> torch.Tensor:
    """First `count` draws of default_rng(seed).uniform(-1, 1), generated on the GPU (test hook)."""
    out = torch.empty(count, dtype=torch.float64, device=device())
    _lib.check(_lib.lib().dash_uniform_pm1(int(seed) & (2**64 - 1), int(count), out.data_ptr(), _lib.stream_ptr()),
               "dash_uniform_pm1")
    return out
