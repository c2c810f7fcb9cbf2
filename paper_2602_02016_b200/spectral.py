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
from .linalg import batched, check_symmetric, device


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
                           seed_index: torch.Tensor | None = None, a_split=None,
                           vec_out: torch.Tensor | None = None) -> None:
    """scale[i] = 2 * lambda_PI(ema[i] + eps I) with per-block seeds block_seed(seed, i) (device).

    With ``a_split`` (the solver's split stack of ema + eps I) and a block size that is a multiple of 128,
    the matvecs run on the tensor cores (dash_power_iteration_split); otherwise the fp32 kernel reads ema."""
    if pool > MAX_POOL:
        raise ValueError(f"the B200 power iteration supports pool <= {MAX_POOL}")
    n, d = ema.shape[0], ema.shape[1]
    if a_split is not None and vec_out is None and d % 128 == 0 and d <= 1024 and not os.environ.get("DASH_PI_FP32"):
        st = _lib.lib().dash_power_iteration_split(a_split.ref(), ema.data_ptr(), float(eps), int(pool), int(iters),
                                                   int(seed) & (2**64 - 1),
                                                   scale.data_ptr(), inv_scale.data_ptr(), status.data_ptr(),
                                                   seed_index.data_ptr() if seed_index is not None else None,
                                                   _lib.stream_ptr())
        _lib.check(st, "dash_power_iteration_split")
        return
    st = _lib.lib().dash_power_iteration(ema.data_ptr(), n, d, float(eps), int(pool), int(iters),
                                         int(seed) & (2**64 - 1), scale.data_ptr(), inv_scale.data_ptr(),
                                         status.data_ptr(),
                                         seed_index.data_ptr() if seed_index is not None else None,
                                         vec_out.data_ptr() if vec_out is not None else None,
                                         _lib.stream_ptr())
    _lib.check(st, "dash_power_iteration")


def rayleigh_quotient(a, x) -> float:
    """x^T a x / x^T x of a symmetric matrix (spectral.py:58-64), reduced in float64."""
    check_symmetric(a)
    ad = a.double() if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a, dtype=np.float64))
    xd = (x.double() if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.float64))).reshape(-1)
    xd = xd.to(ad.device)
    denom = float(xd @ xd)
    if denom == 0.0:
        raise ValueError("rayleigh quotient of the zero vector is undefined")
    return float(xd @ (ad @ xd)) / denom


def batched_multi_power_iteration(a, pool: int, iters: int, seed: int) -> list[SpectralEstimate]:
    """Per-block estimates (lambda and the selected unit vector); block i uses block_seed(seed, i)
    (spectral.py:115-117).  A zero block gives lambda = 0 and its first start vector (spectral.py:99-101)."""
    if pool < 1 or iters < 1:
        raise ValueError("pool and iters must be >= 1")
    is_np = not isinstance(a, torch.Tensor)
    at = batched(a).contiguous()
    n, d = at.shape[0], at.shape[1]
    scale = torch.empty(n, dtype=torch.float32, device=at.device)
    inv = torch.empty_like(scale)
    status = torch.zeros(n, dtype=torch.int32, device=at.device)
    vecs = torch.zeros((n, d), dtype=torch.float32, device=at.device)
    power_iteration_scales(at, 0.0, pool, iters, seed, scale, inv, status, vec_out=vecs)
    if bool((status == 2).any()):
        raise DegenerateSpectrumError("power iteration pool collapsed twice on a nonzero matrix")
    vh = vecs.double().cpu().numpy() if is_np else vecs
    return [SpectralEstimate(lam=0.5 * float(s), vector=vh[i]) for i, s in enumerate(scale.tolist())]


def multi_power_iteration(a, pool: int, iters: int, seed: int) -> SpectralEstimate:
    """Pooled power iteration on one symmetric matrix (spectral.py:87-112): the best Rayleigh quotient of a
    pool of `pool` seeded start vectors after `iters` normalised products, with its vector."""
    check_symmetric(a)
    stack = a[None] if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)[None]
    if pool < 1 or iters < 1:
        raise ValueError("pool and iters must be >= 1")
    if pool > MAX_POOL:
        raise ValueError(f"the B200 power iteration supports pool <= {MAX_POOL}")
    # the batched entry derives block_seed(seed, 0) for block 0; the single-matrix call uses `seed` itself
    scale = torch.empty(1, dtype=torch.float32, device=device())
    inv = torch.empty_like(scale)
    status = torch.zeros(1, dtype=torch.int32, device=device())
    vec = torch.zeros((1, stack.shape[-1]), dtype=torch.float32, device=device())
    at = batched(stack).contiguous()
    _single_seed_power_iteration(at, pool, iters, seed, scale, inv, status, vec)
    if int(status[0]) == 2:
        raise DegenerateSpectrumError("power iteration pool collapsed twice on a nonzero matrix")
    v = vec[0].double().cpu().numpy() if not isinstance(a, torch.Tensor) else vec[0]
    return SpectralEstimate(lam=0.5 * float(scale[0]), vector=v)


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


def _single_seed_power_iteration(at, pool, iters, seed, scale, inv, status, vec) -> None:
    """Block 0 draws its pool from default_rng(seed) itself (multi_power_iteration's seeding, spectral.py:94):
    seed_index = -1 tells the kernel not to derive a child seed."""
    idx = torch.full((1,), -1, dtype=torch.int32, device=at.device)
    power_iteration_scales(at, 0.0, pool, iters, seed, scale, inv, status, seed_index=idx, vec_out=vec)
