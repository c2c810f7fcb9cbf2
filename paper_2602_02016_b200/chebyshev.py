"""Chebyshev-series inverse roots evaluated by matrix Clenshaw on the B200 (drop-in for ``chebyshev.py``).

The coefficient fit (a 1000-point discrete cosine projection, ``chebyshev.py:46-84``) is host setup done
once per (p, degree, points, interval) and cached like the reference's ``_cheb_cache``
(``shampoo.py:281-291``).  The matrix evaluation -- S = 2 a/scale - I, d-1 products
B_k = 2 S B_{k+1} - B_{k+2} + c_k I, out = (S B_1 - B_2 + c_0 I) * scale^(-1/p) -- runs entirely in the
tcgen05 engine with the recurrence fused into each product's epilogue (``csrc/solver.cu: cheb_solve``).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np
import torch

from . import _lib
from .linalg import PrecisionMode, SplitStack, batched, passes_for, tally, workspace


@dataclass(frozen=True)
class ChebCoefficients:
    degree: int
    interval: tuple[float, float]
    coeffs: np.ndarray            # length degree + 1
    power: int | None = None      # inverse-root exponent p, None for generic fits
    num_points: int = 0

    def __post_init__(self) -> None:
        if len(self.coeffs) != self.degree + 1:
            raise ValueError("coefficient vector must have degree + 1 entries")
        a, b = self.interval
        if not a < b:
            raise ValueError(f"invalid interval [{a}, {b}]")


def cheb_fit(f: Callable[[np.ndarray], np.ndarray], degree: int, num_points: int, interval: tuple[float, float],
             power: int | None = None) -> ChebCoefficients:
    """Discrete cosine projection of f at the Chebyshev nodes of [a, b] (host, float64)."""
    a, b = interval
    if not a < b:
        raise ValueError(f"invalid interval [{a}, {b}]")
    if num_points < degree + 1:
        raise ValueError(f"need at least degree+1 = {degree + 1} points, got {num_points}")
    theta = (2.0 * np.arange(num_points) + 1.0) * np.pi / (2.0 * num_points)
    nodes = 0.5 * (b - a) * np.cos(theta) + 0.5 * (b + a)
    basis = np.cos(np.outer(np.arange(degree + 1), theta))
    c = (2.0 / num_points) * (basis @ f(nodes))
    c[0] *= 0.5
    return ChebCoefficients(degree=degree, interval=(a, b), coeffs=c, power=power, num_points=num_points)


def fit_inverse_root(p: int, degree: int = 60, num_points: int = 1000, interval: tuple[float, float] | None = None,
                     epsilon: float = 1e-10) -> ChebCoefficients:
    """Coefficients for x^(-1/p); default interval [eps, 1 + eps]."""
    if p not in (2, 4):
        raise ValueError(f"p must be 2 or 4, got {p}")
    if interval is None:
        interval = (epsilon, 1.0 + epsilon)
    if interval[0] <= 0:
        raise ValueError("inverse-root fits need a strictly positive interval")
    return cheb_fit(lambda x: np.power(x, -1.0 / p), degree, num_points, interval, power=p)


def clenshaw_scalar(x: float, c: ChebCoefficients) -> float:
    """Scalar Clenshaw evaluation (host reference for one point)."""
    a, b = c.interval
    t = (2.0 * float(x) - (b + a)) / (b - a)
    b1 = b2 = 0.0
    for k in range(c.degree, -1, -1):
        b1, b2 = 2.0 * t * b1 - b2 + c.coeffs[k], b1
    return b1 - t * b2


def clenshaw_split(a: SplitStack, c: ChebCoefficients, inv_scale: torch.Tensor | None, mult: torch.Tensor | None,
                   f_out: torch.Tensor | None, out: SplitStack | None, mode: PrecisionMode, *,
                   gate: torch.Tensor | None = None, scratch=None) -> None:
    """Device Clenshaw on a split stack: S = 2 a inv_scale - I, result * mult -> f_out / out (written only
    when the device int ``gate`` is nonzero, if given)."""
    if c.degree < 2:
        raise ValueError("optimized evaluation needs degree >= 2")
    L = _lib.lib()
    coef = np.ascontiguousarray(c.coeffs, dtype=np.float64)
    nbytes = L.dash_cheb_ws_bytes(a.nmat, a.rows)
    ws = scratch.ws("solver", nbytes) if scratch is not None else workspace(nbytes, a.data.device)
    st = L.dash_clenshaw(a.ref(), inv_scale.data_ptr() if inv_scale is not None else None,
                         mult.data_ptr() if mult is not None else None,
                         coef.ctypes.data, int(c.degree), f_out.data_ptr() if f_out is not None else None,
                         out.ref() if out is not None else None, passes_for(mode),
                         gate.data_ptr() if gate is not None else None, ws.data_ptr(), ws.numel(),
                         _lib.stream_ptr())
    _lib.check(st, "dash_clenshaw")
    tally(c.degree - 1)


def batched_clenshaw_matrix(a, c: ChebCoefficients, scales, mode: PrecisionMode = PrecisionMode.FULL64,
                            optimized: bool = True):
    """Per-block Clenshaw evaluation with a per-block scale (chebyshev.py:137-153)."""
    if not optimized:
        raise ValueError("the B200 path implements the optimized (d-1 product) evaluation only")
    is_np = not isinstance(a, torch.Tensor)
    at = batched(a)
    sc = torch.as_tensor(np.asarray(scales, dtype=np.float64) if not isinstance(scales, torch.Tensor) else scales,
                         dtype=torch.float64).to(at.device)
    if tuple(sc.shape) != (at.shape[0],):
        raise ValueError(f"expected {at.shape[0]} scales, got shape {tuple(sc.shape)}")
    if bool((sc <= 0).any()):
        raise ValueError("scales must be positive")
    inv = (1.0 / sc).float()
    mult = (sc ** (-1.0 / c.power)).float() if c.power is not None else torch.ones_like(inv)
    out = torch.empty_like(at)
    clenshaw_split(SplitStack.from_float(at), c, inv, mult, out, None, mode)
    if not bool(torch.isfinite(out).all()):
        raise ValueError("non-finite Clenshaw result; spectrum likely outside the fit interval")
    return out.double().cpu().numpy() if is_np else out


def clenshaw_matrix(a, c: ChebCoefficients, scale: float, mode: PrecisionMode = PrecisionMode.FULL64,
                    optimized: bool = True):
    """Single-matrix variant (chebyshev.py:102-134)."""
    if scale <= 0:
        raise ValueError("scale must be positive")
    is_np = not isinstance(a, torch.Tensor)
    at = a[None] if is_np is False else np.asarray(a, dtype=np.float64)[None]
    out = batched_clenshaw_matrix(at, c, np.array([scale]) if is_np else torch.tensor([scale]), mode, optimized)
    return out[0]
