"""EVD inverse roots with spectrum dampening (drop-in for the reference ``eigensolver.py``).

Reference surface: ``HeuristicKind`` / ``DampeningHeuristic`` (``eigensolver.py:31-44``),
``EigenDecomposition`` (``:47-50``), ``eigh`` (``:120-124``), ``dampen_spectrum`` / ``dampen_corrected``
(``:133-154``), ``evd_inverse_root`` (``:157-172``), ``batched_evd_inverse_root`` (``:175-179``).

The eigendecompositions run on the device in float64, batched over blocks: ``csrc/evd.cu`` restates the
reference's cyclic Jacobi (same round-robin pair schedule, dead-pair skip and stopping rule, IEEE float64
rotations without FMA contraction).  Besides the
EVD solver option / config-2 comparator, the float64 inverse root is the optimizer's fallback for blocks the
fp32-class Newton iterations cannot converge in FULL64 mode (``inverse_root_f64``).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConvergenceError, DegenerateSpectrumError
from .linalg import check_symmetric, device, workspace


class HeuristicKind(enum.Enum):
    LEGACY = "legacy"
    SHIFTED_RELU = "relu"
    ABS = "abs"


@dataclass(frozen=True)
class DampeningHeuristic:
    kind: HeuristicKind
    epsilon: float = 1e-10

    def __post_init__(self) -> None:
        if self.epsilon <= 0:
            raise ValueError("epsilon must be positive")


@dataclass
class EigenDecomposition:
    eigenvalues: np.ndarray   # ascending
    eigenvectors: np.ndarray  # column i pairs with eigenvalues[i]


# ----------------------------------------------------------------------------- device eigensolver
def jacobi(a: torch.Tensor, tol: float = 1e-12, max_sweeps: int = 100):
    """dash_jacobi_eigh on a float64 (n, d, d) CUDA stack: (eigenvalues ascending, eigenvectors in columns,
    sweeps per block, status per block: 0 converged / 1 not converged)."""
    a = a.to(torch.float64).contiguous()
    n, d = a.shape[0], a.shape[-1]
    lam = torch.empty((n, d), dtype=torch.float64, device=a.device)
    q = torch.empty_like(a)
    sweeps = torch.zeros(n, dtype=torch.int32, device=a.device)
    status = torch.zeros(n, dtype=torch.int32, device=a.device)
    L = _lib.lib()
    ws = workspace(L.dash_jacobi_ws_bytes(n, d), a.device)
    _lib.check(L.dash_jacobi_eigh(a.data_ptr(), n, d, float(tol), int(max_sweeps), lam.data_ptr(), q.data_ptr(),
                                  sweeps.data_ptr(), status.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr()),
               "dash_jacobi_eigh")
    return lam, q, sweeps, status


def _eigh_stack(a: torch.Tensor, tol: float = 1e-12, max_sweeps: int = 100) -> tuple[torch.Tensor, torch.Tensor]:
    """Batched symmetric EVD on the device Jacobi kernel (the reference's cyclic round-robin Jacobi,
    eigensolver.py:77-117).  Raises ConvergenceError when a block needs more than max_sweeps sweeps (:112-113)."""
    lam, q, _, status = jacobi(a, tol, max_sweeps)
    if bool(status.any()):
        raise ConvergenceError(f"Jacobi eigensolver did not converge in {max_sweeps} sweeps")
    return lam, q


def _as_stack(a) -> tuple[torch.Tensor, bool]:
    is_np = not isinstance(a, torch.Tensor)
    t = torch.as_tensor(np.asarray(a, dtype=np.float64)).to(device()) if is_np else a.to(device())
    return t.double(), is_np


def eigh(a, tol: float = 1e-12, max_sweeps: int = 100) -> EigenDecomposition:
    """Full symmetric eigendecomposition, eigenvalues ascending (eigensolver.py:120-124)."""
    check_symmetric(a)
    t, _ = _as_stack(a)
    lam, q = _eigh_stack(t[None], tol, max_sweeps)
    return EigenDecomposition(eigenvalues=lam[0].cpu().numpy(), eigenvectors=q[0].cpu().numpy())


# ----------------------------------------------------------------------------- dampening
def dampen_corrected(corrected, heuristic: DampeningHeuristic):
    """SHIFTED_RELU / ABS filters on an eps-corrected spectrum (eigensolver.py:147-154)."""
    eps = heuristic.epsilon
    if heuristic.kind is HeuristicKind.SHIFTED_RELU:
        return _relu(corrected - eps)
    if heuristic.kind is HeuristicKind.ABS:
        return abs(corrected) + eps
    raise ValueError(f"heuristic {heuristic.kind} does not operate on corrected spectra")


def _relu(x):
    return torch.clamp(x, min=0.0) if isinstance(x, torch.Tensor) else np.maximum(x, 0.0)


def dampen_spectrum(lam, heuristic: DampeningHeuristic):
    """Process the spectrum of (A + eps I) (eigensolver.py:133-144); NumPy or torch, 1-D or batched."""
    eps = heuristic.epsilon
    if heuristic.kind is HeuristicKind.LEGACY:
        if isinstance(lam, torch.Tensor):
            return lam - torch.clamp(lam.min(dim=-1, keepdim=True).values, max=0.0) + eps
        lam = np.asarray(lam, dtype=np.float64)
        return lam - np.minimum(lam.min(axis=-1, keepdims=True), 0.0) + eps
    return dampen_corrected(lam - eps, heuristic)


# ----------------------------------------------------------------------------- inverse roots
def evd_inverse_root_torch(a: torch.Tensor, p: int, h: DampeningHeuristic) -> torch.Tensor:
    """Batched inverse p-th root via the eigendecomposition of a + eps I (eigensolver.py:157-179)."""
    if p not in (2, 4):
        raise ValueError(f"p must be 2 or 4, got {p}")
    ad = a.double()
    eye = torch.eye(a.shape[-1], dtype=torch.float64, device=a.device)
    lam, q = _eigh_stack(ad + h.epsilon * eye)
    proc = dampen_spectrum(lam, h)
    if bool((~(proc > 0).any(dim=-1)).any()):
        raise DegenerateSpectrumError("all eigenvalues removed by dampening heuristic")
    inv = torch.where(proc > 0, proc.clamp(min=1e-300).pow(-1.0 / p), torch.zeros_like(proc))
    return ((q * inv[..., None, :]) @ q.transpose(-1, -2)).to(a.dtype)


def evd_inverse_root(a, p: int, heuristic: DampeningHeuristic):
    """Single-block EVD inverse root (eigensolver.py:157-172)."""
    t, is_np = _as_stack(a)
    check_symmetric(t)
    out = evd_inverse_root_torch(t[None], p, heuristic)[0]
    return out.cpu().numpy() if is_np else out


def batched_evd_inverse_root(a, p: int, heuristic: DampeningHeuristic):
    """Per-block EVD inverse roots (eigensolver.py:175-179), batched on the device."""
    t, is_np = _as_stack(a)
    out = evd_inverse_root_torch(t, p, heuristic)
    return out.cpu().numpy() if is_np else out


# Relative resolution of the fp32-class statistics: eigenvalues of ema + eps I below this fraction of the
# largest one are rounding noise of the stored EMA (its products carry ~1e-7 relative error), not spectrum.
STATS_RESOLUTION = 2.0 ** -23


def inverse_root_f64(ema: torch.Tensor, eps: float, p: int) -> torch.Tensor:
    """(ema + eps I)^(-1/p) in float64 (no dampening): the value the reference's float64 Newton iterations
    converge to, up to the resolution of fp32-class statistics -- eigenvalues below
    max(eps, STATS_RESOLUTION * lambda_max) are taken at that floor (below it the stored EMA carries no
    spectral information, and lambda^(-1/p) would amplify its rounding noise).  Returns fp32 (n, d, d)."""
    ad = ema.double()
    ad = 0.5 * (ad + ad.transpose(-1, -2))
    ad.diagonal(dim1=-2, dim2=-1).add_(eps)
    lam, q = _eigh_stack(ad)
    floor = torch.clamp(lam[..., -1:] * STATS_RESOLUTION, min=eps)
    inv = torch.maximum(lam, floor).pow(-1.0 / p)
    return ((q * inv[..., None, :]) @ q.transpose(-1, -2)).float()
