"""EVD inverse roots with spectrum dampening — the comparator solver (``eigensolver.py``).

The reference runs a cyclic Jacobi eigensolver per block (``eigensolver.py:77-124``) and the LEGACY /
SHIFTED_RELU / ABS heuristics (``:133-154``).  On the B200 this comparator uses the batched symmetric
eigensolver of the CUDA math library (``torch.linalg.eigh``, float64) followed by the same dampening and
Q diag(lambda^(-1/p)) Q^T reconstruction; it is not on the DASH hot path.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np
import torch

from .errors import DegenerateSpectrumError


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


def dampen_spectrum_torch(lam: torch.Tensor, h: DampeningHeuristic) -> torch.Tensor:
    """Process the spectrum of (A + eps I) (eigensolver.py:133-154)."""
    eps = h.epsilon
    if h.kind is HeuristicKind.LEGACY:
        return lam - torch.clamp(lam.min(dim=-1, keepdim=True).values, max=0.0) + eps
    corrected = lam - eps
    if h.kind is HeuristicKind.SHIFTED_RELU:
        return torch.clamp(corrected - eps, min=0.0)
    return corrected.abs() + eps


def evd_inverse_root_torch(a: torch.Tensor, p: int, h: DampeningHeuristic) -> torch.Tensor:
    """Batched inverse p-th root via eigendecomposition of a + eps I (eigensolver.py:157-179)."""
    if p not in (2, 4):
        raise ValueError(f"p must be 2 or 4, got {p}")
    ad = a.double()
    eye = torch.eye(a.shape[-1], dtype=torch.float64, device=a.device)
    lam, q = torch.linalg.eigh(ad + h.epsilon * eye)
    proc = dampen_spectrum_torch(lam, h)
    if bool((~(proc > 0).any(dim=-1)).any()):
        raise DegenerateSpectrumError("all eigenvalues removed by dampening heuristic")
    inv = torch.where(proc > 0, proc.clamp(min=1e-300).pow(-1.0 / p), torch.zeros_like(proc))
    return ((q * inv[..., None, :]) @ q.transpose(-1, -2)).to(a.dtype)


def batched_evd_inverse_root(a, p: int, heuristic: DampeningHeuristic):
    is_np = not isinstance(a, torch.Tensor)
    t = torch.as_tensor(np.asarray(a, dtype=np.float64)).cuda() if is_np else a
    out = evd_inverse_root_torch(t, p, heuristic)
    return out.cpu().numpy() if is_np else out
