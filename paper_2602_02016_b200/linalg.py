"""Dense primitives on the B200: precision modes, split-f16 stacks, the batched product.

Mirrors the reference's ``linalg.py`` surface (``PrecisionMode`` ``:23-25``, ``matrix``/``batched``
``:28-47``, ``count_matmuls`` ``:50-72``, ``bmm`` ``:105-114``, ``symmetrize`` ``:121-124``) but every
product runs through the C-ABI tcgen05 engine (``csrc/gemm_tc.cu``).

Precision modes (the reference has FULL64 / EMULATED32; the B200 build adds F16):

* ``EMULATED32`` ("f32") -- split-f16 products: each operand is stored as fp16 hi + fp16 lo with a
  per-matrix power-of-two exponent, and every product issues hi*hi + hi*lo + lo*hi on the tensor
  cores with fp32 accumulation (22-bit significands, fp32-class results).
* ``FULL64`` ("f64", the reference's default) -- the same split-f16 products, accumulated in 16 K ranges per
  output tile that the epilogue sums in fp32 registers (tcgen05's fp32 accumulation truncates, so the error
  grows with the chain length: B = 1024 Newton-DB error ~14x smaller than EMULATED32, ~20% slower); its
  Newton iterations converge at the fp32-class floor and blocks they cannot converge are re-solved in float64
  (see below).  Parity against the float64 reference is by the tolerances stated in DESIGN.md, never bitwise.
* ``F16`` ("f16") -- hi*hi only (fp16 tensor rate, ~11-bit significands).
"""
from __future__ import annotations

import contextlib
import ctypes
import enum
from typing import Iterator

import numpy as np
import torch

from . import _lib

LD_ALIGN = 64


class PrecisionMode(enum.Enum):
    FULL64 = "f64"
    EMULATED32 = "f32"
    F16 = "f16"


def passes_for(mode: PrecisionMode) -> int:
    """The engine's `passes` argument: 1 = fp16 products, 3 = split-f16 (hi*hi + hi*lo + lo*hi, main and
    correction accumulators), 4 = the same split accumulated in 16 K ranges per tile (FULL64)."""
    return {PrecisionMode.F16: 1, PrecisionMode.EMULATED32: 3, PrecisionMode.FULL64: 4}[mode]


# FULL64 promises float64-quality roots on an fp32-class engine.  Its Newton iterations converge "at the
# floor": with a requested tolerance below PRECISION_FLOOR (the reference's default 1e-10 is a float64
# tolerance; measured floors in profiles/r2_floor_f32.log) a block whose residual stops decreasing once it is
# <= STALL_CAP is frozen as converged (include/dash_b200.h), and the optimizer re-solves blocks the iteration
# cannot converge at all in float64 (shampoo.refresh_inverse_roots).  EMULATED32 and F16 keep the
# reference's rules exactly (a tolerance they cannot reach raises ConvergenceError, like the reference's
# EMULATED32).
PRECISION_FLOOR = 1e-5
STALL_CAP = 1e-3


def stall_for(tolerance: float, mode: PrecisionMode) -> float:
    """Stall cap passed to the device solvers: 0 (reference rules) unless FULL64 and 0 < tol < the floor."""
    if mode is PrecisionMode.FULL64 and 0.0 < tolerance < PRECISION_FLOOR:
        return STALL_CAP
    return 0.0


def _ld(cols: int) -> int:
    return (cols + LD_ALIGN - 1) // LD_ALIGN * LD_ALIGN


def device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the DASH B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class SplitStack:
    """A stack of ``nmat`` ``rows x cols`` matrices in split-f16 form (see csrc/types.h).

    ``data``: fp16 tensor (nmat, 2, rows, ld); ``exp``: int32 (nmat,); ``amax``: int32 (nmat,) holding
    float bit patterns.  value = (hi + lo) * 2**exp.
    """

    __slots__ = ("data", "exp", "amax", "rows", "cols", "_c")

    def __init__(self, nmat: int, rows: int, cols: int, dev: torch.device | None = None):
        dev = dev or device()
        self.rows, self.cols = rows, cols
        ld = _ld(cols)
        alloc = torch.empty if ld == cols else torch.zeros  # padding columns must be zero (K-major loads)
        self.data = alloc((nmat, 2, rows, ld), dtype=torch.float16, device=dev)
        self.exp = torch.zeros(nmat, dtype=torch.int32, device=dev)
        self.amax = torch.zeros(nmat, dtype=torch.int32, device=dev)
        self._c = None

    @property
    def nmat(self) -> int:
        return self.data.shape[0]

    @property
    def ld(self) -> int:
        return self.data.shape[3]

    def c(self) -> _lib.dash_stack:
        if self._c is None:
            self._c = _lib.dash_stack(self.data.data_ptr(), self.nmat, self.rows, self.cols, self.ld,
                                      self.exp.data_ptr(), self.amax.data_ptr())
        return self._c

    def ref(self):
        return ctypes.byref(self.c())

    @classmethod
    def from_float(cls, x: torch.Tensor) -> "SplitStack":
        """Split an fp32 (nmat, rows, cols) CUDA tensor."""
        _lib.require_cuda(x, "input")
        x = x.to(torch.float32)
        if x.dim() == 2:
            x = x[None]
        if x.stride(2) != 1:
            x = x.contiguous()
        s = cls(x.shape[0], x.shape[1], x.shape[2], x.device)
        s.load(x)
        return s

    def load(self, x: torch.Tensor) -> "SplitStack":
        if x.stride(2) != 1:
            x = x.contiguous()
        _lib.check(_lib.lib().dash_split(x.data_ptr(), x.stride(0), x.stride(1), self.ref(), _lib.stream_ptr()),
                   "dash_split")
        return self

    def to_float(self) -> torch.Tensor:
        out = torch.empty((self.nmat, self.rows, self.cols), dtype=torch.float32, device=self.data.device)
        _lib.check(_lib.lib().dash_unsplit(self.ref(), out.data_ptr(), out.stride(0), out.stride(1),
                                           _lib.stream_ptr()), "dash_unsplit")
        return out

    def amax_float(self) -> torch.Tensor:
        return self.amax.view(torch.float32)

    def head(self, n: int) -> "SplitStack":
        """The first ``n`` matrices (shares storage)."""
        return self if n == self.nmat else self.slice(0, n)

    def slice(self, start: int, stop: int) -> "SplitStack":
        """Matrices [start, stop) (shares storage)."""
        v = SplitStack.__new__(SplitStack)
        v.rows, v.cols = self.rows, self.cols
        v.data, v.exp, v.amax = self.data[start:stop], self.exp[start:stop], self.amax[start:stop]
        v._c = None
        return v


def workspace(nbytes: int, dev: torch.device | None = None) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev or device())


class Scratch:
    """Device buffers reused across optimizer steps (no allocation on the steady-state step path).

    Buffers are keyed by a name and their per-matrix shape; a request for fewer matrices than the cached
    capacity returns a view of the first ones, a larger request reallocates."""

    def __init__(self, dev: torch.device | None = None):
        self.dev = dev or device()
        self._bufs: dict = {}

    def stack(self, name: str, n: int, rows: int, cols: int) -> SplitStack:
        key = ("stack", name, rows, cols)
        s = self._bufs.get(key)
        if s is None or s.nmat < n:
            s = SplitStack(n, rows, cols, self.dev)
            self._bufs[key] = s
        return s.head(n)

    def tensor(self, name: str, shape: tuple, dtype=torch.float32) -> torch.Tensor:
        key = ("tensor", name, tuple(shape[1:]), dtype)
        t = self._bufs.get(key)
        if t is None or t.shape[0] < shape[0]:
            t = torch.empty(tuple(shape), dtype=dtype, device=self.dev)
            self._bufs[key] = t
        return t[:shape[0]]

    def ws(self, name: str, nbytes: int) -> torch.Tensor:
        key = ("ws", name)
        t = self._bufs.get(key)
        if t is None or t.numel() < nbytes:
            t = workspace(nbytes, self.dev)
            self._bufs[key] = t
        return t


# ----------------------------------------------------------------------------- matmul accounting
class MatmulCounter:
    """Counts matmul/bmm invocations while installed via count_matmuls() (linalg.py:50-67)."""

    def __init__(self) -> None:
        self.count = 0


_ACTIVE_COUNTERS: list[MatmulCounter] = []


@contextlib.contextmanager
def count_matmuls() -> Iterator[MatmulCounter]:
    counter = MatmulCounter()
    _ACTIVE_COUNTERS.append(counter)
    try:
        yield counter
    finally:
        _ACTIVE_COUNTERS.remove(counter)


def tally(n: int = 1) -> None:
    for counter in _ACTIVE_COUNTERS:
        counter.count += n


# ----------------------------------------------------------------------------- validation
def as_device_f32(data, what: str = "tensor") -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        t = data
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(data, dtype=np.float64)))
    return t.to(device=device(), dtype=torch.float32)


def batched(data) -> torch.Tensor:
    """Validate and return an (N, B, B) stack of square blocks as fp32 on the GPU (linalg.py:38-47)."""
    a = as_device_f32(data)
    if a.dim() != 3:
        raise ValueError(f"batched tensor must be 3-D, got shape {tuple(a.shape)}")
    if a.shape[1] != a.shape[2]:
        raise ValueError(f"blocks must be square, got shape {tuple(a.shape)}")
    if not bool(torch.isfinite(a).all()):
        raise ValueError("batched tensor entries must be finite")
    return a


def matrix(data) -> torch.Tensor:
    a = as_device_f32(data)
    if a.dim() != 2:
        raise ValueError(f"matrix must be 2-D, got shape {tuple(a.shape)}")
    if not bool(torch.isfinite(a).all()):
        raise ValueError("matrix entries must be finite")
    return a


# ----------------------------------------------------------------------------- products
def bmm_split(a: SplitStack, b: SplitStack, *, trans_a: bool = False, trans_b: bool = False,
              out: SplitStack | None = None, f_out: torch.Tensor | None = None, alpha: float = 1.0,
              mode: PrecisionMode = PrecisionMode.EMULATED32) -> None:
    """C[m] = alpha * op(A[m]) @ op(B[m]) on the tcgen05 engine, into a split stack and/or fp32."""
    L = _lib.lib()
    ws = workspace(L.dash_bmm_ws_bytes(a.nmat), a.data.device)
    fp, fs, fl = (0, 0, 0) if f_out is None else (f_out.data_ptr(), f_out.stride(0), f_out.stride(1))
    st = L.dash_bmm(a.ref(), int(trans_a), b.ref(), int(trans_b), out.ref() if out is not None else None,
                    fp, fs, fl, float(alpha), passes_for(mode), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    _lib.check(st, "dash_bmm")
    tally()


def bmm(a, b, mode: PrecisionMode = PrecisionMode.FULL64, *, trans_a: bool = False,
        trans_b: bool = False):
    """Blockwise product on the GPU (reference ``bmm``, linalg.py:105-114): block i = a[i] @ b[i].

    NumPy operands give a float64 NumPy result (the reference's types); tensors give an fp32 CUDA tensor."""
    is_np = not isinstance(a, torch.Tensor)
    a = as_device_f32(a)
    b = as_device_f32(b)
    if a.dim() != 3 or b.dim() != 3:
        raise ValueError("bmm expects 3-D operands")
    sa, sb = SplitStack.from_float(a), SplitStack.from_float(b)
    m = a.shape[2] if trans_a else a.shape[1]
    n = b.shape[1] if trans_b else b.shape[2]
    k_a = a.shape[1] if trans_a else a.shape[2]
    k_b = b.shape[2] if trans_b else b.shape[1]
    if a.shape[0] != b.shape[0] or k_a != k_b:
        raise ValueError(f"shape mismatch: {tuple(a.shape)} x {tuple(b.shape)}")
    out = torch.empty((a.shape[0], m, n), dtype=torch.float32, device=a.device)
    bmm_split(sa, sb, trans_a=trans_a, trans_b=trans_b, f_out=out, mode=mode)
    return out.double().cpu().numpy() if is_np else out


def matmul(a, b, mode: PrecisionMode = PrecisionMode.FULL64):
    """Matrix product a @ b on the tcgen05 engine (reference ``matmul``, linalg.py:93-102)."""
    if getattr(a, "ndim", None) != 2 or getattr(b, "ndim", None) != 2:
        raise ValueError("matmul expects 2-D operands")
    if a.shape[1] != b.shape[0]:
        raise ValueError(f"dimension mismatch: {tuple(a.shape)} @ {tuple(b.shape)}")
    out = bmm(a[None], b[None], mode)
    return out[0]


def quantize(a, mode: PrecisionMode):
    """Round values through the storage precision of ``mode`` (linalg.py:75-79): fp32 for EMULATED32,
    fp16 for F16, unchanged for FULL64.  NumPy in -> float64 NumPy out; tensors keep their dtype."""
    dt = {PrecisionMode.EMULATED32: torch.float32, PrecisionMode.F16: torch.float16}.get(mode)
    if isinstance(a, torch.Tensor):
        return a if dt is None else a.to(dt).to(a.dtype)
    a = np.asarray(a, dtype=np.float64)
    if dt is None:
        return a
    return a.astype(np.float32 if dt is torch.float32 else np.float16).astype(np.float64)


def frobenius_norm(a) -> float:
    """||a||_F (linalg.py:117-118); reduced in float64."""
    if isinstance(a, torch.Tensor):
        return float(torch.linalg.vector_norm(a.double()))
    return float(np.linalg.norm(np.asarray(a, dtype=np.float64)))


def check_symmetric(a, rtol: float = 1e-8) -> None:
    """Raise ValueError unless ``a`` is square and symmetric within ``rtol`` (linalg.py:127-133)."""
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {tuple(a.shape)}")
    if isinstance(a, torch.Tensor):
        ad = a.double()
        asym = float(torch.linalg.vector_norm(ad - ad.T))
        nrm = float(torch.linalg.vector_norm(ad))
    else:
        ad = np.asarray(a, dtype=np.float64)
        asym, nrm = float(np.linalg.norm(ad - ad.T)), float(np.linalg.norm(ad))
    if asym > rtol * max(nrm, 1.0):
        raise ValueError(f"matrix is not symmetric (asymmetry norm {asym:.3e})")


def identity_like(a):
    """Identity (2-D input) or stacked identities (3-D input) of ``a``'s type (linalg.py:136-141)."""
    n = a.shape[-1]
    if isinstance(a, torch.Tensor):
        eye = torch.eye(n, dtype=a.dtype, device=a.device)
        return eye.expand(a.shape).clone() if a.dim() == 3 else eye
    eye = np.eye(n)
    return np.broadcast_to(eye, a.shape).copy() if np.ndim(a) == 3 else eye


def symmetrize(a):
    """(a + a^T) / 2 of a square matrix or a stack (linalg.py:121-124)."""
    if isinstance(a, torch.Tensor):
        return (a + a.transpose(-1, -2)) * 0.5
    a = np.asarray(a, dtype=np.float64)
    if a.shape[-1] != a.shape[-2]:
        raise ValueError(f"symmetrize expects a square matrix, got {a.shape}")
    return (a + np.swapaxes(a, -1, -2)) / 2.0


# ----------------------------------------------------------------------------- text matrices (host)
def format_matrix(a) -> str:
    """'rows cols' header + one line of %.17g values per row (linalg.py:150-154), from a 2-D array/tensor."""
    if isinstance(a, torch.Tensor):
        a = a.detach().to("cpu", torch.float64).numpy()
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError(f"format_matrix expects a 2-D array, got shape {a.shape}")
    lines = [f"{a.shape[0]} {a.shape[1]}"]
    lines.extend(" ".join(format(v, ".17g") for v in row) for row in a.tolist())
    return "\n".join(lines) + "\n"


def parse_matrix(text: str) -> np.ndarray:
    """Inverse of format_matrix with the reference's validation (linalg.py:157-173); returns float64."""
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines:
        raise ValueError("empty matrix text")
    header = lines[0].split()
    if len(header) != 2:
        raise ValueError(f"bad matrix header: {lines[0]!r}")
    rows, cols = int(header[0]), int(header[1])
    if len(lines) - 1 != rows:
        raise ValueError(f"expected {rows} data rows, got {len(lines) - 1}")
    out = np.empty((rows, cols), dtype=np.float64)
    for i, ln in enumerate(lines[1:]):
        vals = ln.split()
        if len(vals) != cols:
            raise ValueError(f"expected {cols} values per row, got {len(vals)}")
        out[i] = np.array(vals, dtype=np.float64)
    if not np.isfinite(out).all():
        raise ValueError("matrix entries must be finite")
    return out


def save_matrix(a, path) -> None:
    """Write the text format (linalg.py:144-147)."""
    with open(path, "w") as fh:
        fh.write(format_matrix(a))


def load_matrix(path) -> np.ndarray:
    with open(path) as fh:
        return parse_matrix(fh.read())
