"""ctypes binding of ``libdash_b200.so`` (the C ABI declared in ``include/dash_b200.h``).

The library is the only compute path: there is no CPU or PyTorch fallback.  Loading fails loudly
when the shared object is missing (run ``__graft_entry__.build()``), and every wrapper raises when a
call returns a non-zero status.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

import torch

from .errors import NumericalError

_LIB_PATH = Path(os.environ.get("DASH_LIB") or Path(__file__).resolve().parent / "libdash_b200.so")  # DASH_LIB: A/B builds (dev)
_lib: ctypes.CDLL | None = None

DASH_OK, DASH_EINVAL, DASH_ENONFINITE, DASH_ECUDA = 0, 1, 2, 3

c_int, c_float, c_longlong, c_size_t, c_void_p = (
    ctypes.c_int, ctypes.c_float, ctypes.c_longlong, ctypes.c_size_t, ctypes.c_void_p)


class dash_stack(ctypes.Structure):
    _fields_ = [
        ("data", c_void_p),
        ("nmat", c_int), ("rows", c_int), ("cols", c_int), ("ld", c_int),
        ("exp", c_void_p),
        ("amax", c_void_p),
    ]


class dash_block(ctypes.Structure):
    _fields_ = [
        ("off", c_longlong), ("ld", c_int), ("rows", c_int), ("cols", c_int),
        ("group_l", c_int), ("slot_l", c_int), ("group_r", c_int), ("slot_r", c_int),
    ]


_P = ctypes.POINTER(dash_stack)
_PB = ctypes.POINTER(dash_block)
c_ull = ctypes.c_ulonglong

# name -> (restype, argtypes); mirrors include/dash_b200.h
_SIGNATURES: dict[str, tuple] = {
    "dash_version": (ctypes.c_char_p, []),
    "dash_device_sms": (c_int, []),
    "dash_launch_count": (ctypes.c_ulonglong, []),
    "dash_gemm_timing": (None, [c_int]),
    "dash_gemm_timing_read": (c_int, [ctypes.POINTER(c_int), ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double)]),
    "dash_gemm_timing_list": (c_int, [c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dash_split": (c_int, [c_void_p, c_longlong, c_int, _P, c_void_p]),
    "dash_unsplit": (c_int, [_P, c_void_p, c_longlong, c_int, c_void_p]),
    "dash_bmm_ws_bytes": (c_size_t, [c_int]),
    "dash_bmm": (c_int, [_P, c_int, _P, c_int, _P, c_void_p, c_longlong, c_int, c_float, c_int, c_void_p,
                         c_size_t, c_void_p]),
    "dash_ndb_ws_bytes": (c_size_t, [c_int, c_int]),
    "dash_ndb": (c_int, [_P, c_void_p, _P, _P, c_float, c_float, c_int, c_int, c_void_p, c_void_p, c_void_p,
                         c_void_p, c_size_t, c_void_p]),
    "dash_ndb_upper": (c_int, [_P, c_void_p, _P, _P, c_float, c_float, c_int, c_int, c_int, c_void_p, c_void_p,
                               c_void_p, c_void_p, c_size_t, c_void_p]),
    "dash_fill_lower": (c_int, [_P, c_void_p]),
    "dash_cn_ws_bytes": (c_size_t, [c_int, c_int]),
    "dash_cn": (c_int, [_P, c_void_p, c_int, c_float, _P, c_float, c_float, c_int, c_int, c_void_p, c_void_p,
                        c_void_p, c_void_p, c_size_t, c_void_p]),
    "dash_scale_stack": (c_int, [_P, c_void_p, c_float, c_void_p, c_longlong, c_int, _P, c_void_p, c_int,
                                 c_void_p]),
    "dash_scale_check": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    "dash_cheb_ws_bytes": (c_size_t, [c_int, c_int]),
    "dash_clenshaw": (c_int, [_P, c_void_p, c_void_p, c_void_p, c_int, c_void_p, _P, c_int, c_void_p, c_void_p,
                              c_size_t, c_void_p]),
    "dash_plan_ws_bytes": (c_size_t, [c_int, c_int]),
    "dash_plan_create": (c_void_p, [_PB, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p, _P,
                                    c_void_p, c_void_p, c_void_p, _P, _P, _P, c_void_p, c_void_p, c_void_p,
                                    c_void_p, c_void_p, c_void_p, c_float, c_int, c_void_p, c_size_t, c_void_p,
                                    ctypes.POINTER(c_int)]),
    "dash_plan_destroy": (None, [c_void_p]),
    "dash_plan_set_state_offsets": (c_int, [c_void_p, c_void_p]),
    "dash_plan_un_stride": (c_int, [c_void_p]),
    "dash_prep_parts": (c_int, []),
    "dash_apply_partials": (c_int, [c_int]),
    "dash_plan_accumulate": (c_int, [c_void_p, c_float, c_float, c_int, c_float, c_void_p]),
    "dash_plan_apply": (c_int, [c_void_p, c_void_p, c_void_p, c_float, c_void_p]),
    "dash_group_sym": (c_int, [c_void_p, c_int, c_int, c_float, c_void_p, c_void_p, c_void_p]),
    "dash_group_split_a": (c_int, [c_void_p, c_float, _P, c_void_p]),
    "dash_fro_scale": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
    "dash_power_iteration": (c_int, [c_void_p, c_int, c_int, c_float, c_int, c_int, c_ull, c_void_p, c_void_p,
                                     c_void_p, c_void_p, c_void_p, c_void_p]),
    "dash_power_iteration_split": (c_int, [_P, c_void_p, c_float, c_int, c_int, c_ull, c_void_p, c_void_p,
                                           c_void_p, c_void_p, c_void_p]),
    "dash_block_seed": (c_ull, [c_ull, c_ull]),
    "dash_jacobi_ws_bytes": (c_size_t, [c_int, c_int]),
    "dash_jacobi_eigh": (c_int, [c_void_p, c_int, c_int, ctypes.c_double, c_int, c_void_p, c_void_p, c_void_p,
                                 c_void_p, c_void_p, c_size_t, c_void_p]),
    "dash_pack_blocks": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dash_unpack_blocks": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    "dash_uniform_pm1": (c_int, [c_ull, c_int, c_void_p, c_void_p]),
}


def lib() -> ctypes.CDLL:
    """Load (once) and return the C-ABI library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise RuntimeError(
                f"{_LIB_PATH} not found: the DASH CUDA extension is not built "
                "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback.")
        handle = ctypes.CDLL(str(_LIB_PATH), mode=os.RTLD_LOCAL)
        for name, (res, args) in _SIGNATURES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def check(status: int, what: str) -> None:
    if status == DASH_OK:
        return
    if status == DASH_ENONFINITE:
        raise NumericalError(f"{what}: non-finite values")
    if status == DASH_EINVAL:
        raise ValueError(f"{what}: invalid argument")
    raise RuntimeError(f"{what}: CUDA error (status {status}): {torch.cuda.current_stream()}")


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda(t: torch.Tensor, what: str) -> None:
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (the DASH B200 path has no CPU fallback)")


def launch_count() -> int:
    return int(lib().dash_launch_count())


def gemm_timing(enable: bool) -> None:
    lib().dash_gemm_timing(1 if enable else 0)


def gemm_timing_read() -> tuple[int, float, float]:
    """(launches, total ms, total algorithmic flops) of the GEMM launches since timing was enabled."""
    n, ms, fl = ctypes.c_int(0), ctypes.c_double(0.0), ctypes.c_double(0.0)
    check(lib().dash_gemm_timing_read(ctypes.byref(n), ctypes.byref(ms), ctypes.byref(fl)), "dash_gemm_timing_read")
    return n.value, ms.value, fl.value


def gemm_timing_list(cap: int = 65536) -> list[tuple[float, float, float, int]]:
    """Per-launch (ms, algorithmic flops, issued tensor flops, tiles) of the GEMM launches since timing
    was enabled."""
    import numpy as np

    ms, fl, iss, tl = np.zeros(cap), np.zeros(cap), np.zeros(cap), np.zeros(cap, dtype=np.int32)
    n = lib().dash_gemm_timing_list(cap, ms.ctypes.data, fl.ctypes.data, iss.ctypes.data, tl.ctypes.data)
    if n < 0:
        check(-n, "dash_gemm_timing_list")
    return [(float(ms[i]), float(fl[i]), float(iss[i]), int(tl[i])) for i in range(n)]
