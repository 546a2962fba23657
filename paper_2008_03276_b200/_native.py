"""ctypes binding of libpaqif_b200.so (the C ABI in include/paqif_b200.h).

There is no CPU fallback: if the library is missing or no CUDA device is
present, every compute entry point raises :class:`NativeUnavailableError`.
Device memory and streams come from PyTorch (plumbing only).
"""

from __future__ import annotations

import ctypes
import os

from .errors import PaqifError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PAQIF_LIB") or os.path.join(HERE, "_build", "libpaqif_b200.so")

FLAG_EXACT = 1
FLAG_LINE_SPLIT = 2   # EHL line steps: force the split three-kernel path
FLAG_LINE_FUSED = 4   # EHL line steps: force the fused one-CTA-per-case kernel

LCP_OK = 0
LCP_FACTOR_BREAKDOWN = 1
LCP_ZSOLVE_BREAKDOWN = 2
LCP_NOT_PD = 3
LCP_NONCONVERGED = 4

# every symbol include/paqif_b200.h declares (checked by tests/test_native_abi.py)
EXPORTS = (
    "paqif_version", "paqif_last_error", "paqif_device_count",
    "paqif_factor_batch", "paqif_solve_w_batch", "paqif_solve_z_batch",
    "paqif_band_matvec_batch", "paqif_psor_sweeps", "paqif_solve_r1_batch",
    "paqif_lcp_workspace_bytes", "paqif_lcp_batch", "paqif_lcp_batch_host",
)


class NativeUnavailableError(PaqifError):
    """The CUDA library (or a CUDA device) is not available."""


_lib = None

_i64 = ctypes.c_int64
_u32 = ctypes.c_uint32
_f64 = ctypes.c_double
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t


def lib_path() -> str:
    return LIB_PATH


def load(build_if_missing: bool = False):
    """Load the shared library (no device needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        if build_if_missing:
            from .build import build
            build()
        else:
            raise NativeUnavailableError(
                f"{LIB_PATH} not built; run python -m paper_2008_03276_b200.build")
    L = ctypes.CDLL(LIB_PATH)
    L.paqif_version.restype = ctypes.c_char_p
    L.paqif_last_error.restype = ctypes.c_char_p
    L.paqif_device_count.restype = ctypes.c_int
    L.paqif_factor_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _f64, _vp,
                                     _u32, _vp]
    L.paqif_solve_w_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _u32, _vp]
    L.paqif_solve_z_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _i64, _f64,
                                      _vp, _vp, _u32, _vp]
    L.paqif_band_matvec_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp]
    L.paqif_psor_sweeps.argtypes = [_i64, _i64, _vp, _vp, _vp, _f64, _f64, _i64, _vp, _vp, _vp]
    L.paqif_solve_r1_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _u32, _vp, _sz, _vp]
    L.paqif_lcp_workspace_bytes.argtypes = [_i64, _i64, _i64]
    L.paqif_lcp_workspace_bytes.restype = _sz
    L.paqif_lcp_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _f64, _i64, _u32, _vp, _vp, _vp,
                                  _vp, _vp, _vp, _sz, _vp]
    L.paqif_lcp_batch_host.argtypes = [_i64, _i64, _i64, _vp, _vp, _f64, _i64, _u32, _vp, _vp,
                                       _vp, _vp, _vp]
    if hasattr(L, "paqif_solve_rblock_batch"):
        L.paqif_solve_rblock_workspace_bytes.argtypes = [_i64, _i64, _i64, _i64]
        L.paqif_solve_rblock_workspace_bytes.restype = _sz
        L.paqif_solve_rblock_batch.argtypes = [_i64, _i64, _i64, _i64, _vp, _vp, _vp,
                                               ctypes.c_int32, _vp, _u32, _vp, _sz, _vp]
        L.paqif_lcp_pin_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp]
        L.paqif_lcp_pass_batch.argtypes = [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                           _vp, _vp]
    if hasattr(L, "paqif_ehl_line_step"):
        L.paqif_ehl_line_workspace_bytes.argtypes = [_i64, _i64]
        L.paqif_ehl_line_workspace_bytes.restype = _sz
    for name in EXPORTS:
        if hasattr(L, name):
            fn = getattr(L, name)
            if fn.restype is None or fn.restype is ctypes.c_int:
                fn.restype = fn.restype or ctypes.c_int
    _lib = L
    return L


def lib():
    """The library, with a usable CUDA device (raises otherwise)."""
    L = load()
    if L.paqif_device_count() < 1:
        raise NativeUnavailableError("no CUDA device visible to libpaqif_b200")
    return L


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = _lib.paqif_last_error().decode() if _lib is not None else ""
        raise PaqifError(f"{what} failed (rc={rc}): {msg}")


def torch_cuda():
    """Import torch and return it, requiring CUDA."""
    import torch
    if not torch.cuda.is_available():
        raise NativeUnavailableError("torch reports no CUDA device")
    return torch


def stream_ptr(stream=None) -> int:
    torch = torch_cuda()
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
