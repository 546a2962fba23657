"""Drop-in replacement for the reference's ``paqif._kernels`` module.

Same function names, same batched float64 arrays, same in-place semantics
and status codes as paqif/_kernels.py:62-276 -- but every kernel runs on the
GPU through libpaqif_b200.so.  With the default ``exact=True`` the results
are bit-identical to the reference (no FMA contraction, IEEE division).

Host arrays go up, the kernel runs, results come back into the same numpy
arrays.  ``HAS_NUMBA`` is kept for import compatibility (always False: the
compiled path here is CUDA, not numba).
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import ContractViolationError

HAS_NUMBA = False


def _dev(arr, torch):
    if not isinstance(arr, np.ndarray) or not arr.flags.c_contiguous:
        raise ContractViolationError("kernel buffers must be C-contiguous ndarrays")
    return torch.from_numpy(arr).to("cuda")


def _back(arr, t):
    arr[...] = t.cpu().numpy()


def _flags(exact):
    return _native.FLAG_EXACT if exact else 0


def factor_batch(band, anti, z2x2, zl, zr, ww, tol, status, exact=True):
    """In-place AQIF factorization of a batch (reference _kernels.py:62-149)."""
    torch = _native.torch_cuda()
    L = _native.lib()
    B, d, n = band.shape
    beta = (d - 1) // 2
    ts = [_dev(a, torch) for a in (band, anti, z2x2, zl, zr, ww, status)]
    rc = L.paqif_factor_batch(B, n, beta, *[t.data_ptr() for t in ts[:6]], float(tol),
                              ts[6].data_ptr(), _flags(exact), _native.stream_ptr())
    _native.check(rc, "paqif_factor_batch")
    torch.cuda.current_stream().synchronize()
    for a, t in zip((band, anti, z2x2, zl, zr, ww, status), ts):
        _back(a, t)


def solve_w_batch(ww, rhs, exact=True):
    """Middle-out W solve in place (reference _kernels.py:152-172)."""
    torch = _native.torch_cuda()
    L = _native.lib()
    B, n = rhs.shape
    beta = ww.shape[2] // 2
    tw, tr = _dev(ww, torch), _dev(rhs, torch)
    rc = L.paqif_solve_w_batch(B, n, beta, tw.data_ptr(), tr.data_ptr(), _flags(exact),
                               _native.stream_ptr())
    _native.check(rc, "paqif_solve_w_batch")
    _back(rhs, tr)


def solve_z_batch(z2x2, zl, zr, y, x, start, tol, status, trace, exact=True):
    """Outside-in Z solve (reference _kernels.py:175-225)."""
    torch = _native.torch_cuda()
    L = _native.lib()
    B, n = y.shape
    beta = zl.shape[3] - 1
    ts = [_dev(a, torch) for a in (z2x2, zl, zr, y, x, status, trace)]
    rc = L.paqif_solve_z_batch(B, n, beta, ts[0].data_ptr(), ts[1].data_ptr(), ts[2].data_ptr(),
                               ts[3].data_ptr(), ts[4].data_ptr(), int(start), float(tol),
                               ts[5].data_ptr(), ts[6].data_ptr(), _flags(exact),
                               _native.stream_ptr())
    _native.check(rc, "paqif_solve_z_batch")
    _back(x, ts[4])
    _back(status, ts[5])
    _back(trace, ts[6])


def band_matvec_batch(bands, x, out):
    """out = A x (reference _kernels.py:228-241)."""
    torch = _native.torch_cuda()
    L = _native.lib()
    B, d, n = bands.shape
    tb, tx, to = _dev(bands, torch), _dev(x, torch), _dev(out, torch)
    rc = L.paqif_band_matvec_batch(B, n, (d - 1) // 2, tb.data_ptr(), tx.data_ptr(),
                                   to.data_ptr(), _native.stream_ptr())
    _native.check(rc, "paqif_band_matvec_batch")
    _back(out, to)


def psor_sweeps(bands, f, u, omega, tol, max_sweeps):
    """Projected SOR (reference _kernels.py:244-276); returns (sweeps, change)."""
    import ctypes
    torch = _native.torch_cuda()
    L = _native.lib()
    n = f.shape[0]
    beta = (bands.shape[0] - 1) // 2
    tb, tf, tu = _dev(bands, torch), _dev(f, torch), _dev(u, torch)
    sw = ctypes.c_int64(0)
    ch = ctypes.c_double(0.0)
    rc = L.paqif_psor_sweeps(n, beta, tb.data_ptr(), tf.data_ptr(), tu.data_ptr(), float(omega),
                             float(tol), int(max_sweeps), ctypes.addressof(sw),
                             ctypes.addressof(ch), _native.stream_ptr())
    _native.check(rc, "paqif_psor_sweeps")
    _back(u, tu)
    return int(sw.value), float(ch.value)
