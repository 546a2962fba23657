"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Restatements of the reference algorithm used as the checker by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
arm.  The product package (paper_2008_03276_b200) never imports this.

* ``paqif_oracle.c`` (built to ``oracle/build/libpaqif_oracle.so``): the AQIF
  kernels of ``paqif/_kernels.py`` bit-for-bit, and the r=1 projected LCP
  driver of ``paqif/parallel.py:298-347``.  Pinned against golden vectors the
  reference itself produced (tests/golden/make_golden.py).
* ``ehl_oracle.py``: numpy restatement of the EHL Newton step
  (``paqif/ehl/*``), pinned against reference-generated goldens
  (tests/golden/make_golden_ehl.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libpaqif_oracle.so")

_lib = None

_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int64)
_U8 = ctypes.POINTER(ctypes.c_uint8)
_i64 = ctypes.c_int64
_f64 = ctypes.c_double


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "paqif_oracle.c")
    if force or not os.path.exists(LIB_PATH) or \
            os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.or_factor_batch.argtypes = [_i64, _i64, _i64, _D, _D, _D, _D, _D, _D, _f64, _I]
        L.or_solve_w_batch.argtypes = [_i64, _i64, _i64, _D, _D]
        L.or_solve_z_batch.argtypes = [_i64, _i64, _i64, _D, _D, _D, _D, _D, _i64, _f64, _I, _I]
        L.or_band_matvec_batch.argtypes = [_i64, _i64, _i64, _D, _D, _D]
        L.or_psor_sweeps.argtypes = [_i64, _i64, _D, _D, _D, _f64, _f64, _i64, _D]
        L.or_psor_sweeps.restype = _i64
        L.or_paqif_solve_r1.argtypes = [_i64, _i64, _D, _D, _D]
        L.or_paqif_solve_r1.restype = ctypes.c_int
        L.or_lcp_batch.argtypes = [_i64, _i64, _i64, _D, _D, _f64, _i64, _D, _U8, _I, _D, _I, _i64]
        L.or_paqif_solve_r1_batch.argtypes = [_i64, _i64, _i64, _D, _D, _D, _I, _i64]
        _lib = L
    return _lib


def _p(a, t=_D):
    assert a.flags.c_contiguous
    return a.ctypes.data_as(t)


def _chk(a, dtype=np.float64):
    if a.dtype != dtype or not a.flags.c_contiguous:
        raise TypeError("oracle buffers must be C-contiguous " + str(dtype))
    return a


# -- the reference's _kernels signatures, batched, in place -------------------

def factor_batch(band, anti, z2x2, zl, zr, ww, tol, status):
    for a in (band, anti, z2x2, zl, zr, ww):
        _chk(a)
    _chk(status, np.int64)
    B, d, n = band.shape
    lib().or_factor_batch(B, n, (d - 1) // 2, _p(band), _p(anti), _p(z2x2), _p(zl), _p(zr),
                          _p(ww), float(tol), _p(status, _I))


def solve_w_batch(ww, rhs):
    _chk(ww); _chk(rhs)
    B, n = rhs.shape
    lib().or_solve_w_batch(B, n, ww.shape[2] // 2, _p(ww), _p(rhs))


def solve_z_batch(z2x2, zl, zr, y, x, start, tol, status, trace):
    for a in (z2x2, zl, zr, y, x):
        _chk(a)
    _chk(status, np.int64); _chk(trace, np.int64)
    B, n = y.shape
    lib().or_solve_z_batch(B, n, zl.shape[3] - 1, _p(z2x2), _p(zl), _p(zr), _p(y), _p(x),
                           int(start), float(tol), _p(status, _I), _p(trace, _I))


def band_matvec_batch(bands, x, out):
    _chk(bands); _chk(x); _chk(out)
    B, d, n = bands.shape
    lib().or_band_matvec_batch(B, n, (d - 1) // 2, _p(bands), _p(x), _p(out))


def psor(bands, f, omega=1.0, tol=1e-12, max_sweeps=200_000):
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    n = f.shape[0]
    u = np.zeros(n)
    ch = ctypes.c_double(0.0)
    sweeps = lib().or_psor_sweeps(n, (bands.shape[0] - 1) // 2, _p(bands), _p(f), _p(u),
                                  float(omega), float(tol), int(max_sweeps), ctypes.byref(ch))
    return u, int(sweeps), float(ch.value)


def paqif_solve_r1(bands, f):
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    u = np.zeros(f.shape[0])
    rc = lib().or_paqif_solve_r1(f.shape[0], (bands.shape[0] - 1) // 2, _p(bands), _p(f), _p(u))
    return u, rc


def paqif_solve_r1_batch(bands, f, threads=1):
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    B, d, n = bands.shape
    x = np.zeros((B, n))
    st = np.zeros(B, dtype=np.int64)
    lib().or_paqif_solve_r1_batch(B, n, (d - 1) // 2, _p(bands), _p(f), _p(x), _p(st, _I),
                                  int(threads))
    return x, st


def lcp_batch(bands, f, tol=1e-10, max_outer=100, threads=1):
    """paqif_solve_lcp(LcpProblem(L_b, f_b), r=1) for every b.

    Returns (u, active, passes, res, status); status 0 ok, 1 factor
    breakdown, 2 z-solve breakdown, 3 reduced system not SPD, 4 no convergence.
    """
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    B, d, n = bands.shape
    u = np.zeros((B, n))
    act = np.zeros((B, n), dtype=np.uint8)
    passes = np.zeros(B, dtype=np.int64)
    res = np.zeros(B)
    st = np.zeros(B, dtype=np.int64)
    lib().or_lcp_batch(B, n, (d - 1) // 2, _p(bands), _p(f), float(tol), int(max_outer),
                       _p(u), _p(act, _U8), _p(passes, _I), _p(res), _p(st, _I), int(threads))
    return u, act.astype(bool), passes, res, st
