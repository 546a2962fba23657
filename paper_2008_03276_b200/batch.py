"""Batched device API: many independent banded LCPs / linear systems in one
kernel launch (the config-2 hot path).

Inputs may be torch CUDA tensors (zero-copy; the stream is torch's current
stream) or host numpy arrays (copied in and out).  Layout is the reference's
batched layout: ``bands (B, 2*beta+1, n)`` diagonal-major, ``f (B, n)``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ContractViolationError


@dataclass
class LcpBatchResult:
    u: object          # (B, n) float64 solution (projected)
    active: object     # (B, n) bool, pinned (cavitated) set of the returned pass
    passes: object     # (B,) int64 active-set passes (paqif_solve calls)
    res: object        # (B,) float64 complementarity residual of u
    status: object     # (B,) int64 PAQIF_LCP_* codes


def _shape(bands, f):
    if bands.ndim != 3 or f.ndim != 2:
        raise ContractViolationError("bands must be (B, 2beta+1, n) and f (B, n)")
    B, d, n = bands.shape
    if d % 2 != 1 or f.shape != (B, n):
        raise ContractViolationError("inconsistent batch shapes")
    return B, (d - 1) // 2, n


class LcpSolver:
    """Preallocated device workspace for repeated batches of one shape."""

    def __init__(self, B: int, n: int, beta: int, exact: bool = True):
        torch = _native.torch_cuda()
        self.L = _native.lib()
        self.B, self.n, self.beta = B, n, beta
        self.flags = _native.FLAG_EXACT if exact else 0
        nbytes = self.L.paqif_lcp_workspace_bytes(B, n, beta)
        if nbytes == 0 and B > 0:
            raise ContractViolationError(
                f"unsupported LCP shape B={B} n={n} beta={beta} (n even, n > 2beta+1, beta<=8)")
        self.ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device="cuda")
        self.ws_bytes = nbytes
        dev = "cuda"
        self.u = torch.empty((B, n), dtype=torch.float64, device=dev)
        self.active = torch.empty((B, n), dtype=torch.uint8, device=dev)
        self.passes = torch.empty(B, dtype=torch.int64, device=dev)
        self.res = torch.empty(B, dtype=torch.float64, device=dev)
        self.status = torch.empty(B, dtype=torch.int64, device=dev)

    def launch(self, bands, f, tol: float = 1e-10, max_outer: int = 100, stream=None) -> None:
        """Asynchronous launch on device tensors (results in self.u etc.)."""
        rc = self.L.paqif_lcp_batch(self.B, self.n, self.beta, bands.data_ptr(), f.data_ptr(),
                                    float(tol), int(max_outer), self.flags, self.u.data_ptr(),
                                    self.active.data_ptr(), self.passes.data_ptr(),
                                    self.res.data_ptr(), self.status.data_ptr(),
                                    self.ws.data_ptr(), self.ws_bytes,
                                    _native.stream_ptr(stream))
        _native.check(rc, "paqif_lcp_batch")

    def solve_r1(self, bands, f, stream=None):
        """paqif_solve(L_b, f_b, r=1) for every b; returns (x, status) tensors."""
        rc = self.L.paqif_solve_r1_batch(self.B, self.n, self.beta, bands.data_ptr(),
                                         f.data_ptr(), self.u.data_ptr(), self.status.data_ptr(),
                                         self.flags, self.ws.data_ptr(), self.ws_bytes,
                                         _native.stream_ptr(stream))
        _native.check(rc, "paqif_solve_r1_batch")
        return self.u, self.status


def lcp_batch(bands, f, tol: float = 1e-10, max_outer: int = 100, exact: bool = True,
              solver: LcpSolver | None = None) -> LcpBatchResult:
    """Solve every ``u >= 0, L_b u >= f_b, u.(L_b u - f_b) = 0`` with the
    reference's projected-pass policy (paqif_solve_lcp, parallel.py:298-347)."""
    torch = _native.torch_cuda()
    host = isinstance(bands, np.ndarray)
    if host:
        tb = torch.from_numpy(np.ascontiguousarray(bands, dtype=np.float64)).cuda()
        tf = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).cuda()
    else:
        tb, tf = bands.contiguous(), f.contiguous()
    B, beta, n = _shape(tb, tf)
    s = solver or LcpSolver(B, n, beta, exact)
    s.launch(tb, tf, tol, max_outer)
    if host:
        torch.cuda.current_stream().synchronize()
        return LcpBatchResult(s.u.cpu().numpy(), s.active.cpu().numpy().astype(bool),
                              s.passes.cpu().numpy(), s.res.cpu().numpy(),
                              s.status.cpu().numpy())
    return LcpBatchResult(s.u, s.active.bool(), s.passes, s.res, s.status)


def lcp_batch_host(bands: np.ndarray, f: np.ndarray, tol: float = 1e-10, max_outer: int = 100,
                   exact: bool = True) -> LcpBatchResult:
    """The host-buffer C-ABI entry (paqif_lcp_batch_host): H2D, kernel, D2H."""
    L = _native.lib()
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    f = np.ascontiguousarray(f, dtype=np.float64)
    B, d, n = bands.shape
    u = np.empty((B, n))
    act = np.empty((B, n), dtype=np.uint8)
    passes = np.empty(B, dtype=np.int64)
    res = np.empty(B)
    st = np.empty(B, dtype=np.int64)
    rc = L.paqif_lcp_batch_host(B, n, (d - 1) // 2, bands.ctypes.data, f.ctypes.data, float(tol),
                                int(max_outer), _native.FLAG_EXACT if exact else 0,
                                u.ctypes.data, act.ctypes.data, passes.ctypes.data,
                                res.ctypes.data, st.ctypes.data)
    _native.check(rc, "paqif_lcp_batch_host")
    return LcpBatchResult(u, act.astype(bool), passes, res, st)


def solve_r1_batch(bands, f, exact: bool = True):
    """Batched paqif_solve(L_b, f_b, r=1): returns (x, status) like the inputs."""
    torch = _native.torch_cuda()
    host = isinstance(bands, np.ndarray)
    tb = torch.from_numpy(np.ascontiguousarray(bands, dtype=np.float64)).cuda() if host else bands
    tf = torch.from_numpy(np.ascontiguousarray(f, dtype=np.float64)).cuda() if host else f
    B, beta, n = _shape(tb, tf)
    s = LcpSolver(B, n, beta, exact)
    x, st = s.solve_r1(tb, tf)
    if host:
        torch.cuda.current_stream().synchronize()
        return x.cpu().numpy(), st.cpu().numpy()
    return x, st
