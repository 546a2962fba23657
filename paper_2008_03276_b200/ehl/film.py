"""Film thickness bookkeeping (public surface of paqif/ehl/film.py:35-155).

Line contact: H = h0 + x^2/2 - (1/pi) sum K*u, the Toeplitz convolution
running on the GPU (paqif_line_deformation).  Point contact: H = h0 +
(x^2 + y^2)/2 + sum K*u, the 2-D convolution running as an fp64 FFT on the
GPU (paqif_ehl_point_deformation, csrc/fft_deform.cuh).
"""

from __future__ import annotations

import numpy as np

from ..errors import ContractViolationError
from .kernels import DeformationKernel, kernel_line, kernel_point

__all__ = ["FilmModel"]


class FilmModel:
    def __init__(self, contact: str, intervals: int, h: float, lo: float = -2.5,
                 kernel: DeformationKernel | None = None, lo_y: float | None = None):
        if contact not in ("point", "line"):
            raise ContractViolationError("contact must be 'point' or 'line'")
        self.contact = contact
        self.n = intervals
        self.h = h
        self.x = lo + h * np.arange(intervals + 1)
        if kernel is None:
            kernel = (kernel_point(intervals, intervals, h) if contact == "point"
                      else kernel_line(intervals, h))
        self.kernel = kernel
        # lo_y: the SURVEY 8(c) y-domain adapter, y = (x - x[0]) + lo_y
        self.y = self.x if lo_y is None else (self.x - self.x[0]) + lo_y
        self._device = None
        if contact == "point":
            gx, gy = np.meshgrid(self.x, self.y)
            self.geometry = 0.5 * (gx ** 2 + gy ** 2)
            self.sign = 1.0
        else:
            self.geometry = 0.5 * self.x ** 2
            self.sign = -1.0 / np.pi
        self._base = None
        self._pending = []

    def deformation_full(self, u) -> np.ndarray:
        if self.contact == "point":
            from .point import PointDevice
            if self._device is None:
                self._device = PointDevice(self.kernel.table, self.geometry)
            self._base = self._device.deformation(u)
            self._pending = []
            return self._base
        from .line import line_deformation
        self._base = line_deformation(self.kernel.table, u)
        self._pending = []
        return self._base

    def film_full(self, u, h0: float) -> np.ndarray:
        return h0 + self.geometry + self.deformation_full(u)

    # -- pending line updates (film.py:83-146): the device keeps the list
    # and applies the exact corrections (csrc/ehl_point.cu pt_films) --------

    FOLD_LIMIT = 8

    def note_line_update(self, axis: str, index: int, delta, u) -> None:
        """Record an applied line change; fold into the base once more than
        8 are pending."""
        if axis not in ("row", "col"):
            raise ContractViolationError(f"unknown axis {axis!r}")
        delta = np.asarray(delta, dtype=np.float64)
        if not np.any(delta):
            return
        if self.contact == "point":
            if self._base is None:
                raise ContractViolationError("call deformation_full first")
            self._device.note_update(0 if axis == "row" else 1, index, delta)
        self._pending.append((axis, int(index)))
        if len(self._pending) > self.FOLD_LIMIT:
            self.deformation_full(u)

    def _lines(self, mode: int, idx, h0: float) -> np.ndarray:
        if self._base is None:
            raise ContractViolationError("call deformation_full first")
        if self.contact == "line":
            raise ContractViolationError("line contact has a single row")
        return self._device.film_lines(mode, list(idx), h0)

    def film_rows(self, rows, h0: float) -> np.ndarray:
        """Current film on the requested rows (pending updates included)."""
        return self._lines(0, rows, h0)

    def film_cols(self, cols, h0: float) -> np.ndarray:
        """Current film on the requested columns (pending updates included)."""
        return self._lines(1, cols, h0)

    def sensitivity(self, d: int, axis_offset: int = 0) -> float:
        if self.contact == "line":
            return self.sign * float(self.kernel.table[abs(d)])
        return float(self.kernel.table[abs(d), abs(axis_offset)])
