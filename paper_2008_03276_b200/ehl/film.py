"""Film thickness bookkeeping (public surface of paqif/ehl/film.py:35-155).

Line contact: H = h0 + x^2/2 - (1/pi) sum K*u, the Toeplitz convolution
running on the GPU (paqif_line_deformation).  Point contact grids carry the
geometry and kernel tables; their 2-D deformation path is listed as the next
row in DESIGN.md.
"""

from __future__ import annotations

import numpy as np

from ..errors import ContractViolationError
from .kernels import DeformationKernel, kernel_line, kernel_point

__all__ = ["FilmModel"]


class FilmModel:
    def __init__(self, contact: str, intervals: int, h: float, lo: float = -2.5,
                 kernel: DeformationKernel | None = None):
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
        if contact == "point":
            gx, gy = np.meshgrid(self.x, self.x)
            self.geometry = 0.5 * (gx ** 2 + gy ** 2)
            self.sign = 1.0
        else:
            self.geometry = 0.5 * self.x ** 2
            self.sign = -1.0 / np.pi
        self._base = None
        self._pending = []

    def deformation_full(self, u) -> np.ndarray:
        if self.contact != "line":
            raise NotImplementedError("2-D deformation: next row (DESIGN.md section 7)")
        from .line import line_deformation
        self._base = line_deformation(self.kernel.table, u)
        self._pending = []
        return self._base

    def film_full(self, u, h0: float) -> np.ndarray:
        return h0 + self.geometry + self.deformation_full(u)

    def sensitivity(self, d: int, axis_offset: int = 0) -> float:
        if self.contact == "line":
            return self.sign * float(self.kernel.table[abs(d)])
        return float(self.kernel.table[abs(d), abs(axis_offset)])
