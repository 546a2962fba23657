"""Golden deformation-kernel tables produced by running the REFERENCE's
kernel_line / kernel_point (paqif/ehl/kernels.py:64-100; build container
only):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_kernels.py

Grids: line n_x = 64 / 1024 (h = 0.05 / 6/1024), point 16 x 12 (h = 0.1)
and 128 x 128 (h = 6/128).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
from paqif.ehl.kernels import kernel_line, kernel_point  # noqa: E402

LINE = [(64, 0.05), (1024, 6.0 / 1024)]
POINT = [(16, 12, 0.1), (128, 128, 6.0 / 128)]


def main():
    out = {}
    for k, (n, h) in enumerate(LINE):
        out[f"line{k}_n"], out[f"line{k}_h"] = n, h
        out[f"line{k}_table"] = kernel_line(n, h).table
    for k, (nx, ny, h) in enumerate(POINT):
        out[f"point{k}_nx"], out[f"point{k}_ny"], out[f"point{k}_h"] = nx, ny, h
        out[f"point{k}_table"] = kernel_point(nx, ny, h).table
    np.savez_compressed(os.path.join(HERE, "ehl_kernels.npz"), **out)


if __name__ == "__main__":
    main()
