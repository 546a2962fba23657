"""Deformation kernel tables generated on the device (csrc/ehl_kernels.cu,
kernel_line / kernel_point(device=True)) vs the reference's tables (golden
ehl_kernels.npz, tests/golden/make_golden_kernels.py) and vs the host
tables at config sizes.  The operation order is the reference's; only the
library log / asinh differ in the last bit, so the bound is a few ulp of the
magnitude of the terms the table differences (the closed forms cancel:
an entry is a signed sum of terms up to ~100x larger than itself, so one
ulp of a term is many ulp of the entry -- the same spread two host libms
give)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

K = load_golden("ehl_kernels.npz")
ULP = np.finfo(np.float64).eps


def _line_terms(n, h):
    d = np.arange(n + 1) * h
    t = np.abs(np.concatenate([d + h / 2, d - h / 2]))
    t = t[t > 0]
    return np.abs(t * (np.log(t) - 1.0)).max()


def _point_terms(nx, ny, h):
    a = max(nx, ny) * h + h / 2
    return 2.0 / np.pi ** 2 * a * np.arcsinh(a / (h / 2))


def _close(dev, ref, term):
    err = np.abs(dev - ref).max()
    assert err <= 16 * ULP * term, (err, term)


@pytest.mark.parametrize("k", [0, 1])
def test_kernel_line_device_vs_reference(k):
    from paper_2008_03276_b200.ehl import kernel_line
    n, h = int(K[f"line{k}_n"]), float(K[f"line{k}_h"])
    kl = kernel_line(n, h, device=True)
    assert kl.contact == "line" and kl.h == h and kl.table.shape == (n + 1,)
    _close(kl.table, K[f"line{k}_table"], _line_terms(n, h))


@pytest.mark.parametrize("k", [0, 1])
def test_kernel_point_device_vs_reference(k):
    from paper_2008_03276_b200.ehl import kernel_point
    nx, ny, h = int(K[f"point{k}_nx"]), int(K[f"point{k}_ny"]), float(K[f"point{k}_h"])
    kp = kernel_point(nx, ny, h, device=True)
    assert kp.table.shape == (nx + 1, ny + 1)
    _close(kp.table, K[f"point{k}_table"], _point_terms(nx, ny, h))


@pytest.mark.parametrize("n", [512, 2048])
def test_kernel_point_device_config_sizes(n):
    from paper_2008_03276_b200.ehl import kernel_point
    h = 6.0 / n
    _close(kernel_point(n, n, h, device=True).table, kernel_point(n, n, h).table,
           _point_terms(n, n, h))


def test_kernel_device_args():
    from paper_2008_03276_b200.ehl import kernel_line, kernel_point
    from paper_2008_03276_b200.errors import ContractViolationError
    with pytest.raises(ContractViolationError):
        kernel_point(4, 4, 0.0, device=True)
    with pytest.raises(ContractViolationError):
        kernel_line(4, -1.0, device=True)
    assert kernel_line(0, 0.1, device=True).table.shape == (1,)
