"""The C-ABI library loads without a GPU and exports every symbol the public
headers declare; the kernels are built for sm_100a (no GPU needed)."""

import glob
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_2008_03276_b200 import _native
from paper_2008_03276_b200.build import build


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        for m in re.finditer(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(paqif_[a-z0-9_]+)\s*\(",
                             text, re.M):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    build()
    return _native.load()


def test_headers_declare_symbols():
    names = declared_symbols()
    assert {"paqif_factor_batch", "paqif_lcp_batch", "paqif_lcp_batch_host"} <= names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in sorted(declared_symbols()) if not hasattr(lib, n)]
    assert not missing, missing


def test_version_and_error_strings(lib):
    assert b"sm_100a" in lib.paqif_version()
    assert isinstance(lib.paqif_last_error(), bytes)


def test_argument_errors_need_no_device(lib):
    # odd order is rejected before anything touches the device
    assert lib.paqif_factor_batch(1, 7, 1, None, None, None, None, None, None, 1e-14, None, 1,
                                  None) == -1
    assert b"argument" in lib.paqif_last_error()
    assert lib.paqif_lcp_workspace_bytes(4, 1026, 9) == 0  # beta > 8 unsupported in fused LCP
    assert lib.paqif_lcp_batch(4, 10, 8, None, None, 1e-10, 100, 1, None, None, None, None,
                               None, None, 0, None) == -1  # n <= 2*beta+1


def test_cubin_is_sm100a():
    path = _native.lib_path()
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_cpu_fallback_without_device(monkeypatch):
    import numpy as np
    from paper_2008_03276_b200 import batch
    if _native.load().paqif_device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(_native.NativeUnavailableError):
        batch.lcp_batch(np.zeros((1, 3, 8)), np.zeros((1, 8)))
