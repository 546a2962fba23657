"""The reference's own tests (pkg/tests: test_aqif, test_parallel, test_lcp,
test_bandcore, test_tvdcd), unmodified, run against the device kernels through the
INTEGRATION.md binding (tests/refshim/b200_shim.py).

baseline/_ref holds the unmodified reference package and its tests
(tools/install_ref.sh, git-ignored, shipped to the GPU box).  The shim counts
the device-kernel calls; the test asserts they happened, so a pass cannot
come from the reference's numba kernels.
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, has_gpu

REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "ref_tests")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device"),
              pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                 reason="baseline/_ref not installed (tools/install_ref.sh)")]


def _run(mode, files, tmp_path):
    out = tmp_path / f"calls_{mode}.json"
    env = dict(os.environ)
    env.update({"PAQIF_SHIM": mode, "PAQIF_SHIM_OUT": str(out),
                "PYTHONPATH": os.pathsep.join([os.path.join(ROOT, "tests", "refshim"), ROOT, REF,
                                               REF_TESTS]),
                "NUMBA_CACHE_DIR": str(tmp_path / "numba"), "PYTHONDONTWRITEBYTECODE": "1"})
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "b200_shim", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS] + [os.path.join(REF_TESTS, f) for f in files]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    calls = json.loads(out.read_text())["calls"]
    return calls, tail


def test_reference_suite_on_device_kernels(tmp_path):
    calls, tail = _run("kernels", ["test_aqif.py", "test_parallel.py", "test_lcp.py",
                                   "test_bandcore.py"], tmp_path)
    assert calls.get("factor_batch", 0) > 50 and calls.get("solve_z_batch", 0) > 50, calls
    assert calls.get("psor_sweeps", 0) > 0, calls
    print(tail.splitlines()[-1], calls)


def test_reference_suite_on_fused_entries(tmp_path):
    calls, tail = _run("fused", ["test_parallel.py", "test_lcp.py"], tmp_path)
    assert calls.get("paqif_solve", 0) > 5 and calls.get("paqif_solve_lcp", 0) > 2, calls
    print(tail.splitlines()[-1], calls)


def test_reference_tvd_suite_on_device_sweeps(tmp_path):
    """test_tvdcd.py (the linear TVD study: kappa operators, limiters, the
    line-splitting sweeps) with the sweep entry points on the device sweeps
    and every AQIF call on the device kernels."""
    calls, tail = _run("tvd", ["test_tvdcd.py"], tmp_path)
    assert calls.get("solve_by_sweeps", 0) > 3 and calls.get("sweep_splitting", 0) > 0, calls
    print(tail.splitlines()[-1], calls)
