#!/bin/bash
# Install the UNMODIFIED reference package into baseline/_ref (git-ignored,
# but shipped to the GPU box by gpurun) together with its own test suite, so
# tests/test_reference_suite_gpu.py can run the reference's tests on top of
# the device kernels and bench.py --impl reference can time
# the reference's numba path.  Build container only (reads /root/reference).
set -euo pipefail
cd "$(dirname "$0")/.."
tmp=$(mktemp -d)
cp -r /root/reference/pkg "$tmp/pkg"
rm -rf baseline/_ref
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref "$tmp/pkg" >/dev/null
cp -r /root/reference/pkg/tests baseline/_ref/ref_tests
rm -rf "$tmp"
echo "installed: $(ls baseline/_ref)"
