#!/bin/sh
# One-time offline install of the unmodified reference (femasm) into baseline/_ref (git-ignored,
# travels to the GPU box with gpurun): the package for bench.py's CPU baseline / reference arm,
# and its own test suites (pkg/tests) for tests/test_femasm_suite.py, which runs them against
# this package through tests/femasm_shim.
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/femasm_src && cp -r /root/reference/pkg /tmp/femasm_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$REPO/baseline/_ref" /tmp/femasm_src
rm -rf "$REPO/baseline/_ref/femasm_tests" && cp -r /root/reference/pkg/tests "$REPO/baseline/_ref/femasm_tests"
