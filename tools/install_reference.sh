#!/bin/bash
# Installs the unmodified reference package into baseline/_ref (git-ignored; it
# travels to the GPU box with the snapshot) and copies its test suite next to
# it, so the reference's own engine tests can run against the B200 backend
# (tests/test_gpu_reference_suite.py).  The reference source is never copied
# into the tracked tree.
set -eu
ROOT=$(cd "$(dirname "$0")/.." && pwd)
REF=${1:-/root/reference}
rm -rf /tmp/moe_ref_src && cp -r "$REF/pkg" /tmp/moe_ref_src
rm -rf "$ROOT/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" /tmp/moe_ref_src
mkdir -p "$ROOT/baseline/_ref/ref_tests"
cp -r "$REF/pkg/tests" "$ROOT/baseline/_ref/ref_tests/tests"
touch "$ROOT/baseline/_ref/ref_tests/tests/__init__.py"
echo "reference installed: $ROOT/baseline/_ref"
