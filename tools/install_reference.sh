#!/bin/bash
# Install the unmodified reference package (/root/reference/pkg) into the
# git-ignored baseline/_ref (it travels to the GPU box with the gpurun
# snapshot; /root/reference does not), together with its own test suite, so
# the reference's callers and tests can run against libb200rt through
# paper_2305_07450_b200.install() on a B200 (tests/test_gpu_reference_suite.py).
#   bash tools/install_reference.sh
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=/root/reference/pkg
[ -d "$SRC" ] || { echo "no $SRC here (the GPU box uses the prebuilt baseline/_ref)"; exit 1; }
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"   # the build writes into its source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { cat "$TMP/pip.log"; exit 1; }
# the reference's own tests (pytest rootdir: baseline/_ref/ref_tests)
cp -r "$SRC/tests" "$ROOT/baseline/_ref/ref_tests"
rm -rf "$TMP"
python -c "import sys; sys.path.insert(0, '$ROOT/baseline/_ref'); import raytracer, raytracer.renderer; print('installed', raytracer.__file__)"
