#!/bin/bash
# Install the UNMODIFIED reference (bitunet 0.1.0) into baseline/_ref, with its
# own test suite beside it (baseline/_ref/bitunet_tests). baseline/_ref is
# git-ignored (not repo source) but not gpurun-ignored, so it travels to the
# GPU box, where tests/test_gpu_conformance.py runs that suite with the
# reference's compute functions rebound to this engine (paper_2601_11660_b200/plug.py).
set -e
root=$(cd "$(dirname "$0")/.." && pwd)
src=${1:-/root/reference/pkg}
tmp=$(mktemp -d)
cp -r "$src" "$tmp/pkg"          # the build writes into its source tree; the reference is read-only
rm -rf "$root/baseline/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$root/baseline/_ref" "$tmp/pkg"
cp -r "$src/tests" "$root/baseline/_ref/bitunet_tests"
rm -rf "$tmp"
echo "installed bitunet into $root/baseline/_ref (tests: baseline/_ref/bitunet_tests)"
