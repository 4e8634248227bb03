#!/bin/bash
# Stage the reference package's own test suite (pkg/tests + its data files)
# under baseline/_ref/pkg/ -- git-ignored, but it travels to the GPU box with
# the gpurun snapshot -- so tests/test_gpu_reference_suite.py can run it
# against this package (gridneighbors aliased).  Needs /root/reference (this
# container only); the GPU box uses the staged copy.
set -e
REF=${REF:-/root/reference/pkg}
DST=$(dirname "$0")/../baseline/_ref/pkg
[ -d "$REF/tests" ] || { echo "no reference at $REF"; exit 1; }
mkdir -p "$DST"
rm -rf "$DST/tests" "$DST/data"
cp -r "$REF/tests" "$DST/tests"
cp -r "$REF/data" "$DST/data"
echo "staged $(ls "$DST/tests" | wc -l) files into $DST"
