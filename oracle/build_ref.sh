#!/usr/bin/env bash
# Builds the UNMODIFIED reference `rhosolve` (Python + its Cython kernel
# module) into oracle/_ref/ so it can serve as the checker and as the
# `bench.py --impl reference` CPU arm.  Test infrastructure only: nothing in
# paper_1504_06768_b200/ imports it.
#
# The reference tree is read-only, so the build runs from a copy under /tmp.
# Output goes only to oracle/_ref/ (git-ignored, travels to the GPU box).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REF:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then
  echo "build_ref: $REF not present (GPU box?); keeping prebuilt $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/rhosolve_ref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --no-index --no-build-isolation --no-deps -q \
  --target "$OUT" "$TMP/pkg"
PYTHONPATH="$OUT" python -c "import rhosolve; assert rhosolve.KERNEL_BACKEND == 'c', rhosolve.KERNEL_BACKEND; print('rhosolve reference built, backend', rhosolve.KERNEL_BACKEND)"
