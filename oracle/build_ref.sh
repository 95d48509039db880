#!/usr/bin/env bash
# Build the reference's own compiled lane (txfem/_kernels_cy.pyx) into
# oracle/_ref/ — TEST INFRASTRUCTURE ONLY (checker + CPU reference arm).
#
# Recipe mirrors the reference build flags (pkg/setup.py:14-20: -O3
# -ffp-contract=off) but does NOT run the reference's own build system: the
# single .pyx is translated with cython and compiled with gcc directly.
# Output goes only to oracle/_ref/ (git-ignored, travels to the GPU box).
# /root/reference is read-only and absent on the GPU box, so this runs here.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${TXFEM_REF_PYX:-/root/reference/pkg/src/txfem/_kernels_cy.pyx}"
OUT="$HERE/_ref"
if [ ! -f "$SRC" ]; then
  echo "build_ref: reference source $SRC not present; keeping prebuilt oracle/_ref" >&2
  exit 0
fi
mkdir -p "$OUT"
PY="${PYTHON:-python3}"
EXT_SUFFIX="$($PY -c 'import sysconfig;print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYINC="$($PY -c 'import sysconfig;print(sysconfig.get_paths()["include"])')"
"$PY" -m cython -3 --module-name _kernels_cy "$SRC" -o "$OUT/_kernels_cy.c"
gcc -O3 -ffp-contract=off -shared -fPIC -I"$PYINC" "$OUT/_kernels_cy.c" -o "$OUT/_kernels_cy$EXT_SUFFIX"
echo "built $OUT/_kernels_cy$EXT_SUFFIX"

# A pristine copy of the reference package and its test suite (plus the lane
# just built) for the seam test: oracle/apply_seam.py applies INTEGRATION.md's
# stub to a scratch copy of it and the reference's own tests run on the B200
# through libtxb.so (tests/test_reference_seam.py).  /root/reference is absent
# on the GPU box; this copy travels with the snapshot (git-ignored).
REF_PKG="$(dirname "$(dirname "$(dirname "$SRC")")")"   # .../pkg
rm -rf "$OUT/txfem_pkg"
mkdir -p "$OUT/txfem_pkg/src"
cp -r "$REF_PKG/src/txfem" "$OUT/txfem_pkg/src/txfem"
cp -r "$REF_PKG/tests" "$OUT/txfem_pkg/tests"
rm -rf "$OUT/txfem_pkg/src/txfem/__pycache__" "$OUT/txfem_pkg/tests/__pycache__"
cp "$OUT/_kernels_cy$EXT_SUFFIX" "$OUT/txfem_pkg/src/txfem/"
echo "staged $OUT/txfem_pkg (reference package + tests)"
