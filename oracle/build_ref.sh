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
