#!/usr/bin/env bash
# Build the UNMODIFIED reference kernel set into oracle/_ref/ (git-ignored,
# travels to the GPU box with gpurun).  Test infrastructure only: the product
# never imports anything from here.
#
# Recipe (our own, the reference's setup.py/pip are NOT run):
#   1. copy the reference package sources /root/reference/pkg/src/superpix
#      into oracle/_ref/superpix (build output, never committed);
#   2. cython-translate kernels/_core.pyx with the directives of
#      pkg/setup.py:16-25 (language_level 3, boundscheck/wraparound/
#      initializedcheck off, cdivision on);
#   3. gcc it with the flags of pkg/setup.py:8-14 (-O3 -ffp-contract=off).
set -euo pipefail
REF=${SPX_REFERENCE:-/root/reference}
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
OUT="$HERE/_ref"
SRC="$REF/pkg/src/superpix"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC not present; keeping existing $OUT" >&2
  exit 0
fi
PY=${PYTHON:-python3}
SUFFIX=$("$PY" -c "import sysconfig; print(sysconfig.get_config_var('EXT_SUFFIX'))")
if [ -f "$OUT/superpix/kernels/_core$SUFFIX" ] && [ "$OUT/superpix/kernels/_core$SUFFIX" -nt "$SRC/kernels/_core.pyx" ] && [ "${FORCE:-0}" = "0" ]; then
  echo "build_ref: up to date" >&2
  exit 0
fi
rm -rf "$OUT"
mkdir -p "$OUT/build"
cp -r "$SRC" "$OUT/superpix"
find "$OUT/superpix" -name '__pycache__' -prune -exec rm -rf {} +
"$PY" -m cython -3 \
  -X boundscheck=False -X wraparound=False -X initializedcheck=False -X cdivision=True \
  -o "$OUT/build/_core.c" "$OUT/superpix/kernels/_core.pyx"
PYINC=$("$PY" -c "import sysconfig; print(sysconfig.get_paths()['include'])")
NPINC=$("$PY" -c "import numpy; print(numpy.get_include())")
gcc -shared -fPIC -O3 -ffp-contract=off -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
  -I"$PYINC" -I"$NPINC" "$OUT/build/_core.c" -o "$OUT/superpix/kernels/_core$SUFFIX" -lm
echo "build_ref: built $OUT/superpix/kernels/_core$SUFFIX"
