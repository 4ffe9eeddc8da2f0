#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY -- builds the *unmodified* reference compiled core
# (`rodsim._core`, /root/reference/pkg/src/rodsim/_core.pyx) into oracle/_ref/
# so that tests/ and bench.py's CPU arm can run the reference's own step.
#
# Mirrors the reference build (pkg/setup.py:5-13): Cython -> C, then gcc with
# the interpreter's CFLAGS plus "-O3 -fno-math-errno" and no -march (so the
# object code has no FMA, which is what makes bitwise fp64 parity meaningful).
# Nothing is written outside oracle/_ref/.  The reference source is read in
# place; no reference file is copied into the repository.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${RODSIM_REF_SRC:-/root/reference/pkg/src/rodsim/_core.pyx}"
OUT="$HERE/_ref"
mkdir -p "$OUT"
if [ ! -f "$SRC" ]; then
    echo "build_ref: reference source $SRC not present; skipping" >&2
    exit 0
fi
PY="${PYTHON:-python}"
EXT_SUFFIX="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("EXT_SUFFIX"))')"
PYINC="$($PY -c 'import sysconfig; print(sysconfig.get_paths()["include"])')"
NPINC="$($PY -c 'import numpy; print(numpy.get_include())')"
CFLAGS="$($PY -c 'import sysconfig; print(sysconfig.get_config_var("CFLAGS"))')"
TARGET="$OUT/_core$EXT_SUFFIX"
if [ -f "$TARGET" ] && [ "$TARGET" -nt "$SRC" ] && [ "$TARGET" -nt "$0" ]; then
    exit 0
fi
cython -3 --module-name rodsim._core -o "$OUT/_core.c" "$SRC"
gcc $CFLAGS -fPIC -fwrapv -I"$PYINC" -I"$NPINC" \
    -DNPY_NO_DEPRECATED_API=NPY_1_7_API_VERSION \
    -O3 -fno-math-errno -shared "$OUT/_core.c" -o "$TARGET"
echo "build_ref: built $TARGET"
