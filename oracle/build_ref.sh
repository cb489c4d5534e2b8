#!/usr/bin/env bash
# Build the reference (pivgen, /root/reference/pkg) into oracle/_ref -- test
# infrastructure only. The reference's own setup.py/Cython build is driven from
# a scratch copy (the reference tree is read-only); outputs land only in
# oracle/_ref (git-ignored, travels to the GPU box with the repo snapshot).
# Also builds oracle/_ref/philox_curand_check (NVIDIA curand Philox, host side).
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
REF="${REFERENCE_ROOT:-/root/reference}/pkg"
OUT="$HERE/_ref"
if [ ! -d "$REF" ]; then echo "reference not present at $REF; skipping" >&2; exit 0; fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$REF" "$TMP/pkg"
rm -f "$TMP/pkg/src/pivgen/_native.c"      # regenerate from _native.pyx
mkdir -p "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps --upgrade \
    --target "$OUT" "$TMP/pkg"
mkdir -p "$OUT/h5py"
echo '"""Empty stub: h5py is absent in this image; only pivgen.flowfield.load_hdf5 needs it."""' \
    > "$OUT/h5py/__init__.py"
nvcc -O2 -Wno-deprecated-gpu-targets -o "$OUT/philox_curand_check" "$HERE/philox_curand_check.cu"
PYTHONPATH="$OUT" python -c "import pivgen; assert pivgen.active_backend() == 'native', pivgen.active_backend(); print('oracle/_ref: pivgen', pivgen.__version__, pivgen.active_backend())"
