#!/usr/bin/env bash
# TEST INFRASTRUCTURE ONLY. Builds the UNMODIFIED reference package (drrtrace:
# numpy + one Cython extension, /root/reference/pkg) into oracle/_ref/ so the
# parity tests and bench.py's CPU-baseline / --impl reference leg can import it.
# Nothing is copied into git: oracle/_ref/ is git-ignored but travels to the
# GPU box with the gpurun snapshot. The build runs from a scratch copy because
# /root/reference is read-only.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
OUT="$HERE/_ref"
if [ ! -d "$SRC" ]; then
  echo "build_ref: $SRC not present (GPU box?) - using prebuilt $OUT" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/drrref.XXXXXX)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$OUT"
python -m pip install --no-index --no-build-isolation --no-deps --quiet \
  --target "$OUT" "$TMP/pkg"
# the reference's own test files, so tests/test_gpu_reference_suite.py can run
# them against the "cuda" backend on the GPU box (not committed: _ref/ is ignored)
cp -r "$SRC/tests" "$OUT/tests"
python - "$OUT" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import drrtrace
from drrtrace._kernels import available_backends
assert "native" in available_backends(), available_backends()
print("oracle/_ref: drrtrace", drrtrace.__version__, "backends", available_backends())
PY
