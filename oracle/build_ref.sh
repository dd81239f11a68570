#!/usr/bin/env bash
# Build recipe for oracle/_ref: the UNMODIFIED reference package (toepsolve, pure Python over
# numpy / scipy) installed from /root/reference/pkg into oracle/_ref, so that it travels to the GPU
# box with the repo snapshot (oracle/_ref is git-ignored, not gpurun-ignored).  The reference is not
# compiled code; "building" it is a no-deps, offline pip install of its own sources (copied to /tmp
# first because setuptools writes egg-info next to the sources and /root/reference is read-only).
# Used only as the checker / CPU baseline: bench.py --impl reference and cpu_baseline.
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
if [ ! -f "$SRC/pyproject.toml" ]; then
  echo "build_ref: $SRC not present (GPU box): using the prebuilt oracle/_ref" >&2
  exit 0
fi
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$HERE/_ref" "$TMP/pkg"
python - "$HERE/_ref" <<'PY'
import sys
sys.path.insert(0, sys.argv[1])
import toepsolve.toeplitz  # noqa: F401  (import check)
print("oracle/_ref:", toepsolve.__file__)
PY
