#!/usr/bin/env bash
# Install the UNMODIFIED reference package (pbpqlp) into baseline/_ref — the
# task's one offline install — and stage its own test suite beside it, so the
# GPU box (which has no /root/reference) can run the reference's tests
# through integration.install (tests/test_gpu_reference_suite.py) and the
# stock CPU path for bench.py's reference arm.  baseline/_ref is git-ignored
# (never committed) and travels to the box with gpurun's snapshot.
#
#   bash tools/install_reference.sh            (in the build container)
set -euo pipefail
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${REFERENCE_PKG:-/root/reference/pkg}
[ -d "$SRC" ] || { echo "reference not present at $SRC" >&2; exit 1; }
TMP=$(mktemp -d)
trap 'rm -rf "$TMP"' EXIT
# the build writes egg-info into the source tree, which is read-only: build a copy
cp -r "$SRC" "$TMP/pkg"
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
  --target "$ROOT/baseline/_ref" --no-deps "$TMP/pkg" >/dev/null
mkdir -p "$ROOT/baseline/_ref/_reference_tests"
cp "$SRC"/tests/*.py "$ROOT/baseline/_ref/_reference_tests/"
python - "$ROOT" <<'PY'
import sys, os
sys.path.insert(0, os.path.join(sys.argv[1], "baseline", "_ref"))
import pbpqlp, numpy
print(f"installed pbpqlp {pbpqlp.__version__} from {pbpqlp.__file__} (numpy {numpy.__version__})")
PY
