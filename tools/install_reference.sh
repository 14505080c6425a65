#!/usr/bin/env bash
# Test-only install of the reference package (vtrain 0.1.0) for the live
# drop-in test (tests/test_gpu_protocol_live.py) and the reference CPU legs
# of bench.py.  Run in the build container, where /root/reference exists; the
# result lives in baseline/_ref/ (git-ignored, never part of the product, not
# imported by paper_2403_09603_b200/), which gpurun ships to the GPU box.
#   baseline/_ref/vtrain/           the reference package, unmodified
#   baseline/_ref/vtrain_configs/   the reference's shipped run configs
set -euo pipefail
REPO="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg
TMP="$(mktemp -d)"
trap 'rm -rf "$TMP"' EXIT
cp -r "$SRC" "$TMP/pkg"   # the source tree is read-only; setuptools writes build files
rm -rf "$REPO/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
  --target "$REPO/baseline/_ref" "$TMP/pkg" >/dev/null
mkdir -p "$REPO/baseline/_ref/vtrain_configs"
cp "$SRC"/configs/*.json "$REPO/baseline/_ref/vtrain_configs/"
echo "installed vtrain into $REPO/baseline/_ref"
