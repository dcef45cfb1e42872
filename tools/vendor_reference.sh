#!/bin/bash
# Install the UNMODIFIED reference into baseline/_ref (git-ignored; gpurun
# ships it to the GPU box) and copy its test suite next to it.  Run in the
# build container, where /root/reference exists.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=${1:-/root/reference/pkg}
TMP=$(mktemp -d)
cp -r "$SRC" "$TMP/pkg"            # the build writes into the source tree; /root/reference is read-only
rm -rf "$ROOT/baseline/_ref"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" "$TMP/pkg" > "$TMP/pip.log" 2>&1 || { cat "$TMP/pip.log"; exit 1; }
cp -r "$SRC/tests" "$ROOT/baseline/_ref/tests"
rm -rf "$TMP"
echo "reference installed in $ROOT/baseline/_ref"
