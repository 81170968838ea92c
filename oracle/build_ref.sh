#!/usr/bin/env bash
# Build the reference package (/root/reference/pkg, Python + one Cython file)
# into oracle/_ref with its compiled core, for the oracle pin and the CPU
# baseline.  The sources are copied to a scratch dir under /tmp (the
# reference tree is read-only and setup.py writes next to the sources);
# nothing from the reference is committed.  Output: oracle/_ref/trigbf/...
set -euo pipefail
HERE="$(cd "$(dirname "$0")" && pwd)"
SRC="${1:-/root/reference/pkg}"
if [ ! -d "$SRC" ]; then
  echo "reference not present at $SRC; skipping (prebuilt oracle/_ref is used if shipped)" >&2
  exit 0
fi
TMP="$(mktemp -d /tmp/trigbf_ref.XXXXXX)"
cp -r "$SRC" "$TMP/pkg"
chmod -R u+w "$TMP/pkg"
rm -rf "$HERE/_ref"
python -m pip install --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$HERE/_ref" "$TMP/pkg" >/dev/null
rm -rf "$TMP"
PYTHONPATH="$HERE/_ref" python -c "import trigbf; print('oracle/_ref trigbf backend:', trigbf.backend_name())"
