#!/usr/bin/env bash
# Build the UNMODIFIED reference package (arxiv 2508.10395, `xcache`) into
# oracle/_ref -- test/baseline infrastructure only (see oracle/xq_oracle.py).
#
# The reference tree is read-only, so its pkg/ is copied to a scratch dir under
# /tmp, its own setup.py builds the Cython lane (_native.pyx, -O3
# -ffp-contract=off, setup.py:36-44), and pip installs the result into
# oracle/_ref. Nothing is written anywhere else; oracle/_ref is git-ignored but
# travels to the GPU box with gpurun, where bench.py --impl reference runs it.
set -euo pipefail
HERE="$(cd "$(dirname "${BASH_SOURCE[0]}")" && pwd)"
REF="${XQ_REFERENCE:-/root/reference}"
OUT="$HERE/_ref"
if [ ! -d "$REF/pkg" ]; then
  echo "build_ref: $REF/pkg not present; skipping (prebuilt oracle/_ref is used if it exists)" >&2
  exit 0
fi
SCRATCH="$(mktemp -d /tmp/xq_refbuild.XXXXXX)"
trap 'rm -rf "$SCRATCH"' EXIT
cp -r "$REF/pkg" "$SCRATCH/pkg"
rm -rf "$OUT"
python -m pip install --quiet --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target "$OUT" "$SCRATCH/pkg"
PYTHONPATH="$OUT" python -c "import xcache; assert xcache.kernel_backend()=='native', xcache.kernel_backend(); print('oracle/_ref: xcache', xcache.__version__, 'lane', xcache.kernel_backend())"
