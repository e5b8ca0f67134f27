#!/bin/sh
# Install the unmodified reference package (offsim, pure Python) into
# baseline/_ref (git-ignored; it travels to the GPU box with gpurun) for
# bench.py's python_reference leg.  Offline; the reference mount is
# read-only, so the build runs from a copy under /tmp.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/offsim_ref_copy
cp -r /root/reference/pkg /tmp/offsim_ref_copy
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse --no-deps \
    --target "$ROOT/baseline/_ref" /tmp/offsim_ref_copy
