#!/usr/bin/env bash
# Install the UNMODIFIED reference package (dicmine, /root/reference/pkg) into
# baseline/_ref/ (git-ignored; gpurun ships it to the GPU box), for the
# Option B integration test (tests/test_gpu_integration_ref.py).  The source
# tree is read-only, so the build runs from a copy; numpy / scikit-learn are
# already installed, hence --no-deps.
set -euo pipefail
cd "$(dirname "$0")/.."
tmp=$(mktemp -d)
cp -r /root/reference/pkg "$tmp/"
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref "$tmp/pkg"
rm -rf "$tmp"
