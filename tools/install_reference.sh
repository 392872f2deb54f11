#!/bin/bash
# Offline install of the UNMODIFIED reference into baseline/_ref (git-ignored,
# travels to the GPU box): the reference arm of bench.py and the interop
# tests import sdnnbench from there. /root/reference is read-only, so the
# wheel is built from a copy under /tmp.
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/refcopy baseline/_ref
cp -r /root/reference /tmp/refcopy
python -m pip install --no-index --no-build-isolation --no-deps \
  --find-links /opt/wheelhouse --target baseline/_ref /tmp/refcopy/pkg
