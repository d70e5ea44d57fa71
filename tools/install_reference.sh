#!/bin/bash
# Test-only install of the reference (stalltrace, pure Python) into baseline/_ref
# (git-ignored; travels to the GPU box with the snapshot).  Used ONLY by
# tests/test_ref_suite.py, which runs the reference's own test modules with the
# reference's analyzer functions re-pointed at paper_2604_20032_b200.api (the
# drop-in check of SURVEY §8(b)).  The product never imports it.
set -eu
cd "$(dirname "$0")/.."
REF=${1:-/root/reference/pkg}
rm -rf baseline/_ref
python -m pip install --no-index --no-build-isolation --find-links /opt/wheelhouse \
    --target baseline/_ref "$REF" > /dev/null
cp -r "$REF/tests" baseline/_ref/stalltrace_tests
echo "installed $(ls baseline/_ref | tr '\n' ' ')"
