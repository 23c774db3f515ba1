#!/bin/bash
# Install the UNMODIFIED reference (fzpipe, /root/reference/pkg) into
# baseline/_ref (git-ignored; travels to the GPU box with gpurun), plus a copy
# of its own test suite under baseline/_ref/fzpipe_tests so the drop-in test
# (tests/test_dropin.py) can run the reference's tests with the B200 plugin
# installed.  The build writes into the source tree, so it installs from a
# /tmp copy; dependencies (numpy, numba, scipy) are already in the image.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
rm -rf /tmp/fzpipe_src && cp -r /root/reference/pkg /tmp/fzpipe_src
python -m pip install --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target "$ROOT/baseline/_ref" --upgrade /tmp/fzpipe_src
rm -rf "$ROOT/baseline/_ref/fzpipe_tests" && cp -r /tmp/fzpipe_src/tests "$ROOT/baseline/_ref/fzpipe_tests"
echo "fzpipe installed in $ROOT/baseline/_ref"
