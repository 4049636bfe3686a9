#!/bin/bash
# Stage (copy) the reference package and its test suite into oracle/_ref/pkg
# (git-ignored) so that one gpurun call can run the reference's OWN tests
# against the GPU path (tests/test_gpu_dropin.py).  Never committed; remove
# with `tools/stage_reference.sh --clean` after the run.
set -e
cd "$(dirname "$0")/.."
rm -rf oracle/_ref/pkg
[ "$1" = "--clean" ] && exit 0
mkdir -p oracle/_ref/pkg
cp -r /root/reference/pkg/src oracle/_ref/pkg/src
cp -r /root/reference/pkg/tests oracle/_ref/pkg/tests
find oracle/_ref/pkg -name __pycache__ -prune -exec rm -rf {} \;
echo "staged $(find oracle/_ref/pkg -name '*.py' | wc -l) files"
