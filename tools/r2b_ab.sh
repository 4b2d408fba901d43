#!/bin/bash
# A/B of the working library against libdts_base.so on one box:
#   bash tools/r2b_ab.sh "<configs>" [tests]
# (GPU tests first when a second argument is given)
if [ -n "$2" ]; then
  timeout 900 python -m pytest -m gpu -x -q $2 > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/ab_tests.log
fi
for pass in 1 2; do
  bash tools/ab_libs.sh "libdts_base.so libdts.so" $1
done
