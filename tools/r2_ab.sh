#!/bin/bash
# correctness of the current build on the sort tests, then an A/B of builds
# usage: bash tools/r2_ab.sh "<libs>" "<configs>" [pytest -k expr]
K=${3:-"sort or sizes or variants"}
timeout 1200 python -m pytest -q -x tests/test_gpu_sort.py tests/test_gpu_sizes.py tests/test_gpu_variants.py -k "$K" > gpurun_out/ab_tests.log 2>&1
tail -3 gpurun_out/ab_tests.log
for i in 1 2; do bash tools/ab_libs.sh "$1" $2; done
