#!/bin/bash
# round-2 baseline: bench line + source-level ncu of the scatter and local sort
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/base_bench.json 2> gpurun_out/base_bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_scatter_wc -c 1 -o gpurun_out/base_scatter python tools/prof_sort.py 1e9 > gpurun_out/ncu_sc.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_local_sort -s 1 -c 1 -o gpurun_out/base_local python tools/prof_sort.py 1e9 > gpurun_out/ncu_lo.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_histogram -c 1 -o gpurun_out/base_hist python tools/prof_sort.py 1e9 > gpurun_out/ncu_hi.log 2>&1
ls -la gpurun_out
