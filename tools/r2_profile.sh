#!/bin/bash
# round-2 evidence: bench line, reference arm, launch list, ncu --set full of one C2 sort
mkdir -p gpurun_out/profiles
python bench.py --steps 20 --warmup 5 > gpurun_out/profiles/r2_bench.json 2> gpurun_out/r2_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/profiles/r2_bench_reference.json 2> gpurun_out/r2_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/profiles/r2_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_histogram|k_scatter_wc|k_local_sort|k_sample_plan|k_classify" \
  -o gpurun_out/r2_full python tools/prof_sort.py 1e9 > gpurun_out/r2_full.log 2>&1
ls -la gpurun_out gpurun_out/profiles
