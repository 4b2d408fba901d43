#!/bin/bash
# round-2 evidence (final build, `r2c_*`): bench line, reference arm, every config's
# bench line, launch list, ncu --set full of one C2 sort.  Run on the GPU box:
#   gpurun -- bash tools/r2_profile.sh
P=gpurun_out/profiles; mkdir -p $P
python bench.py --steps 20 --warmup 5 > $P/r2c_bench.json 2> gpurun_out/r2c_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > $P/r2c_bench_reference.json 2> gpurun_out/r2c_ref.err
for c in c1 c3-zipf0.6 c3-zipf1.0 c3-zipf1.2 c3-zipf1.5 c4-exp1e-5 c4-exp1e-7 c4-bexp c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e > $P/r2c_bench_$c.json 2> gpurun_out/r2c_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $P/r2c_launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2c_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_histogram|k_scatter_wc|k_local_sort|k_sample_plan|k_classify" \
  -o gpurun_out/r2c_full python tools/prof_sort.py 1e9 > gpurun_out/r2c_full.log 2>&1
# the heavy-key variants on a skewed input: histogram + WC scatter (wide) of Zipf 1.5's first level
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_histogram|k_scatter_wc" -c 2 \
  -o gpurun_out/r2c_zipf15 python tools/prof_cfg.py c3-zipf1.5 1e9 0 > gpurun_out/r2c_zipf15.log 2>&1
ls -la gpurun_out $P
