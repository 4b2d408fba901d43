#!/bin/bash
# every BASELINE config through bench.py (5 timed steps, CPU oracle beside it),
# one JSON line each into profiles/r2_bench_<config>.json (via gpurun_out/)
mkdir -p gpurun_out/profiles
for c in c1 c3-zipf0.6 c3-zipf1.0 c3-zipf1.2 c3-zipf1.5 c4-exp1e-5 c4-exp1e-7 c4-bexp c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --cpu-budget 10 > gpurun_out/profiles/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err
  echo "$c $(python -c "import json;d=json.load(open('gpurun_out/profiles/r2_bench_$c.json'));print(d['value'],d['ms_per_step'],(d.get('pipeline_roofline') or {}).get('frac_of_peak'),d['cpu_baseline']['value'] if d.get('cpu_baseline') else None)")"
done
