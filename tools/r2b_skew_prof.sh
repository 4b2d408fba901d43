#!/bin/bash
# ncu --set full of the level-0/1 histogram and scatter launches of the skewed configs
for c in c3-zipf1.0 c3-zipf1.5; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_histogram|k_scatter" -c 4 \
    -o gpurun_out/skew_$c python tools/prof_cfg.py $c > gpurun_out/skew_$c.log 2>&1
  echo "$c rc=$?"
done
ls -la gpurun_out
