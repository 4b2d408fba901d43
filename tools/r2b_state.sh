#!/bin/bash
# round 2, session 2: state check on a fresh box — GPU tests, C2 bench line,
# per-launch timelines of C2 and the skewed configs
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/gputests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; cat gpurun_out/bench_c2.json | cut -c1-400
for c in c2 c3-zipf1.0 c3-zipf1.5 c4-bexp; do
  DTS_TIMELINE=1 DTS_TRACE=1 timeout 300 python tools/timeline.py 1e9 $c > gpurun_out/tl_$c.log 2>&1
done
ls gpurun_out
