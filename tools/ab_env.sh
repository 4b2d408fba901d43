# env A/B on one box: VAR=name VALS="a b" bash tools/ab_env.sh config...
for c in "$@"; do
  for e in $VALS; do
    printf "%s %s=%s " $c $VAR $e; env $VAR=$e timeout 300 python bench.py --steps 5 --warmup 3 --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline']['step_share'];print(d['value'],d['ms_per_step'],'scatter',round(r['scatter']*d['ms_per_step'],3),'local',round(r['local_sort']*d['ms_per_step'],3),'hist',round(r['histogram']*d['ms_per_step'],3),'sample',round(r['sample']*d['ms_per_step'],3))"
  done
done
