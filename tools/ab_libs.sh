# A/B of library builds (and env settings) on one box:
#   bash tools/ab_libs.sh "<lib>[:ENV=V] ..." config...
for c in "${@:2}"; do
  for spec in $1; do
    L=${spec%%:*}; E=""; [ "$spec" != "$L" ] && E=${spec#*:}
    printf "%s %s %s " $c $L "$E"; env $E DTS_LIB=paper_2401_00710_b200/_lib/$L timeout 300 python bench.py --steps 5 --warmup 3 --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline']['step_share'];m=d['ms_per_step'];print(d['value'],m,'hist',round(r['histogram']*m,3),'scat',round(r['scatter']*m,3),'local',round(r['local_sort']*m,3),'copy',round(r['copy']*m,3))" 2>/dev/null || echo failed
  done
done
