# per-config comparison of two builds: bash tools/cfgs.sh libA libB cfg...
A=$1; B=$2; shift 2
for C in "$@"; do for L in $A $B; do
  printf "%-12s %-14s " $C $L; DTS_LIB=paper_2401_00710_b200/_lib/$L python bench.py --config $C --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline']['step_share'];print(d['value'],d['ms_per_step'],{k:round(v*d['ms_per_step'],2) for k,v in r.items() if v>0.005})"
done; done
