# A/B timing of two library builds on the same box: bash tools/ab.sh libA libB [rounds] [bench args]
A=$1; B=$2; R=${3:-3}; shift 3; 
for i in $(seq 1 $R); do
  for L in $A $B; do
    printf "%s " $L; DTS_LIB=paper_2401_00710_b200/_lib/$L python bench.py --steps 10 --warmup 3 "$@" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline']['step_share'];print(d['value'],d['ms_per_step'],'scatter',round(r['scatter']*d['ms_per_step'],3),'local',round(r['local_sort']*d['ms_per_step'],3))"
  done
done
