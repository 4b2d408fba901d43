# A/B/... timing of several library builds on one box: bash tools/abn.sh rounds libA libB ... [-- bench args]
R=$1; shift; LIBS=(); while [ $# -gt 0 ] && [ "$1" != "--" ]; do LIBS+=("$1"); shift; done; [ "$1" = "--" ] && shift
for i in $(seq 1 $R); do
  for L in "${LIBS[@]}"; do
    printf "%s " $L; DTS_LIB=paper_2401_00710_b200/_lib/$L python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());r=d['roofline']['step_share'];print(d['value'],d['ms_per_step'],'scatter',round(r['scatter']*d['ms_per_step'],3),'local',round(r['local_sort']*d['ms_per_step'],3))"
  done
done
