for L in 32 64 128 256; do
  echo "LBS=$L"; DTS_WC_LBS=$L python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'],d['ms_per_step'],d['roofline']['step_share']['scatter'])"
  DTS_WC_LBS=$L DTS_LIB=paper_2401_00710_b200/_lib/libdts_phase.so python tools/phase_prof.py | grep -E "stripe|tma|total"
done
