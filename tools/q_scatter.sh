python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
python -c "import json;d=json.load(open('gpurun_out/bench2.json'));print(d['value'],d['ms_per_step'],d['roofline']['step_share'])"
DTS_LIB=paper_2401_00710_b200/_lib/libdts_phase.so python tools/phase_prof.py
