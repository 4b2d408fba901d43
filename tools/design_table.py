"""Markdown table of the per-config bench lines: python tools/design_table.py profiles/r2c_bench"""
import json, sys
pre = sys.argv[1]
rows = [("C1 (10^6 keys, launch-bound)", "_c1"), ("C2 (headline, 20 steps)", ""), ("C3 Zipf 0.6", "_c3-zipf0.6"),
        ("C3 Zipf 1.0", "_c3-zipf1.0"), ("C3 Zipf 1.2", "_c3-zipf1.2"), ("C3 Zipf 1.5", "_c3-zipf1.5"),
        ("C4 exp 1e-5", "_c4-exp1e-5"), ("C4 exp 1e-7", "_c4-exp1e-7"), ("C4 bit-exp", "_c4-bexp"),
        ("C5 (2^32 R-MAT edges, one GPU)", "_c5")]
print("| config | Gkeys/s | ms | pipeline frac | CPU Gkeys/s |\n|---|---|---|---|---|")
for name, suf in rows:
    d = json.loads(open(f"{pre}{suf}.json").read().strip().splitlines()[-1])
    p = d.get("pipeline_roofline") or {}
    fr = p.get("frac_of_peak")
    frs = f"{100 * fr:.1f} %" if fr and suf not in ("_c1", "_c5") else "—"
    cpu = (d.get("cpu_baseline") or {}).get("value")
    print(f"| {name} | {d['value']:.2f} | {d['ms_per_step']:.2f} | {frs} | {cpu:.3f} |")
