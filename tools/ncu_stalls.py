"""Per-CUDA-line stall breakdown. Usage: python tools/ncu_stalls.py rep kernel_regex [N]"""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--kernel-name",f"regex:{kre}","--launch-count","1","--print-source","cuda,sass"],capture_output=True,text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None; fname='?'; agg = collections.defaultdict(lambda: collections.Counter()); text = {}; tot = collections.Counter()
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split('/')[-1]; continue
    if r[0] == "Function Name": continue
    if r[0] == "Line No": hdr = r; idx = {h: i for i, h in enumerate(hdr) if h.startswith('stall_') and '(Not' not in h}; continue
    if hdr is None or not r[0]: continue
    k = (fname, int(r[0])); text[k] = r[1].strip()
    for h, i in idx.items():
        try: v = float(r[i]); agg[k][h] += v; tot[h] += v
        except: pass
T = sum(tot.values())
print("overall:", ", ".join(f"{h[6:]}={v/T*100:.0f}%" for h, v in tot.most_common(8)))
for k, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:N]:
    s = sum(c.values())
    print(f"{s/T*100:5.1f}% {k[0]}:{k[1]:<4} {', '.join(f'{h[6:]}={v/s*100:.0f}' for h, v in c.most_common(3))}  | {text[k][:60]}")
