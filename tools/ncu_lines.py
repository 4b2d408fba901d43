"""Per-CUDA-source-line instruction / stall totals from an ncu report
(--print-source cuda,sass).  Usage: python tools/ncu_lines.py rep kernel_regex [N]"""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
inst = collections.Counter(); samp = collections.Counter(); text = {}
fname = "?"; hdr = None; seen_fn = set()
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]; continue
    if row[0] == "Function Name":
        continue
    if row[0] == "Line No":
        hdr = row; iS = 4; iI = 7; continue
    if hdr is None or len(row) < 8: continue
    if row[0]:
        key = (fname, int(row[0])); text[key] = row[1].strip()
        try:
            inst[key] += float(row[iI]); samp[key] += float(row[iS])
        except ValueError:
            pass
ti = sum(inst.values()); ts = sum(samp.values())
print(f"total inst {ti:.3e}  samples {ts:.0f}")
for key, v in sorted(samp.items(), key=lambda kv: -kv[1])[:N]:
    print(f"{v/ts*100:5.1f}% samp {inst[key]/ti*100:5.1f}% inst  {key[0]}:{key[1]}  {text[key][:80]}")
