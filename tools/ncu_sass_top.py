"""Summarise an ncu SASS source page: top instructions by stall samples and
instruction mix.  Usage: python tools/ncu_sass_top.py rep.ncu-rep kernel_regex [N]"""
import csv, subprocess, sys, collections, io
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
# first line is kernel name header; may contain multiple kernels (launch-count)
rows = list(csv.reader(io.StringIO("\n".join(l for l in lines if not l.startswith('"Kernel Name"')))))
hdr = rows[0]
data = [r for r in rows[1:] if len(r) == len(hdr) and r[0] != "Address"]
iS = hdr.index("Warp Stall Sampling (All Samples)"); iI = hdr.index("Instructions Executed"); iSrc = hdr.index("Source")
tot_s = sum(float(r[iS] or 0) for r in data); tot_i = sum(float(r[iI] or 0) for r in data)
print(f"instructions={tot_i:.3e} samples={tot_s:.0f}")
mix = collections.Counter()
for r in data:
    op = r[iSrc].strip().split()[0] if r[iSrc].strip() else "?"
    if op.startswith("@"): op = r[iSrc].strip().split()[1]
    mix[op.split(".")[0]] += float(r[iI] or 0)
print("mix:", ", ".join(f"{k}:{v/tot_i*100:.1f}%" for k, v in mix.most_common(18)))
top = sorted(data, key=lambda r: -float(r[iS] or 0))[:N]
for r in top:
    print(f"{float(r[iS] or 0)/tot_s*100:5.1f}%  {r[0][-5:]}  {r[iSrc].strip()[:90]}")
