"""Per-CUDA-line shared-memory wavefronts (actual / ideal) from an ncu source page.
Usage: python tools/ncu_smem_lines.py rep kernel_regex records [N] [launch_skip]"""
import collections, csv, io, subprocess, sys
rep, kre, recs = sys.argv[1], sys.argv[2], float(sys.argv[3])
N = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
wf = collections.Counter(); ideal = collections.Counter(); text = {}; fname = "?"; hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0] == "File Path": fname = row[1].split("/")[-1]; continue
    if row[0] == "Function Name": continue
    if row[0] == "Line No": hdr = row; iw = hdr.index("L1 Wavefronts Shared"); ii = hdr.index("L1 Wavefronts Shared Ideal"); continue
    if hdr is None or not row[0] or len(row) < len(hdr): continue
    k = (fname, int(row[0])); text[k] = row[1].strip()
    try:
        wf[k] += float(row[iw]); ideal[k] += float(row[ii])
    except ValueError:
        pass
tw = sum(wf.values()); ti = sum(ideal.values())
print(f"total {tw/recs:.3f} wavefronts/record (ideal {ti/recs:.3f})")
for k, v in wf.most_common(N):
    print(f"{v/recs:6.3f}/rec (ideal {ideal[k]/recs:5.3f})  {k[0]}:{k[1]}  {text[k][:70]}")
