"""Per-CUDA-line warp-instruction counts (normalised per record) and stall samples.
Usage: python tools/ncu_inst_lines.py rep kernel_regex records [N]"""
import csv, io, subprocess, sys, collections
rep, kre, recs = sys.argv[1], sys.argv[2], float(sys.argv[3])
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu","-i",rep,"--page","source","--csv","--kernel-name",f"regex:{kre}","--launch-count","1","--print-source","cuda,sass"],capture_output=True,text=True).stdout
inst=collections.Counter(); samp=collections.Counter(); text={}; fname='?'; hdr=None
for row in csv.reader(io.StringIO(out)):
    if not row: continue
    if row[0]=="File Path": fname=row[1].split('/')[-1]; continue
    if row[0]=="Function Name": continue
    if row[0]=="Line No": hdr=row; continue
    if hdr is None or len(row)<8: continue
    if row[0]:
        k=(fname,int(row[0])); text[k]=row[1].strip()
        try: inst[k]+=float(row[7]); samp[k]+=float(row[4])
        except: pass
ti=sum(inst.values()); ts=sum(samp.values())
print(f"total {ti/recs:.2f} warp-inst/record")
for k,v in sorted(inst.items(), key=lambda kv:-kv[1])[:N]:
    print(f"{v/recs:6.3f}/rec {samp[k]/ts*100:5.1f}%smp  {k[0]}:{k[1]} {text[k][:75]}")
