"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.
Usage: python tools/launch_summary.py launches.csv"""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0]
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"].replace(",", "")) * scale[d["Metric Unit"]]
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k[:60]:60s} {v[0]:8d} {v[1]/1e3:10.3f} {v[1]/v[0]:10.1f} {v[1]/tot*100:5.1f}%")
print(f"{'total':60s} {sum(v[0] for v in agg.values()):8d} {tot/1e3:10.3f}")
