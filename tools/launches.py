"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list by kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("pf::", "").replace("(anonymous namespace)::", "")
    agg[name][0] += 1
    agg[name][1] += float(d["Metric Value"]) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
tot = sum(v[1] for v in agg.values())
print("%-45s %6s %12s %7s" % ("kernel", "calls", "total us", "share"))
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%-45s %6d %12.1f %6.1f%%" % (k[:45], v[0], v[1], 100 * v[1] / tot))
print("%-45s %6d %12.1f" % ("TOTAL", sum(v[0] for v in agg.values()), tot))
