"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel (share of device
time; cold-cache, serialised launches: compare SHARES, not absolutes)."""
import collections
import csv
import sys

src, dst, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(src)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
agg = collections.OrderedDict()
for r in data:
    if len(r) <= iv or not r[iv]:
        continue
    k = r[ik].split("(")[0]
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1e-6)
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
lines = ["# ncu --metrics gpu__time_duration.sum --clock-control none launch list of:", f"# {cmd}",
         "%-60s %8s %10s %7s" % ("kernel", "launches", "total_ms", "share")]
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    lines.append("%-60s %8d %10.3f %7.3f" % (k[:60], n, ms, ms / tot))
open(dst, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[:20]))
