"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, total device time and share (cold-cache, serialised
times: shares are what to compare, not absolutes)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows:
    if r and r[0] == "ID":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr is None or len(r) < len(hdr) or r[hdr["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[hdr["Kernel Name"]]
    name = name.split("(")[0][:90]
    agg[name][0] += 1
    agg[name][1] += float(r[hdr["Metric Value"]].replace(",", "")) * scale.get(r[hdr["Metric Unit"]], 1.0)
tot = sum(v[1] for v in agg.values())
print(f"{'total device time (us)':>24}: {tot:.1f}   launches: {sum(v[0] for v in agg.values())}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t:12.1f} us {100 * t / tot:5.1f}%  n={n:5d}  {k}")
