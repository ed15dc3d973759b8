"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per-kernel
launches, total ms and share (cold-cache, serialised: compare shares, not absolutes).

    python tools/launch_summary.py LAUNCHES.csv "HEADER LINE" > OUT.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
order = []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"].replace(",", ""))
    u = d.get("Metric Unit", "")
    ms = v * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u, 1e-6)
    k = d["Kernel Name"]
    k = k[:k.index("(")] if "(" in k else k
    k = k.replace("void ", "").split("::")[-1] if "<" not in k.split("::")[-1] else k.replace("void ", "").split("::")[-1]
    if k not in agg:
        order.append(k)
    agg[k][0] += 1
    agg[k][1] += ms
tot = sum(v[1] for v in agg.values())
if len(sys.argv) > 2:
    print("# " + sys.argv[2])
print(f"# {sum(v[0] for v in agg.values())} launches, {tot:.3f} ms total")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{k:45s} launches={c:5d} total_ms={t:9.3f} share={t / tot:.3f}")
