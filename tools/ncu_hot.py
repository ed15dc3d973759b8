"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`
output, with the dominant stall reasons of each.  Usage: python tools/ncu_hot.py src.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    data.append((s, r))
tot = sum(s for s, _ in data)
print(f"total samples {tot}")
for pos, (s, r) in enumerate(data):
    r.append(str(pos))
for s, r in sorted(data, key=lambda x: -x[0])[:top]:
    st = sorted(((int(r[ix[c]]) if r[ix[c]].isdigit() else 0, c[6:]) for c in stall_cols), reverse=True)[:3]
    print(f"{s:7d} {100.0 * s / tot:5.1f}% #{r[-1]:>5} {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in st if v))
