"""Stall-reason totals and top instructions of one kernel from an ncu source-page CSV.

    ncu -i rep --page source --csv --launch-skip S --launch-count 1 > src.csv
    python tools/stalls.py src.csv [top]
"""
import csv
import sys

r = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
print(r[0][1][:100])
h = r[1]
rows = [x for x in r[2:] if len(x) == len(h)]
seen, u = set(), []
for x in rows:
    if x[0] in seen:
        continue
    seen.add(x[0])
    u.append(x)
f = lambda v: int(v) if v.strip().isdigit() else 0  # noqa: E731
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = {c: sum(f(x[h.index(c)]) for x in u) for c in reasons}
allS = sum(tot.values())
print("samples", allS)
for c, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {c:24s} {v:7d} {100.0 * v / max(allS, 1):5.1f}%")
si = h.index("Warp Stall Sampling (All Samples)")
ei = h.index("Instructions Executed")
idx = {x[0]: i for i, x in enumerate(u)}
for x in sorted(u, key=lambda x: -f(x[si]))[:top]:
    i = idx[x[0]]
    why = max(reasons, key=lambda c: f(x[h.index(c)]))
    print(f"{x[si]:>6} {x[ei]:>8} {x[0][-5:]} {why[6:]:12s} {x[1][:70]:70s} <= {u[i - 1][1][:40]}")
