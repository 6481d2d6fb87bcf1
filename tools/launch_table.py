"""Per-launch durations of the last bench step from an ncu --csv launch list."""
import csv
import io
import sys

txt = open(sys.argv[1]).read().splitlines()
start = [i for i, l in enumerate(txt) if l.startswith('"ID"')][0]
rows = list(csv.reader(io.StringIO("\n".join(txt[start:]))))
h = rows[0]
ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
data = [(r[ki], float(r[vi].replace(",", "")), r[gi]) for r in rows[1:] if len(r) == len(h)]
# the last step: from the last fwd_prologue launch on
last = max(i for i, d in enumerate(data) if "prologue" in d[0] and "fwd" in d[0]) if any(
    "fwd_prologue" in d[0] for d in data) else 0
tot = 0.0
for name, ns, grid in data[last:]:
    tot += ns
    print(f"{ns / 1000:8.1f} us  {grid:>14}  {name.replace('hxm::<unnamed>::', '')[:70]}")
print(f"{tot / 1000:8.1f} us  total")
