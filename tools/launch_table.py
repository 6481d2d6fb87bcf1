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
# the last complete step: between the last two fwd_prologue launches
starts = [i for i, d in enumerate(data) if "fwd_prologue" in d[0]]
lo, hi = (starts[-2], starts[-1]) if len(starts) >= 2 else (starts[-1] if starts else 0, len(data))
tot = 0.0
for name, ns, grid in data[lo:hi]:
    tot += ns
    print(f"{ns / 1000:8.1f} us  {grid:>14}  {name.replace('hxm::<unnamed>::', '')[:70]}")
print(f"{tot / 1000:8.1f} us  total")
