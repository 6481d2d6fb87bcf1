"""Summarise an ncu --set full report (raw page CSV) into a markdown table.

    ncu -i rep.ncu-rep --page raw --csv > raw.csv; python tools/ncu_summary.py raw.csv
"""
import csv
import sys

COLS = [
    ("us", "gpu__time_duration.sum", 1e-3),
    ("DRAM rd MB", "dram__bytes_read.sum", None),
    ("DRAM wr MB", "dram__bytes_write.sum", None),
    ("tensor %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L1 %", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("regs", "launch__registers_per_thread", 1),
]


def to_mb(v, unit):
    f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    return v * f


def main(path):
    r = list(csv.reader(open(path)))
    h, units = r[0], r[1]
    ix = {name: h.index(name) for _, name, _ in COLS if name in h}
    kn = h.index("Kernel Name")
    print("| kernel | " + " | ".join(c for c, _, _ in COLS) + " |")
    print("|---" * (len(COLS) + 1) + "|")
    for row in r[2:]:
        cells = []
        for label, name, scale in COLS:
            if name not in ix:
                cells.append("-")
                continue
            v = float(row[ix[name]].replace(",", "") or 0)
            u = units[ix[name]]
            if "MB" in label:
                v = to_mb(v, u)
            elif name == "gpu__time_duration.sum":
                v = v * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
            cells.append(f"{v:.1f}")
        name = row[kn].replace("(anonymous namespace)::", "").split("(")[0][:48]
        print(f"| `{name}` | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main(sys.argv[1])
