"""Summarise bench.py JSON lines (stdin) into a per-kernel table (experiments)."""
import json
import sys

for line in sys.stdin:
    if not line.startswith("{"):
        continue
    d = json.loads(line)
    if "kernels" not in d:
        print(line.strip())
        continue
    c = d.get("clocks", {})
    print("ms %.3f (profiled %s) tok/s %.2fM e2e %.2fM sm %s/%s %s" % (
        d["ms_per_step"], d.get("ms_per_step_profiled"), d["value"] / 1e6,
        d["e2e"]["value"] / 1e6, c.get("sm_mhz"), c.get("sm_max_mhz"), c.get("reasons")))
    for k, v in d["kernels"].items():
        extra = ""
        if "tflops" in v and "gbs" in v:
            extra = " (%.0f TF/s %.2f | %.0f GB/s %.2f)" % (v["tflops"], v["frac_tensor"], v["gbs"], v["frac_hbm"])
        print("  %-14s %7.1f us %7.1f %s %.2f %s%s" % (k, v["avg_us"], v["achieved"], v["unit"],
                                                   v["frac"], v.get("bound", ""), extra))
