"""Per-CTA timeline of one tcgen05 kernel (debug): HXM_TRACE=<label> python tools/trace_kernel.py"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2411_01288_b200 as H  # noqa: E402
from paper_2411_01288_b200 import _lib  # noqa: E402
from paper_2411_01288_b200.runner import LayerRunner  # noqa: E402

E, k, D, Hd, N = 32, 2, 384, 1536, 16384
dev = torch.device("cuda")
p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=1, n_tokens=N, dtype=torch.bfloat16, device=dev)
a = H.synthesize_routing(N, E, k, "uniform", 1).to_device(dev)
gy = torch.ones(N, D, dtype=torch.bfloat16, device=dev)
run = LayerRunner(p, N, k, dev, torch.bfloat16)
for _ in range(4):
    run.step(x, a, gy)
torch.cuda.synchronize()
L = _lib.lib()
buf = (ctypes.c_ulonglong * (148 * 64 * 8))()
L.hxm_debug_trace(buf)
t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 64, 8).astype(np.int64)
ts = t[:, :, :6]
if not (ts > 0).any():
    sys.exit("no trace recorded: build with -DHXM_TRACE_BUILD (python tools/trace_build.py)")
t0 = ts[ts > 0].min()
print("label", os.environ.get("HXM_TRACE"), "kernel span us", (ts[ts > 0].max() - t0) / 1e3)
for cta in (0, 2, 74):
    print(f"CTA {cta}: item  mma[wait_tempty->got, loop_end]   epi[wait_tfull->got, end]  (us from start)")
    for i in range(64):
        r = t[cta, i]
        if not r.any():
            break
        f = lambda v: (v - t0) / 1e3 if v else float("nan")  # noqa: E731
        print(f"  {i:2d}  mma {f(r[0]):7.2f} {f(r[1]):7.2f} {f(r[2]):7.2f}   epi {f(r[3]):7.2f} {f(r[4]):7.2f} {f(r[5]):7.2f}"
              f"   mma-waits-full {r[6] / 1965:6.2f}  producer-waits-empty {r[7] / 1965:6.2f}")
