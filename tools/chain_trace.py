"""Per-CTA wait totals of the chained layer GEMMs (HXM_CHAIN_TRACE=1):
HXM_CHAIN_TRACE=1 python tools/chain_trace.py [E k D H N]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.getcwd())
import paper_2411_01288_b200 as H  # noqa: E402
from paper_2411_01288_b200 import _lib  # noqa: E402
from paper_2411_01288_b200.runner import LayerRunner  # noqa: E402

E, k, D, Hd, N = (int(v) for v in sys.argv[1:6]) if len(sys.argv) > 5 else (32, 2, 384, 1536, 16384)
dev = torch.device("cuda")
p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=1, n_tokens=N, dtype=torch.bfloat16, device=dev)
a = H.synthesize_routing(N, E, k, "uniform", 1).to_device(dev)
gy = torch.ones(N, D, dtype=torch.bfloat16, device=dev)
run = LayerRunner(p, N, k, dev, torch.bfloat16)
for _ in range(4):
    run.step(x, a, gy)
torch.cuda.synchronize()
L = _lib.lib()
names = ["mma:acc1_empty", "mma:full(G1)", "mma:f_full", "mma:full(G2)", "mma:acc2_empty",
         "mma:a1full", "prod:empty", "prod:a1empty", "epi:acc1_full", "epi:math", "epi:B1",
         "epi:f_empty", "epi:Fwrite+B2", "epi:acc2_full", "epi:y-epilogue", "total", "epi:loop-top"]
for bwd in (0, 1):
    buf = (ctypes.c_ulonglong * (148 * 20))()
    if L.hxm_debug_chain_trace(bwd, buf, 148) != 0:
        print("no trace for", "bwd" if bwd else "fwd")
        continue
    t = np.frombuffer(buf, dtype=np.uint64).reshape(148, 20).astype(np.float64) / 1965.0
    print("== chain", "bwd" if bwd else "fwd", "(us, mean / max over CTAs; leader-only MMA slots use even CTAs)")
    for i, nm in enumerate(names):
        col = t[0::2, i] if i < 6 else t[:, i]
        print(f"  {nm:16s} {col.mean():8.2f} {col.max():8.2f}")
