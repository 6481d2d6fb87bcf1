"""Worker for test_gpu_chain.py: one layer fwd + bwd under the chain switches
of the environment (read once per process), outputs saved to argv[1]."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_01288_b200 as H  # noqa: E402

CASES = [(32, 2, 384, 1536, 2500, "gelu", True), (8, 2, 384, 512, 900, "relu", False),
         (16, 2, 192, 256, 1300, "identity", True), (4, 1, 384, 384, 200, "gelu", True)]

out = {}
for ci, (E, k, D, Hd, N, act, b2) in enumerate(CASES):
    p, x = H.make_random_params(E, D, Hd, D, act, seed=20 + ci, n_tokens=N)
    if not b2:
        p.b2 = None
    r = H.synthesize_routing(N, E, k, "uniform", 30 + ci)
    fw = H.moe_forward(x, p, r)
    g = torch.randn(N, D, device="cuda",
                    generator=torch.Generator("cuda").manual_seed(ci)).to(torch.bfloat16)
    gr = H.moe_backward(fw.stash, p, g)
    out[f"{ci}_y"] = fw.y.cpu()
    for c in range(k):
        d1, f1 = fw.stash.export(c)
        out[f"{ci}_dact{c}"] = d1.cpu()
        out[f"{ci}_fact{c}"] = f1.cpu()
    for nm in ("gw1", "gb1", "gw2", "gx"):
        out[f"{ci}_{nm}"] = getattr(gr, nm).cpu()
torch.save(out, sys.argv[1])
