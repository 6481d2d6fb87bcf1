"""Bit-identity of the chained forward (HXM_CHAIN=1) against the two-kernel
forward (HXM_CHAIN=0): run `python tools/chain_check.py save <tag>` under each
setting (the switch is read once per process), then `compare a b`."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2411_01288_b200 as H  # noqa: E402

CASES = [
    # (E, k, D, Hd, N, act, dist, bias2)
    (32, 2, 384, 1536, 16384, "gelu", "uniform", True),
    (32, 2, 384, 1536, 1000, "gelu", "uniform", True),
    (8, 2, 384, 512, 3000, "relu", "uniform", False),
    (16, 2, 192, 256, 2500, "identity", "uniform", True),
    (64, 2, 384, 1536, 16384, "gelu", "skew90", True),
]


def run(tag):
    out = {}
    for ci, (E, k, D, Hd, N, act, dist, b2) in enumerate(CASES):
        p, x = H.make_random_params(E, D, Hd, D, act, seed=3 + ci, n_tokens=N)
        if not b2:
            p.b2 = None
        if dist == "skew90":
            from bench import skew90_routing
            r = skew90_routing(N, E, k, 5 + ci)
        else:
            r = H.synthesize_routing(N, E, k, dist, 5 + ci)
        fw = H.moe_forward(x, p, r)
        g = torch.randn(N, D, device="cuda", generator=torch.Generator("cuda").manual_seed(ci)).to(torch.bfloat16)
        gr = H.moe_backward(fw.stash, p, g)
        torch.cuda.synchronize()
        out[f"{ci}_y"] = fw.y.cpu()
        for c in range(k):
            d1, f1 = fw.stash.export(c)
            out[f"{ci}_dact{c}"] = d1.cpu()
            out[f"{ci}_fact{c}"] = f1.cpu()
        for nm in ("gw1", "gb1", "gw2", "gx"):
            out[f"{ci}_{nm}"] = getattr(gr, nm).cpu()
    os.makedirs("gpurun_out", exist_ok=True)
    torch.save(out, f"/tmp/chain_{tag}.pt")


def compare(a, b):
    A = torch.load(f"/tmp/chain_{a}.pt")
    B = torch.load(f"/tmp/chain_{b}.pt")
    bad = 0
    for key in A:
        x, y = A[key].float(), B[key].float()
        same = torch.equal(A[key], B[key])
        d = (x - y).abs().max().item() if x.numel() else 0.0
        print(f"{key:12s} {'bit-identical' if same else 'DIFF'} maxabs {d:.3e} "
              f"(max |ref| {x.abs().max().item() if x.numel() else 0:.3e})")
        bad += not same
    print("mismatching tensors:", bad)


if __name__ == "__main__":
    if sys.argv[1] == "save":
        run(sys.argv[2])
    else:
        compare(sys.argv[2], sys.argv[3])
