"""Run under compute-sanitizer by tests/test_gpu_sanitizer.py: one small
layer forward + backward on each device path (bf16 tcgen05 CTA pairs, the
whole-tile d 384 kernels -- and, with HXM_CHAIN=1 / HXM_CHAIN_BWD=1 in the
environment, the chained kernels -- bf16 single-CTA tiles, fp32 SIMT) and
the operator API, so memcheck / racecheck / synccheck see every kernel
family of the library."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2411_01288_b200 as H  # noqa: E402


def layer(E, k, D, Hd, N, dtype):
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=3, n_tokens=N, dtype=dtype)
    r = H.synthesize_routing(N, E, k, "uniform", 5)
    gy = torch.randn(N, D, generator=torch.Generator().manual_seed(2)).to("cuda", dtype)
    fw = H.moe_forward(x, p, r)
    g = H.moe_backward(fw.stash, p, gy)
    torch.cuda.synchronize()
    assert torch.isfinite(fw.y).all() and torch.isfinite(g.gx).all()


def ops(dtype):
    E, N, d1, d2 = 4, 200, 128, 64
    r = H.synthesize_routing(N, E, 1, "uniform", 7)
    rx = H.build_reindex(r.assignments[0], E, 8)
    gen = torch.Generator().manual_seed(1)
    x = torch.randn(N, d1, generator=gen).to("cuda", dtype)
    g = torch.randn(N, d2, generator=gen).to("cuda", dtype)
    w = torch.randn(E, d1, d2, generator=gen).to("cuda", dtype)
    H.esmm(x, w, None, rx)
    H.ess(g, rx)
    H.estmm(x, g, rx)
    H.esfk(x, g, w, rx, w_transposed=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    torch.cuda.set_device(0)
    layer(8, 2, 128, 256, 300, torch.bfloat16)   # CTA-pair tcgen05 path
    layer(6, 2, 384, 512, 300, torch.bfloat16)   # whole-tile fwd2 / gx / gW2 / gW1 (d 384)
    layer(4, 2, 64, 192, 150, torch.bfloat16)    # single-CTA / fallback tiles
    layer(4, 1, 96, 384, 200, torch.float32)     # fp32 SIMT path
    ops(torch.bfloat16)
    ops(torch.float32)
    print("sanitize worker: ok")
