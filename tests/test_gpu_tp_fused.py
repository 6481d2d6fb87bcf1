"""Fused GEMM -> reduce-scatter over peer memory (model-centric TP along H):
the ESMM epilogues reduce y / g_x rows straight into the token owners'
buffers (hxm_moe_forward_tp / hxm_moe_backward_tp).  Checked against the
single-GPU layer (same device kernels, different fp32 summation order):
simulated ranks in one process, and two real processes on one GPU exchanging
CUDA IPC handles (gloo for the handle exchange, the device barrier over peer
flags)."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def scaled(a, b):
    a = a.detach().double().cpu().numpy()
    b = b.detach().double().cpu().numpy()
    return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b))))


def _problem(P, seed=3):
    import paper_2411_01288_b200 as H
    E, k, D, Hd, N = 8, 2, 128, 256 * P, 256 * P
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=seed, n_tokens=N)
    r = H.synthesize_routing(N, E, k, "uniform", seed + 1)
    gy = torch.randn(N, D, generator=torch.Generator().manual_seed(seed + 2)).to(
        "cuda", torch.bfloat16)
    return p, x, r, gy


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
@pytest.mark.parametrize("P", [1, 2, 4])
def test_fused_reduce_scatter_simulated_ranks(P):
    import paper_2411_01288_b200 as H
    from paper_2411_01288_b200 import dist as D
    p, x, r, gy = _problem(P)
    N, Dm = x.shape
    ref = H.moe_forward(x, p, r)
    gref = H.moe_backward(ref.stash, p, gy)
    sp = D.shard_params(p, D.even_split(p.hidden(), P))
    ybufs = [torch.zeros(N // P, Dm, device="cuda") for _ in range(P)]
    gxbufs = [torch.zeros(N // P, Dm, device="cuda") for _ in range(P)]
    yb, gxb = D.PeerBuffers.local(ybufs), D.PeerBuffers.local(gxbufs)
    a = r.to_device()
    errs = {}
    for rr in range(P):
        sh = sp.shards[rr]
        prm = H.MoeLayerParams(sh.w1, sh.b1, sh.w2, sp.b2 if rr == 0 else None, "gelu")
        st = D.layer_forward_tp(x, prm, a, yb, rr == 0)
        g = D.layer_backward_tp(st, prm, gy, gxb)
        off, h = sh.hidden_offset, sp.hidden_sizes[rr]
        errs[f"gw1_{rr}"] = scaled(g.gw1, gref.gw1[:, :, off:off + h])
        errs[f"gw2_{rr}"] = scaled(g.gw2, gref.gw2[:, off:off + h, :])
        errs[f"gb1_{rr}"] = scaled(g.gb1, gref.gb1[:, off:off + h])
        if rr == 0:
            errs["gb2"] = scaled(g.gb2, gref.gb2)
    torch.cuda.synchronize()
    errs["y"] = scaled(torch.cat(ybufs), ref.y)
    errs["gx"] = scaled(torch.cat(gxbufs), gref.gx)
    bad = {k: v for k, v in errs.items() if not v <= 1e-3}
    assert not bad, bad


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
def test_fused_tp_rejects_bad_peer_tables():
    import paper_2411_01288_b200 as H
    from paper_2411_01288_b200 import dist as D
    p, x, r, _ = _problem(1)
    yb = D.PeerBuffers.local([torch.zeros(8, x.shape[1], device="cuda")])  # too few rows
    with pytest.raises(ValueError):
        D.layer_forward_tp(x, p, r.to_device(), yb, True)
    p32, x32 = H.make_random_params(4, 64, 128, 64, "gelu", seed=1, n_tokens=64,
                                    dtype=torch.float32)
    yb = D.PeerBuffers.local([torch.zeros(64, 64, device="cuda")])
    with pytest.raises(ValueError):  # fp32 layers have no tcgen05 path
        D.layer_forward_tp(x32, p32, H.synthesize_routing(64, 4, 2, "uniform", 1).to_device(),
                           yb, True, dtype=torch.float32)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
def test_fused_reduce_scatter_two_processes_ipc():
    import torch.multiprocessing as mp
    import _gpu_ipc_worker as W
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=W.run, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = {}
    for _ in range(2):
        rank, errs = q.get(timeout=300)
        out[rank] = errs
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    for rank, errs in out.items():
        bad = {k: v for k, v in errs.items() if not v <= 1e-3}
        assert not bad, (rank, bad)


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
@pytest.mark.parametrize("P,Dm", [(1, 128), (2, 128), (4, 128), (2, 384), (3, 384)])
def test_fused_grad_reduce_scatter_simulated_ranks(P, Dm):
    """Data-centric: each simulated rank runs the full layer on its own tokens
    and reduces gW1 / gW2 into the H-shard owners' buffers; the shards must
    equal the H-slices of the summed single-GPU gradients.  Dm = 384: the
    whole-tile ESTMM kernels (gW2 rows and the transposed gW1 reduced into the
    owners' H spans)."""
    import paper_2411_01288_b200 as H
    from paper_2411_01288_b200 import dist as D
    E, k, Hd, n = 8, 2, 256 * P, 256
    p, _ = H.make_random_params(E, Dm, Hd, Dm, "gelu", seed=9, n_tokens=0)
    span = Hd // P
    gw1s = [torch.zeros(E, Dm, span, device="cuda") for _ in range(P)]
    gw2s = [torch.zeros(E, span, Dm, device="cuda") for _ in range(P)]
    b1 = D.PeerBuffers.local(gw1s, span=span)
    b2 = D.PeerBuffers.local(gw2s, span=span)
    tot_w1 = torch.zeros(E, Dm, Hd, device="cuda")
    tot_w2 = torch.zeros(E, Hd, Dm, device="cuda")
    for rr in range(P):
        _, x = H.make_random_params(E, Dm, Hd, Dm, "gelu", seed=100 + rr, n_tokens=n)
        r = H.synthesize_routing(n, E, k, "uniform", 200 + rr)
        gy = torch.randn(n, Dm, generator=torch.Generator().manual_seed(rr)).to("cuda",
                                                                             torch.bfloat16)
        fw = H.moe_forward(x, p, r)
        g = H.moe_backward(fw.stash, p, gy)
        tot_w1 += g.gw1
        tot_w2 += g.gw2
        fw2 = H.moe_forward(x, p, r)
        gb1, gb2, gx = D.layer_backward_dc(fw2.stash, p, gy, b1, b2)
        assert scaled(gb1, g.gb1) <= 1e-5 and scaled(gx, g.gx) <= 1e-5
    torch.cuda.synchronize()
    for rr in range(P):
        sl = slice(rr * span, (rr + 1) * span)
        assert scaled(gw1s[rr], tot_w1[:, :, sl]) <= 1e-4, rr
        assert scaled(gw2s[rr], tot_w2[:, sl, :]) <= 1e-4, rr
