"""Worker of tests/test_gpu_tp_fused.py: one of two processes on the SAME GPU.
Handles are exchanged over gloo; the fused reduce-scatter reduces into the
peer process's buffer through CUDA IPC; hxm_peer_barrier orders it."""
import os
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)


def run(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2411_01288_b200 as H
        from paper_2411_01288_b200 import dist as D
        from test_gpu_tp_fused import _problem, scaled
        p, x, r, gy = _problem(world)
        N, Dm = x.shape
        n_local = N // world
        ref = H.moe_forward(x, p, r)
        gref = H.moe_backward(ref.stash, p, gy)
        sp = D.shard_params(p, D.even_split(p.hidden(), world))
        sh = sp.shards[rank]
        prm = H.MoeLayerParams(sh.w1, sh.b1, sh.w2, sp.b2 if rank == 0 else None, "gelu")
        yb = D.PeerBuffers(n_local, Dm)
        gxb = D.PeerBuffers(n_local, Dm)
        errs = {}
        for it in range(2):  # twice: the epochs advance, buffers are re-zeroed
            yb.view().zero_()
            yb.barrier()
            st = D.layer_forward_tp(x, prm, r.to_device(), yb, rank == 0)
            yb.barrier()
            y = yb.view().clone()
            gxb.view().zero_()
            gxb.barrier()
            g = D.layer_backward_tp(st, prm, gy, gxb)
            gxb.barrier()
            gx = gxb.view().clone()
            torch.cuda.synchronize()
            lo = rank * n_local
            errs[f"y{it}"] = scaled(y, ref.y[lo:lo + n_local])
            errs[f"gx{it}"] = scaled(gx, gref.gx[lo:lo + n_local])
            off, h = sh.hidden_offset, sp.hidden_sizes[rank]
            errs[f"gw1_{it}"] = scaled(g.gw1, gref.gw1[:, :, off:off + h])
        dist.barrier()  # nobody closes its mappings while a peer still reduces
        yb.close()
        gxb.close()
        q.put((rank, errs))
    finally:
        dist.destroy_process_group()
