"""Worker for tests/test_dist_gloo.py: one process per rank over gloo.

Checks the TP choreography of paper_2411_01288_b200.dist (sharding, b2
ownership, which tensors are gathered / reduced) against the single-device
result, in the spirit of the reference's test_dist_sim.cpp:176-259 and
acceptance criterion 8.  The per-rank local layer math is the fp64 CPU oracle
(test infrastructure); the collectives are real torch.distributed calls.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


class _G:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def oracle_compute():
    import oracle as O
    from paper_2411_01288_b200.dist import LocalCompute

    def fwd(x, p, a, add_b2):
        b2 = p.b2 if (add_b2 and p.b2 is not None) else torch.zeros(p.w2.shape[0], p.w2.shape[2],
                                                                   dtype=torch.float64)
        a = a.numpy()
        y, y1, y2 = O.moe_forward(x.numpy(), p.w1.numpy(), p.b1.numpy(), p.w2.numpy(),
                                  b2.numpy(), a, 4, p.activation)
        return torch.from_numpy(y), (x, a, y1, y2)

    def bwd(stash, p, gy):
        x, a, y1, y2 = stash
        g = O.moe_backward(x.numpy(), p.w1.numpy(), p.w2.numpy(), a, y1, y2, gy.numpy(), 4,
                           p.activation)
        return _G(**{k: torch.from_numpy(v) for k, v in g.items()})

    return LocalCompute(fwd, bwd)


def problem(seed, n_tokens, E=4, din=5, hid=12, dout=5, k=2):
    import oracle as O
    from paper_2411_01288_b200.moe_layer import MoeLayerParams
    x, w1, b1, w2, b2 = O.ref_make_inputs(seed, E, din, hid, dout, n_tokens) \
        if O.ref_available() else _np_inputs(seed, E, din, hid, dout, n_tokens)
    a = O.synthesize_routing(n_tokens, E, k, "uniform", seed + 1)
    gy = np.random.default_rng(seed).standard_normal((n_tokens, dout))
    t = torch.from_numpy
    p = MoeLayerParams(t(w1), t(b1), t(w2), t(b2), "gelu")
    return p, t(x), t(a), t(gy)


def _np_inputs(seed, E, din, hid, dout, n):
    r = np.random.default_rng(seed)
    return (r.standard_normal((n, din)), 0.5 * r.standard_normal((E, din, hid)),
            0.5 * r.standard_normal((E, hid)), 0.5 * r.standard_normal((E, hid, dout)),
            0.5 * r.standard_normal((E, dout)))


def scaled(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b)))) if b.size else 0.0


def run(rank, world, port, batches, hidden_alloc, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_01288_b200 import dist as D
        comp = oracle_compute()
        total = sum(batches)
        p, x, a, gy = problem(20240608, total, hid=sum(hidden_alloc))
        # single-device reference (the oracle on the whole batch)
        y_ref, stash = comp.forward(x, p, a, True)
        g_ref = comp.backward(stash, p, gy)
        lo = sum(batches[:rank])
        hi = lo + batches[rank]
        lx, la, lgy = x[lo:hi], a[:, lo:hi], gy[lo:hi]
        sp = D.shard_params(p, hidden_alloc)
        shard = sp.shards[rank]
        errs = {}
        # data-centric, grads all-reduced (reference semantics)
        cache = D.PipelineSharedCache(sp.full_param_elements())
        r = D.data_centric_step(lx, la, lgy, shard, sp.b2 if rank == 0 else None, hidden_alloc,
                                "gelu", cache, comp, grad_reduce="all_reduce")
        errs["dc_y"] = scaled(r.y, y_ref[lo:hi])
        errs["dc_gx"] = scaled(r.grads.gx, g_ref.gx[lo:hi])
        for key in ("gw1", "gb1", "gw2", "gb2"):
            errs["dc_" + key] = scaled(getattr(r.grads, key), getattr(g_ref, key))
        # data-centric, grads reduce-scattered to the shard owners
        r = D.data_centric_step(lx, la, lgy, shard, sp.b2 if rank == 0 else None, hidden_alloc,
                                "gelu", cache, comp, grad_reduce="reduce_scatter")
        off, h = shard.hidden_offset, hidden_alloc[rank]
        errs["dcrs_gw1"] = scaled(r.grads.gw1, g_ref.gw1[:, :, off:off + h])
        errs["dcrs_gb1"] = scaled(r.grads.gb1, g_ref.gb1[:, off:off + h])
        errs["dcrs_gw2"] = scaled(r.grads.gw2, g_ref.gw2[:, off:off + h, :])
        if rank == 0:
            errs["dcrs_gb2"] = scaled(r.grads.gb2, g_ref.gb2)
        # model-centric, all-reduce (reference semantics: global y / gx)
        r = D.model_centric_step(lx, la, lgy, shard, sp.b2, "gelu", comp, reduce="all_reduce")
        errs["mc_y"] = scaled(r.y, y_ref)
        errs["mc_gx"] = scaled(r.grads.gx, g_ref.gx)
        errs["mc_gw1"] = scaled(r.grads.gw1, g_ref.gw1[:, :, off:off + h])
        errs["mc_gb1"] = scaled(r.grads.gb1, g_ref.gb1[:, off:off + h])
        errs["mc_gw2"] = scaled(r.grads.gw2, g_ref.gw2[:, off:off + h, :])
        if rank == 0:
            errs["mc_gb2"] = scaled(r.grads.gb2, g_ref.gb2)
        else:
            errs["mc_gb2_none"] = 0.0 if r.grads.gb2 is None else 1.0
        # model-centric, reduce-scatter back to the token owners
        r = D.model_centric_step(lx, la, lgy, shard, sp.b2, "gelu", comp, reduce="reduce_scatter")
        errs["mcrs_y"] = scaled(r.y, y_ref[lo:hi])
        errs["mcrs_gx"] = scaled(r.grads.gx, g_ref.gx[lo:hi])
        # unshard(shard) is exact (dist_sim.hpp:50-52)
        back = D.unshard_params(sp)
        errs["unshard"] = float((back.w1 - p.w1).abs().max() + (back.w2 - p.w2).abs().max()
                                + (back.b1 - p.b1).abs().max())
        out_q.put((rank, errs))
    finally:
        dist.destroy_process_group()


def run_pipeline(rank, world, port, batches, hidden_alloc, n_layers, out_q):
    """Multi-layer data-centric pipeline (dist_sim.cpp:410-433) vs the
    single-device sequential stack: y, every layer's gradients, 2L - 1 gathers."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2411_01288_b200 import dist as D
        comp = oracle_compute()
        total = sum(batches)
        H = sum(hidden_alloc)
        layers, assigns = [], []
        x = gy = None
        for l in range(n_layers):
            p, xl, a, gyl = problem(777 + 13 * l, total, din=5, hid=H, dout=5)
            layers.append(p)
            assigns.append(a)
            if l == 0:
                x, gy = xl, gyl
        # single-device sequential reference
        stashes, h = [], x
        for l in range(n_layers):
            h, st = comp.forward(h, layers[l], assigns[l], True)
            stashes.append(st)
        y_ref = h
        g_ref = [None] * n_layers
        g = gy
        for l in reversed(range(n_layers)):
            g_ref[l] = comp.backward(stashes[l], layers[l], g)
            g = g_ref[l].gx
        lo = sum(batches[:rank])
        hi = lo + batches[rank]
        sps = [D.shard_params(p, hidden_alloc) for p in layers]
        shards = [sp.shards[rank] for sp in sps]
        b2s = [sp.b2 if rank == 0 else None for sp in sps]
        la = [a[:, lo:hi] for a in assigns]
        errs = {}
        for how in ("all_reduce", "reduce_scatter"):
            cache = D.PipelineSharedCache(sps[0].full_param_elements(), slots=2)
            r = D.data_centric_pipeline(x[lo:hi], la, gy[lo:hi], shards, b2s, hidden_alloc,
                                        "gelu", cache, comp, grad_reduce=how)
            errs[f"{how}_gathers"] = 0.0 if r.gathers == 2 * n_layers - 1 else 1.0
            errs[f"{how}_y"] = scaled(r.y, y_ref[lo:hi])
            off, hh = shards[0].hidden_offset, hidden_alloc[rank]
            for l in range(n_layers):
                gl, gr = r.grads[l], g_ref[l]
                if how == "all_reduce":
                    for key in ("gw1", "gb1", "gw2", "gb2"):
                        errs[f"{how}_{key}{l}"] = scaled(getattr(gl, key), getattr(gr, key))
                else:
                    errs[f"{how}_gw1{l}"] = scaled(gl.gw1, gr.gw1[:, :, off:off + hh])
                    errs[f"{how}_gb1{l}"] = scaled(gl.gb1, gr.gb1[:, off:off + hh])
                    errs[f"{how}_gw2{l}"] = scaled(gl.gw2, gr.gw2[:, off:off + hh, :])
                    if rank == 0:
                        errs[f"{how}_gb2{l}"] = scaled(gl.gb2, gr.gb2)
                errs[f"{how}_gx{l}"] = scaled(gl.gx, gr.gx[lo:hi])
        # the prefetching schedule refuses a one-slot cache
        try:
            D.data_centric_pipeline(x[lo:hi], la, gy[lo:hi], shards, b2s, hidden_alloc, "gelu",
                                    D.PipelineSharedCache(sps[0].full_param_elements()), comp)
            errs["one_slot_rejected"] = 1.0 if n_layers > 1 else 0.0
        except D.CacheError:
            errs["one_slot_rejected"] = 0.0
        out_q.put((rank, errs))
    finally:
        dist.destroy_process_group()
