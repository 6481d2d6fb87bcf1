"""The C ABI's NCCL collectives (include/hexamoe.h, csrc/nccl.cu) on a
one-rank communicator (this pool has one GPU per box; NCCL refuses two ranks
on one device): the data-centric cache fill feeds the layer bit-identically,
a too-small cache raises CacheError (dist_sim.cpp:104-125), and the
gradient / token collectives are the identity at P = 1."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def comm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2411_01288_b200._lib import check, lib
    torch.cuda.set_device(0)
    L = lib()
    uid = (C.c_ubyte * 128)()
    check(L.hxm_nccl_get_unique_id(uid), "nccl id")
    c = C.c_void_p()
    check(L.hxm_nccl_comm_init(C.byref(c), 1, uid, 0), "nccl init")
    yield c
    check(L.hxm_nccl_comm_destroy(c), "nccl destroy")


def test_dc_cache_fill_feeds_layer(comm):
    import paper_2411_01288_b200 as H
    from paper_2411_01288_b200._lib import check, lib, CacheError
    from paper_2411_01288_b200.runner import LayerRunner
    L = lib()
    E, k, D, Hd, N = 8, 2, 128, 512, 600
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=3, n_tokens=N, dtype=torch.bfloat16)
    r = H.synthesize_routing(N, E, k, "uniform", 4).to_device()
    gy = torch.randn(N, D, generator=torch.Generator().manual_seed(5)).to("cuda", torch.bfloat16)
    ref = LayerRunner(p, N, k, "cuda", torch.bfloat16)
    ref.step(x, r, gy)
    run = LayerRunner(p, N, k, "cuda", torch.bfloat16)
    pd = C.byref(run.desc)
    nb = L.hxm_dc_cache_bytes(pd)
    cache = torch.empty(nb, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    b1 = p.b1.float().contiguous()
    with pytest.raises(CacheError):
        check(L.hxm_dc_fill_cache(comm, pd, p.w1.data_ptr(), b1.data_ptr(), p.w2.data_ptr(),
                                  cache.data_ptr(), nb - 1, st), "fill")
    check(L.hxm_dc_fill_cache(comm, pd, p.w1.data_ptr(), b1.data_ptr(), p.w2.data_ptr(),
                              cache.data_ptr(), nb, st), "fill")
    w1p, b1p, w2p = C.c_void_p(), C.c_void_p(), C.c_void_p()
    check(L.hxm_dc_cache_views(pd, cache.data_ptr(), C.byref(w1p), C.byref(b1p), C.byref(w2p)))
    base = cache.data_ptr()
    w1 = cache[w1p.value - base:].view(torch.bfloat16)[:E * D * Hd].view(E, D, Hd)
    b1c = cache[b1p.value - base:][:E * Hd * 4].view(torch.float32).view(E, Hd)
    w2 = cache[w2p.value - base:].view(torch.bfloat16)[:E * Hd * D].view(E, Hd, D)
    run.set_weights(w1, b1c, w2)
    run.step(x, r, gy)
    torch.cuda.synchronize()
    assert torch.equal(run.y, ref.y)
    for key in ("gw1", "gb1", "gw2", "gb2", "gx"):
        assert torch.equal(getattr(run.grads, key), getattr(ref.grads, key)), key
    g = run.grads
    before = [t.clone() for t in (g.gw1, g.gb1, g.gw2, g.gb2)]
    check(L.hxm_dc_allreduce_grads(comm, pd, g.gw1.data_ptr(), g.gb1.data_ptr(),
                                   g.gw2.data_ptr(), g.gb2.data_ptr(), st), "allreduce")
    torch.cuda.synchronize()
    for a, b in zip(before, (g.gw1, g.gb1, g.gw2, g.gb2)):
        assert torch.equal(a, b)


def test_tp_collectives_identity_at_one_rank(comm):
    from paper_2411_01288_b200._lib import check, lib
    L = lib()
    st = torch.cuda.current_stream().cuda_stream
    x = torch.randn(37, 24, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(x)
    check(L.hxm_tp_allgather_rows(comm, x.data_ptr(), 37, 24 * 2, out.data_ptr(), st))
    a = torch.randint(0, 8, (2, 37), dtype=torch.int32, device="cuda")
    ao = torch.empty_like(a)
    check(L.hxm_tp_allgather_assignments(comm, a.data_ptr(), 2, 37, ao.data_ptr(), st))
    y = torch.randn(37, 24, device="cuda")
    y0 = y.clone()
    check(L.hxm_tp_allreduce_sum(comm, y.data_ptr(), y.numel(), st))
    torch.cuda.synchronize()
    assert torch.equal(out, x) and torch.equal(ao, a) and torch.equal(y, y0)


def test_nccl_errors_are_typed(comm):
    from paper_2411_01288_b200._lib import check, lib
    L = lib()
    with pytest.raises(ValueError):
        check(L.hxm_tp_allreduce_sum(None, None, 4, None), "null comm")
