"""Shard-major weights (hxm_layer_desc.weight_shards): the data-centric TP
cache is filled by all_gather_into_tensor of the P hidden shards, i.e.
w1 (P*E) x D_i x h, b1 (P*E) x h, w2 (P*E) x h x D_o, and the layer's GEMMs
read that buffer in place (SURVEY.md §7 hard part 5; dist_sim.cpp:367-368)
instead of repacking it into the reference layout.

The kernels see the same bf16 operands in the same order either way, so the
layer run from a shard-major copy must be BIT-identical to the reference
layout run -- y and all five gradients."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def shard_major(p, P):
    """What all_gather_into_tensor of shard_params(p, even_split(H, P)) lands."""
    E, Di, H = p.w1.shape
    Do = p.w2.shape[2]
    h = H // P
    w1 = p.w1.view(E, Di, P, h).permute(2, 0, 1, 3).reshape(P * E, Di, h).contiguous()
    b1 = p.b1.float().view(E, P, h).permute(1, 0, 2).reshape(P * E, h).contiguous()
    w2 = p.w2.view(E, P, h, Do).permute(1, 0, 2, 3).reshape(P * E, h, Do).contiguous()
    return w1, b1, w2


@pytest.mark.parametrize("E,k,D,Hd,N,P", [(8, 2, 128, 1024, 700, 2), (8, 2, 128, 1024, 700, 4),
                                          (16, 2, 1024, 4096, 1024, 8),
                                          (32, 2, 384, 1536, 2048, 3)])
def test_layer_shard_major_bit_identical(E, k, D, Hd, N, P):
    import paper_2411_01288_b200 as H
    from paper_2411_01288_b200.runner import LayerRunner
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=5, n_tokens=N, dtype=torch.bfloat16)
    r = H.synthesize_routing(N, E, k, "uniform", 6).to_device()
    gy = torch.randn(N, D, generator=torch.Generator().manual_seed(7)).to("cuda", torch.bfloat16)
    ref = LayerRunner(p, N, k, "cuda", torch.bfloat16)
    ref.step(x, r, gy)
    run = LayerRunner(p, N, k, "cuda", torch.bfloat16)
    w1, b1, w2 = shard_major(p, P)
    ev = torch.cuda.Event()
    ev.record()
    run.set_weights(w1, b1, w2, shards=P, ready=ev)
    assert run.desc.weight_shards == P
    run.step(x, r, gy)
    torch.cuda.synchronize()
    assert torch.equal(run.y, ref.y)
    for key in ("gw1", "gb1", "gw2", "gb2", "gx"):
        assert torch.equal(getattr(run.grads, key), getattr(ref.grads, key)), key


def test_shard_major_unsupported_shape_rejected():
    import paper_2411_01288_b200 as H
    from paper_2411_01288_b200.runner import LayerRunner
    E, k, D, Hd, N, P = 8, 2, 384, 1536, 256, 8  # h = 192: not a multiple of the 128-col halves
    p, _ = H.make_random_params(E, D, Hd, D, "gelu", seed=5, n_tokens=N, dtype=torch.bfloat16)
    run = LayerRunner(p, N, k, "cuda", torch.bfloat16)
    w1, b1, w2 = shard_major(p, P)
    with pytest.raises(ValueError, match="split 8 ways"):
        run.set_weights(w1, b1, w2, shards=P)
