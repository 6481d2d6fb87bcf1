"""Heterogeneous allocation (reference tests/test_hetero_alloc.cpp KATs and
properties) -- host arithmetic on CPU; the GPU probe under -m gpu."""
import numpy as np
import pytest

from paper_2411_01288_b200 import hetero as HA


def test_capacity_proportions_paper_cases():
    # test_hetero_alloc.cpp:10-23 (the paper's three measured cases)
    for lat, want in (([4.58, 3.06], [0.40, 0.60]), ([3.20, 3.18], [0.50, 0.50]),
                      ([3.28, 9.42], [0.74, 0.26])):
        r = HA.capacity_proportions(lat)
        assert all(abs(a - b) <= 0.005 for a, b in zip(r, want))


def test_proportions_sum_and_errors():
    r = HA.capacity_proportions([1.0, 2.0, 5.0])
    assert abs(sum(r) - 1.0) <= 1e-12
    for bad in ([1.0, 0.0], [-1.0], []):
        with pytest.raises(ValueError):
            HA.capacity_proportions(bad)


def test_allocate_kats():
    # test_hetero_alloc.cpp:33-56
    assert HA.allocate_batches([4.58, 3.06], 100).shares == [40, 60]
    assert HA.allocate_batches([2.0] * 4, 100).shares == [25, 25, 25, 25]
    assert HA.allocate_batches([3.3], 17).shares == [17]
    assert HA.allocate_hidden([3.28, 9.42], 100).shares == [74, 26]
    ex = HA.allocate_hidden([1.0, 3.0], 8)
    assert abs(ex.ideal[0] - 6.0) <= 1e-12 and abs(ex.ideal[1] - 2.0) <= 1e-12
    assert ex.shares == [6, 2]
    assert HA.allocate_hidden([2.5, 2.5], 64).shares == [32, 32]
    assert HA.allocate_batches([1.0], 0).shares == [0]
    with pytest.raises(ValueError):
        HA.allocate_batches([1.0], -1)


def test_round_preserving_sum_kats():
    # test_hetero_alloc.cpp:58-67
    assert HA.round_preserving_sum([2.5, 2.5], 5) == [3, 2]
    assert HA.round_preserving_sum([1.9, 1.9, 1.2], 5) == [2, 2, 1]
    assert HA.round_preserving_sum([3.0, 1.0, 4.0], 8) == [3, 1, 4]
    with pytest.raises(ValueError):
        HA.round_preserving_sum([-0.5, 5.5], 5)
    with pytest.raises(ValueError):
        HA.round_preserving_sum([1.0, 1.0], 5)


def test_allocation_properties_random():
    # test_hetero_alloc.cpp:69-101: sum, |share - ideal| < 1, monotone, scale invariant
    rng = np.random.default_rng(61)
    for _ in range(1000):
        n = 1 + int(rng.integers(8))
        lat = list(0.1 + 10.0 * rng.random(n))
        total = int(rng.integers(5000))
        plan = HA.allocate_batches(lat, total)
        assert sum(plan.shares) == total
        assert all(abs(s - i) < 1.0 and s >= 0 for s, i in zip(plan.shares, plan.ideal))
        for i in range(n):
            for j in range(n):
                if lat[i] < lat[j]:
                    assert plan.shares[i] >= plan.shares[j]
        assert HA.allocate_batches([t * 37.5 for t in lat], total).shares == plan.shares


def test_plan_serialisation():
    p = HA.allocate_hidden([1.0, 3.0], 8)
    import json
    assert json.loads(p.to_json()) == {"kind": "hidden", "total": 8, "shares": [6, 2],
                                       "ideal": p.ideal}
    assert p.to_csv().splitlines()[0] == "device,ideal,share"


def test_allocate_hidden_feeds_uneven_shards():
    import torch
    from paper_2411_01288_b200 import MoeLayerParams
    from paper_2411_01288_b200 import dist as D
    plan = HA.allocate_hidden([3.28, 9.42], 12)
    p = MoeLayerParams(torch.randn(2, 3, 12), torch.randn(2, 12), torch.randn(2, 12, 3),
                       torch.randn(2, 3))
    sp = D.shard_params(p, plan.shares)
    assert [s.w1.shape[2] for s in sp.shards] == plan.shares
    back = D.unshard_params(sp)
    assert torch.equal(back.w1, p.w1) and torch.equal(back.w2, p.w2)


@pytest.mark.gpu
def test_gpu_probe_scales_with_work():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    assert HA.probe_capacity_seconds(0, 256) == 0.0
    light = HA.probe_capacity_seconds(2, 2048)
    heavy = HA.probe_capacity_seconds(16, 2048)
    assert 0.0 < light < heavy
    with pytest.raises(ValueError):
        HA.probe_capacity_seconds(1, 0)
    lat = HA.measure_latencies(4, 1024)
    assert len(lat) == 1 and lat[0] > 0
