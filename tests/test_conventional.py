"""Conventional dispatch/combine + capacity-factor baseline (SURVEY.md §8(f)
row 2; reference core/src/gemm_oracle.cpp).  Host accounting against the
reference's KATs (tests/test_gemm_oracle.cpp:151-223) on CPU; the device
baseline (hxm_layer_desc.capacity) against the oracle under -m gpu."""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O
import paper_2411_01288_b200 as H
from paper_2411_01288_b200 import conventional as CV


def test_balanced_factor_one_has_no_overhead():
    for k in (1, 2):
        r = H.synthesize_routing(32, 8, k, "balanced", 1)
        rep = CV.count_redundancy(r, 4, 16, 4, 1.0)
        assert rep.padded_rows == 0 and rep.dropped_tokens == 0
        assert rep.token_macs_oracle == rep.token_macs_expert_specific


def test_all_to_one_expert_drops_three_quarters():
    r = H.synthesize_routing(16, 4, 1, "fixed:0", 1)
    rep = CV.count_redundancy(r, 2, 4, 2, 1.0)
    assert rep.capacity_per_expert == 4
    assert rep.dropped_tokens == 12 and rep.padded_rows == 12


def test_matches_brute_force_counting():
    n, e, k, f = 1024, 8, 2, 1.25
    r = H.synthesize_routing(n, e, k, "uniform", 2024)
    rep = CV.count_redundancy(r, 8, 32, 8, f)
    cap = int(np.ceil(f * k * n / e))
    load = np.bincount(r.assignments.ravel(), minlength=e)
    kept = np.minimum(load, cap)
    per_row = 8 * 32 + 32 * 8
    assert rep.capacity_per_expert == cap
    assert rep.padded_rows == int((cap - kept).sum())
    assert rep.dropped_tokens == int((load - kept).sum()) == 0
    assert rep.token_macs_oracle == e * cap * per_row
    assert rep.token_macs_expert_specific == k * n * per_row
    assert rep.token_macs_oracle > rep.token_macs_expert_specific


def test_report_schema_keys_and_errors():
    r = H.synthesize_routing(64, 4, 2, "uniform", 7)
    d = json.loads(CV.count_redundancy(r, 4, 8, 4, 1.25).to_json())
    # schemas/redundancy_report.schema.json: required keys, no extras, ints >= 0
    assert set(d) == {"token_macs_expert_specific", "token_macs_oracle", "padded_rows",
                      "dropped_tokens", "capacity_per_expert"}
    assert all(isinstance(v, int) and v >= 0 for v in d.values())
    with pytest.raises(ValueError):
        CV.count_redundancy(H.synthesize_routing(8, 2, 1, "uniform", 1), 2, 2, 2, 0.0)


def test_kept_slots_keep_lowest_slot_ids():
    r = H.RoutingChoice(4, 2, 2, np.array([[0, 0, 0, 1], [1, 1, 1, 0]], np.int32))
    m = CV.kept_slots(r, 2)
    # expert 0: slots 0,1,2,7 -> keep 0,1 ; expert 1: slots 3,4,5,6 -> keep 3,4
    assert m.ravel().tolist() == [True, True, False, True, True, False, False, False]
    assert H.moe_layer.capacity_rows(1000, 8, 2, 1.25) == 320
    with pytest.raises(ValueError):
        H.moe_layer.capacity_rows(10, 2, 1, 0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("E,k,din,hid,dout,n,cap", [
    (4, 2, 64, 128, 64, 256, 64),     # about half of every expert's slots dropped
    (8, 2, 128, 192, 128, 512, 192),  # headroom: pads, no drops
    (4, 1, 64, 64, 64, 300, 64),
])
def test_gpu_capacity_baseline_vs_oracle(E, k, din, hid, dout, n, cap):
    """The device baseline equals the exact layer with the dropped slots
    rerouted to all-zero experts E + i (zero weights and bias: no
    contribution to y, zero gradient flow) -- computed by the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    p, x = H.make_random_params(E, din, hid, dout, "gelu", seed=5, n_tokens=n,
                                dtype=torch.bfloat16)
    r = H.synthesize_routing(n, E, k, "uniform", 6)
    gy = torch.as_tensor(np.random.default_rng(7).standard_normal((n, dout))).to(
        "cuda", torch.bfloat16)
    fw = H.moe_forward(x, p, r, capacity=cap)
    g = H.moe_backward(fw.stash, p, gy)
    keep = CV.kept_slots(r, cap)
    a2 = np.where(keep, r.assignments, E + np.arange(k)[:, None]).astype(np.int32)
    f64 = lambda t: t.detach().double().cpu().numpy()  # noqa: E731
    z = lambda *s: np.zeros(s)  # noqa: E731
    w1 = np.concatenate([f64(p.w1), z(k, din, hid)])
    b1 = np.concatenate([f64(p.b1), z(k, hid)])
    w2 = np.concatenate([f64(p.w2), z(k, hid, dout)])
    b2 = np.concatenate([f64(p.b2), z(k, dout)])
    y_ref, y1, y2 = O.moe_forward(f64(x), w1, b1, w2, b2, a2, 8, "gelu")
    go = O.moe_backward(f64(x), w1, w2, a2, y1, y2, f64(gy), 8, "gelu")
    errs = {"y": O.scaled_err(f64(fw.y), y_ref),
            "gx": O.scaled_err(f64(g.gx), go["gx"])}
    for key in ("gw1", "gb1", "gw2", "gb2"):
        errs[key] = O.scaled_err(f64(getattr(g, key)), go[key][:E])
    assert max(errs.values()) <= 2e-2, errs
    # work accounting: E x capacity rows per weight
    import ctypes
    assert H.lib().hxm_layer_forward_macs(ctypes.byref(fw.stash.desc)) == \
        E * cap * (din * hid + hid * dout)
