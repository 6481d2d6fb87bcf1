"""GPU parity: the CUDA path (through the C ABI) against the pinned CPU oracle.

Bars (BASELINE.json north_star; scaled error = max|a-b| / (1 + max|ref|),
reference tests/support/test_oracles.hpp:60-62):
  * routing index: bit-exact;
  * integer-valued known-answer tests: exact in fp32 and bf16;
  * fp32 path: scaled error <= 1e-4;
  * bf16 path: scaled error <= 2e-2, with the oracle fed the same
    bf16-rounded inputs so only accumulation / stash rounding is measured.
"""
import json
import os

import numpy as np
import pytest
import torch

import oracle as O

pytestmark = pytest.mark.gpu

RTOL_F32 = 1e-4
RTOL_BF16 = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def hx():
    import paper_2411_01288_b200 as H
    return H


def dev(a, dtype=torch.float32):
    return torch.as_tensor(np.asarray(a, dtype=np.float64)).to("cuda", dtype)


def host(t):
    return t.detach().to(torch.float64).cpu().numpy()


def rounded(a, dtype):
    """The values the device sees, as float64 for the oracle."""
    return host(dev(a, dtype))


def kat():
    with open(os.path.join(os.path.dirname(__file__), "golden", "kat.json")) as f:
        return json.load(f)


def dact_ref(act, y1):
    """F'(y1) of the reference activations (tensor.cpp:48-53, 72), fp64."""
    y1 = np.asarray(y1, dtype=np.float64)
    if act == "gelu":
        c = 0.7978845608028654
        t = np.tanh(c * (y1 + 0.044715 * y1 ** 3))
        return 0.5 * (1 + t) + 0.5 * y1 * (1 - t * t) * c * (1 + 3 * 0.044715 * y1 * y1)
    if act == "relu":
        return (y1 > 0).astype(np.float64)
    return np.ones_like(y1)


# ----------------------------------------------------------------- routing --
def test_reindex_kats_bitexact():
    H = hx()
    for c in kat()["reindex"]:
        rx = H.build_reindex(c["assignment"], c["E"], c["blk"])
        assert rx.idx.cpu().tolist() == c["idx"], c["cite"]
        assert rx.v.cpu().tolist() == c["v"], c["cite"]


def test_reindex_errors():
    H = hx()
    for c in kat()["reindex_errors"]:
        with pytest.raises(ValueError):
            H.build_reindex(c["assignment"], c["E"], c["blk"])


def test_reindex_reference_fixtures_bitexact(golden_dir):
    H = hx()
    d = np.load(os.path.join(golden_dir, "ref_reindex.npz"))
    for i in range(40):
        E, blk = d[f"r{i}_meta"].tolist()
        rx = H.build_reindex(d[f"r{i}_a"], E, blk)
        assert np.array_equal(rx.v.cpu().numpy(), d[f"r{i}_v"]), i
        assert np.array_equal(rx.idx.cpu().numpy(), d[f"r{i}_idx"]), i
    for c in range(2):
        rx = H.build_reindex(d["c2_assign"][c], 32, 8)
        assert np.array_equal(rx.v.cpu().numpy(), d[f"c2_v{c}"])
        assert np.array_equal(rx.idx.cpu().numpy(), d[f"c2_idx{c}"])


@pytest.mark.parametrize("n,E,blk,dist", [
    (131072, 64, 8, "uniform"),      # c4 routing size
    (16384, 64, 1, "zipf:1.5"),
    (100000, 7, 128, "uniform"),
    (5000, 300, 3, "uniform"),       # many experts, odd blk
    (1, 1, 1, "uniform"),
    (3000, 16, 16, "fixed:0"),       # all tokens to one expert
])
def test_reindex_random_bitexact(n, E, blk, dist):
    H = hx()
    a = O.synthesize_routing(n, E, 1, dist, n + E)[0]
    want = O.build_reindex(a, E, blk)
    rx = H.build_reindex(a, E, blk)
    assert np.array_equal(rx.idx.cpu().numpy(), want.idx)
    assert np.array_equal(rx.v.cpu().numpy(), want.v)


def test_reindex_500_random_instances():
    """acceptance criterion 7 style (verify_suites.cpp:166-218)."""
    H = hx()
    rng = np.random.default_rng(20240607)
    for _ in range(500):
        n = int(rng.integers(1, 65)); E = int(rng.integers(1, 9))
        blk = int(rng.choice([2, 4, 8]))
        a = rng.integers(0, E, size=n).astype(np.int32)
        want = O.build_reindex(a, E, blk)
        rx = H.build_reindex(a, E, blk)
        assert np.array_equal(rx.v.cpu().numpy(), want.v)
        assert np.array_equal(rx.idx.cpu().numpy(), want.idx)


# ---------------------------------------------------------------- operators --
@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_operator_kats_exact(dtype):
    H = hx()
    k = kat()
    for c in k["esmm"]:
        rx = H.build_reindex(c["assignment"], c["E"], c["blk"])
        y = H.esmm(dev(c["x"], dtype), dev(c["w"], dtype), dev(c["b"]), rx)
        assert host(y).tolist() == c["y"], c["cite"]
    for c in k["ess"]:
        rx = H.build_reindex(c["assignment"], c["E"], c["blk"])
        assert host(H.ess(dev(c["x"], dtype), rx)).tolist() == c["out"], c["cite"]
    for c in k["estmm"]:
        rx = H.build_reindex(c["assignment"], c["E"], c["blk"])
        got = H.estmm(dev(c["x1"], dtype), dev(c["x2"], dtype), rx)
        assert host(got).tolist() == c["out"], c["cite"]


def test_esmm_accumulate_and_errors():
    H = hx()
    rng = np.random.default_rng(6)
    x = rng.standard_normal((10, 3)); w = rng.standard_normal((2, 3, 4))
    b = rng.standard_normal((2, 4))
    rx_a = H.build_reindex([0, 1, 0, 1, 0, 1, 0, 1, 0, 1], 2, 2)
    rx_b = H.build_reindex([1, 1, 1, 0, 0, 0, 1, 1, 0, 0], 2, 2)
    pa = H.esmm(dev(x), dev(w), dev(b), rx_a)
    pb = H.esmm(dev(x), dev(w), dev(b), rx_b)
    dest = pa.clone()
    H.esmm(dev(x), dev(w), dev(b), rx_b, H.ACCUMULATE, dest)
    assert torch.equal(dest, pa + pb)  # test_es_ops.cpp:60-77
    with pytest.raises(ValueError):
        H.esmm(dev(x), dev(w), None, rx_a, H.ACCUMULATE, None)
    with pytest.raises(H.ShapeError):
        H.esmm(dev(x), dev(w), None, rx_a, H.ACCUMULATE, torch.zeros(3, 4, device="cuda"))
    with pytest.raises(H.ShapeError):  # test_es_ops.cpp:289-298
        H.esmm(dev(np.zeros((2, 3))), dev(np.zeros((2, 4, 2))), None,
               H.build_reindex([0, 1], 2, 2))
    with pytest.raises(H.ShapeError):
        H.estmm(dev(np.zeros((2, 3))), dev(np.zeros((3, 2))), H.build_reindex([0, 1], 2, 2))
    with pytest.raises(H.ShapeError):
        H.ess(dev(np.zeros((5, 2))), H.build_reindex([0, 1], 2, 2))


@pytest.mark.parametrize("dtype,rtol", [(torch.float32, RTOL_F32), (torch.bfloat16, RTOL_BF16)])
def test_operators_vs_reference_fixtures(golden_dir, dtype, rtol):
    H = hx()
    d = np.load(os.path.join(golden_dir, "ref_ops.npz"))
    for i in range(16):
        g = lambda k: d[f"o{i}_{k}"]
        E, blk = g("meta").tolist()
        rx = H.build_reindex(g("a"), E, blk)
        x, x2, w, b = (rounded(g(k), dtype) for k in ("x", "x2", "w", "b"))
        orx = O.build_reindex(g("a"), E, blk)
        if dtype == torch.float32:  # fixtures are the reference's own outputs
            want_mm, want_ss, want_tm = g("esmm"), g("ess"), g("estmm")
        else:                        # oracle on the bf16-rounded inputs
            want_mm = O.esmm(x, w, g("b"), orx)
            want_ss, want_tm = O.ess(x, orx), O.estmm(x, x2, orx)
        got = H.esmm(dev(x, dtype), dev(w, dtype), dev(g("b")), rx)
        assert O.scaled_err(host(got), want_mm) <= rtol, (i, "esmm")
        assert O.scaled_err(host(H.ess(dev(x, dtype), rx)), want_ss) <= rtol, (i, "ess")
        got_tm = H.estmm(dev(x, dtype), dev(x2, dtype), rx)
        assert O.scaled_err(host(got_tm), want_tm) <= rtol, (i, "estmm")
        f = H.esfk(dev(x, dtype), dev(x2, dtype), dev(w, dtype), rx, w_transposed=True)
        want_gx = O.esmm(x2, np.ascontiguousarray(np.transpose(w, (0, 2, 1))), None, orx)
        assert O.scaled_err(host(f.grad_x), want_gx) <= rtol, (i, "esfk grad_x")
        # es_ops.cpp:210-247: grad_b = ess(g), grad_w = estmm(x, g)
        assert O.scaled_err(host(f.grad_b), O.ess(x2, orx)) <= rtol, (i, "esfk grad_b")
        assert O.scaled_err(host(f.grad_w), O.estmm(x, x2, orx)) <= rtol, (i, "esfk grad_w")


@pytest.mark.parametrize("E,n,d1,d2,blk", [
    (32, 4096, 384, 1536, 8),    # c2 first GEMM shape (token subsample)
    (32, 4096, 1536, 384, 8),    # c2 second GEMM shape
    (8, 1000, 128, 256, 3),      # ragged segments, odd blk
    (64, 3000, 64, 192, 8),      # many experts, some empty
    (4, 20000, 512, 384, 8),     # whole-tile ESTMM with split (> 8192-slot) experts
])
def test_bf16_operators_at_scale(E, n, d1, d2, blk):
    H = hx()
    rng = np.random.default_rng(E * n)
    a = O.synthesize_routing(n, E, 1, "zipf:1.1", 5)[0]
    x = rounded(rng.standard_normal((n, d1)), torch.bfloat16)
    x2 = rounded(rng.standard_normal((n, d2)), torch.bfloat16)
    w = rounded(0.5 * rng.standard_normal((E, d1, d2)), torch.bfloat16)
    b = rng.standard_normal((E, d2))
    orx = O.build_reindex(a, E, blk)
    rx = H.build_reindex(a, E, blk)
    bf = torch.bfloat16
    got = H.esmm(dev(x, bf), dev(w, bf), dev(b), rx)
    assert O.scaled_err(host(got), O.esmm(x, w, b, orx)) <= RTOL_BF16
    gt = H.esmm(dev(x2, bf), dev(w, bf), None, rx, w_transposed=True)
    want_t = O.esmm(x2, np.ascontiguousarray(np.transpose(w, (0, 2, 1))), None, orx)
    assert O.scaled_err(host(gt), want_t) <= RTOL_BF16
    assert O.scaled_err(host(H.estmm(dev(x, bf), dev(x2, bf), rx)), O.estmm(x, x2, orx)) <= RTOL_BF16
    assert O.scaled_err(host(H.ess(dev(x, bf), rx)), O.ess(x, orx)) <= RTOL_BF16


# -------------------------------------------------------------------- layer --
def _layer_case(E, k, din, hid, dout, n, act, dtype, seed, dist="uniform"):
    H = hx()
    p, x = H.make_random_params(E, din, hid, dout, act, seed=seed, n_tokens=n, dtype=dtype)
    r = H.synthesize_routing(n, E, k, dist, seed + 1)
    gy = torch.as_tensor(np.random.default_rng(seed).standard_normal((n, dout))).to("cuda", dtype)
    return p, x, r, gy


def _check_layer(p, x, r, gy, rtol, act):
    H = hx()
    fw = H.moe_forward(x, p, r)
    g = H.moe_backward(fw.stash, p, gy)
    y_ref, y1_ref, y2_ref = O.moe_forward(host(x), host(p.w1), host(p.b1), host(p.w2),
                                          host(p.b2), r.assignments, 8, act)
    go = O.moe_backward(host(x), host(p.w1), host(p.w2), r.assignments, y1_ref, y2_ref,
                        host(gy), 8, act)
    errs = {"y": O.scaled_err(host(fw.y), y_ref)}
    for i in range(r.k):
        dact, y2 = fw.stash.export(i)
        errs[f"dact_{i}"] = O.scaled_err(host(dact), dact_ref(act, y1_ref[i]))
        errs[f"y2_{i}"] = O.scaled_err(host(y2), y2_ref[i])
    for key in ("gw1", "gb1", "gw2", "gb2", "gx"):
        errs[key] = O.scaled_err(host(getattr(g, key)), go[key])
    bad = {k: v for k, v in errs.items() if not v <= rtol}
    assert not bad, bad
    return errs


def test_layer_chain_rule_kat():
    H = hx()
    c = kat()["layer_chain_rule"]
    for dtype in (torch.float32, torch.bfloat16):
        p = H.MoeLayerParams(dev(c["w1"], dtype), dev(c["b1"]), dev(c["w2"], dtype),
                             dev(c["b2"]), c["act"])
        r = H.RoutingChoice(1, 1, 1, np.array(c["assignments"], np.int32))
        fw = H.moe_forward(dev(c["x"], dtype), p, r, c["blk"])
        assert host(fw.y).tolist() == c["y"]
        g = H.moe_backward(fw.stash, p, dev(c["g_y"], dtype))
        for key in ("gx", "gw1", "gw2", "gb1", "gb2"):
            assert host(getattr(g, key)).tolist() == c[key], (dtype, key)


def test_layer_reference_fixtures_fp32(golden_dir):
    H = hx()
    d = np.load(os.path.join(golden_dir, "ref_layer.npz"))
    for i in range(5):
        g = lambda k: d[f"l{i}_{k}"]
        E, k, din, hid, dout, n, blk, act = g("meta").tolist()
        actn = {v: kk for kk, v in O.ACT.items()}[act]
        p = H.MoeLayerParams(dev(g("w1")), dev(g("b1")), dev(g("w2")), dev(g("b2")), actn)
        r = H.RoutingChoice(n, E, k, g("a"))
        fw = H.moe_forward(dev(g("x")), p, r, blk)
        assert O.scaled_err(host(fw.y), g("y")) <= RTOL_F32, i
        gr = H.moe_backward(fw.stash, p, dev(g("gy")))
        for key in ("gw1", "gb1", "gw2", "gb2", "gx"):
            assert O.scaled_err(host(getattr(gr, key)), g(key)) <= RTOL_F32, (i, key)


def test_layer_c1_fp32_full_size():
    """BASELINE.json configs[0]: 8 experts top-1, d=96, ffn=384, 3136 tokens, fp32."""
    p, x, r, gy = _layer_case(8, 1, 96, 384, 96, 3136, "gelu", torch.float32, 1)
    _check_layer(p, x, r, gy, RTOL_F32, "gelu")


@pytest.mark.parametrize("E,k,din,hid,dout,n,act,dist", [
    (32, 2, 384, 1536, 384, 1024, "gelu", "uniform"),  # c2 dims, token subsample
    (8, 2, 64, 128, 64, 777, "relu", "uniform"),
    (16, 3, 128, 256, 192, 500, "identity", "zipf:1.3"),
    (64, 2, 128, 192, 128, 600, "gelu", "uniform"),    # many empty experts
    (4, 2, 12, 20, 6, 50, "gelu", "uniform"),          # unaligned dims
    (8, 2, 640, 512, 640, 512, "gelu", "uniform"),     # K > 512: 8-warp stash epilogues
    (8, 2, 128, 256, 256, 300, "relu", "uniform"),     # K <= 512: 16-warp stash epilogues
    # d = 384 with H a multiple of 256: the whole-tile kernels (fwd2 / gx and
    # gW2 / transposed gW1, umma_wide.cu), incl. empty experts and top-1
    (12, 2, 384, 256, 384, 300, "gelu", "uniform"),
    (40, 1, 384, 512, 384, 200, "relu", "uniform"),
    (6, 2, 384, 768, 384, 900, "identity", "zipf:1.3"),
])
def test_layer_bf16_vs_oracle(E, k, din, hid, dout, n, act, dist):
    p, x, r, gy = _layer_case(E, k, din, hid, dout, n, act, torch.bfloat16, E + n, dist)
    _check_layer(p, x, r, gy, RTOL_BF16, act)


def test_layer_skewed_split_k():
    """c5-style skew: most slots on two experts, so their ESTMM is split over
    several 8192-position chunks (fp32 reductions into zeroed slices), others
    have a few tokens or none."""
    H = hx()
    E, k, D, Hd, N = 16, 2, 128, 256, 20000
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=5, n_tokens=N)
    r = H.synthesize_routing(N, E, k, "uniform", 6)
    a = r.assignments.copy()
    hot = np.random.default_rng(7).random(N) < 0.9
    a[0, hot], a[1, hot] = 0, 1
    a[:, :] = np.where(a == 15, 14, a)  # expert 15 empty
    bad = a[0] == a[1]
    a[1, bad] = (a[0, bad] + 1) % 15
    r = H.RoutingChoice(N, E, k, a)
    gy = torch.as_tensor(np.random.default_rng(8).standard_normal((N, D))).to("cuda", torch.bfloat16)
    errs = _check_layer(p, x, r, gy, RTOL_BF16, "gelu")
    assert errs["gw1"] <= RTOL_BF16


def test_layer_c2_full_size_properties():
    """c2 at full N: exact integer properties that do not need the CPU oracle.
    With g_y = ones, gb2[e] = number of (token, choice) slots routed to e
    exactly, and two runs give bit-identical outputs (k = 2 reductions
    commute)."""
    H = hx()
    E, k, D, Hd, N = 32, 2, 384, 1536, 16384
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=1, n_tokens=N)
    r = H.synthesize_routing(N, E, k, "uniform", 1)
    ones = torch.ones(N, D, dtype=torch.bfloat16, device="cuda")
    fw = H.moe_forward(x, p, r)
    g = H.moe_backward(fw.stash, p, ones)
    counts = np.bincount(r.assignments.ravel(), minlength=E).astype(np.float64)
    assert np.array_equal(host(g.gb2), np.repeat(counts[:, None], D, axis=1))
    fw2 = H.moe_forward(x, p, r)
    assert torch.equal(fw.y, fw2.y)
    assert torch.isfinite(g.gw1).all() and torch.isfinite(g.gx).all()


def test_layer_backward_repeatable_gb2_combine():
    """The backward prologue combines gb2 per expert in the block that brings
    the expert's ESS items to completion (per-expert arrival counters that
    reset themselves): repeated backward passes on one stash give
    bit-identical bias gradients, an expert without tokens gets gb2 = 0, and
    with g_y = ones gb2[e] is the exact slot count."""
    H = hx()
    E, k, D, Hd, N = 16, 2, 128, 256, 3000
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=11, n_tokens=N)
    r = H.synthesize_routing(N, E, k, "uniform", 12)
    a = r.assignments.copy()
    a[:, :] = np.where(a == 15, 14, a)  # expert 15 empty
    bad = a[0] == a[1]
    a[1, bad] = (a[0, bad] + 1) % 15
    r = H.RoutingChoice(N, E, k, a)
    ones = torch.ones(N, D, dtype=torch.bfloat16, device="cuda")
    fw = H.moe_forward(x, p, r)
    runs = [H.moe_backward(fw.stash, p, ones) for _ in range(3)]
    counts = np.bincount(a.ravel(), minlength=E).astype(np.float64)
    assert counts[15] == 0
    for g in runs:
        assert np.array_equal(host(g.gb2), np.repeat(counts[:, None], D, axis=1))
        assert torch.equal(g.gb1, runs[0].gb1)
        assert torch.equal(g.gx, runs[0].gx)


def test_layer_c4_full_size_properties():
    """BASELINE.json c4 at its full 131072 tokens on one GPU (64 experts
    top-2, d 1024, ffn 4096): size-independent exact properties instead of
    the CPU oracle (hours at this size).  gb2 counts the routed slots exactly
    for g_y = ones; the backward is linear in g_y and scaling by 2 is exact in
    floating point, so every gradient of 2 g_y is bitwise twice that of g_y
    (deterministic reductions: k = 2 reductions commute); a 64-token
    subsample of the batch matches the oracle."""
    H = hx()
    E, k, D, Hd, N = 64, 2, 1024, 4096, 131072
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=4, n_tokens=N)
    r = H.synthesize_routing(N, E, k, "uniform", 4)
    ones = torch.ones(N, D, dtype=torch.bfloat16, device="cuda")
    fw = H.moe_forward(x, p, r)
    g1 = H.moe_backward(fw.stash, p, ones)
    counts = np.bincount(r.assignments.ravel(), minlength=E).astype(np.float64)
    assert np.array_equal(host(g1.gb2), np.repeat(counts[:, None], D, axis=1))
    g2 = H.moe_backward(fw.stash, p, 2 * ones)
    for key in ("gw1", "gb1", "gw2", "gb2", "gx"):
        assert torch.equal(getattr(g2, key), 2 * getattr(g1, key)), key
    del g2
    # token subsample against the oracle (the rows of y depend only on
    # their own token)
    sub = np.arange(0, N, N // 64)
    y_ref, _, _ = O.moe_forward(host(x)[sub], host(p.w1), host(p.b1), host(p.w2), host(p.b2),
                                r.assignments[:, sub], 8, "gelu")
    assert O.scaled_err(host(fw.y)[sub], y_ref) <= RTOL_BF16


@pytest.mark.parametrize("E,k,D,Hd,N,dtype", [
    (1, 1, 64, 128, 1, torch.bfloat16),     # one token, one expert
    (3, 3, 64, 128, 5, torch.bfloat16),     # k == E
    (2, 1, 8, 16, 0, torch.float32),        # no tokens
    (2, 1, 64, 64, 0, torch.bfloat16),
    (5, 2, 64, 256, 130, torch.bfloat16),   # segments straddling 64/128/256 rows
    (1, 1, 384, 256, 3, torch.bfloat16),    # whole-tile kernels, 3 tokens
    (3, 2, 384, 512, 0, torch.bfloat16),    # whole-tile kernels, no tokens
])
def test_layer_edge_cases(E, k, D, Hd, N, dtype):
    H = hx()
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=E + N, n_tokens=max(N, 1), dtype=dtype)
    x = x[:N]
    r = H.synthesize_routing(N, E, k, "uniform", 3) if N else \
        H.RoutingChoice(0, E, k, np.zeros((k, 0), np.int32))
    gy = torch.as_tensor(np.random.default_rng(1).standard_normal((N, D))).to("cuda", dtype)
    fw = H.moe_forward(x, p, r)
    g = H.moe_backward(fw.stash, p, gy)
    torch.cuda.synchronize()
    if N == 0:
        assert fw.y.shape == (0, D)
        for key in ("gw1", "gb1", "gw2", "gb2"):
            assert torch.count_nonzero(getattr(g, key)) == 0, key  # es_ops.cpp:202 zeros
        return
    _check_layer(p, x, r, gy, RTOL_BF16 if dtype == torch.bfloat16 else RTOL_F32, "gelu")


def test_layer_routing_validation():
    H = hx()
    p, x = H.make_random_params(2, 8, 16, 8, "gelu", seed=28, n_tokens=4)
    bad = H.RoutingChoice(4, 2, 3, np.zeros((3, 4), np.int32))  # k > E
    with pytest.raises(ValueError):
        H.moe_forward(x, p, bad)
    ok = H.synthesize_routing(4, 2, 1, "uniform", 1)
    with pytest.raises(H.ShapeError):
        H.moe_forward(x[:3], p, ok)


def test_cpp_dropin():
    """The reference's own C++ types and KATs through include/hexamoe_moekit.hpp
    (C++ shim over the C ABI) -- built by oracle/Makefile from the reference
    headers, see INTEGRATION.md."""
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(__file__)), "oracle", "_ref", "dropin_test")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_test not built (needs /root/reference at build time)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout


@pytest.mark.parametrize("n,E,k,blk,dist", [
    (16384, 32, 2, 8, "uniform"),    # c2 routing
    (131072, 64, 2, 8, "uniform"),   # c4 routing
    (777, 5, 3, 3, "zipf:1.2"),
    (10, 4, 4, 1, "uniform"),        # k == E
])
def test_build_reindex_all_bitexact(n, E, k, blk, dist):
    """build_reindex_all (routing.cpp:72-80): one index per choice, all k in
    one batched call, each bit-exact with the reference order."""
    H = hx()
    a = O.synthesize_routing(n, E, k, dist, n + k)
    out = H.build_reindex_all(H.RoutingChoice(n, E, k, a), blk)
    assert len(out) == k
    for i in range(k):
        want = O.build_reindex(a[i], E, blk)
        assert np.array_equal(out[i].idx.cpu().numpy(), want.idx), i
        assert np.array_equal(out[i].v.cpu().numpy(), want.v), i
    bad = a.copy()
    bad[k - 1, n // 2] = E
    with pytest.raises(ValueError):
        H.build_reindex_all(H.RoutingChoice(n, E, k, bad), blk)


def test_op_stats_counters():
    """OpStats (es_ops.hpp:17-24): macs == N*D1*D2 for esmm / estmm, adds ==
    N*D for ess, padding_slots == rx.padding() per operator pass; esfk counts
    its three passes (test_es_ops.cpp:270-287)."""
    H = hx()
    rng = np.random.default_rng(3)
    n, E, d1, d2 = 37, 3, 5, 4
    a = rng.integers(0, E, size=n).astype(np.int32)
    rx = H.build_reindex(a, E, 8)
    pads = rx.padding()
    x = dev(rng.standard_normal((n, d1)))
    g = dev(rng.standard_normal((n, d2)))
    w = dev(rng.standard_normal((E, d1, d2)))
    s = H.OpStats()
    H.esmm(x, w, None, rx, stats=s)
    assert (s.macs, s.adds, s.padding_slots) == (n * d1 * d2, 0, pads)
    s.reset()
    H.ess(g, rx, stats=s)
    assert (s.macs, s.adds, s.padding_slots) == (0, n * d2, pads)
    s.reset()
    H.estmm(x, g, rx, stats=s)
    assert (s.macs, s.adds, s.padding_slots) == (n * d1 * d2, 0, pads)
    s.reset()
    f = H.esfk(x, g, w, rx, w_transposed=True, stats=s)
    assert (s.macs, s.adds, s.padding_slots) == (2 * n * d1 * d2, n * d2, 3 * pads)
    assert s.total_ops() == 2 * n * d1 * d2 + n * d2
    orx = O.build_reindex(a, E, 8)
    assert O.scaled_err(host(f.grad_w), O.estmm(host(x), host(g), orx)) <= RTOL_F32
