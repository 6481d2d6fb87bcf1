"""Pins the C oracle (oracle/moe_oracle.c) before anything is checked against it.

1. the reference's own known-answer tests (tests/golden/kat.json, each entry
   cites the reference test file:line it was transcribed from);
2. bit-for-bit equality with fixtures produced by the unmodified reference
   sources (tests/golden/ref_*.npz, oracle/make_golden.py);
3. when oracle/_ref/libmoekit_ref.so is present, fresh random instances run
   through both.
"""
import json
import os

import numpy as np
import pytest

import oracle as O


@pytest.fixture(scope="module")
def kat(golden_dir):
    with open(os.path.join(golden_dir, "kat.json")) as f:
        return json.load(f)


def test_reindex_kats(kat):
    for c in kat["reindex"]:
        rx = O.build_reindex(c["assignment"], c["E"], c["blk"])
        assert rx.idx.tolist() == c["idx"], c["cite"]
        assert rx.v.tolist() == c["v"], c["cite"]


def test_reindex_errors(kat):
    for c in kat["reindex_errors"]:
        with pytest.raises(ValueError):
            O.build_reindex(c["assignment"], c["E"], c["blk"])


def _rx(c):
    return O.build_reindex(c["assignment"], c["E"], c["blk"])


def test_op_kats(kat):
    for c in kat["esmm"]:
        y = O.esmm(c["x"], c["w"], c["b"], _rx(c))
        assert y.tolist() == c["y"], c["cite"]
    for c in kat["ess"]:
        assert O.ess(c["x"], _rx(c)).tolist() == c["out"], c["cite"]
    for c in kat["estmm"]:
        assert O.estmm(c["x1"], c["x2"], _rx(c)).tolist() == c["out"], c["cite"]


def test_layer_chain_rule(kat):
    c = kat["layer_chain_rule"]
    y, y1, y2 = O.moe_forward(c["x"], c["w1"], c["b1"], c["w2"], c["b2"],
                              c["assignments"], c["blk"], c["act"])
    assert y.tolist() == c["y"]
    g = O.moe_backward(c["x"], c["w1"], c["w2"], c["assignments"], y1, y2, c["g_y"],
                       c["blk"], c["act"])
    for key in ("gx", "gw1", "gw2", "gb1", "gb2"):
        assert g[key].tolist() == c[key], key


def test_rng_stream_matches_reference(golden_dir):
    d = np.load(os.path.join(golden_dir, "ref_rng.npz"))
    lib = O.c_lib()
    import ctypes as C
    r = (C.c_uint64 * 313)()  # orc_rng: 312 words + int
    lib.orc_rng_seed(r, C.c_uint64(1))
    lib.orc_rng_next_u64.restype = C.c_uint64
    got = np.array([lib.orc_rng_next_u64(r) for _ in range(1000)], dtype=np.uint64)
    assert np.array_equal(got, d["u64_seed1"])
    lib.orc_rng_gaussian.restype = C.c_double
    lib.orc_rng_seed(r, C.c_uint64(20240601))
    g = np.array([lib.orc_rng_gaussian(r) for _ in range(200)])
    assert np.array_equal(g, d["gauss_seed20240601"])


def test_reindex_bitexact_vs_reference_fixtures(golden_dir):
    d = np.load(os.path.join(golden_dir, "ref_reindex.npz"))
    for i in range(40):
        E, blk = d[f"r{i}_meta"].tolist()
        rx = O.build_reindex(d[f"r{i}_a"], E, blk)
        assert np.array_equal(rx.v, d[f"r{i}_v"])
        assert np.array_equal(rx.idx, d[f"r{i}_idx"])
    a = d["c2_assign"]
    assert np.array_equal(a, O.synthesize_routing(16384, 32, 2, "uniform", 1))
    for c in range(2):
        rx = O.build_reindex(a[c], 32, 8)
        assert np.array_equal(rx.v, d[f"c2_v{c}"])
        assert np.array_equal(rx.idx, d[f"c2_idx{c}"])
    assert np.array_equal(d["zipf_assign"], O.synthesize_routing(4096, 64, 2, "zipf:1.2", 7))
    assert np.array_equal(d["fixed_assign"], O.synthesize_routing(512, 8, 3, "fixed:2", 5))
    assert np.array_equal(d["balanced_assign"], O.synthesize_routing(100, 7, 2, "balanced", 3))


def test_ops_bitexact_vs_reference_fixtures(golden_dir):
    d = np.load(os.path.join(golden_dir, "ref_ops.npz"))
    for i in range(16):
        g = lambda k: d[f"o{i}_{k}"]
        E, blk = g("meta").tolist()
        rx = O.build_reindex(g("a"), E, blk)
        assert np.array_equal(rx.v, g("v"))
        assert np.array_equal(O.esmm(g("x"), g("w"), g("b"), rx), g("esmm"))
        assert np.array_equal(O.esmm(g("x"), g("w"), None, rx, 1, g("x2")), g("esmm_acc"))
        assert np.array_equal(O.ess(g("x"), rx), g("ess"))
        assert np.array_equal(O.estmm(g("x"), g("x2"), rx), g("estmm"))


def test_layer_bitexact_vs_reference_fixtures(golden_dir):
    d = np.load(os.path.join(golden_dir, "ref_layer.npz"))
    for i in range(5):
        g = lambda k: d[f"l{i}_{k}"]
        E, k, din, hid, dout, n, blk, act = g("meta").tolist()
        actn = {v: kk for kk, v in O.ACT.items()}[act]
        y, y1, y2 = O.moe_forward(g("x"), g("w1"), g("b1"), g("w2"), g("b2"), g("a"), blk, actn)
        assert np.array_equal(y, g("y"))
        assert np.array_equal(y1, g("y1")) and np.array_equal(y2, g("y2"))
        gr = O.moe_backward(g("x"), g("w1"), g("w2"), g("a"), y1, y2, g("gy"), blk, actn)
        for key in ("gw1", "gb1", "gw2", "gb2", "gx"):
            assert np.array_equal(gr[key], g(key)), (i, key)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_random_layers_vs_live_reference():
    rng = np.random.default_rng(20240601)
    for it in range(10):
        E = int(rng.integers(1, 9)); k = int(rng.integers(1, min(E, 3) + 1))
        din, hid, dout = (int(v) for v in rng.integers(1, 13, size=3))
        n = int(rng.integers(1, 65)); blk = int(rng.choice([2, 4, 8]))
        act = ["gelu", "relu", "identity"][it % 3]
        x, w1, b1, w2, b2 = O.ref_make_inputs(it, E, din, hid, dout, n)
        a = O.ref_synthesize_routing(n, E, k, "uniform", 1000 + it)
        assert np.array_equal(a, O.synthesize_routing(n, E, k, "uniform", 1000 + it))
        gy = rng.standard_normal((n, dout))
        ry, ry1, ry2, rg = O.ref_moe_step(x, w1, b1, w2, b2, a, gy, blk, act, fused=bool(it % 2))
        y, y1, y2 = O.moe_forward(x, w1, b1, w2, b2, a, blk, act)
        assert np.array_equal(y, ry)
        gr = O.moe_backward(x, w1, w2, a, y1, y2, gy, blk, act)
        for key in rg:
            assert np.array_equal(gr[key], rg[key]), key


def test_routing_validation_matches_reference():
    ok = O.synthesize_routing(10, 4, 2, "uniform", 3)
    assert O.c_lib().orc_validate_routing(ok, 2, 10, 4) == 0
    dup = ok.copy(); dup[1, 3] = dup[0, 3]
    assert O.c_lib().orc_validate_routing(dup, 2, 10, 4) == 2
    with pytest.raises(ValueError):
        O.synthesize_routing(4, 2, 3)  # k > E (test_routing.cpp:103-106)


# ------------------------------------------------ fast (BLAS) restatement --
@pytest.mark.parametrize("E,k,din,hid,dout,n,act,dist,seed", [
    (8, 1, 24, 40, 16, 300, "gelu", "uniform", 1),
    (16, 2, 32, 48, 32, 500, "gelu", "zipf:1.3", 2),
    (5, 3, 12, 20, 6, 77, "relu", "uniform", 3),
    (32, 2, 16, 16, 16, 40, "identity", "uniform", 4),   # many empty experts
    (4, 2, 8, 8, 8, 0, "gelu", "uniform", 5),            # no tokens
])
def test_fast_oracle_matches_c_oracle(E, k, din, hid, dout, n, act, dist, seed):
    """oracle/fast.py (one BLAS GEMM per expert segment) is pinned to the
    loop-order C oracle at 1e-12 scaled error before the GPU parity tests use
    it at the BASELINE shapes."""
    import fast as F
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, din))
    w1 = 0.5 * rng.standard_normal((E, din, hid)); b1 = rng.standard_normal((E, hid))
    w2 = 0.5 * rng.standard_normal((E, hid, dout)); b2 = rng.standard_normal((E, dout))
    a = O.synthesize_routing(n, E, k, dist, seed) if n else np.zeros((k, 0), np.int32)
    gy = rng.standard_normal((n, dout))
    y, y1, y2 = O.moe_forward(x, w1, b1, w2, b2, a, 8, act)
    g = O.moe_backward(x, w1, w2, a, y1, y2, gy, 8, act)
    fy, fy1, fy2 = F.moe_forward(x, w1, b1, w2, b2, a, act)
    fg = F.moe_backward(x, w1, w2, a, fy1, fy2, gy, act)
    assert O.scaled_err(fy, y) <= 1e-12
    assert O.scaled_err(fy1, y1) <= 1e-12 and O.scaled_err(fy2, y2) <= 1e-12
    for key in ("gw1", "gb1", "gw2", "gb2", "gx"):
        assert O.scaled_err(fg[key], g[key]) <= 1e-12, key
    if n:
        rx = O.build_reindex(a[0], E, 8)
        assert O.scaled_err(F.esmm(x, w1, b1, a[0], E), O.esmm(x, w1, b1, rx)) <= 1e-12
        assert O.scaled_err(F.ess(x, a[0], E), O.ess(x, rx)) <= 1e-12
        assert O.scaled_err(F.estmm(x, gy, a[0], E), O.estmm(x, gy, rx)) <= 1e-12
