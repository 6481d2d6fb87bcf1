"""make_golden.py -- TEST INFRASTRUCTURE ONLY.

Regenerates tests/golden/ref_*.npz by running the UNMODIFIED reference
sources (oracle/_ref/libmoekit_ref.so, built by `make -C oracle` from
/root/reference).  The fixtures travel with the repo so the GPU box (which has
no /root/reference) can check the CUDA path against reference outputs.

    python oracle/make_golden.py
"""
from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def gen_rng():
    lib = O.ref_lib()
    u = np.empty(1000, dtype=np.uint64)
    lib.ref_rng_u64(1, u, 1000)
    g = np.empty(200)
    lib.ref_rng_gaussian(20240601, g, 200)
    np.savez_compressed(os.path.join(OUT, "ref_rng.npz"), u64_seed1=u, gauss_seed20240601=g)


def gen_reindex():
    """Random instances in the style of test_routing.cpp:108-147 plus the c2/c5
    routing at full size (seed 1, synthesize_routing uniform)."""
    d = {}
    rng = np.random.default_rng(321)
    for i in range(40):
        n = int(rng.integers(1, 300))
        E = int(rng.integers(1, 40))
        blk = int(rng.choice([1, 2, 4, 8, 16, 128]))
        a = rng.integers(0, E, size=n).astype(np.int32)
        rx = O.ref_build_reindex(a, E, blk)
        d[f"r{i}_a"], d[f"r{i}_meta"] = a, np.array([E, blk], dtype=np.int64)
        d[f"r{i}_v"], d[f"r{i}_idx"] = rx.v, rx.idx
    # BASELINE.json c2: 32 experts top-2, 16384 tokens, blk 8 (commands.hpp:28)
    a = O.ref_synthesize_routing(16384, 32, 2, "uniform", 1)
    d["c2_assign"] = a
    for c in range(2):
        rx = O.ref_build_reindex(a[c], 32, 8)
        d[f"c2_v{c}"], d[f"c2_idx{c}"] = rx.v, rx.idx
    d["zipf_assign"] = O.ref_synthesize_routing(4096, 64, 2, "zipf:1.2", 7)
    d["fixed_assign"] = O.ref_synthesize_routing(512, 8, 3, "fixed:2", 5)
    d["balanced_assign"] = O.ref_synthesize_routing(100, 7, 2, "balanced", 3)
    np.savez_compressed(os.path.join(OUT, "ref_reindex.npz"), **d)


def gen_ops():
    """Operator instances in the style of test_es_ops.cpp:191-215, outputs from
    the reference esmm / ess / estmm."""
    lib = O.ref_lib()
    d = {}
    rng = np.random.default_rng(11)
    for i in range(16):
        n = int(rng.integers(1, 100))
        E = int(rng.integers(1, 9))
        blk = int(rng.choice([2, 4, 8]))
        d1 = int(rng.integers(1, 40))
        d2 = int(rng.integers(1, 40))
        a = rng.integers(0, E, size=n).astype(np.int32)
        x = rng.standard_normal((n, d1))
        x2 = rng.standard_normal((n, d2))
        w = rng.standard_normal((E, d1, d2))
        b = rng.standard_normal((E, d2))
        rx = O.ref_build_reindex(a, E, blk)
        np_ = len(rx.v)
        mm = np.zeros((n, d2))
        assert lib.ref_esmm(x, n, d1, w, E, d2, b.ctypes.data, rx.v, np_, rx.idx, blk, 0, mm) == 0
        acc = x2.copy()  # accumulate onto a nonzero destination
        assert lib.ref_esmm(x, n, d1, w, E, d2, None, rx.v, np_, rx.idx, blk, 1, acc) == 0
        ss = np.zeros((E, d1))
        assert lib.ref_ess(x, n, d1, rx.v, np_, rx.idx, E, blk, ss) == 0
        tm = np.zeros((E, d1, d2))
        assert lib.ref_estmm(x, x2, n, d1, d2, rx.v, np_, rx.idx, E, blk, tm) == 0
        for key, val in dict(a=a, x=x, x2=x2, w=w, b=b, v=rx.v, idx=rx.idx,
                             meta=np.array([E, blk]), esmm=mm, esmm_acc=acc,
                             ess=ss, estmm=tm).items():
            d[f"o{i}_{key}"] = val
    np.savez_compressed(os.path.join(OUT, "ref_ops.npz"), **d)


def gen_layer():
    """Layer fwd+bwd instances through moe_forward / moe_backward."""
    d = {}
    shapes = [  # (E, k, din, hid, dout, n, blk, act, dist)
        (4, 2, 8, 16, 8, 40, 2, "gelu", "uniform"),
        (8, 1, 12, 24, 12, 64, 8, "gelu", "uniform"),
        (6, 3, 5, 7, 9, 33, 4, "relu", "uniform"),
        (5, 2, 16, 32, 16, 70, 8, "identity", "zipf:1.5"),
        (8, 2, 32, 64, 32, 96, 8, "gelu", "uniform"),
    ]
    for i, (E, k, din, hid, dout, n, blk, act, dist) in enumerate(shapes):
        x, w1, b1, w2, b2 = O.ref_make_inputs(100 + i, E, din, hid, dout, n)
        a = O.ref_synthesize_routing(n, E, k, dist, 200 + i)
        gy = np.random.default_rng(300 + i).standard_normal((n, dout))
        y, y1, y2, g = O.ref_moe_step(x, w1, b1, w2, b2, a, gy, blk, act)
        meta = np.array([E, k, din, hid, dout, n, blk, O.ACT[act]])
        for key, val in dict(x=x, w1=w1, b1=b1, w2=w2, b2=b2, a=a, gy=gy, y=y,
                             y1=y1, y2=y2, meta=meta, **g).items():
            d[f"l{i}_{key}"] = val
    np.savez_compressed(os.path.join(OUT, "ref_layer.npz"), **d)


if __name__ == "__main__":
    O.build()
    os.makedirs(OUT, exist_ok=True)
    gen_rng()
    gen_reindex()
    gen_ops()
    gen_layer()
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)))
