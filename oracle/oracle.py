"""oracle.py -- TEST INFRASTRUCTURE ONLY.

numpy/ctypes front end to the two CPU checkers built by oracle/Makefile:

* ``C``   -- oracle/_build/libmoe_oracle.so, the plain-C fp64 restatement
             (oracle/moe_oracle.c) of the reference hot path;
* ``REF`` -- oracle/_ref/libmoekit_ref.so, the unmodified reference sources
             (/root/reference/proj/core/src/{tensor,routing,es_ops,moe_layer}.cpp)
             behind an extern "C" shim (oracle/ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs import this module.  The product package
(paper_2411_01288_b200/) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_C_PATH = os.path.join(_HERE, "_build", "libmoe_oracle.so")
_REF_PATH = os.path.join(_HERE, "_ref", "libmoekit_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(dtype=np.uint64, flags="C_CONTIGUOUS")
_sz = C.c_size_t

ACT = {"relu": 0, "gelu": 1, "identity": 2}
DIST = {"uniform": 0, "zipf": 1, "fixed": 2, "balanced": 3}


def build() -> None:
    """Compile both checkers (no-op when up to date)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _load(path: str) -> C.CDLL:
    if not os.path.exists(path):
        build()
    return C.CDLL(path)


_c_lib = None
_ref_lib = None


def c_lib() -> C.CDLL:
    global _c_lib
    if _c_lib is None:
        lib = _load(_C_PATH)
        lib.orc_reindex_bound.restype = _sz
        lib.orc_reindex_bound.argtypes = [_sz, _sz, _sz]
        lib.orc_build_reindex.restype = C.c_int64
        lib.orc_build_reindex.argtypes = [_i32p, _sz, _sz, _sz, _i64p, _i64p]
        lib.orc_synthesize_routing.restype = C.c_int
        lib.orc_synthesize_routing.argtypes = [_sz, _sz, _sz, C.c_int, C.c_double,
                                               _sz, C.c_uint64, _i32p]
        lib.orc_validate_routing.restype = C.c_int
        lib.orc_validate_routing.argtypes = [_i32p, _sz, _sz, _sz]
        lib.orc_act_value.restype = C.c_double
        lib.orc_act_value.argtypes = [C.c_int, C.c_double]
        lib.orc_act_derivative.restype = C.c_double
        lib.orc_act_derivative.argtypes = [C.c_int, C.c_double]
        lib.orc_esmm.restype = None
        lib.orc_esmm.argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, C.c_void_p,
                                 _i64p, _i64p, _sz, C.c_int, _dp]
        lib.orc_ess.restype = None
        lib.orc_ess.argtypes = [_dp, _sz, _sz, _i64p, _i64p, _sz, _sz, _dp]
        lib.orc_estmm.restype = None
        lib.orc_estmm.argtypes = [_dp, _dp, _sz, _sz, _sz, _i64p, _i64p, _sz,
                                  _sz, _dp]
        lib.orc_moe_forward.restype = C.c_int
        lib.orc_moe_forward.argtypes = [_dp, _sz, _sz, _sz, _sz, _sz, _dp, _dp,
                                        _dp, _dp, C.c_int, _i32p, _sz, _sz, _dp,
                                        _dp, _dp]
        lib.orc_moe_backward.restype = C.c_int
        lib.orc_moe_backward.argtypes = [_dp, _sz, _sz, _sz, _sz, _sz, _dp, _dp,
                                         C.c_int, _i32p, _sz, _sz, _dp, _dp, _dp,
                                         _dp, _dp, _dp, _dp, _dp]
        lib.orc_random_fill.restype = None
        _c_lib = lib
    return _c_lib


def ref_available() -> bool:
    return os.path.exists(_REF_PATH)


def ref_lib() -> C.CDLL:
    global _ref_lib
    if _ref_lib is None:
        if not os.path.exists(_REF_PATH):
            raise FileNotFoundError(
                f"{_REF_PATH} missing: run `make -C oracle` where /root/reference exists")
        lib = C.CDLL(_REF_PATH)
        lib.ref_last_error.restype = C.c_char_p
        lib.ref_rng_u64.argtypes = [C.c_uint64, _u64p, _sz]
        lib.ref_rng_gaussian.argtypes = [C.c_uint64, _dp, _sz]
        lib.ref_make_inputs.argtypes = [C.c_uint64, _sz, _sz, _sz, _sz, _sz,
                                        C.c_double, _dp, _dp, _dp, _dp, _dp]
        lib.ref_synthesize_routing.restype = C.c_int
        lib.ref_synthesize_routing.argtypes = [_sz, _sz, _sz, C.c_char_p,
                                               C.c_uint64, _i32p]
        lib.ref_validate_routing.restype = C.c_int
        lib.ref_validate_routing.argtypes = [_i32p, _sz, _sz, _sz]
        lib.ref_build_reindex.restype = C.c_int64
        lib.ref_build_reindex.argtypes = [_i32p, _sz, _sz, _sz, _i64p, _i64p]
        lib.ref_esmm.restype = C.c_int
        lib.ref_esmm.argtypes = [_dp, _sz, _sz, _dp, _sz, _sz, C.c_void_p, _i64p,
                                 _sz, _i64p, _sz, C.c_int, _dp]
        lib.ref_ess.restype = C.c_int
        lib.ref_ess.argtypes = [_dp, _sz, _sz, _i64p, _sz, _i64p, _sz, _sz, _dp]
        lib.ref_estmm.restype = C.c_int
        lib.ref_estmm.argtypes = [_dp, _dp, _sz, _sz, _sz, _i64p, _sz, _i64p,
                                  _sz, _sz, _dp]
        lib.ref_moe_step.restype = C.c_int
        lib.ref_moe_step.argtypes = [_dp, _sz, _sz, _sz, _sz, _sz, _dp, _dp, _dp,
                                     _dp, C.c_int, _i32p, _sz, _sz, C.c_void_p,
                                     C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                     _dp]
        lib.ref_time_layer.restype = C.c_double
        lib.ref_time_layer.argtypes = [_sz, _sz, _sz, _sz, _sz, _sz, _sz, C.c_int,
                                       C.c_uint64]
        _ref_lib = lib
    return _ref_lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------- C oracle --
class ReIndex:
    """Host mirror of moekit::ReIndex (routing.hpp:29-38)."""

    def __init__(self, v: np.ndarray, idx: np.ndarray, blk: int, n_tokens: int):
        self.v, self.idx, self.blk, self.n_tokens = v, idx, blk, n_tokens

    @property
    def num_experts(self) -> int:
        return len(self.idx) - 1

    def padding(self) -> int:
        return len(self.v) - self.n_tokens


def build_reindex(assignment, n_experts: int, blk: int) -> ReIndex:
    a = np.ascontiguousarray(assignment, dtype=np.int32)
    lib = c_lib()
    bound = lib.orc_reindex_bound(len(a), n_experts, max(blk, 1))
    v = np.empty(max(bound, 1), dtype=np.int64)
    idx = np.empty(n_experts + 1, dtype=np.int64)
    np_ = lib.orc_build_reindex(a, len(a), n_experts, blk, v, idx)
    if np_ < 0:
        raise ValueError("build_reindex: blk must be >= 1 and ids in range")
    return ReIndex(v[:np_].copy(), idx, blk, len(a))


def synthesize_routing(n, n_experts, k, dist="uniform", seed=1) -> np.ndarray:
    kind, s, fixed = DIST["uniform"], 1.0, 0
    if dist.startswith("zipf:"):
        kind, s = DIST["zipf"], float(dist[5:])
    elif dist.startswith("fixed:"):
        kind, fixed = DIST["fixed"], int(dist[6:])
    elif dist == "balanced":
        kind = DIST["balanced"]
    out = np.empty((k, n), dtype=np.int32)
    if c_lib().orc_synthesize_routing(n, n_experts, k, kind, s, fixed, seed, out) != 0:
        raise ValueError("synthesize_routing: invalid arguments")
    return out


def esmm(x, w, bias, rx: ReIndex, mode=0, dest=None) -> np.ndarray:
    x, w = _f64(x), _f64(w)
    n, d1 = x.shape
    E, _, d2 = w.shape
    out = np.zeros((n, d2)) if dest is None else _f64(dest).copy()
    b = None if bias is None else _f64(bias)
    c_lib().orc_esmm(x, n, d1, w, E, d2, None if b is None else b.ctypes.data,
                     rx.v, rx.idx, rx.blk, mode, out)
    return out


def ess(x, rx: ReIndex) -> np.ndarray:
    x = _f64(x)
    n, d = x.shape
    out = np.zeros((rx.num_experts, d))
    c_lib().orc_ess(x, n, d, rx.v, rx.idx, rx.num_experts, rx.blk, out)
    return out


def estmm(x1, x2, rx: ReIndex) -> np.ndarray:
    x1, x2 = _f64(x1), _f64(x2)
    n, d1 = x1.shape
    d2 = x2.shape[1]
    out = np.zeros((rx.num_experts, d1, d2))
    c_lib().orc_estmm(x1, x2, n, d1, d2, rx.v, rx.idx, rx.num_experts, rx.blk, out)
    return out


def moe_forward(x, w1, b1, w2, b2, assignments, blk=8, act="gelu"):
    """Returns (y, y1[k,n,H], y2[k,n,H])."""
    x, w1, b1, w2, b2 = map(_f64, (x, w1, b1, w2, b2))
    a = np.ascontiguousarray(assignments, dtype=np.int32)
    k, n = a.shape
    E, din, hid = w1.shape
    dout = w2.shape[2]
    y = np.zeros((n, dout))
    y1 = np.zeros((k, n, hid))
    y2 = np.zeros((k, n, hid))
    rc = c_lib().orc_moe_forward(x, n, din, hid, dout, E, w1, b1, w2, b2, ACT[act],
                                 a, k, blk, y, y1, y2)
    if rc != 0:
        raise ValueError("moe_forward: invalid routing")
    return y, y1, y2


def moe_backward(x, w1, w2, assignments, y1, y2, g_y, blk=8, act="gelu"):
    """Returns dict gw1, gb1, gw2, gb2, gx."""
    x, w1, w2, y1, y2, g_y = map(_f64, (x, w1, w2, y1, y2, g_y))
    a = np.ascontiguousarray(assignments, dtype=np.int32)
    k, n = a.shape
    E, din, hid = w1.shape
    dout = w2.shape[2]
    g = dict(gw1=np.zeros((E, din, hid)), gb1=np.zeros((E, hid)),
             gw2=np.zeros((E, hid, dout)), gb2=np.zeros((E, dout)),
             gx=np.zeros((n, din)))
    c_lib().orc_moe_backward(x, n, din, hid, dout, E, w1, w2, ACT[act], a, k, blk,
                             y1, y2, g_y, g["gw1"], g["gb1"], g["gw2"], g["gb2"],
                             g["gx"])
    return g


def act_value(act: str, x: float) -> float:
    return c_lib().orc_act_value(ACT[act], x)


def act_derivative(act: str, x: float) -> float:
    return c_lib().orc_act_derivative(ACT[act], x)


def scaled_err(a, ref) -> float:
    """Reference tolerance form max|a-b| / (1 + max|b|) (tests/support/test_oracles.hpp:60-62)."""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(a - ref)) / (1.0 + np.max(np.abs(ref))))


# ------------------------------------------------------ reference (REF) --
def ref_make_inputs(seed, E, din, hid, dout, n, scale=0.5):
    """make_random_params(..., scale) then random_matrix(n, din) (moe_layer.cpp:136-147)."""
    w1 = np.empty((E, din, hid)); b1 = np.empty((E, hid))
    w2 = np.empty((E, hid, dout)); b2 = np.empty((E, dout)); x = np.empty((n, din))
    ref_lib().ref_make_inputs(seed, E, din, hid, dout, n, scale, w1, b1, w2, b2, x)
    return x, w1, b1, w2, b2


def ref_synthesize_routing(n, E, k, dist="uniform", seed=1) -> np.ndarray:
    out = np.empty((k, n), dtype=np.int32)
    rc = ref_lib().ref_synthesize_routing(n, E, k, dist.encode(), seed, out)
    if rc != 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return out


def ref_build_reindex(assignment, E, blk):
    a = np.ascontiguousarray(assignment, dtype=np.int32)
    bound = len(a) + E * max(blk - 1, 0)
    v = np.empty(max(bound, 1), dtype=np.int64)
    idx = np.empty(E + 1, dtype=np.int64)
    r = ref_lib().ref_build_reindex(a, len(a), E, blk, v, idx)
    if r < 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return ReIndex(v[:r].copy(), idx, blk, len(a))


def ref_moe_step(x, w1, b1, w2, b2, assignments, g_y, blk=8, act="gelu", fused=False):
    x, w1, b1, w2, b2 = map(_f64, (x, w1, b1, w2, b2))
    a = np.ascontiguousarray(assignments, dtype=np.int32)
    k, n = a.shape
    E, din, hid = w1.shape
    dout = w2.shape[2]
    y = np.zeros((n, dout)); y1 = np.zeros((k, n, hid)); y2 = np.zeros((k, n, hid))
    g = dict(gw1=np.zeros((E, din, hid)), gb1=np.zeros((E, hid)),
             gw2=np.zeros((E, hid, dout)), gb2=np.zeros((E, dout)),
             gx=np.zeros((n, din)))
    gy = None if g_y is None else _f64(g_y)
    rc = ref_lib().ref_moe_step(x, n, din, hid, dout, E, w1, b1, w2, b2, ACT[act], a,
                                k, blk, None if gy is None else gy.ctypes.data,
                                int(fused), y, y1, y2, g["gw1"], g["gb1"], g["gw2"],
                                g["gb2"], g["gx"])
    if rc != 0:
        raise ValueError(ref_lib().ref_last_error().decode())
    return y, y1, y2, g


def ref_time_layer(E, k, din, hid, dout, n_sample, blk=8, threads=1, seed=1) -> float:
    return ref_lib().ref_time_layer(E, k, din, hid, dout, n_sample, blk, threads, seed)
