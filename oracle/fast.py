"""fast.py -- TEST INFRASTRUCTURE ONLY: a numpy fp64 restatement of the
reference MoE layer for parity checks at the BASELINE.json shapes.

The C restatement (moe_oracle.c) keeps the reference's loop order so it can be
pinned bit-for-bit against the reference itself; that order streams W[e] once
per token (es_ops.cpp:61-72) and runs at ~1 GMAC/s, i.e. minutes to hours at
c2 full N and at the d1024 / ffn4096 dims.  This module computes the same
functions with one BLAS GEMM per expert segment (numpy fp64): only the
summation order differs, so it agrees with the C oracle to ~1e-13 scaled
error (pinned by tests/test_oracle.py::test_fast_oracle_matches_c_oracle at
1e-12) -- nine orders of magnitude inside the 2e-2 bf16 bar it checks.

Semantics followed (reference file:line):
  * routing / grouping: build_reindex (routing.cpp:42-70): per expert, the
    tokens routed to it in ascending token order; pads contribute nothing.
  * ESMM (es_ops.cpp:47-81): row_t = b[e] + x[t] . W[e].
  * activations (tensor.cpp:39-104): GELU-tanh and its exact derivative,
    ReLU, identity.
  * moe_forward (moe_layer.cpp:30-67): y = sum_i ESMM(F(ESMM(x, W1, b1, R_i)),
    W2, b2, R_i) -- unweighted, b2 once per choice.
  * moe_backward (moe_layer.cpp:69-122): per choice gb2 += ESS(g_y),
    gW2 += ESTMM(y2_i, g_y), g_y2 = ESMM(g_y, W2^T), g_y1 = g_y2 * F'(y1_i),
    gb1 += ESS(g_y1), gW1 += ESTMM(x, g_y1), gx += ESMM(g_y1, W1^T).
Nothing in the product package imports this module.
"""
from __future__ import annotations

import numpy as np

_C = 0.7978845608028654  # sqrt(2/pi), tensor.cpp:39
_K = 0.044715            # tensor.cpp:40


def act_value(act: str, x: np.ndarray) -> np.ndarray:
    """activation_value (tensor.cpp:56-67)."""
    if act == "gelu":
        return 0.5 * x * (1.0 + np.tanh(_C * (x + _K * x * x * x)))
    if act == "relu":
        return np.where(x > 0.0, x, 0.0)
    return x.copy()


def act_derivative(act: str, x: np.ndarray) -> np.ndarray:
    """activation_derivative (tensor.cpp:48-53, 69-80)."""
    if act == "gelu":
        t = np.tanh(_C * (x + _K * x * x * x))
        return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * (_C * (1.0 + 3.0 * _K * x * x))
    if act == "relu":
        return (x > 0.0).astype(np.float64)
    return np.ones_like(x)


def segments(assignment: np.ndarray, n_experts: int):
    """Per expert, its tokens in ascending order (build_reindex's segment
    contents without the -1 pads, routing.cpp:64-68)."""
    a = np.asarray(assignment, dtype=np.int64)
    order = np.argsort(a, kind="stable")
    bounds = np.searchsorted(a[order], np.arange(n_experts + 1))
    return [order[bounds[e]:bounds[e + 1]] for e in range(n_experts)]


def moe_forward(x, w1, b1, w2, b2, assignments, act="gelu"):
    """Returns (y, y1[k, n, H], y2[k, n, H]) like oracle.moe_forward."""
    x = np.asarray(x, np.float64)
    w1, b1 = np.asarray(w1, np.float64), np.asarray(b1, np.float64)
    w2 = np.asarray(w2, np.float64)
    b2 = None if b2 is None else np.asarray(b2, np.float64)
    a = np.asarray(assignments)
    k, n = a.shape
    E, _, H = w1.shape
    Do = w2.shape[2]
    y = np.zeros((n, Do))
    y1 = np.zeros((k, n, H))
    y2 = np.zeros((k, n, H))
    for i in range(k):
        for e, tok in enumerate(segments(a[i], E)):
            if tok.size == 0:
                continue
            pre = x[tok] @ w1[e] + b1[e]
            post = act_value(act, pre)
            y1[i, tok] = pre
            y2[i, tok] = post
            out = post @ w2[e]
            if b2 is not None:
                out += b2[e]
            y[tok] += out
    return y, y1, y2


def moe_backward(x, w1, w2, assignments, y1, y2, g_y, act="gelu", add_b2=True):
    """Returns dict gw1, gb1, gw2, gb2, gx like oracle.moe_backward."""
    x = np.asarray(x, np.float64)
    w1, w2 = np.asarray(w1, np.float64), np.asarray(w2, np.float64)
    g_y = np.asarray(g_y, np.float64)
    a = np.asarray(assignments)
    k, n = a.shape
    E, Di, H = w1.shape
    Do = w2.shape[2]
    g = dict(gw1=np.zeros((E, Di, H)), gb1=np.zeros((E, H)), gw2=np.zeros((E, H, Do)),
             gb2=np.zeros((E, Do)), gx=np.zeros((n, Di)))
    for i in range(k):
        for e, tok in enumerate(segments(a[i], E)):
            if tok.size == 0:
                continue
            gy = g_y[tok]
            if add_b2:
                g["gb2"][e] += gy.sum(axis=0)
            g["gw2"][e] += y2[i, tok].T @ gy
            gy1 = (gy @ w2[e].T) * act_derivative(act, y1[i, tok])
            g["gb1"][e] += gy1.sum(axis=0)
            g["gw1"][e] += x[tok].T @ gy1
            g["gx"][tok] += gy1 @ w1[e].T
    return g


def esmm(x, w, bias, assignment, n_experts):
    """Single-choice ESMM (es_ops.cpp:47-81), write mode."""
    x, w = np.asarray(x, np.float64), np.asarray(w, np.float64)
    out = np.zeros((x.shape[0], w.shape[2]))
    for e, tok in enumerate(segments(assignment, n_experts)):
        if tok.size:
            out[tok] = x[tok] @ w[e] + (0.0 if bias is None else np.asarray(bias)[e])
    return out


def ess(x, assignment, n_experts):
    """ESS (es_ops.cpp:86-102)."""
    x = np.asarray(x, np.float64)
    out = np.zeros((n_experts, x.shape[1]))
    for e, tok in enumerate(segments(assignment, n_experts)):
        if tok.size:
            out[e] = x[tok].sum(axis=0)
    return out


def estmm(x1, x2, assignment, n_experts):
    """ESTMM (es_ops.cpp:106-128)."""
    x1, x2 = np.asarray(x1, np.float64), np.asarray(x2, np.float64)
    out = np.zeros((n_experts, x1.shape[1], x2.shape[1]))
    for e, tok in enumerate(segments(assignment, n_experts)):
        if tok.size:
            out[e] = x1[tok].T @ x2[tok]
    return out
