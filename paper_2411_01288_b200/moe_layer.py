"""MoE FFN layer forward / backward on the GPU.

Mirrors core/include/moekit/moe_layer.hpp:13-89: ``MoeLayerParams``,
``ForwardStash``, ``MoeGrads``, ``moe_forward`` (moe_layer.cpp:30-67),
``moe_backward`` (moe_layer.cpp:69-122), ``estimate_activation_memory``
(moe_layer.cpp:124-134) and ``make_random_params`` (moe_layer.cpp:136-147).
All compute is the C ABI hxm_moe_forward / hxm_moe_backward (layer.cu).
"""
from __future__ import annotations

import math

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import ACT, LayerDesc, ShapeError, check, lib
from .routing import RoutingChoice, _require_cuda, _stream

SCHEMES = ("naive", "memory_efficient")


def moe_scheme_from_name(name: str) -> str:
    if name not in SCHEMES:
        raise ValueError("unknown scheme: " + name)
    return name


@dataclass
class MoeLayerParams:
    """w1 E x D_i x H, b1 E x H, w2 E x H x D_o, b2 E x D_o (moe_layer.hpp:20-37)."""
    w1: torch.Tensor
    b1: torch.Tensor
    w2: torch.Tensor
    b2: Optional[torch.Tensor]
    activation: str = "gelu"

    def experts(self) -> int:
        return self.w1.shape[0]

    def d_in(self) -> int:
        return self.w1.shape[1]

    def hidden(self) -> int:
        return self.w1.shape[2]

    def d_out(self) -> int:
        return self.w2.shape[2]

    def param_elements(self) -> int:
        n = self.w1.numel() + self.b1.numel() + self.w2.numel()
        return n + (self.b2.numel() if self.b2 is not None else 0)

    def validate(self) -> None:
        """moe_layer.cpp:17-28."""
        e = self.w1.shape[0]
        if self.b1.shape[0] != e or self.w2.shape[0] != e or (
                self.b2 is not None and self.b2.shape[0] != e):
            raise ShapeError("MoeLayerParams: expert counts disagree")
        if self.b1.shape[1] != self.w1.shape[2] or self.w2.shape[1] != self.w1.shape[2]:
            raise ShapeError("MoeLayerParams: hidden sizes disagree")
        if self.b2 is not None and self.b2.shape[1] != self.w2.shape[2]:
            raise ShapeError("MoeLayerParams: b2 cols != W2 output dim")
        if self.activation not in ACT:
            raise ValueError("unknown activation: " + self.activation)


@dataclass
class ForwardStash:
    """Device stash: x, the combined index and y1/y2 in expert-sorted order
    (inside ``workspace``), as moekit::ForwardStash (moe_layer.hpp:39-46)."""
    desc: LayerDesc
    workspace: torch.Tensor
    x: torch.Tensor
    scheme: str
    blk: int

    def export(self, choice: int):
        """(F'(y1_i), y2_i) in token order, fp32 N x H (for parity checks).
        The device stash keeps F'(y1) instead of y1: it is all the backward
        needs of y1 (moe_layer.cpp:108) and saves recomputing F'."""
        d = self.desc
        y1 = torch.empty(d.n_tokens, d.hidden, dtype=torch.float32, device=self.x.device)
        y2 = torch.empty_like(y1)
        check(lib().hxm_moe_stash_export(C.byref(d), self.workspace.data_ptr(), choice,
                                         y1.data_ptr(), y2.data_ptr(), _stream()),
              "stash_export")
        return y1, y2


@dataclass
class MoeGrads:
    gw1: torch.Tensor
    gb1: torch.Tensor
    gw2: torch.Tensor
    gb2: Optional[torch.Tensor]
    gx: torch.Tensor


@dataclass
class MoeForwardResult:
    y: torch.Tensor
    stash: ForwardStash


def _dtype_code(t):
    if t.dtype == torch.bfloat16:
        return _lib.HXM_BF16
    if t.dtype == torch.float32:
        return _lib.HXM_F32
    raise ValueError(f"unsupported dtype {t.dtype}")


def make_desc(n_tokens, n_experts, k, d_in, hidden, d_out, activation="gelu",
              dtype=torch.bfloat16, add_b2=True, capacity: int = 0) -> LayerDesc:
    """capacity > 0 selects the conventional dispatch/combine baseline
    (per-expert buffers of exactly ``capacity`` rows; see capacity_rows())."""
    d = LayerDesc()
    d.n_tokens, d.n_experts, d.k = n_tokens, n_experts, k
    d.d_in, d.hidden, d.d_out = d_in, hidden, d_out
    d.activation = ACT[activation]
    d.dtype = _lib.HXM_BF16 if dtype == torch.bfloat16 else _lib.HXM_F32
    d.add_b2 = int(add_b2)
    d.capacity = int(capacity)
    return d


def capacity_rows(n_tokens: int, n_experts: int, k: int, capacity_factor: float) -> int:
    """Per-expert rows of the conventional formulation: ceil(cf * k * N / E)
    (gemm_oracle.cpp:268-271), rounded up to the 64-row segment granule of
    the device layout (the extra rows are padding too)."""
    if capacity_factor <= 0.0:
        raise ValueError("count_redundancy: capacity_factor must be > 0")
    c = int(math.ceil(capacity_factor * k * n_tokens / n_experts))
    return max(64, (c + 63) // 64 * 64)


def layer_workspace(desc: LayerDesc, device="cuda") -> torch.Tensor:
    b = lib().hxm_layer_workspace_bytes(C.byref(desc))
    if b == 0:
        raise ValueError("invalid layer descriptor")
    return torch.empty(b, dtype=torch.uint8, device=device)


def moe_forward(x: torch.Tensor, p: MoeLayerParams, r, blk: int = 8,
                scheme: str = "memory_efficient", validate: bool = True,
                workspace: Optional[torch.Tensor] = None,
                y: Optional[torch.Tensor] = None, capacity: int = 0) -> MoeForwardResult:
    """y = sum_i ESMM(F(ESMM(x, W1, b1, R_i)), W2, b2, R_i) (moe_layer.cpp:30-67).

    ``r`` is a RoutingChoice (host) or a device int32 k x N tensor.  Both
    schemes give the same result; on the device both accumulate (the
    memory-efficient scheme, moe_layer.cpp:61-63).  ``blk`` is the reference
    re-index tile size; results do not depend on it (padding neutrality,
    test_es_ops.cpp:250-268) and it is only validated.

    ``capacity`` > 0 runs the conventional dispatch/combine baseline instead
    (fixed per-expert buffers of ``capacity`` rows, overflow dropped; see
    conventional.py) -- for measurement against the expert-specific path.
    """
    p.validate()
    moe_scheme_from_name(scheme)
    if blk <= 0:
        raise ValueError("build_reindex: blk must be >= 1")
    if isinstance(r, RoutingChoice):
        if validate:
            r.validate()
        a = r.to_device(x.device)
        k, n, n_experts = r.k, r.n_tokens, r.n_experts
    else:
        a = r
        k, n = a.shape
        n_experts = p.experts()
    _require_cuda(x, "x")
    if x.shape[0] != n:
        raise ShapeError("moe_forward: x rows != routed token count")
    if x.shape[1] != p.d_in():
        raise ShapeError("moe_forward: x cols != layer input size")
    if n_experts != p.experts():
        raise ShapeError("moe_forward: routing expert count != layer experts")
    desc = make_desc(n, p.experts(), k, p.d_in(), p.hidden(), p.d_out(), p.activation,
                     x.dtype, p.b2 is not None, capacity)
    ws = workspace if workspace is not None else layer_workspace(desc, x.device)
    if y is None:
        y = torch.empty(n, p.d_out(), dtype=torch.float32, device=x.device)
    status = torch.zeros(1, dtype=torch.int32, device=x.device) if validate else None
    b1 = p.b1.to(torch.float32).contiguous()
    b2 = p.b2.to(torch.float32).contiguous() if p.b2 is not None else None
    check(lib().hxm_moe_forward(C.byref(desc), x.contiguous().data_ptr(), p.w1.data_ptr(),
                                b1.data_ptr(), p.w2.data_ptr(),
                                None if b2 is None else b2.data_ptr(),
                                a.to(torch.int32).contiguous().data_ptr(), y.data_ptr(),
                                ws.data_ptr(), ws.numel(),
                                None if status is None else status.data_ptr(), _stream()),
          "moe_forward")
    if status is not None and int(status.item()) != 0:
        raise ValueError("RoutingChoice: expert id out of range or duplicate expert")
    return MoeForwardResult(y, ForwardStash(desc, ws, x, scheme, blk))


def moe_backward(stash: ForwardStash, p: MoeLayerParams, g_y: torch.Tensor,
                 use_fused: bool = False, grads: Optional[MoeGrads] = None) -> MoeGrads:
    """All five gradients for upstream g_y (moe_layer.cpp:69-122).  ``use_fused``
    is accepted for API parity: the device backward always runs the fused
    schedule (the reference proves both bit-identical)."""
    p.validate()
    d = stash.desc
    if g_y.shape[0] != stash.x.shape[0] or g_y.shape[1] != p.d_out():
        raise ShapeError("moe_backward: g_y shape must be N x D_o")
    if stash.x.shape[1] != p.d_in() or d.hidden != p.hidden():
        raise ShapeError("moe_backward: stash does not match params")
    dev = g_y.device
    if grads is None:
        E, Di, H, Do = p.experts(), p.d_in(), p.hidden(), p.d_out()
        f = dict(dtype=torch.float32, device=dev)
        grads = MoeGrads(torch.empty(E, Di, H, **f), torch.empty(E, H, **f),
                         torch.empty(E, H, Do, **f),
                         torch.empty(E, Do, **f) if d.add_b2 else None,
                         torch.empty(stash.x.shape[0], Di, **f))
    g_y = g_y.to(stash.x.dtype).contiguous()
    check(lib().hxm_moe_backward(C.byref(d), stash.x.data_ptr(), p.w1.data_ptr(),
                                 p.w2.data_ptr(), g_y.data_ptr(), stash.workspace.data_ptr(),
                                 stash.workspace.numel(), grads.gw1.data_ptr(),
                                 grads.gb1.data_ptr(), grads.gw2.data_ptr(),
                                 None if grads.gb2 is None else grads.gb2.data_ptr(),
                                 grads.gx.data_ptr(), _stream()), "moe_backward")
    return grads


def estimate_activation_memory(n_tokens: int, k: int, hidden_ratio: float = 4.0,
                               scheme: str = "memory_efficient") -> float:
    """moe_layer.cpp:124-134 (token units)."""
    if n_tokens == 0:
        return 0.0
    hidden = k * hidden_ratio * n_tokens
    return hidden + k * n_tokens + n_tokens if scheme == "naive" else hidden + n_tokens


def make_random_params(experts, d_in, hidden, d_out, activation="gelu", seed=1, scale=0.5,
                       n_tokens=0, dtype=torch.bfloat16, device="cuda"):
    """make_random_params (moe_layer.cpp:136-147) from Rng(seed), then
    random_matrix(n_tokens, d_in) from the same stream (commands.cpp:174-176).
    Returns (MoeLayerParams, x or None).  Weights and x are rounded to
    ``dtype``; biases stay fp32."""
    w1 = np.empty((experts, d_in, hidden), np.float32)
    b1 = np.empty((experts, hidden), np.float32)
    w2 = np.empty((experts, hidden, d_out), np.float32)
    b2 = np.empty((experts, d_out), np.float32)
    x = np.empty((max(n_tokens, 0), d_in), np.float32)
    lib().hxm_make_layer_inputs(seed, experts, d_in, hidden, d_out, n_tokens, scale,
                                w1.ctypes.data, b1.ctypes.data, w2.ctypes.data,
                                b2.ctypes.data, x.ctypes.data)
    t = lambda a, dt: torch.from_numpy(a).to(device=device, dtype=dt)
    p = MoeLayerParams(t(w1, dtype), t(b1, torch.float32), t(w2, dtype), t(b2, torch.float32),
                       activation)
    return p, (t(x, dtype) if n_tokens > 0 else None)
