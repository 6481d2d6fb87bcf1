"""Expert-specific operators: ESMM, ESS, ESTMM, ESFK on the GPU.

Mirrors the reference operator API (core/include/moekit/es_ops.hpp:37-65):
same names, argument meaning, output shapes and exception types
(ShapeError for shape mismatches, ValueError for domain errors), checked in
the reference's order (es_ops.cpp:140-165, 180-186, 193-201, 210-221).
Tensors are CUDA tensors; bf16 inputs run on the tcgen05 tensor cores with
fp32 accumulation, fp32 inputs on fp32 FMA.  Outputs are fp32.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import HXM_ACCUMULATE, HXM_WRITE, ShapeError, check, lib
from .routing import ReIndex, _require_cuda, _stream

WRITE, ACCUMULATE = "write", "accumulate"  # moekit::EsOutputMode (es_ops.hpp:13)

HXM_OP_ESMM, HXM_OP_ESS, HXM_OP_ESTMM, HXM_OP_ESFK = range(4)


class _CStats(C.Structure):
    _fields_ = [("macs", C.c_uint64), ("adds", C.c_uint64), ("padding_slots", C.c_uint64)]


@dataclass
class OpStats:
    """moekit::OpStats (es_ops.hpp:17-24): token-granular work counters.
    Padding slots contribute nothing, so ``macs`` counts real-token MACs only.
    Pass one as ``stats=`` to an operator to accumulate its counts (the
    counters follow the index, computed by hxm_op_stats_add)."""
    macs: int = 0
    adds: int = 0
    padding_slots: int = 0

    def total_ops(self) -> int:
        return self.macs + self.adds

    def reset(self) -> None:
        self.macs = self.adds = self.padding_slots = 0


def _count(stats, op: int, rx: ReIndex, d1: int, d2: int) -> None:
    if stats is None:
        return
    c = _CStats(stats.macs, stats.adds, stats.padding_slots)
    pad = rx.padded_len() - rx.n_tokens
    lib().hxm_op_stats_add(op, rx.n_tokens, pad, d1, d2, C.byref(c))
    stats.macs, stats.adds, stats.padding_slots = c.macs, c.adds, c.padding_slots


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return _lib.HXM_BF16
    if t.dtype == torch.float32:
        return _lib.HXM_F32
    raise ValueError(f"unsupported dtype {t.dtype} (bf16 or fp32)")


def _ws(rx: ReIndex, d1: int, d2: int) -> torch.Tensor:
    b = lib().hxm_op_workspace_bytes(rx.n_tokens, rx.num_experts(), _bound(rx), d1, d2)
    return torch.empty(max(b, 1), dtype=torch.uint8, device=rx.idx.device)


def _bound(rx: ReIndex) -> int:
    return max(rx.bound, rx.v.numel())


def _check_reindex(rx: ReIndex) -> None:
    # check_reindex (es_ops.cpp:12-17): structural part checkable without a sync
    if rx.idx.numel() < 2:
        raise ShapeError("es-ops: malformed re-index vector")


def esmm(x: torch.Tensor, weights: torch.Tensor, bias, rx: ReIndex, mode=WRITE, dest=None,
         w_transposed: bool = False, stats: OpStats | None = None) -> torch.Tensor:
    """y[t] = x[t] . W[e(t)] + b[e(t)]  (es_ops.hpp:39-46).

    mode "write" returns a new N x D2 fp32 tensor (or writes ``dest``);
    "accumulate" adds into ``dest`` (required).  ``w_transposed`` reads
    ``weights`` (E x D2 x D1) as W^T instead of materialising
    transpose_experts.
    """
    _check_reindex(rx)
    for t, nm in ((x, "x"), (weights, "weights")):
        _require_cuda(t, nm)
    if x.dim() != 2 or x.shape[0] != rx.n_tokens:
        raise ShapeError("esmm: token count does not match re-index vector")
    if weights.dim() != 3 or weights.shape[0] != rx.num_experts():
        raise ShapeError("esmm: expert count mismatch between weights and rx")
    d1 = weights.shape[2] if w_transposed else weights.shape[1]
    d2 = weights.shape[1] if w_transposed else weights.shape[2]
    if x.shape[1] != d1:
        raise ShapeError("esmm: x cols != weights dim1")
    if bias is not None and tuple(bias.shape) != (weights.shape[0], d2):
        raise ShapeError("esmm: bias shape must be E x D2")
    if mode == ACCUMULATE and dest is None:
        raise ValueError("esmm: Accumulate mode requires a destination")
    if dest is None:
        dest = torch.empty(x.shape[0], d2, dtype=torch.float32, device=x.device)
    elif tuple(dest.shape) != (x.shape[0], d2) or dest.dtype != torch.float32:
        raise ShapeError("esmm: destination shape must be N x D2")
    if weights.dtype != x.dtype:
        raise ValueError("esmm: x and weights must share a dtype")
    x, weights = x.contiguous(), weights.contiguous()
    b = None if bias is None else bias.to(torch.float32).contiguous()
    ws = _ws(rx, d1, d2)
    check(lib().hxm_esmm(_dtype_code(x), x.data_ptr(), x.shape[0], d1, weights.data_ptr(),
                         weights.shape[0], d2, int(w_transposed),
                         None if b is None else b.data_ptr(), rx.v.data_ptr(),
                         rx.idx.data_ptr(), _bound(rx),
                         HXM_ACCUMULATE if mode == ACCUMULATE else HXM_WRITE,
                         dest.data_ptr(), ws.data_ptr(), ws.numel(), _stream()), "esmm")
    _count(stats, HXM_OP_ESMM, rx, d1, d2)
    return dest


def ess(x: torch.Tensor, rx: ReIndex, stats: OpStats | None = None) -> torch.Tensor:
    """out[e] = sum of rows routed to e (es_ops.hpp:49)."""
    _check_reindex(rx)
    _require_cuda(x, "x")
    if x.dim() != 2 or x.shape[0] != rx.n_tokens:
        raise ShapeError("ess: token count does not match re-index vector")
    x = x.contiguous()
    E, d = rx.num_experts(), x.shape[1]
    out = torch.empty(E, d, dtype=torch.float32, device=x.device)
    ws = _ws(rx, d, d)
    check(lib().hxm_ess(_dtype_code(x), x.data_ptr(), x.shape[0], d, rx.v.data_ptr(),
                        rx.idx.data_ptr(), E, _bound(rx), out.data_ptr(), ws.data_ptr(),
                        ws.numel(), _stream()), "ess")
    _count(stats, HXM_OP_ESS, rx, d, 0)
    return out


def estmm(x1: torch.Tensor, x2: torch.Tensor, rx: ReIndex,
          stats: OpStats | None = None) -> torch.Tensor:
    """out[e] = sum_{t in e} outer(x1[t], x2[t]) (es_ops.hpp:52-53)."""
    _check_reindex(rx)
    _require_cuda(x1, "x1")
    _require_cuda(x2, "x2")
    if x1.shape[0] != x2.shape[0]:
        raise ShapeError("estmm: x1 and x2 token counts differ")
    if x1.shape[0] != rx.n_tokens:
        raise ShapeError("estmm: token count does not match re-index vector")
    if x1.dtype != x2.dtype:
        raise ValueError("estmm: x1 and x2 must share a dtype")
    x1, x2 = x1.contiguous(), x2.contiguous()
    E, d1, d2 = rx.num_experts(), x1.shape[1], x2.shape[1]
    out = torch.empty(E, d1, d2, dtype=torch.float32, device=x1.device)
    ws = _ws(rx, d1, d2)
    check(lib().hxm_estmm(_dtype_code(x1), x1.data_ptr(), x2.data_ptr(), x1.shape[0], d1, d2,
                          rx.v.data_ptr(), rx.idx.data_ptr(), E, _bound(rx), out.data_ptr(),
                          ws.data_ptr(), ws.numel(), _stream()), "estmm")
    _count(stats, HXM_OP_ESTMM, rx, d1, d2)
    return out


@dataclass
class EsfkResult:
    grad_x: torch.Tensor  # esmm(g, w_t, null)
    grad_b: torch.Tensor  # ess(g)
    grad_w: torch.Tensor  # estmm(x, g)


def esfk(x: torch.Tensor, g: torch.Tensor, w_t: torch.Tensor, rx: ReIndex,
         w_transposed: bool = False, stats: OpStats | None = None) -> EsfkResult:
    """Fused backward of one MLP (es_ops.hpp:55-65).  ``w_t`` is E x D2 x D1
    as in the reference; with ``w_transposed`` pass the forward weights
    E x D1 x D2 instead (no transpose copy)."""
    _check_reindex(rx)
    if x.shape[0] != g.shape[0]:
        raise ShapeError("esfk: x and g token counts differ")
    if x.shape[0] != rx.n_tokens:
        raise ShapeError("esfk: token count does not match re-index vector")
    wd1 = w_t.shape[2] if w_transposed else w_t.shape[1]
    if w_t.shape[0] != rx.num_experts() or wd1 != g.shape[1]:
        raise ShapeError("esfk: w_t must be E x D2 x D1 for g of width D2")
    for t, nm in ((x, "x"), (g, "g"), (w_t, "w_t")):
        _require_cuda(t, nm)
    if x.dtype != g.dtype or w_t.dtype != g.dtype:
        raise ValueError("esfk: x, g and w_t must share a dtype")
    x, g, w_t = x.contiguous(), g.contiguous(), w_t.contiguous()
    n, d1, d2, E = x.shape[0], x.shape[1], g.shape[1], rx.num_experts()
    wd2 = w_t.shape[1] if w_transposed else w_t.shape[2]
    if wd2 != d1:
        raise ShapeError("esfk: w_t must be E x D2 x D1 for g of width D2")
    f = dict(dtype=torch.float32, device=x.device)
    res = EsfkResult(torch.empty(n, d1, **f), torch.empty(E, d2, **f), torch.empty(E, d1, d2, **f))
    ws = _ws(rx, d1, d2)
    check(lib().hxm_esfk(_dtype_code(x), x.data_ptr(), g.data_ptr(), n, d1, d2, w_t.data_ptr(),
                         int(w_transposed), rx.v.data_ptr(), rx.idx.data_ptr(), E, _bound(rx),
                         res.grad_x.data_ptr(), res.grad_b.data_ptr(), res.grad_w.data_ptr(),
                         ws.data_ptr(), ws.numel(), _stream()), "esfk")
    _count(stats, HXM_OP_ESFK, rx, d1, d2)
    return res
