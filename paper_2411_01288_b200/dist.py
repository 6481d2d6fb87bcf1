"""Tensor parallelism along the FFN hidden dimension H (one process per GPU).

Re-designs the reference's in-process simulator (core/src/dist_sim.cpp) as real
collectives over torch.distributed (NCCL over NVLink on B200; gloo for the
CPU tests).  The numerics follow the reference exactly:

* ``shard_params`` / ``unshard_params`` (dist_sim.cpp:29-102): rank r owns
  W1[:, :, h_r], b1[:, h_r], W2[:, h_r, :]; b2 is owned by rank 0
  (dist_sim.hpp:33-36).  Shards are stored contiguous per rank.
* ``PipelineSharedCache`` (dist_sim.hpp:60-82, dist_sim.cpp:104-125): one
  layer's full parameters per device; CacheError on overflow or
  read-before-fill.
* ``data_centric_step`` (dist_sim.cpp:352-452): the parameter shards are
  all-gathered into the cache -- on a side stream, so the gather of the
  next layer overlaps the current compute -- every rank runs the full layer on
  its own tokens, then parameter gradients are summed across ranks
  (all-reduce as in the reference, or reduce-scatter to the owners).
* ``model_centric_step`` (dist_sim.cpp:454-601): tokens (and routing, and in
  backward g_y) are all-gathered, every rank computes the global batch on its
  H-slice (rank 0 alone adds b2 and computes gb2, dist_sim.cpp:486, 520-522),
  the partial y and partial gx are all-reduce-summed (or reduce-scattered back
  to the token owners).

Compute is injected as a ``LocalCompute`` so the same choreography runs with
the CUDA layer in production and with a CPU reference in the gloo tests.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import torch
import torch.distributed as dist

from ._lib import CacheError


# ------------------------------------------------------------ sharding ----
@dataclass
class ParamShard:
    w1: torch.Tensor  # E x D_i x h_r
    b1: torch.Tensor  # E x h_r
    w2: torch.Tensor  # E x h_r x D_o
    hidden_offset: int

    def elements(self) -> int:
        return self.w1.numel() + self.b1.numel() + self.w2.numel()


@dataclass
class ShardedParams:
    shards: List[ParamShard]
    b2: Optional[torch.Tensor]  # owned by rank 0
    activation: str
    hidden_sizes: List[int]

    def n_devices(self) -> int:
        return len(self.shards)

    def full_param_elements(self) -> int:
        s = self.shards[0]
        E, Di, Do = s.w1.shape[0], s.w1.shape[1], s.w2.shape[2]
        H = sum(self.hidden_sizes)
        return E * (Di * H + H + H * Do + Do)

    def shard_elements(self, d: int) -> int:
        n = self.shards[d].elements()
        return n + (self.b2.numel() if d == 0 and self.b2 is not None else 0)


def even_split(hidden: int, n: int) -> List[int]:
    base, rem = divmod(hidden, n)
    return [base + (1 if i < rem else 0) for i in range(n)]


def shard_params(p, hidden_alloc: Sequence[int]) -> ShardedParams:
    """dist_sim.cpp:29-78 (same checks and messages)."""
    p.validate()
    if len(hidden_alloc) == 0:
        raise ValueError("shard_params: need at least one device")
    if sum(hidden_alloc) != p.hidden():
        raise ValueError("shard_params: hidden allocation does not sum to the hidden size")
    if any(h <= 0 for h in hidden_alloc):
        raise ValueError("shard_params: hidden shares must be > 0")
    shards, off = [], 0
    for h in hidden_alloc:
        shards.append(ParamShard(p.w1[:, :, off:off + h].contiguous(),
                                 p.b1[:, off:off + h].contiguous(),
                                 p.w2[:, off:off + h, :].contiguous(), off))
        off += h
    return ShardedParams(shards, p.b2, p.activation, list(hidden_alloc))


def unshard_params(s: ShardedParams):
    """dist_sim.cpp:80-102: exact inverse of shard_params."""
    from .moe_layer import MoeLayerParams
    w1 = torch.cat([sh.w1 for sh in s.shards], dim=2)
    b1 = torch.cat([sh.b1 for sh in s.shards], dim=1)
    w2 = torch.cat([sh.w2 for sh in s.shards], dim=1)
    return MoeLayerParams(w1, b1, w2, s.b2, s.activation)


class PipelineSharedCache:
    """Full-layer parameter buffers per device (dist_sim.hpp:60-82).

    ``slots=1`` is the reference's cache: at most one layer resident, fill()
    replaces it.  The multi-layer pipeline uses ``slots=2`` (current layer +
    the one being prefetched by the side-stream all-gather): fill() replaces
    the least recently filled slot.  ``capacity_elements`` bounds one slot
    (CacheError on overflow or on reading a layer that is not resident)."""

    def __init__(self, capacity_elements: int, slots: int = 1):
        if slots < 1:
            raise ValueError("PipelineSharedCache: slots must be >= 1")
        self.capacity = capacity_elements
        self.slots = slots
        self._res = []  # [(layer_id, params)], oldest first
        self.fills = 0

    @property
    def layer(self) -> int:
        return self._res[-1][0] if self._res else -1

    def fill(self, layer_id: int, params) -> None:
        n = params.param_elements()
        if n > self.capacity:
            raise CacheError(f"pipeline-shared cache: layer parameters ({n} elements) exceed "
                             f"cache capacity ({self.capacity})")
        self._res = [r for r in self._res if r[0] != layer_id]
        if len(self._res) >= self.slots:
            self._res.pop(0)
        self._res.append((layer_id, params))
        self.fills += 1

    def clear(self) -> None:
        self._res = []

    def filled(self) -> bool:
        return bool(self._res)

    def resident(self) -> List[int]:
        return [r[0] for r in self._res]

    def params(self, layer_id: Optional[int] = None):
        if not self._res:
            raise CacheError("pipeline-shared cache: read before fill")
        if layer_id is None:
            return self._res[-1][1]
        for lid, p in self._res:
            if lid == layer_id:
                return p
        raise CacheError(f"pipeline-shared cache: layer {layer_id} is not resident "
                         f"(resident: {self.resident()})")


# ------------------------------------------------------------- compute ----
@dataclass
class LocalCompute:
    """forward(x, params, assignments, add_b2) -> (y fp32, stash);
    backward(stash, params, g_y) -> MoeGrads-like object (gw1, gb1, gw2, gb2, gx)."""
    forward: Callable
    backward: Callable


def cuda_compute() -> LocalCompute:
    from .moe_layer import moe_backward, moe_forward

    def fwd(x, params, assignments, add_b2):
        p = params if add_b2 else _without_b2(params)
        res = moe_forward(x, p, assignments, validate=False)
        return res.y, res.stash

    def bwd(stash, params, g_y):
        return moe_backward(stash, params if stash.desc.add_b2 else _without_b2(params), g_y)

    return LocalCompute(fwd, bwd)


def _without_b2(p):
    from .moe_layer import MoeLayerParams
    return MoeLayerParams(p.w1, p.b1, p.w2, None, p.activation)


# ---------------------------------------------------------- collectives ---
def _ws(group) -> int:
    return dist.get_world_size(group)


def _rank(group) -> int:
    return dist.get_rank(group)


def all_gather_rows(local: torch.Tensor, counts: Sequence[int], group=None) -> torch.Tensor:
    """Rank-order row concatenation (dist_sim.cpp:127-145) for uneven row
    counts: pad to the largest count, all_gather_into_tensor, drop padding."""
    P = _ws(group)
    m = max(counts)
    if local.shape[0] < m:
        pad = torch.zeros((m - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        local = torch.cat([local, pad])
    out = torch.empty((P * m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, local.contiguous(), group=group)
    if all(c == m for c in counts):
        return out
    return torch.cat([out[r * m:r * m + counts[r]] for r in range(P)])


def _row_counts(n_local: int, group=None, device=None) -> List[int]:
    t = torch.tensor([n_local], dtype=torch.int64, device=device)
    out = torch.empty(_ws(group), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, t, group=group)
    return [int(v) for v in out.tolist()]


def gather_params(shard: ParamShard, b2, hidden_sizes: Sequence[int], activation: str,
                  group=None, stream: Optional[torch.cuda.Stream] = None):
    """All-gather every rank's hidden-slice into full parameters (the cache
    fill of dist_sim.cpp:367-368).  Shards are padded to the largest share so
    one all_gather_into_tensor moves them; b2 is broadcast from rank 0."""
    from .moe_layer import MoeLayerParams
    P = _ws(group)
    hmax = max(hidden_sizes)
    E, Di, hr = shard.w1.shape
    Do = shard.w2.shape[2]

    def padded(t, dim):
        if t.shape[dim] == hmax:
            return t.contiguous()
        shp = list(t.shape)
        shp[dim] = hmax - t.shape[dim]
        return torch.cat([t, torch.zeros(shp, dtype=t.dtype, device=t.device)], dim=dim)

    ctx = torch.cuda.stream(stream) if stream is not None else _nullctx()
    with ctx:
        # rank-major flat outputs (gloo requires dim-0 concatenation)
        w1g = torch.empty((P * E, Di, hmax), dtype=shard.w1.dtype, device=shard.w1.device)
        w2g = torch.empty((P * E, hmax, Do), dtype=shard.w2.dtype, device=shard.w2.device)
        b1g = torch.empty((P * E, hmax), dtype=shard.b1.dtype, device=shard.b1.device)
        dist.all_gather_into_tensor(w1g, padded(shard.w1, 2), group=group)
        dist.all_gather_into_tensor(w2g, padded(shard.w2, 1), group=group)
        dist.all_gather_into_tensor(b1g, padded(shard.b1, 1), group=group)
        w1g, w2g = w1g.view(P, E, Di, hmax), w2g.view(P, E, hmax, Do)
        b1g = b1g.view(P, E, hmax)
        b2f = b2
        if b2f is None or _rank(group) != 0:
            b2f = torch.empty((E, Do), dtype=shard.b1.dtype, device=shard.w1.device) \
                if b2 is None else b2
        b2f = b2f.contiguous()
        dist.broadcast(b2f, src=dist.get_global_rank(group, 0) if group is not None else 0,
                       group=group)
        w1 = torch.cat([w1g[r, :, :, :hidden_sizes[r]] for r in range(P)], dim=2)
        w2 = torch.cat([w2g[r, :, :hidden_sizes[r], :] for r in range(P)], dim=1)
        b1 = torch.cat([b1g[r, :, :hidden_sizes[r]] for r in range(P)], dim=1)
    return MoeLayerParams(w1, b1, w2, b2f, activation)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


# -------------------------------------------------------------- steps -----
@dataclass
class DistStepResult:
    y: torch.Tensor            # local rows (data-centric / reduce-scatter) or global (all-reduce)
    grads: object              # gw1, gb1, gw2, gb2, gx
    collectives: List[str] = field(default_factory=list)


def data_centric_step(local_x, local_assign, local_gy, shard: ParamShard, b2, hidden_sizes,
                      activation: str, cache: PipelineSharedCache, compute: LocalCompute,
                      group=None, grad_reduce: str = "all_reduce",
                      side_stream: Optional[torch.cuda.Stream] = None) -> DistStepResult:
    """dist_sim.cpp:352-452 with real collectives.  Returns this rank's y
    rows and the summed parameter gradients (all_reduce: full tensors on every
    rank, as the reference; reduce_scatter: each rank's H-slice of gw1 / gb1 /
    gw2, and gb2 on rank 0)."""
    log = ["param_all_gather"]
    full = gather_params(shard, b2, hidden_sizes, activation, group, side_stream)
    if side_stream is not None:
        torch.cuda.current_stream().wait_stream(side_stream)
    cache.fill(0, full)
    p = cache.params()
    y, stash = compute.forward(local_x, p, local_assign, True)
    g = compute.backward(stash, p, local_gy)
    g = _reduce_param_grads(g, shard, hidden_sizes, group, grad_reduce)
    log.append("grad_all_reduce" if grad_reduce == "all_reduce" else "grad_reduce_scatter")
    return DistStepResult(y, g, log)


def model_centric_step(local_x, local_assign, local_gy, shard: ParamShard, b2, activation: str,
                       compute: LocalCompute, group=None,
                       reduce: str = "all_reduce") -> DistStepResult:
    """dist_sim.cpp:454-601 with real collectives.  ``reduce`` = "all_reduce"
    returns global y / gx on every rank (reference semantics);
    "reduce_scatter" returns this rank's token rows only."""
    from .moe_layer import MoeGrads, MoeLayerParams
    r = _rank(group)
    log = []
    counts = _row_counts(local_x.shape[0], group, local_x.device)
    x = all_gather_rows(local_x, counts, group)
    a = all_gather_rows(local_assign.t().contiguous(), counts, group).t().contiguous()
    log.append("token_all_gather")
    p = MoeLayerParams(shard.w1, shard.b1, shard.w2, b2 if r == 0 else None, activation)
    y_part, stash = compute.forward(x, p, a, r == 0)
    y = _reduce_rows(y_part, counts, group, reduce)
    log.append("output_" + reduce)
    gy = all_gather_rows(local_gy, counts, group)
    log.append("grad_all_gather")
    g = compute.backward(stash, p, gy)
    gx = _reduce_rows(g.gx, counts, group, reduce)
    log.append("input_grad_" + reduce)
    return DistStepResult(y, MoeGrads(g.gw1, g.gb1, g.gw2, g.gb2 if r == 0 else None, gx), log)


class DataCentricRunner:
    """Preallocated data-centric TP step for one process per GPU (the fast
    path behind bench.py --gpus N; the choreography is data_centric_step's).

    Each rank owns an even H-slice of the layer.  The pipeline-shared cache
    (dist_sim.cpp:104-125, 367-368) has two slots; each slot is one
    shard-major buffer per tensor -- w1 (P*E) x D_i x h, b1 (P*E) x h,
    w2 (P*E) x h x D_o -- which is exactly what ``all_gather_into_tensor`` of
    the P shards produces, and the CUDA layer reads it in place
    (hxm_layer_desc.weight_shards): no repacking copy.  step():
      (1) the slot for this step was filled on the side stream (NCCL) by the
          previous step's prefetch() -- or now, for the first step; the
          forward waits on its fill event only after the routing prologue;
      (2) with ``overlap`` the NEXT step's fill of the other slot is issued on
          the side stream right after this forward is enqueued, so it runs
          under this step's compute (the steady state of data_centric_pipeline,
          where layer l + 1's gather hides under layer l);
      (3) fwd+bwd of the full layer on this rank's tokens, then the fp32
          parameter gradients reduce-scattered to the shard owners (gb2, owned
          by rank 0, all-reduced).
    Shapes the kernels cannot read shard-major (H / P not a multiple of the
    tile widths) fall back to one repacked reference-layout slot."""

    def __init__(self, shard: ParamShard, b2, hidden_sizes: Sequence[int], activation: str,
                 n_tokens: int, k: int, group=None, dtype=torch.bfloat16, overlap: bool = True):
        from .moe_layer import MoeLayerParams
        from .runner import LayerRunner
        self.group = group
        self.P, self.rank = _ws(group), _rank(group)
        if len(set(hidden_sizes)) != 1:
            raise ValueError("DataCentricRunner: even hidden shares only (use data_centric_step)")
        self.h = hidden_sizes[0]
        self.shard = shard
        E, Di, h = shard.w1.shape
        Do = shard.w2.shape[2]
        dev = shard.w1.device
        P = self.P
        self.b2 = (b2 if b2 is not None else torch.zeros((E, Do), device=dev)).float().contiguous()
        full = MoeLayerParams(torch.empty((E, Di, P * h), dtype=shard.w1.dtype, device=dev),
                              torch.empty((E, P * h), dtype=torch.float32, device=dev),
                              torch.empty((E, P * h, Do), dtype=shard.w2.dtype, device=dev),
                              self.b2, activation)
        self.cache = PipelineSharedCache(full.param_elements(), slots=2)
        self.cache.fill(0, full)
        self.runner = LayerRunner(full, n_tokens, k, dev, dtype)
        L = self.runner._L
        self.shard_major = P == 1 or bool(L.hxm_layer_weight_shards_ok(
            C.byref(self.runner.desc), P))
        self.overlap = overlap and self.shard_major
        self.side = torch.cuda.Stream(device=dev)
        # cache slots: gather targets (rank-major == shard-major)
        nslot = 2 if self.shard_major else 1
        self.slots = []
        for i in range(nslot):
            if P == 1 and i == 0:
                w1g, w2g, b1g = full.w1, full.w2, self.runner.b1
            else:
                w1g = torch.empty((P * E, Di, h), dtype=shard.w1.dtype, device=dev)
                w2g = torch.empty((P * E, h, Do), dtype=shard.w2.dtype, device=dev)
                b1g = torch.empty((P * E, h), dtype=torch.float32, device=dev)
            self.slots.append(dict(w1=w1g, w2=w2g, b1=b1g, ready=torch.cuda.Event(),
                                   free=torch.cuda.Event(), filled=False))
        for sl in self.slots:  # "free" starts recorded
            sl["free"].record(torch.cuda.current_stream())
        self.cur = 0
        self.fills = 0
        self.gw1 = torch.empty((E, Di, h), dtype=torch.float32, device=dev)
        self.gb1 = torch.empty((E, h), dtype=torch.float32, device=dev)
        self.gw2 = torch.empty((E, h, Do), dtype=torch.float32, device=dev)

    def _fill(self, i: int) -> None:
        """Cache fill of slot i (dist_sim.cpp:367-368) on the side stream."""
        sl = self.slots[i]
        P, E = self.P, self.shard.w1.shape[0]
        self.side.wait_event(sl["free"])  # the last step that read slot i is done
        with torch.cuda.stream(self.side):
            dist.all_gather_into_tensor(sl["w1"], self.shard.w1.contiguous(), group=self.group)
            dist.all_gather_into_tensor(sl["w2"], self.shard.w2.contiguous(), group=self.group)
            dist.all_gather_into_tensor(sl["b1"], self.shard.b1.float().contiguous(),
                                        group=self.group)
            dist.broadcast(self.b2, src=dist.get_global_rank(self.group, 0)
                           if self.group is not None else 0, group=self.group)
            if not self.shard_major and P > 1:
                # fallback: rank-major gather buffers -> the reference layout
                p = self.cache.params()
                Di, h, Do = sl["w1"].shape[1], self.h, sl["w2"].shape[2]
                p.w1.view(E, Di, P, h).copy_(sl["w1"].view(P, E, Di, h).permute(1, 2, 0, 3))
                p.w2.view(E, P, h, Do).copy_(sl["w2"].view(P, E, h, Do).permute(1, 0, 2, 3))
                self.runner.b1.view(E, P, h).copy_(sl["b1"].view(P, E, h).permute(1, 0, 2))
            sl["ready"].record(self.side)
        sl["filled"] = True
        self.fills += 1

    def gather(self) -> None:
        """Fill the current slot now (blocking the compute stream on it)."""
        self._fill(self.cur)
        torch.cuda.current_stream().wait_event(self.slots[self.cur]["ready"])

    def _use_slot(self) -> dict:
        sl = self.slots[self.cur]
        if not sl["filled"]:
            self._fill(self.cur)
        if self.shard_major:
            self.runner.set_weights(sl["w1"], sl["b1"], sl["w2"], shards=self.P,
                                    ready=sl["ready"])
        else:
            torch.cuda.current_stream().wait_event(sl["ready"])
        return sl

    def _release(self, sl) -> None:
        sl["free"].record(torch.cuda.current_stream())
        sl["filled"] = False
        self.cur = (self.cur + 1) % len(self.slots)

    def enable_fused_grads(self) -> None:
        """Reduce-scatter gW1 / gW2 inside the ESTMM epilogues into the shard
        owners' peer-mapped buffers (hxm_moe_backward_dc) instead of NCCL
        reduce-scatters of permuted copies; gb1 / gb2 stay NCCL (tiny)."""
        E, Di, h = self.shard.w1.shape
        Do = self.shard.w2.shape[2]
        self._w1b = PeerBuffers(h, Di, self.group, shape=(E, Di, h))
        self._w2b = PeerBuffers(h, Do, self.group, shape=(E, h, Do))
        self.gw1, self.gw2 = self._w1b.view(), self._w2b.view()

    def step(self, x, assignments, g_y):
        sl = self._use_slot()
        self.runner.forward(x, assignments)
        if self.overlap:  # next step's cache fill under this step's compute
            self._fill((self.cur + 1) % len(self.slots))
        if getattr(self, "_w1b", None) is not None:
            y = self._step_fused_bwd(x, g_y)
        else:
            y = self._step_nccl_bwd(x, g_y)
        self._release(sl)
        return y

    def _step_nccl_bwd(self, x, g_y):
        self.runner.backward(x, g_y)
        g = self.runner.grads
        E = g.gw1.shape[0]
        P, h = self.P, self.h
        # reduce-scatter along H: rank-major views of the H axis
        w1 = g.gw1.view(E, g.gw1.shape[1], P, h).permute(2, 0, 1, 3).contiguous()
        dist.reduce_scatter_tensor(self.gw1, w1, group=self.group)
        b1 = g.gb1.view(E, P, h).permute(1, 0, 2).contiguous()
        dist.reduce_scatter_tensor(self.gb1, b1, group=self.group)
        w2 = g.gw2.view(E, P, h, g.gw2.shape[2]).permute(1, 0, 2, 3).contiguous()
        dist.reduce_scatter_tensor(self.gw2, w2, group=self.group)
        if g.gb2 is not None:
            dist.all_reduce(g.gb2, group=self.group)
        return self.runner.y


# ------------------------------------------- multi-layer data-centric ------
@dataclass
class PipelineResult:
    y: torch.Tensor            # this rank's output rows of the last layer
    grads: List[object]        # per layer: gw1, gb1, gw2, gb2, gx (gx: this rank's rows)
    gathers: int               # parameter all-gathers issued (2L - 1)
    log: List[str] = field(default_factory=list)


def data_centric_pipeline(local_x, local_assigns: Sequence, local_gy,
                          shards: Sequence[ParamShard], b2s: Sequence, hidden_sizes,
                          activation: str, cache: PipelineSharedCache, compute: LocalCompute,
                          group=None, grad_reduce: str = "all_reduce",
                          side_stream: Optional[torch.cuda.Stream] = None) -> PipelineResult:
    """L stacked MoE layers (d_in == d_out), data-centric TP along H, with
    the pipeline-shared cache schedule of dist_sim.cpp:410-433 executed for
    real instead of accounted: forward all-gathers layer l + 1's shards (on
    ``side_stream`` with NCCL, overlapping layer l's compute) while layer l
    runs from the cache; backward starts from the still-resident last layer
    (no re-gather) and prefetches layer l - 1 while layer l runs -- 2L - 1
    gathers in total (test_dist_sim.cpp:329-336).  Layer l + 1's input is
    layer l's output cast to the input dtype; layer l's g_y is layer l + 1's
    g_x, likewise.  The cache needs two slots (current + prefetch).

    Returns the last layer's local y and every layer's gradients reduced as
    in data_centric_step (all_reduce: full tensors; reduce_scatter: each
    rank's H-slices, gb2 on rank 0)."""
    L = len(shards)
    if L < 1 or len(local_assigns) != L or len(b2s) != L:
        raise ValueError("data_centric_pipeline: one shard, routing and b2 per layer")
    if cache.slots < 2 and L > 1:
        raise CacheError("data_centric_pipeline: the prefetching schedule needs a two-slot "
                         "pipeline-shared cache")
    log: List[str] = []
    gathers = 0
    cur = torch.cuda.current_stream() if side_stream is not None else None

    def gather(l):
        nonlocal gathers
        gathers += 1
        log.append(f"param_gather_layer{l}")
        p = gather_params(shards[l], b2s[l], hidden_sizes, activation, group, side_stream)
        ev = None
        if side_stream is not None:
            ev = torch.cuda.Event()
            ev.record(side_stream)
        return l, p, ev

    def land(pending):
        l, p, ev = pending
        if ev is not None:
            cur.wait_event(ev)
        cache.fill(l, p)
        return p

    # ---- forward: layer l computes while layer l + 1 is gathered ----------
    stashes = []
    x = local_x
    pending = gather(0)
    for l in range(L):
        p = land(pending)
        if l + 1 < L:
            if side_stream is not None:
                side_stream.wait_stream(cur)  # the slot being refilled is idle
            pending = gather(l + 1)
        y, stash = compute.forward(x, p, local_assigns[l], True)
        stashes.append(stash)
        log.append(f"forward_layer{l}")
        x = y.to(local_x.dtype) if l + 1 < L else y
    y_out = x
    # ---- backward: the last layer is still resident -----------------------
    grads = [None] * L
    g_in = local_gy
    pending = None
    for l in reversed(range(L)):
        if l == L - 1:
            p = cache.params(l)
            log.append(f"reuse_cached_layer{l}")
        else:
            p = land(pending)
        if l > 0:
            if side_stream is not None:
                side_stream.wait_stream(cur)
            pending = gather(l - 1)
        g = compute.backward(stashes[l], p, g_in)
        log.append(f"backward_layer{l}")
        grads[l] = _reduce_param_grads(g, shards[l], hidden_sizes, group, grad_reduce)
        log.append(f"grad_{grad_reduce}_layer{l}")
        if l > 0:
            g_in = g.gx.to(local_gy.dtype)
    return PipelineResult(y_out, grads, gathers, log)


def _reduce_param_grads(g, shard: ParamShard, hidden_sizes, group, how: str):
    from .moe_layer import MoeGrads
    if how == "all_reduce":
        for t in (g.gw1, g.gb1, g.gw2, g.gb2):
            dist.all_reduce(t, group=group)
        return g
    r = _rank(group)
    h, hmax = hidden_sizes[r], max(hidden_sizes)
    outs = []
    for t, dim in ((g.gw1, 2), (g.gb1, 1), (g.gw2, 1)):
        parts, o = [], 0
        for hr in hidden_sizes:
            sl = t.narrow(dim, o, hr)
            if hr < hmax:
                shp = list(sl.shape)
                shp[dim] = hmax - hr
                sl = torch.cat([sl, torch.zeros(shp, dtype=t.dtype, device=t.device)], dim=dim)
            parts.append(sl.movedim(dim, 0).contiguous())
            o += hr
        out = torch.empty_like(parts[0])
        dist.reduce_scatter_tensor(out, torch.cat(parts), group=group)
        outs.append(out[:h].movedim(0, dim).contiguous())
    dist.reduce(g.gb2, dst=dist.get_global_rank(group, 0) if group is not None else 0,
                group=group)
    return MoeGrads(outs[0], outs[1], outs[2], g.gb2 if r == 0 else None, g.gx)


def _dc_step_fused_bwd(self, x, g_y):
    run = self.runner
    self._w1b.view().zero_()
    self._w2b.view().zero_()
    self._w1b.barrier()  # every owner's shards are zero before any rank reduces
    self._w2b.barrier()
    gb1, gb2 = run.grads.gb1, run.grads.gb2
    run.backward_dc(x, g_y, self._w1b, self._w2b)
    self._w1b.barrier()  # all contributions landed
    self._w2b.barrier()
    E, P, h = gb1.shape[0], self.P, self.h
    b1 = gb1.view(E, P, h).permute(1, 0, 2).contiguous()
    dist.reduce_scatter_tensor(self.gb1, b1, group=self.group)
    if gb2 is not None:
        dist.all_reduce(gb2, group=self.group)
    return run.y


DataCentricRunner._step_fused_bwd = _dc_step_fused_bwd


def _reduce_rows(t: torch.Tensor, counts: Sequence[int], group, how: str) -> torch.Tensor:
    if how == "all_reduce":
        dist.all_reduce(t, group=group)
        return t
    P, r, m = _ws(group), _rank(group), max(counts)
    if all(c == m for c in counts):
        out = torch.empty((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        dist.reduce_scatter_tensor(out, t.contiguous(), group=group)
        return out
    parts, o = [], 0
    for c in counts:
        sl = t[o:o + c]
        if c < m:
            sl = torch.cat([sl, torch.zeros((m - c,) + tuple(t.shape[1:]), dtype=t.dtype,
                                            device=t.device)])
        parts.append(sl)
        o += c
    out = torch.empty((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    dist.reduce_scatter_tensor(out, torch.cat(parts), group=group)
    return out[:counts[r]]


# ------------------------------------ fused GEMM -> reduce-scatter (peer) ---
class _CudaArray:
    """__cuda_array_interface__ view of a raw device pointer (torch.as_tensor)."""

    def __init__(self, ptr: int, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3}


class PeerBuffers:
    """Per-rank receive buffers (rows x cols fp32) mapped into every rank, plus
    a barrier flag array: the targets of hxm_moe_forward_tp /
    hxm_moe_backward_tp, whose ESMM epilogues reduce each token's output row
    into its owner's buffer over NVLink peer memory (CUDA IPC handles
    exchanged through ``group``).  ``PeerBuffers.local`` builds the same table
    from buffers of one process (single-GPU tests, no IPC)."""

    def __init__(self, rows_per_rank: int, cols: int, group=None, shape=None):
        """rows_per_rank x cols fp32 per rank; or any per-rank ``shape`` with
        ``rows_per_rank`` the H span each rank owns (weight-gradient shards)."""
        from ._lib import PeerFlags, PeerRows, check, lib
        L = lib()
        self.rows, self.cols = rows_per_rank, cols
        self.shape = tuple(shape) if shape is not None else (rows_per_rank, cols)
        self.P, self.rank = _ws(group), _rank(group)
        if self.P > 8:
            raise ValueError("PeerBuffers: at most 8 ranks (HXM_MAX_PEERS)")
        self._own = []
        buf, flg = C.c_void_p(), C.c_void_p()
        nelem = 1
        for v in self.shape:
            nelem *= v
        check(L.hxm_peer_malloc(nelem * 4, C.byref(buf)), "peer_malloc")
        check(L.hxm_peer_malloc(8 * 4, C.byref(flg)), "peer_malloc")
        self._own = [buf.value, flg.value]
        hb, hf = C.create_string_buffer(64), C.create_string_buffer(64)
        check(L.hxm_ipc_get_handle(buf, hb), "ipc_get_handle")
        check(L.hxm_ipc_get_handle(flg, hf), "ipc_get_handle")
        handles = [None] * self.P
        dist.all_gather_object(handles, (hb.raw, hf.raw), group=group)
        self._opened = []
        bufs, flags = [], []
        for r, (b, f) in enumerate(handles):
            if r == self.rank:
                bufs.append(buf.value)
                flags.append(flg.value)
                continue
            pb, pf = C.c_void_p(), C.c_void_p()
            check(L.hxm_ipc_open_handle(b, C.byref(pb)), "ipc_open_handle")
            check(L.hxm_ipc_open_handle(f, C.byref(pf)), "ipc_open_handle")
            self._opened += [pb.value, pf.value]
            bufs.append(pb.value)
            flags.append(pf.value)
        self._tables(bufs, flags, PeerRows, PeerFlags)

    @classmethod
    def local(cls, tensors: Sequence[torch.Tensor], rank: int = 0, span: Optional[int] = None):
        """Table over same-process fp32 buffers (simulated ranks on one GPU);
        ``span``: the H extent each buffer owns (default: its row count)."""
        from ._lib import PeerFlags, PeerRows
        self = cls.__new__(cls)
        self.shape = tuple(tensors[0].shape)
        self.rows = span if span is not None else tensors[0].shape[0]
        self.cols = tensors[0].shape[-1]
        self.P, self.rank = len(tensors), rank
        self._own, self._opened = [], []
        self._keep = list(tensors)
        self._flags = torch.zeros(self.P, 8, dtype=torch.int32, device=tensors[0].device)
        self._tables([t.data_ptr() for t in tensors],
                     [self._flags[r].data_ptr() for r in range(self.P)], PeerRows, PeerFlags)
        return self

    def _tables(self, bufs, flags, PeerRows, PeerFlags):
        self.bufs = bufs
        self.rows_struct = PeerRows()
        self.rows_struct.n_ranks, self.rows_struct.rows_per_rank = self.P, self.rows
        self.flags_struct = PeerFlags()
        self.flags_struct.n_ranks, self.flags_struct.rank = self.P, self.rank
        for r in range(self.P):
            self.rows_struct.ptrs[r] = bufs[r]
            self.flags_struct.ptrs[r] = flags[r]
        self.epoch = 0

    def view(self, rank: Optional[int] = None) -> torch.Tensor:
        """torch view of rank's buffer (default: this rank's own rows)."""
        r = self.rank if rank is None else rank
        return torch.as_tensor(_CudaArray(self.bufs[r], self.shape), device="cuda")

    def barrier(self, stream=None) -> None:
        from ._lib import check, lib
        self.epoch += 1
        st = (stream or torch.cuda.current_stream()).cuda_stream
        check(lib().hxm_peer_barrier(C.byref(self.flags_struct), self.epoch, st), "peer_barrier")

    def close(self) -> None:
        from ._lib import lib
        L = lib()
        for p in self._opened:
            L.hxm_ipc_close_handle(C.c_void_p(p))
        for p in self._own:
            L.hxm_peer_free(C.c_void_p(p))
        self._opened, self._own = [], []


def layer_forward_tp(x, params, assignments, y_rows: "PeerBuffers", add_b2: bool,
                     workspace=None, dtype=torch.bfloat16):
    """One rank's model-centric forward with y reduce-scattered inside the
    ESMM epilogue (hxm_moe_forward_tp).  Returns the stash handle for
    layer_backward_tp.  The caller orders the owners' zeroing and reads with
    PeerBuffers.barrier."""
    from ._lib import check, lib
    from .moe_layer import ForwardStash, layer_workspace, make_desc
    k, n = assignments.shape
    p = params
    desc = make_desc(n, p.experts(), k, p.d_in(), p.hidden(), p.d_out(), p.activation, dtype,
                     add_b2 and p.b2 is not None)
    ws = workspace if workspace is not None else layer_workspace(desc, x.device)
    b1 = p.b1.to(torch.float32).contiguous()
    b2 = p.b2.to(torch.float32).contiguous() if (add_b2 and p.b2 is not None) else None
    check(lib().hxm_moe_forward_tp(C.byref(desc), x.contiguous().data_ptr(), p.w1.data_ptr(),
                                   b1.data_ptr(), p.w2.data_ptr(),
                                   None if b2 is None else b2.data_ptr(),
                                   assignments.to(torch.int32).contiguous().data_ptr(),
                                   C.byref(y_rows.rows_struct), ws.data_ptr(), ws.numel(), None,
                                   torch.cuda.current_stream().cuda_stream), "moe_forward_tp")
    return ForwardStash(desc, ws, x, "memory_efficient", 8)


def layer_backward_tp(stash, params, g_y, gx_rows: "PeerBuffers"):
    """The matching backward: parameter gradients of this rank's H-slice
    (local), g_x reduce-scattered to the token owners inside the ESMM epilogue."""
    from ._lib import check, lib
    from .moe_layer import MoeGrads
    p, d = params, stash.desc
    f = dict(dtype=torch.float32, device=g_y.device)
    E, Di, H, Do = p.experts(), p.d_in(), p.hidden(), p.d_out()
    g = MoeGrads(torch.empty(E, Di, H, **f), torch.empty(E, H, **f), torch.empty(E, H, Do, **f),
                 torch.empty(E, Do, **f) if d.add_b2 else None, None)
    check(lib().hxm_moe_backward_tp(C.byref(d), stash.x.data_ptr(), p.w1.data_ptr(),
                                    p.w2.data_ptr(), g_y.contiguous().data_ptr(),
                                    stash.workspace.data_ptr(), stash.workspace.numel(),
                                    g.gw1.data_ptr(), g.gb1.data_ptr(), g.gw2.data_ptr(),
                                    None if g.gb2 is None else g.gb2.data_ptr(),
                                    C.byref(gx_rows.rows_struct),
                                    torch.cuda.current_stream().cuda_stream), "moe_backward_tp")
    return g


def model_centric_step_fused(local_x, local_assign, local_gy, shard: ParamShard, b2,
                             activation: str, ybuf: "PeerBuffers", gxbuf: "PeerBuffers",
                             group=None) -> DistStepResult:
    """dist_sim.cpp:454-601 with the two activation reductions fused into the
    GEMMs: every rank computes the global batch on its H-slice and its ESMM
    epilogues reduce y (forward) and g_x (backward) straight into the token
    owners' buffers over peer memory -- no NCCL reduce-scatter afterwards.
    Token shares must be even (rows_per_rank = local batch)."""
    from .moe_layer import MoeGrads, MoeLayerParams
    r = _rank(group)
    counts = _row_counts(local_x.shape[0], group, local_x.device)
    if len(set(counts)) != 1 or counts[0] != ybuf.rows:
        raise ValueError("model_centric_step_fused: even token shares of ybuf.rows required")
    x = all_gather_rows(local_x, counts, group)
    a = all_gather_rows(local_assign.t().contiguous(), counts, group).t().contiguous()
    p = MoeLayerParams(shard.w1, shard.b1, shard.w2, b2 if r == 0 else None, activation)
    ybuf.view().zero_()
    ybuf.barrier()  # every owner's rows are zero before any rank reduces
    stash = layer_forward_tp(x, p, a, ybuf, r == 0, dtype=x.dtype)
    ybuf.barrier()  # every rank's contributions have landed
    y = ybuf.view().clone()
    gy = all_gather_rows(local_gy, counts, group)
    gxbuf.view().zero_()
    gxbuf.barrier()
    g = layer_backward_tp(stash, p, gy, gxbuf)
    gxbuf.barrier()
    gx = gxbuf.view().clone()
    log = ["token_all_gather", "output_fused_reduce_scatter", "grad_all_gather",
           "input_grad_fused_reduce_scatter"]
    return DistStepResult(y, MoeGrads(g.gw1, g.gb1, g.gw2, g.gb2 if r == 0 else None, gx), log)


def layer_backward_dc(stash, params, g_y, gw1_shards: "PeerBuffers", gw2_shards: "PeerBuffers"):
    """Data-centric backward with the weight gradients reduce-scattered along
    H inside the ESTMM epilogues (hxm_moe_backward_dc): gW1 columns / gW2 rows
    land, summed over ranks, in their owner's E x D_i x span / E x span x D_o
    shard.  Returns this rank's full gb1, gb2 and g_x (reduced by the caller)."""
    from ._lib import check, lib
    p, d = params, stash.desc
    f = dict(dtype=torch.float32, device=g_y.device)
    gb1 = torch.empty(p.experts(), p.hidden(), **f)
    gb2 = torch.empty(p.experts(), p.d_out(), **f) if d.add_b2 else None
    gx = torch.empty(g_y.shape[0], p.d_in(), **f)
    check(lib().hxm_moe_backward_dc(C.byref(d), stash.x.data_ptr(), p.w1.data_ptr(),
                                    p.w2.data_ptr(), g_y.contiguous().data_ptr(),
                                    stash.workspace.data_ptr(), stash.workspace.numel(),
                                    C.byref(gw1_shards.rows_struct), gb1.data_ptr(),
                                    C.byref(gw2_shards.rows_struct),
                                    None if gb2 is None else gb2.data_ptr(), gx.data_ptr(),
                                    torch.cuda.current_stream().cuda_stream), "moe_backward_dc")
    return gb1, gb2, gx


def data_centric_step_fused(local_x, local_assign, local_gy, shard: ParamShard, b2, hidden_sizes,
                            activation: str, gw1_shards: "PeerBuffers", gw2_shards: "PeerBuffers",
                            group=None, side_stream: Optional[torch.cuda.Stream] = None):
    """dist_sim.cpp:352-452 with the weight-gradient reduce-scatter fused into
    the ESTMM epilogues: parameters all-gathered (NCCL) into the cache, the
    full layer run on this rank's tokens, gW1 / gW2 reduced straight into the
    shard owners' buffers over peer memory; the small gb1 / gb2 are reduced
    with NCCL.  Even hidden shares; returns this rank's shards (as
    data_centric_step(grad_reduce="reduce_scatter"))."""
    from .moe_layer import MoeGrads
    from .moe_layer import moe_forward
    if len(set(hidden_sizes)) != 1:
        raise ValueError("data_centric_step_fused: even hidden shares required")
    r, h = _rank(group), hidden_sizes[0]
    full = gather_params(shard, b2, hidden_sizes, activation, group, side_stream)
    if side_stream is not None:
        torch.cuda.current_stream().wait_stream(side_stream)
    fw = moe_forward(local_x, full, local_assign, validate=False)
    gw1_shards.view().zero_()
    gw2_shards.view().zero_()
    gw1_shards.barrier()  # every owner's shards are zero before any rank reduces
    gw2_shards.barrier()
    gb1, gb2, gx = layer_backward_dc(fw.stash, full, local_gy, gw1_shards, gw2_shards)
    gw1_shards.barrier()  # all contributions landed
    gw2_shards.barrier()
    dist.all_reduce(gb1, group=group)
    dist.reduce(gb2, dst=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    off = shard.hidden_offset
    return DistStepResult(fw.y, MoeGrads(gw1_shards.view().clone(), gb1[:, off:off + h].contiguous(),
                                         gw2_shards.view().clone(), gb2 if r == 0 else None, gx),
                          ["param_all_gather", "grad_fused_reduce_scatter", "bias_grad_reduce"])
