"""Heterogeneous workload allocation (reference core/src/hetero_alloc.cpp).

The paper's adaptive schemes split the batch (data-centric) or the FFN hidden
dimension (model-centric) across devices in proportion to measured device
capacity.  The arithmetic is the reference's exactly:

* ``capacity_proportions`` -- R_i = (1/t_i) / sum_j 1/t_j (hetero_alloc.cpp:66-83)
* ``round_preserving_sum`` -- largest-remainder rounding, ties to the lower
  index, float-drift repair (hetero_alloc.cpp:85-126)
* ``allocate_batches`` / ``allocate_hidden`` -- ideal = R_i * total, then
  rounded (hetero_alloc.cpp:128-156)

B200-native part: ``probe_capacity_seconds`` times the proxy workload ON THE
GPU (the tcgen05 ESMM of this package over a fixed synthetic routing, CUDA
events on the launch stream) instead of the reference's scalar fp64 CPU
triple loop, and ``measure_latencies`` all-gathers every rank's probe so all
ranks derive the same plan; ``allocate_hidden`` feeds ``dist.shard_params``
(uneven H-slices) and ``allocate_batches`` the per-rank token counts.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from typing import List, Sequence


def capacity_proportions(latencies: Sequence[float]) -> List[float]:
    if len(latencies) == 0:
        raise ValueError("capacity_proportions: no devices")
    inv = 0.0
    for t in latencies:
        if not (t > 0.0):
            raise ValueError("capacity_proportions: latency must be > 0")
        inv += 1.0 / t
    return [(1.0 / t) / inv for t in latencies]


def round_preserving_sum(ideal: Sequence[float], total: int) -> List[int]:
    s = 0.0
    for v in ideal:
        if v < 0.0:
            raise ValueError("round_preserving_sum: negative ideal share")
        s += v
    if abs(s - float(total)) > 1e-9 * (1.0 + abs(s)):
        raise ValueError("round_preserving_sum: ideals do not sum to total")
    shares = [int(math.floor(v)) for v in ideal]
    frac = [v - sh for v, sh in zip(ideal, shares)]
    # stable sort by descending fractional part: ties keep the lower index
    order = sorted(range(len(ideal)), key=lambda i: -frac[i])
    remaining = total - sum(shares)
    for i in order:
        if remaining <= 0:
            break
        shares[i] += 1
        remaining -= 1
    for i in reversed(order):  # float drift only: take units back
        if remaining >= 0:
            break
        if shares[i] > 0:
            shares[i] -= 1
            remaining += 1
    return shares


@dataclass
class AllocationPlan:
    kind: str  # "batch" | "hidden"
    shares: List[int]
    total: int
    ideal: List[float] = field(default_factory=list)

    def to_json(self) -> str:
        return json.dumps({"kind": self.kind, "total": self.total, "shares": self.shares,
                           "ideal": self.ideal})

    def to_csv(self) -> str:
        rows = ["device,ideal,share"]
        rows += [f"{i},{self.ideal[i]!r},{self.shares[i]}" for i in range(len(self.shares))]
        return "\n".join(rows) + "\n"


def _allocate(latencies, total: int, kind: str) -> AllocationPlan:
    if total < 0:
        raise ValueError("allocate: total must be >= 0")
    r = capacity_proportions(latencies)
    ideal = [ri * float(total) for ri in r]
    return AllocationPlan(kind, round_preserving_sum(ideal, total), total, ideal)


def allocate_batches(latencies: Sequence[float], b_global: int) -> AllocationPlan:
    return _allocate(latencies, b_global, "batch")


def allocate_hidden(latencies: Sequence[float], hidden_total: int) -> AllocationPlan:
    return _allocate(latencies, hidden_total, "hidden")


def probe_capacity_seconds(iterations: int, matrix_size: int, seed: int = 1,
                           device=None) -> float:
    """Device seconds of ``iterations`` tcgen05 ESMM launches of the proxy
    problem (matrix_size tokens x matrix_size features, 8 experts, top-1,
    seeded), timed with CUDA events on the current stream after one warm-up.
    The GPU analogue of hetero_alloc.cpp:35-64's timed dense loop."""
    if matrix_size < 1:
        raise ValueError("probe_capacity: matrix size must be >= 1")
    import torch

    from .es_ops import esmm
    from .routing import build_reindex, synthesize_routing
    dev = torch.device(device if device is not None else "cuda")
    if iterations <= 0:
        return 0.0
    g = torch.Generator().manual_seed(seed)
    d = max(64, (matrix_size + 63) // 64 * 64)  # tcgen05 needs 64-multiples
    x = torch.randn(matrix_size, d, generator=g).to(dev, torch.bfloat16)
    w = (0.5 * torch.randn(8, d, d, generator=g)).to(dev, torch.bfloat16)
    r = synthesize_routing(matrix_size, 8, 1, "uniform", seed)
    rx = build_reindex(torch.as_tensor(r.assignments[0]).to(dev), 8, 8)
    esmm(x, w, None, rx)  # warm-up (tensor maps, kernel attributes)
    s = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(iterations):
        esmm(x, w, None, rx)
    e1.record(s)
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3


def measure_latencies(iterations: int = 20, matrix_size: int = 4096, group=None) -> List[float]:
    """Every rank probes its own GPU; the timings are all-gathered so all
    ranks compute the same allocation plan."""
    import torch
    import torch.distributed as dist
    t = probe_capacity_seconds(iterations, matrix_size)
    if not (dist.is_available() and dist.is_initialized()):
        return [t]
    P = dist.get_world_size(group)
    dev = "cuda" if dist.get_backend(group) == "nccl" else "cpu"
    out = torch.empty(P, dtype=torch.float64, device=dev)
    dist.all_gather_into_tensor(out, torch.tensor([t], dtype=torch.float64, device=dev),
                                group=group)
    return [float(v) for v in out.tolist()]
