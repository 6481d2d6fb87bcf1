"""Routing choices and the device routing-index build.

Mirrors the reference header core/include/moekit/routing.hpp:
``RoutingChoice`` (routing.hpp:14-21), ``ReIndex`` (routing.hpp:29-38),
``build_reindex`` / ``build_reindex_all`` (routing.hpp:42-46, routing.cpp:42-80),
``synthesize_routing`` (routing.cpp:121-200) and the routing CSV fixture format
(routing.cpp:202-282).  The index build runs on the GPU (routing.cu) and is
bit-exact with the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import ShapeError, check, lib


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _require_cuda(t: torch.Tensor, name: str) -> None:
    if not (isinstance(t, torch.Tensor) and t.is_cuda):
        raise _lib.HexaMoeCudaError(f"{name} must be a CUDA tensor (no CPU fallback)")


@dataclass
class RoutingChoice:
    """k vectors of n_tokens expert ids; per token the k experts are distinct."""
    n_tokens: int
    n_experts: int
    k: int
    assignments: np.ndarray  # int32 [k, n_tokens]

    def validate(self) -> None:
        """routing.cpp:13-40 (same exception types and order)."""
        a = np.asarray(self.assignments)
        if self.k == 0 or a.ndim != 2 or a.shape[0] != self.k:
            raise ShapeError("RoutingChoice: expected k assignment vectors")
        if self.k > self.n_experts:
            raise ValueError("RoutingChoice: k exceeds expert count")
        if a.shape[1] != self.n_tokens:
            raise ShapeError("RoutingChoice: assignment length != n_tokens")
        if a.size and (a.min() < 0 or a.max() >= self.n_experts):
            raise ValueError("RoutingChoice: expert id out of range")
        for i in range(self.k):
            for j in range(i + 1, self.k):
                dup = np.nonzero(a[i] == a[j])[0]
                if dup.size:
                    raise ValueError(f"RoutingChoice: duplicate expert for token {int(dup[0])}")

    def to_device(self, device="cuda") -> torch.Tensor:
        return torch.from_numpy(np.ascontiguousarray(self.assignments, dtype=np.int32)).to(device)


def synthesize_routing(n_tokens: int, n_experts: int, k: int, dist: str = "uniform",
                       seed: int = 1) -> RoutingChoice:
    """Deterministic synthetic routing with the reference's seeded stream."""
    out = np.empty((k, n_tokens), dtype=np.int32)
    check(lib().hxm_synthesize_routing(n_tokens, n_experts, k, dist.encode(), seed,
                                       out.ctypes.data), "synthesize_routing")
    return RoutingChoice(n_tokens, n_experts, k, out)


def routing_to_csv(r: RoutingChoice) -> str:
    """routing.cpp:202-211: header then token_index,choice_index,expert_id."""
    lines = ["token_index,choice_index,expert_id"]
    a = np.asarray(r.assignments)
    for t in range(r.n_tokens):
        for i in range(r.k):
            lines.append(f"{t},{i},{int(a[i, t])}")
    return "\n".join(lines) + "\n"


def routing_from_csv(text: str) -> RoutingChoice:
    """routing.cpp:213-268 (holes rejected, then validate())."""
    rows = []
    first = True
    for line in text.splitlines():
        if not line:
            continue
        if first and "token_index" in line:
            first = False
            continue
        first = False
        try:
            t, c, e = (int(f) for f in line.split(",")[:3])
        except ValueError:
            raise ValueError("routing CSV: bad field in line: " + line) from None
        rows.append((t, c, e))
    if not rows:
        raise ValueError("routing CSV: no data rows")
    arr = np.array(rows, dtype=np.int64)
    n, k, E = int(arr[:, 0].max()) + 1, int(arr[:, 1].max()) + 1, int(arr[:, 2].max()) + 1
    a = np.full((k, n), -1, dtype=np.int32)
    a[arr[:, 1], arr[:, 0]] = arr[:, 2]
    if (a == -1).any():
        raise ValueError("routing CSV: missing (token, choice) rows")
    r = RoutingChoice(n, E, k, a)
    r.validate()
    return r


def write_routing_csv(path: str, r: RoutingChoice) -> None:
    with open(path, "w") as f:
        f.write(routing_to_csv(r))


def read_routing_csv(path: str) -> RoutingChoice:
    with open(path) as f:
        return routing_from_csv(f.read())


@dataclass
class ReIndex:
    """Device ReIndex: v int64 [N'] (-1 pads), idx int64 [E+1] (routing.hpp:29-38)."""
    v: torch.Tensor
    idx: torch.Tensor
    blk: int
    n_tokens: int
    bound: int = field(default=0)

    def num_experts(self) -> int:
        return self.idx.numel() - 1

    def padded_len(self) -> int:
        return int(self.idx[-1].item())

    def padding(self) -> int:
        return self.padded_len() - self.n_tokens


def build_reindex(assignment, n_experts: int, blk: int, validate: bool = True) -> ReIndex:
    """Device build_reindex (routing.cpp:42-70), bit-exact with the reference.

    ``validate`` synchronises once to surface an out-of-range expert id as
    ValueError (the reference throws std::invalid_argument) and trims v to N'.
    """
    if blk <= 0:
        raise ValueError("build_reindex: blk must be >= 1")
    if not isinstance(assignment, torch.Tensor):
        assignment = torch.as_tensor(np.asarray(assignment, dtype=np.int32)).cuda()
    _require_cuda(assignment, "assignment")
    a = assignment.to(torch.int32).contiguous()
    n = a.numel()
    L = lib()
    bound = L.hxm_reindex_bound(n, n_experts, blk)
    dev = a.device
    v = torch.empty(max(bound, 1), dtype=torch.int64, device=dev)
    idx = torch.empty(n_experts + 1, dtype=torch.int64, device=dev)
    wsb = L.hxm_reindex_workspace_bytes(n, n_experts)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    check(L.hxm_build_reindex(a.data_ptr(), n, n_experts, blk, v.data_ptr(), idx.data_ptr(),
                              ws.data_ptr(), wsb, status.data_ptr(), _stream()),
          "build_reindex")
    rx = ReIndex(v, idx, blk, n, bound)
    if validate:
        if int(status.item()) != 0:
            raise ValueError("build_reindex: expert id out of range")
        rx.v = v[: int(idx[-1].item())]
    return rx


def build_reindex_all(r: RoutingChoice, blk: int, validate: bool = True):
    """One ReIndex per routing choice (routing.cpp:72-80), all k built by one
    hxm_build_reindex_all call (three launches, choice = grid y)."""
    if blk <= 0:
        raise ValueError("build_reindex: blk must be >= 1")
    # (no r.validate(): the reference builds each choice's index as given)
    a = r.to_device() if not isinstance(r.assignments, torch.Tensor) else r.assignments
    _require_cuda(a, "assignments")
    a = a.to(torch.int32).contiguous()
    k, n, E = r.k, r.n_tokens, r.n_experts
    L = lib()
    bound = max(L.hxm_reindex_bound(n, E, blk), 1)
    dev = a.device
    v = torch.empty(k, bound, dtype=torch.int64, device=dev)
    idx = torch.empty(k, E + 1, dtype=torch.int64, device=dev)
    wsb = L.hxm_reindex_all_workspace_bytes(n, E, k)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    check(L.hxm_build_reindex_all(a.data_ptr(), k, n, E, blk, v.data_ptr(), bound,
                                  idx.data_ptr(), ws.data_ptr(), wsb, status.data_ptr(),
                                  _stream()), "build_reindex_all")
    out = [ReIndex(v[i], idx[i], blk, n, bound) for i in range(k)]
    if validate:
        if int(status.item()) != 0:
            raise ValueError("build_reindex: expert id out of range")
        ends = idx[:, -1].tolist()
        for i, rx in enumerate(out):
            rx.v = v[i, :ends[i]]
    return out
