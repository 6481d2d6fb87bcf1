"""The conventional dispatch -> per-expert dense GEMM -> combine formulation
with a capacity factor (reference core/src/gemm_oracle.cpp), as the GPU
baseline the expert-specific path is measured against.

Semantics follow count_redundancy (gemm_oracle.cpp:251-285, whose comment
at :269 says "all k*N (token, choice) pairs compete for the same per-expert
buffers"): the k*N slots compete for E per-expert buffers of
C = ceil(capacity_factor * k * N / E) rows; the lowest slot ids are kept
(dispatch()'s keep-lowest policy, gemm_oracle.cpp:88-95, applied to the
combined slot order choice-major, token-ascending), overflow slots are
dropped (zero contribution to y and to every gradient), and shortfall rows
are zero padding that the GEMMs really compute.

Deliberate divergence: the reference's oracle_forward calls dispatch() once
per choice (gemm_oracle.cpp:154-156), so there each choice has its own
capacity-C buffer and for k > 1 fewer slots are dropped.  The device baseline
follows count_redundancy's combined competition -- the accounting the bench
columns (padded_rows, dropped_tokens, macs_oracle) report -- so its drops and
its MAC count agree with those columns; for k = 1 the two coincide.

On the device the baseline is the same layer with a fixed-capacity index
(hxm_layer_desc.capacity): the dispatch is the expert-sorted gather, the
per-expert GEMMs run over exactly C rows each (C rounded up to the 64-row
segment granule), the combine is the scatter-reduction epilogue.  Only the
index differs, so a timing difference is the cost of padding (and the
accuracy difference the cost of dropping).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np

from .moe_layer import capacity_rows  # noqa: F401  (re-export: device capacity)


@dataclass
class RedundancyReport:
    token_macs_expert_specific: int
    token_macs_oracle: int
    padded_rows: int
    dropped_tokens: int
    capacity_per_expert: int

    def to_json(self) -> str:
        return json.dumps(self.__dict__)


def count_redundancy(r, d_in: int, hidden: int, d_out: int,
                     capacity_factor: float) -> RedundancyReport:
    """gemm_oracle.cpp:251-285 (same arithmetic, same exception)."""
    r.validate()
    if not capacity_factor > 0.0:
        raise ValueError("count_redundancy: capacity_factor must be > 0")
    per_row = d_in * hidden + hidden * d_out
    cap = int(math.ceil(capacity_factor * r.k * r.n_tokens / r.n_experts))
    load = np.bincount(np.asarray(r.assignments).ravel(), minlength=r.n_experts)
    kept = np.minimum(load, cap)
    return RedundancyReport(
        token_macs_expert_specific=int(r.k * r.n_tokens * per_row),
        token_macs_oracle=int(r.n_experts * cap * per_row),
        padded_rows=int((cap - kept).sum()),
        dropped_tokens=int((load - kept).sum()),
        capacity_per_expert=cap)


def kept_slots(r, capacity: int) -> np.ndarray:
    """Boolean k x N mask of the slots the capacity-C baseline keeps (lowest
    slot ids per expert, slot = choice * N + token)."""
    a = np.asarray(r.assignments)
    flat = a.ravel()  # slot order
    mask = np.zeros(flat.shape, dtype=bool)
    for e in range(r.n_experts):
        idx = np.nonzero(flat == e)[0]
        mask[idx[:capacity]] = True
    return mask.reshape(a.shape)
