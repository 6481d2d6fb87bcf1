"""LayerRunner: a preallocated, low-overhead fwd+bwd driver of one MoE layer.

Holds the workspace, outputs and gradients for a fixed (N, E, k, D_i, H, D_o,
dtype) and calls the C ABI (hxm_moe_forward / hxm_moe_backward) directly with
cached pointers, so a training loop (or bench.py) issues a step with a few
microseconds of host work.  All buffers are laid out once in HBM.
"""
from __future__ import annotations

import ctypes as C

import torch

from ._lib import check, lib
from .moe_layer import MoeGrads, MoeLayerParams, layer_workspace, make_desc


class LayerRunner:
    def __init__(self, p: MoeLayerParams, n_tokens: int, k: int, device="cuda",
                 dtype=torch.bfloat16, add_b2: bool = True, capacity: int = 0):
        p.validate()
        self.p = p
        self.dtype = dtype
        self.desc = make_desc(n_tokens, p.experts(), k, p.d_in(), p.hidden(), p.d_out(),
                              p.activation, dtype, add_b2 and p.b2 is not None, capacity)
        self.ws = layer_workspace(self.desc, device)
        f = dict(dtype=torch.float32, device=device)
        E, Di, H, Do = p.experts(), p.d_in(), p.hidden(), p.d_out()
        self.y = torch.empty(n_tokens, Do, **f)
        self.grads = MoeGrads(torch.empty(E, Di, H, **f), torch.empty(E, H, **f),
                              torch.empty(E, H, Do, **f),
                              torch.empty(E, Do, **f) if self.desc.add_b2 else None,
                              torch.empty(n_tokens, Di, **f))
        self.b1 = p.b1.to(torch.float32).contiguous()
        self.b2 = p.b2.to(torch.float32).contiguous() if p.b2 is not None else None
        self._w1, self._w2 = p.w1, p.w2
        self._pd = C.byref(self.desc)
        self._L = lib()

    def set_weights(self, w1: torch.Tensor, b1: torch.Tensor, w2: torch.Tensor,
                    shards: int = 0, ready: torch.cuda.Event | None = None) -> None:
        """Point the layer at another copy of its weights (a pipeline-shared
        cache slot).  shards <= 1: reference layout (E x D_i x H, E x H,
        E x H x D_o).  shards = P > 1: shard-major, as an all-gather of P
        hidden shards lands -- w1 (P*E) x D_i x h, b1 (P*E) x h (fp32),
        w2 (P*E) x h x D_o with h = H / P -- read in place by the GEMMs (no
        repacking copy).  ``ready``: an event recorded after the cache fill;
        the forward waits on it only after its routing prologue."""
        d = self.desc
        E, Di, H, Do = d.n_experts, d.d_in, d.hidden, d.d_out
        P = max(1, int(shards))
        if H % P:
            raise ValueError("set_weights: H must split evenly into the shards")
        h = H // P
        want = ((P * E, Di, h), (P * E, h), (P * E, h, Do)) if P > 1 else \
            ((E, Di, H), (E, H), (E, H, Do))
        for t, shp, nm in ((w1, want[0], "w1"), (b1, want[1], "b1"), (w2, want[2], "w2")):
            if tuple(t.shape) != shp or not t.is_contiguous():
                raise ValueError(f"set_weights: {nm} must be a contiguous {shp} tensor")
        if b1.dtype != torch.float32:
            raise ValueError("set_weights: b1 must be fp32")
        if P > 1 and not self._L.hxm_layer_weight_shards_ok(C.byref(d), P):
            raise ValueError(f"set_weights: this layer cannot read weights split {P} ways "
                             "(H / P must be a multiple of 64 and of the tile widths)")
        d.weight_shards = P if P > 1 else 0
        d.weights_ready = ready.cuda_event if ready is not None else None
        self._w1, self.b1, self._w2 = w1, b1, w2

    def forward(self, x: torch.Tensor, assignments: torch.Tensor, stream=None,
                status: torch.Tensor | None = None) -> torch.Tensor:
        st = (stream or torch.cuda.current_stream()).cuda_stream
        check(self._L.hxm_moe_forward(
            self._pd, x.data_ptr(), self._w1.data_ptr(), self.b1.data_ptr(),
            self._w2.data_ptr(), None if self.b2 is None else self.b2.data_ptr(),
            assignments.data_ptr(), self.y.data_ptr(), self.ws.data_ptr(), self.ws.numel(),
            None if status is None else status.data_ptr(), st), "moe_forward")
        return self.y

    def backward(self, x: torch.Tensor, g_y: torch.Tensor, stream=None) -> MoeGrads:
        st = (stream or torch.cuda.current_stream()).cuda_stream
        g = self.grads
        check(self._L.hxm_moe_backward(
            self._pd, x.data_ptr(), self._w1.data_ptr(), self._w2.data_ptr(), g_y.data_ptr(),
            self.ws.data_ptr(), self.ws.numel(), g.gw1.data_ptr(), g.gb1.data_ptr(),
            g.gw2.data_ptr(), None if g.gb2 is None else g.gb2.data_ptr(), g.gx.data_ptr(), st),
            "moe_backward")
        return g

    def backward_dc(self, x: torch.Tensor, g_y: torch.Tensor, gw1_shards, gw2_shards, stream=None):
        """Data-centric backward: gW1 / gW2 reduce-scattered along H into the
        shard owners' peer buffers (dist.PeerBuffers) inside the ESTMM
        epilogues; gb1, gb2, gx land in this runner's grads."""
        st = (stream or torch.cuda.current_stream()).cuda_stream
        g = self.grads
        check(self._L.hxm_moe_backward_dc(
            self._pd, x.data_ptr(), self._w1.data_ptr(), self._w2.data_ptr(), g_y.data_ptr(),
            self.ws.data_ptr(), self.ws.numel(), C.byref(gw1_shards.rows_struct),
            g.gb1.data_ptr(), C.byref(gw2_shards.rows_struct),
            None if g.gb2 is None else g.gb2.data_ptr(), g.gx.data_ptr(), st),
            "moe_backward_dc")
        return g

    def step(self, x, assignments, g_y, stream=None):
        self.forward(x, assignments, stream)
        return self.backward(x, g_y, stream)

    # ---- CUDA graph: the whole fwd+bwd step as one launch -----------------
    def capture(self, x, assignments, g_y, warm: bool = True) -> None:
        """Record step(x, assignments, g_y) into a CUDA graph.  x / assignments /
        g_y become the graph's static input buffers: refill them in place
        (copy_) before replay()."""
        if warm:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self.step(x, assignments, g_y)  # kernel attributes, tensor maps
            torch.cuda.current_stream().wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.step(x, assignments, g_y)

    def replay(self) -> MoeGrads:
        self.graph.replay()
        return self.grads


class HostPipeline:
    """Layer steps fed from (pinned) HOST memory with the PCIe traffic
    overlapped: step i's H2D copies, step i-1's compute and step i-2's D2H of
    y run concurrently on three streams, double-buffered (two LayerRunners
    sharing the parameters, each replaying its own CUDA graph).

    push(x_h, a_h, gy_h, y_h, gx_h=None, grads_h=None): enqueue one step;
    y_h (pinned) receives y, gx_h (optional, pinned N x D_i fp32) g_x, and
    grads_h (optional: a MoeGrads of pinned host tensors) the parameter
    gradients -- what a caller of the reference's moe_backward receives in
    host memory (moe_layer.hpp:70-73).
    drain(): wait for everything enqueued."""

    def __init__(self, p: MoeLayerParams, n_tokens: int, k: int, d_in: int, d_out: int,
                 device="cuda", dtype=torch.bfloat16, capacity: int = 0):
        self.runners = [LayerRunner(p, n_tokens, k, device, dtype, capacity=capacity)
                        for _ in range(2)]
        f = dict(device=device)
        self.x = [torch.empty(n_tokens, d_in, dtype=dtype, **f) for _ in range(2)]
        self.a = [torch.zeros(k, n_tokens, dtype=torch.int32, **f) for _ in range(2)]
        self.gy = [torch.empty(n_tokens, d_out, dtype=dtype, **f) for _ in range(2)]
        self.s_in, self.s_out = torch.cuda.Stream(), torch.cuda.Stream()
        self.s_comp = torch.cuda.current_stream()
        self.ev_in = [torch.cuda.Event() for _ in range(2)]
        self.ev_comp = [torch.cuda.Event() for _ in range(2)]
        self.ev_out = [torch.cuda.Event() for _ in range(2)]
        self.i = 0
        self.captured = False

    def _capture(self, a_init):
        for b in range(2):
            self.a[b].copy_(a_init)
            self.x[b].zero_()
            self.gy[b].zero_()
            self.runners[b].capture(self.x[b], self.a[b], self.gy[b])
        torch.cuda.synchronize()
        for b in range(2):  # events start "recorded"
            self.ev_comp[b].record(self.s_comp)
            self.ev_out[b].record(self.s_comp)
        self.captured = True

    def push(self, x_h, a_h, gy_h, y_h, gx_h=None, grads_h=None):
        if not self.captured:
            self._capture(a_h.to(self.a[0].device))
        b = self.i % 2
        self.i += 1
        with torch.cuda.stream(self.s_in):
            self.s_in.wait_event(self.ev_comp[b])  # step i-2 done reading buffer b
            self.x[b].copy_(x_h, non_blocking=True)
            self.a[b].copy_(a_h, non_blocking=True)
            self.gy[b].copy_(gy_h, non_blocking=True)
            self.ev_in[b].record(self.s_in)
        self.s_comp.wait_event(self.ev_in[b])
        self.s_comp.wait_event(self.ev_out[b])  # y_b of step i-2 copied out
        self.runners[b].replay()
        self.ev_comp[b].record(self.s_comp)
        with torch.cuda.stream(self.s_out):
            self.s_out.wait_event(self.ev_comp[b])
            y_h.copy_(self.runners[b].y, non_blocking=True)
            g = self.runners[b].grads
            if gx_h is not None:
                gx_h.copy_(g.gx, non_blocking=True)
            if grads_h is not None:
                for key in ("gw1", "gb1", "gw2", "gb2"):
                    dst = getattr(grads_h, key)
                    if dst is not None and getattr(g, key) is not None:
                        dst.copy_(getattr(g, key), non_blocking=True)
            self.ev_out[b].record(self.s_out)

    def drain(self):
        self.s_comp.wait_stream(self.s_in)
        self.s_comp.wait_stream(self.s_out)
