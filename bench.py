#!/usr/bin/env python
"""bench.py -- MoE-layer fwd+bwd tokens/s of the B200-native HEXA-MoE hot path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One step = one fwd+bwd pass (routing-index build, ESMM x4, ESTMM x2, ESS x2)
of the layer over one synthetic batch: the reference's own generators
(make_random_params scale 0.5, x ~ N(0,1), uniform top-k routing, seed 1,
g_y = ones as in tools/commands.cpp:220-221).

value   : whole-job tokens/s with inputs resident in HBM, each step timed with
          CUDA events on the launch stream, L2 flushed (256 MiB write) between
          steps outside the timed events, max over ranks.
e2e     : the same metric through the public API (paper_2411_01288_b200.HostPipeline /
          LayerRunner) with x, g_y and the routing in pinned HOST memory: H2D
          copies, fwd+bwd and the D2H reads of y and g_x are inside the timed
          region every step (e2e_full_grads: plus gW1, gb1, gW2, gb2 D2H).
roofline: the dominant kernel's algorithmic FLOP (or bytes) per launch over its
          live CUDA-event duration inside the timed region, against
          MEASURED_PEAKS.json.
cpu_baseline: the reference's own CPU path (oracle/_ref, compiled unmodified
          from /root/reference) on the host cores, rank 0, bounded sample.
--impl reference: times that same reference CPU path as the reference arm.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs; N for c3/c5 is not given there
    "c1": dict(E=8, k=1, D=96, H=384, N=3136, dtype="f32", dist="uniform",
               desc="single MoE-MLP layer 8E top-1 d96 ffn384 3136 tok fp32"),
    "c2": dict(E=32, k=2, D=384, H=1536, N=16384, dtype="bf16", dist="uniform",
               desc="Swin-MoE-S stage-3 layer 32E top-2 d384 ffn1536 16384 tok bf16"),
    "c3": dict(E=32, k=2, D=1024, H=4096, N=16384, dtype="bf16", dist="uniform",
               desc="Swin-MoE-B stage-4 layer 32E top-2 d1024 ffn4096, 16384 tok per GPU"),
    "c4": dict(E=64, k=2, D=1024, H=4096, N=131072, dtype="bf16", dist="uniform",
               desc="64E top-2 d1024 ffn4096 131072 tok"),
    "c5": dict(E=64, k=2, D=768, H=3072, N=16384, dtype="bf16", dist="skew90",
               desc="64E top-2 d768 ffn3072, 90% of tokens to experts {0,1}"),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return dict(hbm=d["hbm_gbs"], tensor=d["bf16_tflops"],
                    tensor_sustained=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    source="measured")
    except (OSError, KeyError, ValueError):
        return dict(hbm=6650.0, tensor=1590.0, tensor_sustained=1400.0, source="fallback")


def skew90_routing(N, E, k, seed):
    """c5: 90% of tokens choose {0, 1} (choice i -> expert i), the rest uniform
    distinct pairs from the reference generator."""
    import numpy as np
    from paper_2411_01288_b200 import RoutingChoice, synthesize_routing
    r = synthesize_routing(N, E, k, "uniform", seed)
    a = r.assignments.copy()
    rng = np.random.default_rng(seed)
    hot = rng.random(N) < 0.9
    for i in range(k):
        a[i, hot] = i
    return RoutingChoice(N, E, k, a)


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling during the timed region."""

    def __init__(self, index=0, period=0.1):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self.period, self._stop = period, threading.Event()
        try:
            import pynvml as N
            N.nvmlInit()
            self.N, self.h = N, N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001 - clocks are best effort
            self.N = None

    def _run(self):
        N = self.N
        names = {getattr(N, a): a for a in dir(N) if a.startswith("nvmlClocksThrottleReason")
                 and isinstance(getattr(N, a), int)}
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                bits = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for v, nm in names.items():
                    if v and bits & v and v != N.nvmlClocksThrottleReasonGpuIdle:
                        self.reasons.add(nm.replace("nvmlClocksThrottleReason", ""))
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.N:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.N:
            self._stop.set()
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_init(args):
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1 or args.mode in ("data_centric", "model_centric"):
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(ws))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, ws, local


def max_over_ranks(v, ws):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    import torch
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()


def cpu_model():
    """lscpu's model name of this host."""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _ref_rate(O, cfg, n, threads):
    E, k, D, H = cfg["E"], cfg["k"], cfg["D"], cfg["H"]
    return n / O.ref_time_layer(E, k, D, H, D, n, 8, threads, 1)


def ref_sample_tokens(O, cfg, threads, seconds):
    """Tokens per reference step: at least REF_MIN_PER_THREAD tokens per thread
    (so the per-call fixed costs -- transpose_experts of the whole weight set,
    moe_layer.cpp:91-92 -- are amortised as in one full-batch call), grown to
    about `seconds` of work, never above N.  Independent of --steps, and the
    same sample for the reference arm and the cpu_baseline leg."""
    probe = min(cfg["N"], threads * 64)
    rate = _ref_rate(O, cfg, probe, threads)
    n = max(threads * REF_MIN_PER_THREAD, int(rate * seconds))
    n = min(cfg["N"], n)
    return max(threads, n // threads * threads)


REF_MIN_PER_THREAD = 1024
REF_SAMPLE_SECONDS = 20.0   # work per reference step (c2: the full 16384-token batch)
REF_RUN_BUDGET_S = 150.0    # --impl reference: timed steps stop once this is spent


def cpu_baseline(cfg):
    """Reference CPU path (oracle/_ref) on the reference arm's sample: all host
    threads on disjoint token shards, plus a 1-core figure (the reference is
    single-threaded)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.ref_available():
        return None
    threads = max(1, min(os.cpu_count() or 1, 64))
    n = ref_sample_tokens(O, cfg, threads, REF_SAMPLE_SECONDS)
    E, k, D, H = cfg["E"], cfg["k"], cfg["D"], cfg["H"]
    t = O.ref_time_layer(E, k, D, H, D, n, 8, threads, 1)
    # one core: a single moe_forward + moe_backward call of ~10 s of work
    n1 = max(64, min(cfg["N"], int(n / t / threads * 10.0)))
    t1 = O.ref_time_layer(E, k, D, H, D, n1, 8, 1, 1)
    return {"value": n / t, "unit": "tokens/s", "cores": threads, "kind": "reference",
            "sample": f"{n} of {cfg['N']} tokens, fwd+bwd via moekit::moe_forward/"
                      f"moe_backward, {threads} threads on disjoint token shards "
                      f"({n // threads} tokens each)",
            "seconds": t, "cpu_model": cpu_model(),
            "single_core": {"value": n1 / t1, "unit": "tokens/s", "cores": 1,
                            "sample": f"{n1} tokens, one call", "seconds": t1}}


def run_reference(args, cfg, rank, ws):
    """--impl reference: the reference's CPU implementation of the same path
    (oracle/_ref = the unmodified moekit sources), all host threads on
    disjoint token shards.  Every timed step is the same sample as the
    cpu_baseline leg (>= 1024 tokens per thread, c2: the full batch),
    independent of --steps; the timed steps stop after REF_RUN_BUDGET_S so a
    large --steps still ends within a few minutes (steps_timed says how many
    ran).  Warm-up steps are small samples (page faults / caches only)."""
    if rank != 0:
        return
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built"}))
        return
    threads = max(1, min(os.cpu_count() or 1, 64))
    E, k, D, H = cfg["E"], cfg["k"], cfg["D"], cfg["H"]
    n = ref_sample_tokens(O, cfg, threads, REF_SAMPLE_SECONDS)
    nw = max(threads, min(n, threads * 32))
    for _ in range(args.warmup):
        O.ref_time_layer(E, k, D, H, D, nw, 8, threads, 1)
    times = []
    while len(times) < args.steps and (not times or sum(times) < REF_RUN_BUDGET_S):
        times.append(O.ref_time_layer(E, k, D, H, D, n, 8, threads, 1))
    total = sum(times)
    val = n * len(times) / total
    sample = (f"{n} of {cfg['N']} tokens per step ({n // threads} per thread), {threads} "
              f"threads on disjoint token shards; {len(times)} of {args.steps} steps timed "
              f"(run budget {REF_RUN_BUDGET_S:.0f} s); warm-up steps {nw} tokens")
    out = {
        "impl": "reference", "metric": "MoE layer fwd+bwd tokens/sec", "value": val,
        "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "steps_timed": len(times),
        "ms_per_step": 1000 * total / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "E": E, "k": k, "d": D,
                   "ffn": H, "tokens": cfg["N"]},
        "cpu_baseline": {"value": val, "unit": "tokens/s", "cores": threads,
                         "kind": "reference", "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": val, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def _redundancy(args, r, D, Hd):
    """count_redundancy (gemm_oracle.cpp:251-285) of the baseline run."""
    from paper_2411_01288_b200 import conventional as CV
    rep = CV.count_redundancy(r, D, Hd, D, args.capacity_factor)
    out = dict(rep.__dict__)
    out["capacity_factor"] = args.capacity_factor
    out["device_capacity_rows"] = CV.capacity_rows(r.n_tokens, r.n_experts, r.k,
                                                   args.capacity_factor)
    return out


def run_ours(args, cfg, rank, ws, local):
    cap = 0  # conventional-baseline capacity rows (single mode)
    import numpy as np
    import torch

    import paper_2411_01288_b200 as H
    from paper_2411_01288_b200 import _lib
    from paper_2411_01288_b200.runner import LayerRunner

    dtype = torch.bfloat16 if cfg["dtype"] == "bf16" else torch.float32
    E, k, D, Hd, N = cfg["E"], cfg["k"], cfg["D"], cfg["H"], cfg["N"]
    dev = torch.device("cuda", torch.cuda.current_device())
    seed = 1 + rank  # each rank its own token batch (weak scaling)
    p, x = H.make_random_params(E, D, Hd, D, "gelu", seed=1, n_tokens=N, dtype=dtype,
                                device=dev)
    if rank:
        _, x = H.make_random_params(E, D, Hd, D, "gelu", seed=seed, n_tokens=N, dtype=dtype,
                                    device=dev)
    r = skew90_routing(N, E, k, seed) if cfg["dist"] == "skew90" else \
        H.synthesize_routing(N, E, k, cfg["dist"], seed)
    a = r.to_device(dev)
    gy = torch.ones(N, D, dtype=dtype, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    L = _lib.lib()
    mode = args.mode if args.mode != "auto" else ("single" if ws == 1 else "data_centric")
    use_graph = mode == "single" and not args.no_graph

    if mode == "model_centric":
        # model-centric TP along H (dist_sim.cpp:454-601): tokens / routing /
        # g_y all-gathered, each rank runs the global batch on its H-slice,
        # partial y and g_x reduce-scattered back to the token owners
        from paper_2411_01288_b200 import dist as HD
        sp = HD.shard_params(p, HD.even_split(Hd, ws))
        shard, b2 = sp.shards[rank], sp.b2
        del p, sp
        comp = HD.cuda_compute()
        mc_out = {}
        fused = not args.no_fused and cfg["dtype"] == "bf16"
        if fused:
            # y / g_x reduce-scattered inside the ESMM epilogues over peer
            # memory (CUDA IPC handles, device barrier) -- no NCCL afterwards
            ybuf = HD.PeerBuffers(N, D)
            gxbuf = HD.PeerBuffers(N, D)

        def mc_step():
            if fused:
                res = HD.model_centric_step_fused(x, a, gy, shard, b2, "gelu", ybuf, gxbuf)
            else:
                res = HD.model_centric_step(x, a, gy, shard, b2, "gelu", comp,
                                            reduce="reduce_scatter")
            mc_out["y"] = res.y
            return res
        mc_step()
        torch.cuda.synchronize()
        y_out = mc_out["y"]
    elif mode == "single":
        cap = 0
        if args.capacity_factor > 0:
            from paper_2411_01288_b200.moe_layer import capacity_rows
            cap = capacity_rows(N, E, k, args.capacity_factor)
        run = LayerRunner(p, N, k, dev, dtype, capacity=cap)
        # warm-up (also validates routing once)
        status = torch.zeros(1, dtype=torch.int32, device=dev)
        run.forward(x, a, status=status)
        run.backward(x, gy)
        torch.cuda.synchronize()
        assert int(status.item()) == 0
        y_out = run.y
    else:
        # data-centric TP along H (dist_sim.cpp:352-452): rank r owns an even
        # H-slice; every step all-gathers it into the pipeline-shared cache,
        # runs the full layer on this rank's 16384 tokens and reduce-scatters
        # the gradients to the shard owners
        from paper_2411_01288_b200 import dist as HD
        sp = HD.shard_params(p, HD.even_split(Hd, ws))
        dc = HD.DataCentricRunner(sp.shards[rank], sp.b2 if rank == 0 else None,
                                  sp.hidden_sizes, "gelu", N, k, None, dtype)
        if not args.no_fused and cfg["dtype"] == "bf16":
            dc.enable_fused_grads()  # gW reduce-scatter inside the ESTMM epilogues
        del p, sp
        run = dc.runner
        y_out = run.y
    if mode == "single":
        step_fn = lambda: run.step(x, a, gy)  # noqa: E731
    elif mode == "data_centric":
        step_fn = lambda: dc.step(x, a, gy)  # noqa: E731
    else:
        step_fn = mc_step
    for _ in range(max(0, args.warmup - 1)):
        step_fn()
    graph_kernels = 0
    L.hxm_profile_reset()
    if use_graph:
        # two graphs of the same step: the timed one carries no event nodes;
        # the profiled one (per-kernel event pairs recorded as graph nodes)
        # gives the kernel durations in a second pass of K steps
        c0 = L.hxm_launch_count()
        run.capture(x, a, gy)
        graph_kernels = (L.hxm_launch_count() - c0) // 2  # capture() warms once
        g_plain = run.graph
        L.hxm_profile_enable(1)
        run.capture(x, a, gy, warm=False)
        L.hxm_profile_enable(0)
        g_prof = run.graph
        step_fn = g_plain.replay
        for _ in range(2):
            g_plain.replay()
            g_prof.replay()
    barrier(ws)

    def timed(fn, profile_eager):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
        barrier(ws)
        if profile_eager:
            L.hxm_profile_reset()
            L.hxm_profile_enable(1)
        for i in range(args.steps):
            flush.zero_()  # L2 flush outside the step's events
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        L.hxm_profile_enable(0)
        barrier(ws)
        return sum(s.elapsed_time(e) for s, e in evs)

    # ---- device-resident timed region ------------------------------------
    launches0 = L.hxm_launch_count()
    clocks = ClockSampler(local, period=0.005)
    with clocks:
        # the value pass never carries per-kernel events (eager modes too)
        total_ms = max_over_ranks(timed(step_fn, False), ws)
        launches = L.hxm_launch_count() - launches0
        if use_graph:
            launches = graph_kernels * args.steps  # each replay runs the captured kernels
            # second pass: the profiled graph (its event nodes hold the last
            # replay's per-kernel durations)
            prof_ms = max_over_ranks(timed(g_prof.replay, False), ws)
        else:
            # second pass of the eager step with an event pair per launch
            prof_ms = max_over_ranks(timed(step_fn, True), ws)
    prof = _lib.profile_read()
    L.hxm_profile_reset()
    value = N * ws * args.steps / (total_ms / 1000.0)

    # ---- end-to-end through the public API with host buffers --------------
    # every step: x, g_y and the routing copied in from pinned host memory,
    # fwd+bwd, and the per-token outputs y AND g_x read back (what a layer
    # inside a network hands its neighbours); a second variant also reads
    # back the parameter gradients gW1, gb1, gW2, gb2 -- everything the
    # reference's moe_backward returns in host memory (moe_layer.hpp:70-73)
    xh = x.cpu().pin_memory()
    gyh = gy.cpu().pin_memory()
    ah = a.cpu().pin_memory()
    yh = torch.empty(N, D, dtype=torch.float32).pin_memory()
    gxh = torch.empty(N, D, dtype=torch.float32).pin_memory()
    e2e_steps = max(3, args.steps, 40)  # amortise the 3-stage pipeline fill / drain

    def run_e2e(full_grads):
        if use_graph:
            # public API HostPipeline: H2D of step i, compute of step i-1 and
            # D2H of step i-2 overlap on three streams (double-buffered)
            from paper_2411_01288_b200.moe_layer import MoeGrads
            from paper_2411_01288_b200.runner import HostPipeline
            pipe = HostPipeline(run.p, N, k, D, D, dev, dtype, capacity=cap)
            gh = None
            if full_grads:
                g0 = run.grads
                gh = MoeGrads(*(None if t is None else torch.empty_like(t, device="cpu")
                                .pin_memory() for t in (g0.gw1, g0.gb1, g0.gw2, g0.gb2, g0.gx)))

            def e2e_step():
                pipe.push(xh, ah, gyh, yh, gxh, gh)
            drain = pipe.drain
        else:
            gsrc = None if mode == "model_centric" else run.grads

            def e2e_step():
                # the step's static inputs are x / a / gy: refill them from the host
                x.copy_(xh, non_blocking=True)
                a.copy_(ah, non_blocking=True)
                gy.copy_(gyh, non_blocking=True)
                res = step_fn()
                yh.copy_(mc_out["y"] if mode == "model_centric" else y_out, non_blocking=True)
                gxs = res.grads.gx if mode == "model_centric" else gsrc.gx
                gxh[:gxs.shape[0]].copy_(gxs, non_blocking=True)
            drain = None
        for _ in range(2):
            e2e_step()
        if drain:
            drain()
        barrier(ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e2e_steps):
            e2e_step()
        if drain:
            drain()  # the last D2H lands before e1
        e1.record(stream)
        barrier(ws)
        ms = max_over_ranks(e0.elapsed_time(e1), ws)
        return N * ws * e2e_steps / (ms / 1000.0)

    e2e_val = run_e2e(False)
    h2d = xh.numel() * xh.element_size() + gyh.numel() * gyh.element_size() + \
        ah.numel() * ah.element_size()
    d2h = yh.numel() * yh.element_size() + gxh.numel() * gxh.element_size()
    e2e_full = None
    if use_graph:
        e2e_full = run_e2e(True)
        g0 = run.grads
        d2h_full = d2h + sum(t.numel() * 4 for t in (g0.gw1, g0.gb1, g0.gw2, g0.gb2)
                             if t is not None)

    if rank != 0:
        return
    pk = peaks()
    kernels = {}
    # each kernel under its own roofline: GEMM regions state FLOP and
    # algorithmic HBM bytes, the bound is whichever floor is longer (at
    # c2's K = 384 the stash GEMMs are HBM-bound, not tensor-bound)
    t_peak = pk["tensor"]  # burst: the step is short and clocks stay at max
    for nm, (ms, n, work, kind, nbytes) in prof.items():
        avg_s = ms / max(n, 1) / 1e3
        flop = work / max(n, 1) if kind == 0 else 0.0
        byts = (nbytes if kind == 0 else work) / max(n, 1)
        kd = {"avg_us": 1e6 * avg_s, "launches": n}
        if flop:
            kd["tflops"] = flop / avg_s / 1e12
            kd["frac_tensor"] = kd["tflops"] / t_peak
        if byts:
            kd["gbs"] = byts / avg_s / 1e9
            kd["frac_hbm"] = kd["gbs"] / pk["hbm"]
        tensor = flop and (not byts or flop / (t_peak * 1e12) >= byts / (pk["hbm"] * 1e9))
        kd["bound"] = "tensor" if tensor else "hbm"
        kd["achieved"] = kd["tflops"] if tensor else kd["gbs"]
        kd["unit"] = "TFLOP/s" if tensor else "GB/s"
        kd["frac"] = kd["frac_tensor"] if tensor else kd["frac_hbm"]
        kd["work_per_launch"] = flop if tensor else byts
        kernels[nm] = kd
    dom = max(prof.items(), key=lambda kv: kv[1][0])[0] if prof else None
    roof = None
    if dom:
        kd = kernels[dom]
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tf) and not args.shape:
            with open(tf) as f:
                traffic = json.load(f).get(args.config, {}).get(dom)
        tensor = kd["bound"] == "tensor"
        roof = {"kernel": dom, "bound": kd["bound"], "achieved": kd["achieved"],
                "peak": t_peak if tensor else pk["hbm"], "unit": kd["unit"], "frac": kd["frac"],
                "traffic": traffic,
                "peak_source": f"{pk['source']} ({'bf16 dense burst' if tensor else 'HBM copy'})",
                "work_per_launch": kd["work_per_launch"],
                "share_of_step": prof[dom][0] / max(sum(v[0] for v in prof.values()), 1e-9)}
    flop_step = 6.0 * k * N * (D * Hd + Hd * D)
    cpu = None
    if ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg)
    out = {
        "metric": "MoE layer fwd+bwd tokens/sec", "value": value, "unit": "tokens/s",
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "E": E, "k": k, "d": D,
                   "ffn": Hd, "tokens_per_gpu": N, "routing": cfg["dist"],
                   "parallelism": (f"{mode}_tp{ws}" + ("_fused_rs" if not args.no_fused else ""))
                   if mode != "single" else "single",
                   "formulation": (f"conventional dispatch/combine, capacity factor "
                                   f"{args.capacity_factor}") if args.capacity_factor > 0
                   else "expert-specific (no padding, no dropping)",
                   "cuda_graph": use_graph,
                   "kernel_times": "second K-step pass of the same step captured with per-kernel "
                                   "event nodes" if use_graph else
                                   "second K-step pass with events around each launch",
                   "l2": "flushed between steps (256 MiB write, outside the timed events)"},
        "ms_per_step_profiled": (prof_ms / args.steps) if prof_ms else None,
        "layer_tflops": flop_step * args.steps * ws / (total_ms / 1e3) / 1e12,
        "layer_frac_of_bf16_peak": flop_step * args.steps / (total_ms / 1e3) / 1e12 / pk["tensor"],
        "roofline": roof, "kernels": kernels,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                "copies": "H2D x, g_y, routing; D2H y and g_x (fp32), every step"},
        "e2e_full_grads": None if e2e_full is None else {
            "value": e2e_full, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h_full, "steps": e2e_steps,
            "copies": "as e2e plus gW1, gb1, gW2, gb2 (fp32) D2H every step"},
        "gpu_launches": int(launches),
        "redundancy": _redundancy(args, r, D, Hd) if args.capacity_factor > 0 else None,
        "clocks": clocks.summary(),
    }
    print(json.dumps(out))


def relaunch(args):
    """--gpus N without a torchrun environment: re-exec this command as N
    ranks (one process per GPU, NCCL over NVLink) -- or fail loudly when the
    box has fewer GPUs, never silently measure one."""
    import subprocess

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} requested but only {have} CUDA device(s) visible")
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--mode", default="auto",
                    choices=["auto", "single", "data_centric", "model_centric"],
                    help="auto: single GPU at N=1, data-centric TP along H at N>1")
    ap.add_argument("--no-fused", action="store_true",
                    help="model-centric: NCCL reduce-scatter instead of the fused GEMM epilogues")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the step eagerly instead of replaying its CUDA graph")
    ap.add_argument("--capacity-factor", type=float, default=0.0,
                    help="> 0: the conventional dispatch/combine baseline with this capacity "
                         "factor (gemm_oracle.cpp) instead of the expert-specific path")
    ap.add_argument("--shape", default=None,
                    help="experiment override E,k,D,H,N of the chosen config (not a bench line)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = dict(CONFIGS[args.config])
    if args.shape:
        E, k, D, H, N = (int(v) for v in args.shape.split(","))
        cfg.update(E=E, k=k, D=D, H=H, N=N, desc=f"experiment shape {args.shape}")
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, cfg, rank, int(os.environ.get("WORLD_SIZE", "1")))
        return
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch(args)  # does not return
    env_ws = int(os.environ.get("WORLD_SIZE", "1"))
    if env_ws != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={env_ws}: launch one rank per GPU "
                 f"(python -m torch.distributed.run --nproc-per-node {args.gpus} bench.py ...)")
    if args.gpus > 1:
        # communicator init lines (rank counts) on stderr for the driver
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    rank, ws, local = dist_init(args)
    try:
        run_ours(args, cfg, rank, ws, local)
    finally:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
