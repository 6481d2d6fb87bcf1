"""Reference-compatible front end (reference
tools/main.cpp, tools/commands.cpp, core/src/dist_sim.cpp:756-817).

    python -m paper_2411_01288_b200.cli bench    [CommonOptions] [--distribution D] [--routing-csv F]
    python -m paper_2411_01288_b200.cli allocate --latencies T... --total N [--kind batch|hidden]
    python -m paper_2411_01288_b200.cli probe    [--iterations I] [--size S] [--seed S]

The flags, their defaults and validation are moekit's CommonOptions
(commands.hpp:21-38, commands.cpp:42-58); usage errors exit 2 (kExitUsage).
``bench`` emits the reference's bench report columns (commands.cpp:234-279,
schemas/bench_report.schema.json) -- deterministic work / memory counts plus
timings -- except that every timing is the device time of this package's
CUDA kernels (CUDA events, microseconds), one row per top-k in 1..topk exactly
as run_bench does.  ``--config`` reads a JSON file with the CommonOptions /
SimScenario keys (load_scenario, dist_sim.cpp:756-817).
"""
from __future__ import annotations

import argparse
import json
import sys
from dataclasses import dataclass, field
from typing import List, Optional

EXIT_OK, EXIT_VERIFY_FAIL, EXIT_USAGE = 0, 1, 2

BENCH_COLUMNS = [
    "n", "experts", "topk", "din", "hidden", "dout", "blk", "distribution",
    "capacity_factor", "seed", "macs_expert_specific", "macs_counted", "macs_oracle",
    "capacity_per_expert", "padded_rows", "dropped_tokens", "mem_units_naive",
    "mem_units_efficient", "wall_esmm_us", "wall_ess_us", "wall_estmm_us", "wall_esfk_us",
    "wall_forward_us", "wall_backward_us"]


class UsageError(RuntimeError):
    """Invalid flags / unreadable configs (commands.hpp:15-19) -> exit 2."""


@dataclass
class CommonOptions:  # commands.hpp:21-38 (same defaults)
    n: int = 64
    experts: int = 8
    topk: int = 2
    d_in: int = 16
    hidden: int = 32
    d_out: int = 16
    blk: int = 8
    seed: int = 1
    scheme: str = "memory_efficient"
    activation: str = "gelu"
    capacity_factor: float = 1.0
    config_path: str = ""
    out_path: str = ""
    format: str = "json"

    def validate(self) -> None:  # commands.cpp:42-58
        if 0 in (self.n, self.experts, self.topk, self.d_in, self.hidden, self.d_out, self.blk):
            raise UsageError("all dimensions must be positive")
        if self.topk > self.experts:
            raise UsageError("--topk must not exceed --experts")
        if self.format not in ("json", "csv"):
            raise UsageError("--format must be json or csv")
        if not self.capacity_factor > 0.0:
            raise UsageError("--capacity-factor must be > 0")
        if self.scheme not in ("naive", "memory_efficient"):
            raise UsageError(f"unknown scheme: {self.scheme}")
        if self.activation not in ("relu", "gelu", "identity"):
            raise UsageError(f"unknown activation: {self.activation}")


@dataclass
class SimScenario:  # dist_sim.hpp SimScenario (keys of load_scenario)
    devices: List[dict] = field(default_factory=list)
    n: int = 64
    experts: int = 8
    k: int = 2
    d_in: int = 16
    hidden: int = 32
    d_out: int = 16
    blk: int = 8
    seed: int = 1
    mode: str = "data_centric"
    moe_scheme: str = "memory_efficient"
    activation: str = "gelu"
    distribution: str = "uniform"
    use_fused: bool = False
    non_moe_seconds: float = 0.0
    n_layers: int = 1
    workloads: List[int] = field(default_factory=list)
    batch_shares: List[int] = field(default_factory=list)
    hidden_shares: List[int] = field(default_factory=list)
    device_latencies: List[float] = field(default_factory=list)


def load_scenario(path: str) -> SimScenario:
    """dist_sim.cpp:756-817: same keys, same defaults, device specs validated."""
    try:
        with open(path) as f:
            j = json.load(f)
    except OSError:
        raise UsageError(f"{path}: cannot open config") from None
    except ValueError as e:
        raise UsageError(f"{path}: invalid JSON: {e}") from None
    s = SimScenario()
    if "devices" not in j:
        raise UsageError(f"{path}: missing key 'devices'")
    for dj in j["devices"]:
        d = {"id": dj.get("id", len(s.devices)), "compute_rate": dj.get("compute_rate", 1e9),
             "link_bandwidth": dj.get("link_bandwidth", 1e8),
             "link_latency": dj.get("link_latency", 0.0)}
        if not (d["compute_rate"] > 0 and d["link_bandwidth"] > 0 and d["link_latency"] >= 0):
            raise UsageError(f"{path}: invalid device spec {dj}")
        s.devices.append(d)
    for key, attr in (("n", "n"), ("experts", "experts"), ("topk", "k"), ("din", "d_in"),
                      ("hidden", "hidden"), ("dout", "d_out"), ("blk", "blk"), ("seed", "seed"),
                      ("mode", "mode"), ("moe_scheme", "moe_scheme"),
                      ("activation", "activation"), ("distribution", "distribution"),
                      ("use_fused", "use_fused"), ("non_moe_seconds", "non_moe_seconds"),
                      ("n_layers", "n_layers"), ("workloads", "workloads"),
                      ("batch_shares", "batch_shares"), ("hidden_shares", "hidden_shares"),
                      ("device_latencies", "device_latencies")):
        if key in j:
            setattr(s, attr, j[key])
    return s


def _common_from_config(c: CommonOptions) -> CommonOptions:
    if not c.config_path:
        return c
    try:
        with open(c.config_path) as f:
            j = json.load(f)
    except OSError:
        raise UsageError(f"{c.config_path}: cannot open config") from None
    except ValueError as e:
        raise UsageError(f"{c.config_path}: invalid JSON: {e}") from None
    for key, attr in (("n", "n"), ("experts", "experts"), ("topk", "topk"), ("din", "d_in"),
                      ("hidden", "hidden"), ("dout", "d_out"), ("blk", "blk"), ("seed", "seed"),
                      ("scheme", "scheme"), ("moe_scheme", "scheme"),
                      ("activation", "activation"), ("capacity_factor", "capacity_factor")):
        if key in j:
            setattr(c, attr, j[key])
    return c


def _emit(text: str, out_path: str) -> None:
    if out_path:
        with open(out_path, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text if text.endswith("\n") else text + "\n")


def _dev_us(fn, reps: int = 3) -> float:
    """Mean device microseconds of fn() (CUDA events on the current stream,
    after one warm-up call)."""
    import torch
    fn()
    s = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fn()
    b.record(s)
    b.synchronize()
    return 1e3 * a.elapsed_time(b) / reps


def run_bench(c: CommonOptions, distribution: str = "uniform",
              routing_csv: str = "") -> List[dict]:
    """commands.cpp:153-281 on the device: one row per k in 1..topk."""
    import torch

    from . import conventional as CV
    from .es_ops import esfk, esmm, ess, estmm
    from .moe_layer import (estimate_activation_memory, make_desc, make_random_params,
                            moe_backward, moe_forward)
    from .routing import RoutingChoice, build_reindex, read_routing_csv, synthesize_routing
    c.validate()
    if not torch.cuda.is_available():
        raise RuntimeError("bench: no CUDA device (there is no CPU fallback)")
    dtype = torch.bfloat16
    rows = []
    for k in range(1, c.topk + 1):
        if routing_csv:
            full = read_routing_csv(routing_csv)
            if full.k < k:
                break
            r = RoutingChoice(full.n_tokens, full.n_experts, k, full.assignments[:k].copy())
        else:
            r = synthesize_routing(c.n, c.experts, k, distribution, c.seed)
        p, x = make_random_params(r.n_experts, c.d_in, c.hidden, c.d_out, c.activation,
                                  seed=c.seed, n_tokens=r.n_tokens, dtype=dtype)
        a0 = torch.as_tensor(r.assignments[0]).cuda()
        rx = build_reindex(a0, r.n_experts, c.blk)
        rep = CV.count_redundancy(r, c.d_in, c.hidden, c.d_out, c.capacity_factor)
        ratio = c.hidden / c.d_in
        row = {"n": r.n_tokens, "experts": r.n_experts, "topk": k, "din": c.d_in,
               "hidden": c.hidden, "dout": c.d_out, "blk": c.blk,
               "distribution": distribution if not routing_csv else "csv",
               "capacity_factor": c.capacity_factor, "seed": c.seed,
               "macs_expert_specific": rep.token_macs_expert_specific,
               "macs_oracle": rep.token_macs_oracle,
               "capacity_per_expert": rep.capacity_per_expert,
               "padded_rows": rep.padded_rows, "dropped_tokens": rep.dropped_tokens,
               "mem_units_naive": estimate_activation_memory(r.n_tokens, k, ratio, "naive"),
               "mem_units_efficient": estimate_activation_memory(r.n_tokens, k, ratio,
                                                                 "memory_efficient")}
        y1 = esmm(x, p.w1, p.b1, rx)
        y1b = y1.to(dtype)
        row["wall_esmm_us"] = _dev_us(lambda: esmm(x, p.w1, p.b1, rx))
        row["wall_ess_us"] = _dev_us(lambda: ess(y1b, rx))
        row["wall_estmm_us"] = _dev_us(lambda: estmm(x, y1b, rx))
        row["wall_esfk_us"] = _dev_us(lambda: esfk(x, y1b, p.w1, rx, w_transposed=True))
        fw = moe_forward(x, p, r, c.blk, c.scheme)
        row["wall_forward_us"] = _dev_us(lambda: moe_forward(x, p, r, c.blk, c.scheme,
                                                             validate=False))
        gy = torch.ones(r.n_tokens, c.d_out, dtype=dtype, device="cuda")
        row["wall_backward_us"] = _dev_us(lambda: moe_backward(fw.stash, p, gy))
        import ctypes
        from ._lib import lib
        desc = make_desc(r.n_tokens, r.n_experts, k, c.d_in, c.hidden, c.d_out, c.activation,
                         dtype)
        row["macs_counted"] = int(lib().hxm_layer_forward_macs(ctypes.byref(desc)))
        rows.append({key: row[key] for key in BENCH_COLUMNS})
    return rows


def format_rows(rows: List[dict], fmt: str) -> str:
    if fmt == "json":
        return json.dumps({"rows": rows}, indent=2)
    out = [",".join(BENCH_COLUMNS)]
    for r in rows:
        out.append(",".join(str(r[c]) for c in BENCH_COLUMNS))
    return "\n".join(out) + "\n"


def _add_common(ap: argparse.ArgumentParser) -> None:
    d = CommonOptions()
    ap.add_argument("--n", type=int, default=d.n)
    ap.add_argument("--experts", type=int, default=d.experts)
    ap.add_argument("--topk", type=int, default=d.topk)
    ap.add_argument("--din", type=int, default=d.d_in)
    ap.add_argument("--hidden", type=int, default=d.hidden)
    ap.add_argument("--dout", type=int, default=d.d_out)
    ap.add_argument("--seed", type=int, default=d.seed)
    ap.add_argument("--scheme", default=d.scheme)
    ap.add_argument("--activation", default=d.activation)
    ap.add_argument("--capacity-factor", type=float, default=d.capacity_factor)
    ap.add_argument("--config", default="")
    ap.add_argument("--out", default="")
    ap.add_argument("--format", default=d.format)
    ap.add_argument("--blk", type=int, default=d.blk)


def _common(ns) -> CommonOptions:
    return _common_from_config(CommonOptions(
        n=ns.n, experts=ns.experts, topk=ns.topk, d_in=ns.din, hidden=ns.hidden,
        d_out=ns.dout, blk=ns.blk, seed=ns.seed, scheme=ns.scheme, activation=ns.activation,
        capacity_factor=ns.capacity_factor, config_path=ns.config, out_path=ns.out,
        format=ns.format))


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse errors are usage errors (exit 2)
        raise UsageError(message)


def main(argv: Optional[List[str]] = None) -> int:
    ap = _Parser(prog="paper_2411_01288_b200.cli")
    sub = ap.add_subparsers(dest="cmd")
    b = sub.add_parser("bench", help="work/memory counts plus device timings")
    _add_common(b)
    b.add_argument("--distribution", default="uniform")
    b.add_argument("--routing-csv", default="")
    al = sub.add_parser("allocate", help="heterogeneous batch / hidden allocation")
    al.add_argument("--latencies", type=float, nargs="+", default=[])
    al.add_argument("--total", type=int, default=0)
    al.add_argument("--kind", default="batch")
    al.add_argument("--config", default="")
    al.add_argument("--out", default="")
    al.add_argument("--format", default="json")
    pr = sub.add_parser("probe", help="GPU capacity probe (seconds)")
    pr.add_argument("--device-id", type=int, default=0)
    pr.add_argument("--iterations", type=int, default=8)
    pr.add_argument("--size", type=int, default=192)
    pr.add_argument("--seed", type=int, default=1)
    pr.add_argument("--out", default="")
    try:
        ns = ap.parse_args(argv)
        if ns.cmd == "bench":
            c = _common(ns)
            c.validate()
            rows = run_bench(c, ns.distribution, ns.routing_csv)
            _emit(format_rows(rows, c.format), c.out_path)
        elif ns.cmd == "allocate":
            from . import hetero as HA
            lat, total, kind = ns.latencies, ns.total, ns.kind
            if ns.config:
                try:
                    with open(ns.config) as f:
                        j = json.load(f)
                except (OSError, ValueError) as e:
                    raise UsageError(f"{ns.config}: cannot read config: {e}") from None
                lat = j.get("device_latencies", j.get("latencies", lat))
                total = j.get("total", total)
                kind = j.get("kind", kind)
            if kind not in ("batch", "hidden"):
                raise UsageError("--kind must be batch or hidden")
            if ns.format not in ("json", "csv"):
                raise UsageError("--format must be json or csv")
            try:
                plan = (HA.allocate_batches if kind == "batch" else HA.allocate_hidden)(lat, total)
            except ValueError as e:
                raise UsageError(str(e)) from None
            _emit(plan.to_json() if ns.format == "json" else plan.to_csv(), ns.out)
        elif ns.cmd == "probe":
            from . import hetero as HA
            try:
                t = HA.probe_capacity_seconds(ns.iterations, ns.size, ns.seed)
            except ValueError as e:
                raise UsageError(str(e)) from None
            _emit(json.dumps({"device_id": ns.device_id, "iterations": ns.iterations,
                              "matrix_size": ns.size, "seconds": t}), ns.out)
        else:
            ap.print_help()
            return EXIT_USAGE
    except UsageError as e:
        print(f"usage error: {e}", file=sys.stderr)
        return EXIT_USAGE
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
