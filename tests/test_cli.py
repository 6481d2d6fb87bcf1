"""Reference-compatible front end (tools/main.cpp, tools/commands.cpp,
dist_sim.cpp:756-817): flags, validation, exit codes, report columns."""
import json
import os

import pytest

from paper_2411_01288_b200 import cli


def test_common_options_defaults_and_validation():
    c = cli.CommonOptions()
    assert (c.n, c.experts, c.topk, c.d_in, c.hidden, c.d_out, c.blk, c.seed) == \
        (64, 8, 2, 16, 32, 16, 8, 1)
    c.validate()
    for bad in (dict(n=0), dict(topk=9), dict(format="xml"), dict(capacity_factor=0.0),
                dict(scheme="fast"), dict(activation="tanh")):
        with pytest.raises(cli.UsageError):
            cli.CommonOptions(**bad).validate()


def test_usage_errors_exit_2(capsys):
    assert cli.main(["bench", "--topk", "9", "--experts", "4"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--format", "xml"]) == cli.EXIT_USAGE
    assert cli.main(["allocate", "--latencies", "1", "0", "--total", "5"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--no-such-flag"]) == cli.EXIT_USAGE
    assert cli.main(["bench", "--config", "/nonexistent.json"]) == cli.EXIT_USAGE
    assert cli.main([]) == cli.EXIT_USAGE


def test_allocate_json_and_csv(capsys, tmp_path):
    assert cli.main(["allocate", "--latencies", "4.58", "3.06", "--total", "100"]) == 0
    out = json.loads(capsys.readouterr().out)
    assert out["kind"] == "batch" and out["shares"] == [40, 60] and out["total"] == 100
    assert cli.main(["allocate", "--latencies", "3.28", "9.42", "--total", "100", "--kind",
                     "hidden", "--format", "csv"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0] == "device,ideal,share" and lines[1].endswith(",74")
    cfg = tmp_path / "a.json"
    cfg.write_text(json.dumps({"device_latencies": [1.0, 3.0], "total": 8, "kind": "hidden"}))
    out = tmp_path / "plan.json"
    assert cli.main(["allocate", "--config", str(cfg), "--out", str(out)]) == 0
    assert json.loads(out.read_text())["shares"] == [6, 2]


def test_load_scenario_keys(tmp_path):
    p = tmp_path / "s.json"
    p.write_text(json.dumps({"devices": [{"compute_rate": 2e9}, {"id": 7}], "n": 128,
                             "topk": 1, "din": 8, "mode": "model_centric", "n_layers": 3,
                             "hidden_shares": [20, 12], "device_latencies": [1.0, 2.0]}))
    s = cli.load_scenario(str(p))
    assert [d["id"] for d in s.devices] == [0, 7] and s.devices[0]["compute_rate"] == 2e9
    assert (s.n, s.k, s.d_in, s.mode, s.n_layers) == (128, 1, 8, "model_centric", 3)
    assert s.hidden_shares == [20, 12] and s.experts == 8  # default kept
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    with pytest.raises(cli.UsageError):
        cli.load_scenario(str(bad))
    nodev = tmp_path / "nodev.json"
    nodev.write_text("{}")
    with pytest.raises(cli.UsageError):
        cli.load_scenario(str(nodev))
    neg = tmp_path / "neg.json"
    neg.write_text(json.dumps({"devices": [{"compute_rate": -1}]}))
    with pytest.raises(cli.UsageError):
        cli.load_scenario(str(neg))


def test_bench_csv_header_matches_reference_columns():
    # commands.cpp:256-260 column order
    hdr = cli.format_rows([], "csv").splitlines()[0].split(",")
    assert hdr == cli.BENCH_COLUMNS
    assert hdr[:10] == ["n", "experts", "topk", "din", "hidden", "dout", "blk",
                        "distribution", "capacity_factor", "seed"]


@pytest.mark.gpu
def test_gpu_bench_rows_follow_the_schema(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = tmp_path / "bench.json"
    assert cli.main(["bench", "--n", "512", "--experts", "8", "--topk", "2", "--din", "64",
                     "--hidden", "128", "--dout", "64", "--capacity-factor", "1.25",
                     "--out", str(out)]) == 0
    rows = json.loads(out.read_text())["rows"]
    assert [r["topk"] for r in rows] == [1, 2]
    for r in rows:
        assert list(r) == cli.BENCH_COLUMNS
        assert r["macs_counted"] == r["macs_expert_specific"]  # zero redundancy
        assert r["macs_oracle"] >= r["macs_expert_specific"]
        assert all(r[k] > 0 for k in cli.BENCH_COLUMNS if k.startswith("wall_"))
    # routing CSV fixture drives the run (routing.cpp:202-282)
    import paper_2411_01288_b200 as H
    rc = tmp_path / "r.csv"
    H.write_routing_csv(str(rc), H.synthesize_routing(256, 4, 2, "uniform", 3))
    assert cli.main(["bench", "--experts", "4", "--din", "64", "--hidden", "64", "--dout", "64",
                     "--routing-csv", str(rc), "--format", "csv", "--out",
                     str(tmp_path / "b.csv")]) == 0
    lines = (tmp_path / "b.csv").read_text().splitlines()
    assert lines[0].split(",") == cli.BENCH_COLUMNS and len(lines) == 3
