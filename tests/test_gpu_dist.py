"""TP choreography with the CUDA layer and NCCL (torchrun, one process per
visible GPU; the pool gives one GPU per call, where the collectives are
identities but every view / permute / stream of the NCCL path runs)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
def test_tp_nccl_matches_single_gpu():
    n = min(torch.cuda.device_count(), 8)
    cmd = [sys.executable, "-m", "torch.distributed.run", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(HERE, "_gpu_dist_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("OK") == n, r.stdout


@pytest.mark.skipif(not torch.cuda.is_available(), reason="no CUDA device")
@pytest.mark.parametrize("mode", ["data_centric", "model_centric"])
def test_bench_tp_modes_run(mode):
    """bench.py's N>1 code paths, exercised at world size 1 under torchrun."""
    root = os.path.dirname(HERE)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nproc-per-node=1",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", os.path.join(root, "bench.py"),
           "--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--mode", mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    import json
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1]
    d = json.loads(line)
    assert d["value"] > 0 and d["config"]["parallelism"].startswith(mode)
