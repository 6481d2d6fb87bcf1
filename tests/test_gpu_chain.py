"""Chained layer GEMMs (umma_chain.cu): the forward fwd1 -> fwd2 chain and
the backward bwd_act -> gx chain compute every output with the same MMA
order and the same epilogue arithmetic as the two-kernel path, so y, the
F'(y1) / F(y1) stash and all gradients must be BIT-identical with the chains
on and off (ragged segments, relu / identity, no b2, top-1 included).  The
switches are read once per process, hence one worker process per setting."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _run(tmp_path, tag, env):
    path = str(tmp_path / f"{tag}.pt")
    e = dict(os.environ)
    e.update(env)
    subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_chain_worker.py"), path],
                   check=True, env=e, timeout=600)
    return torch.load(path)


@pytest.mark.parametrize("fpt", ["0", "1"])
def test_chain_bit_identical(tmp_path, fpt):
    off = _run(tmp_path, "off", {"HXM_CHAIN": "0", "HXM_CHAIN_BWD": "0"})
    on = _run(tmp_path, "on", {"HXM_CHAIN": "1", "HXM_CHAIN_BWD": "1", "HXM_CHAIN_FPT": fpt})
    assert off.keys() == on.keys()
    bad = [k for k in off if not torch.equal(off[k], on[k])]
    assert not bad, f"chained outputs differ: {bad}"
