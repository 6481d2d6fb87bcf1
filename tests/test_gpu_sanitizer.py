"""compute-sanitizer memcheck / racecheck / synccheck over every kernel
family: the tcgen05 GEMMs (mbarrier rings, CTA-pair
multicast commits), the cooperative prologues, the backward prologue's
arrival counters, the ESS / gather kernels, esfk and the SIMT path.

racecheck and tcgen05.alloc.cta_group::2: the pair allocation is one
collective of both CTAs' allocator warps and writes the TMEM base address
into the smem slot of each CTA; racecheck reports that as a cross-CTA
write/read hazard on the alloc instruction itself (both writes carry the
same value, and every read of the slot follows the cluster barrier).  The
racecheck test therefore runs twice: single-CTA tiles (HXM_CTA_PAIR=0) must
be hazard-free; with CTA pairs every reported hazard must sit on the
tcgen05.alloc line and nowhere else."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2411_01288_b200", "csrc")


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    return None


def _run(tool, env_extra=None):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cs = _sanitizer()
    if cs is None:
        pytest.skip("compute-sanitizer not installed")
    env = dict(os.environ, **(env_extra or {}))
    cmd = [cs, "--tool", tool, "--error-exitcode", "3", "--print-limit", "50",
           sys.executable, os.path.join(ROOT, "tests", "_sanitize_worker.py")]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=1500)
    out = r.stdout + r.stderr
    assert "sanitize worker: ok" in out, out[-6000:]
    return r.returncode, out


@pytest.mark.parametrize("tool", ["memcheck", "synccheck"])
def test_sanitizer_clean(tool):
    rc, out = _run(tool)
    assert rc == 0, out[-6000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]


def test_memcheck_chained_kernels_clean():
    """The opt-in chained fwd1 -> fwd2 / bwd_act -> gx kernels (umma_chain.cu)."""
    rc, out = _run("memcheck", {"HXM_CHAIN": "1", "HXM_CHAIN_BWD": "1"})
    assert rc == 0, out[-6000:]
    assert "ERROR SUMMARY: 0 errors" in out, out[-4000:]


def test_racecheck_single_cta_clean():
    rc, out = _run("racecheck", {"HXM_CTA_PAIR": "0"})
    assert rc == 0, out[-6000:]
    assert "RACECHECK SUMMARY: 0 hazards" in out, out[-4000:]


def _source_line(fname, line):
    """The statement around fname:line (an asm statement spans a few lines;
    -lineinfo attributes it to its last one)."""
    path = os.path.join(CSRC, os.path.basename(fname))
    with open(path) as f:
        lines = f.read().splitlines()
    return "\n".join(lines[max(0, line - 4):line])


def test_racecheck_cta_pairs_only_alloc():
    rc, out = _run("racecheck")
    sites = re.findall(r"access at .*? in ([\w./-]+\.cuh?):(\d+)", out)
    bad = [(f, l, _source_line(f, int(l))) for f, l in sites
           if "tcgen05.alloc" not in _source_line(f, int(l))]
    assert not bad, (bad[:10], out[-4000:])
    if rc != 0:  # every hazard is the pair allocation's result slot
        assert sites, out[-4000:]
