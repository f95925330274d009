"""compute-sanitizer over a tiny forward: every kernel of the
path (stem, tcgen05 convs and tconvs with their mbarrier / TMEM / TMA
pipelines, pools, head), once through the eager runner with trace buffers
and once through the CUDA-graph Engine, checked against the dense oracle.
memcheck: no out-of-bounds or misaligned global / shared access; racecheck:
no shared-memory hazard reported. (synccheck is not run: its mbarrier
"missing wait" heuristic flags every arrive-only role of a producer /
consumer pipeline -- here the epilogue warps that release accumulators they
never wait on -- which is the intended use of an mbarrier.) racecheck runs
with one-CTA tiles (MBU_PAIR=0); with CTA pairs its only reports are the
cta_group::2 TMEM allocation's own handshake (test below)."""

from __future__ import annotations

import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    return exe


def _run(tool, env=None, exit_code=True):
    import os
    cmd = [_sanitizer(), "--tool", tool, "--print-limit", "20"]
    if exit_code:
        cmd += ["--error-exitcode", "3"]
    cmd += [sys.executable, str(ROOT / "tools" / "tiny_forward.py"), "32", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT,
                       env={**os.environ, **(env or {})})
    out = r.stdout + r.stderr
    print(out[-4000:])
    if "closed on this pool" in out:
        # the GPU pool's compute-sanitizer wrapper refuses every run (it has
        # left GPUs needing a reset elsewhere); the clean runs of this test on
        # the round-2 build are in profiles/r2d_pytest_gpu.log (107 passed)
        pytest.skip("compute-sanitizer closed on this GPU pool: " + out.strip().splitlines()[-1][:200])
    return r, out


@pytest.mark.parametrize("tool,env", [("memcheck", {}), ("memcheck", {"MBU_PAIR": "0"}),
                                      ("racecheck", {"MBU_PAIR": "0"})])
def test_tiny_forward_is_sanitizer_clean(cuda, tool, env):
    r, out = _run(tool, env)
    assert r.returncode == 0, out[-4000:]
    assert "tiny forward ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out


def test_cta_pair_racecheck_hazards_are_the_pair_tmem_alloc(cuda):
    """With CTA pairs (cta_group::2) racecheck reports hazards between a write
    from outside the kernel's code and the SYNCS wait / arrive that ptxas emits
    for `tcgen05.alloc.cta_group::2` (its handshake with the peer CTA in the
    compiler-reserved static shared memory) -- and nowhere else: every
    reported access must sit on the alloc's source line."""
    import re
    src = (ROOT / "paper_2601_11660_b200" / "csrc" / "conv_tc.cu").read_text().splitlines()
    alloc = set()  # every source line of the alloc's asm statement (lineinfo may name any)
    for i, l in enumerate(src):
        if "tcgen05.alloc.cta_group::2" in l:
            j = i
            while ");" not in src[j]:
                j += 1
            alloc |= set(range(i + 1, j + 2))
    assert alloc
    r, out = _run("racecheck", exit_code=False)
    assert r.returncode == 0, out[-4000:]
    assert "tiny forward ok" in out
    lines = {int(m) for m in re.findall(r"Read access at .*? in conv_tc\.cu:(\d+)", out)}
    lines |= {int(m) for m in re.findall(r"Write access at .*? in conv_tc\.cu:(\d+)", out)}
    assert lines <= alloc, (sorted(lines), sorted(alloc))
    # every reported race names the pair kernel (no other kernel has a hazard)
    for m in re.findall(r"Race reported between .*? at (.*?)\+0x", out):
        assert "(bool)1, (bool)1, (bool)1>" in m, m
