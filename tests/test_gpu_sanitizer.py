"""compute-sanitizer over a tiny forward: every kernel of the
path (stem, tcgen05 convs and tconvs with their mbarrier / TMEM / TMA
pipelines, pools, head), once through the eager runner with trace buffers
and once through the CUDA-graph Engine, checked against the dense oracle.
memcheck: no out-of-bounds or misaligned global / shared access; racecheck:
no shared-memory hazard reported. (synccheck is not run: its mbarrier
"missing wait" heuristic flags every arrive-only role of a producer /
consumer pipeline -- here the epilogue warps that release accumulators they
never wait on -- which is the intended use of an mbarrier.)"""

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


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_tiny_forward_is_sanitizer_clean(cuda, tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "3", "--print-limit", "20",
           sys.executable, str(ROOT / "tools" / "tiny_forward.py"), "32", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    out = r.stdout + r.stderr
    print(out[-4000:])
    assert r.returncode == 0, out[-4000:]
    assert "tiny forward ok" in out
    assert "ERROR SUMMARY: 0 errors" in out or "RACECHECK SUMMARY: 0 hazards" in out
