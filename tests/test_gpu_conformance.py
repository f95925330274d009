"""The reference's own test suite, run through the plug point on the B200.

``baseline/_ref`` holds the unmodified reference package and its tests
(``tools/install_reference.sh``; git-ignored, shipped to the GPU box with the
snapshot). Each case runs a pytest subprocess over those tests with
``tests/conformance/mbu_conformance.py`` loaded, which rebinds ``bitunet``'s
compute functions (``conv_forward`` ... ``graph.forward``) to this engine
(``paper_2601_11660_b200/plug.py``). The reference's verifier and dense
oracle stay the reference's, so e.g. ``test_engine_matches_dense_replay``
(test_graph.py:204-217) and acceptance criteria 1-5 (test_acceptance.py:91-293)
now certify the GPU results.

Deselected: criterion 9 (the reference's own CPU throughput floor,
test_acceptance.py:400-409 — it fails on the reference too) and the
JIT-vs-numpy fallback checks of the reference's private kernels, which
exercise reference internals rather than the rebound API.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"
SUITE = REF / "bitunet_tests"

pytestmark = pytest.mark.gpu

FILES = ["test_acceptance.py", "test_graph.py", "test_layers.py", "test_bitcore.py",
         "test_kernels.py", "test_oracle.py", "test_verify_bench.py"]
DESELECT = "not criterion_09"


def _run(level: str, files, timeout=1800):
    if not (REF / "bitunet").is_dir() or not SUITE.is_dir():
        pytest.fail("reference not installed in baseline/_ref (run tools/install_reference.sh)")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests" / "conformance")])
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env.setdefault("NUMBA_CACHE_DIR", "/tmp/mbu_numba_cache")
    env["MBU_PLUG"] = level
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "mbu_conformance", "-p", "no:cacheprovider",
           "-k", DESELECT, *files]
    r = subprocess.run(cmd, cwd=SUITE, env=env, capture_output=True, text=True, timeout=timeout)
    tail = (r.stdout + r.stderr)[-6000:]
    print(tail)
    assert r.returncode == 0, tail
    assert "rebound to the GPU engine" in r.stdout + r.stderr
    return tail


@pytest.mark.parametrize("level", ["layers", "forward"])
def test_reference_suite_through_plug(cuda, level):
    _run(level, FILES)
