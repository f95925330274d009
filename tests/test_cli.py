"""Front end (paper_2601_11660_b200.cli): flags and exit codes of the
reference CLI (pkg/src/bitunet/cli.py:3-13); the GPU infer run is checked
against the reference ``bitunet infer`` outputs (mask byte for byte)."""

from __future__ import annotations

import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from paper_2601_11660_b200 import read_tensor
from paper_2601_11660_b200.cli import main


def test_usage_errors_exit_2(capsys):
    assert main([]) == 2
    assert main(["infer", "--model", "x"]) == 2
    assert main(["bench", "--extent", "3x4x5"]) == 2
    assert main(["--version"]) == 0


def test_missing_or_bad_files_exit_3(tmp_path):
    assert main(["infer", "--model", str(tmp_path / "none.mbun"), "--image", "x.ppm"]) == 3
    bad = tmp_path / "bad.mbun"
    bad.write_bytes(b"NOPE" + bytes(60))
    assert main(["infer", "--model", str(bad), "--image", "x.ppm"]) == 3
    img = tmp_path / "x.ppm"
    img.write_bytes(b"P3 1 1 255\n")
    assert main(["infer", "--model", str(GOLDEN / "tiny_masked.mbun"), "--image", str(img)]) == 3


def test_shape_mismatch_exit_5():
    # img_rgb8.ppm is 24x40, tiny_masked.mbun wants 32x32
    assert main(["infer", "--model", str(GOLDEN / "tiny_masked.mbun"),
                 "--image", str(GOLDEN / "img_rgb8.ppm")]) == 5


@pytest.mark.gpu
def test_infer_matches_reference_cli(tmp_path):
    out = subprocess.run(
        [sys.executable, "-m", "paper_2601_11660_b200", "infer", "--model", str(GOLDEN / "tiny_masked.mbun"),
         "--image", str(GOLDEN / "img_32.ppm"), "--mask-out", str(tmp_path / "m.pgm"),
         "--logits-out", str(tmp_path / "l.rten"), "--device", "cuda:0"],
        cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    assert (tmp_path / "m.pgm").read_bytes() == (GOLDEN / "cli_mask.pgm").read_bytes()
    # logits: same file layout, values within the reference's float tolerance (verify.py:23)
    got, ref = read_tensor(tmp_path / "l.rten"), read_tensor(GOLDEN / "cli_logits.rten")
    assert got.dtype == ref.dtype and got.shape == ref.shape
    assert np.allclose(got, ref, rtol=1e-9, atol=1e-9)
    assert (tmp_path / "l.rten").stat().st_size == (GOLDEN / "cli_logits.rten").stat().st_size


@pytest.mark.gpu
def test_bench_runs(capsys):
    assert main(["bench", "--extent", "64x128", "--batch", "2", "--reps", "2", "--csv"]) == 0
    lines = capsys.readouterr().out.strip().splitlines()
    assert lines[0].startswith("extent,batch") and lines[1].startswith("64x128,2,")
