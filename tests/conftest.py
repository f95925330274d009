"""Shared fixtures. GPU tests carry @pytest.mark.gpu and run on the B200 box."""

from __future__ import annotations

import json
import sys
from dataclasses import replace
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")


@pytest.fixture
def rng() -> np.random.Generator:
    return np.random.default_rng(0xBADC0DE)


def tiny_config(divisor: int = 4, extent: int = 64, **overrides):
    """Default architecture shrunk to test scale (reference conftest.py:23-26)."""
    import paper_2601_11660_b200 as mb

    cfg = replace(mb.scale_config(mb.UNetConfig(), divisor), height=extent, width=extent)
    return replace(cfg, **overrides) if overrides else cfg


def load_golden(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def golden_cases():
    z = load_golden("layers.npz")
    return z, json.loads(bytes(z["cases_json"]).decode())


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test ran without a CUDA device")
    return torch.device("cuda", 0)


@pytest.fixture(params=["fp4", "i8"])
def conv_engine(request):
    """Run the test once per tcgen05 operand kind of the 3x3 convs: kind::mxf4
    (e2m1, default) and kind::i8 (MBU_OPT_CONV_I8)."""
    from paper_2601_11660_b200 import _lib

    _lib.call("mbu_set_option", 3, 1 if request.param == "i8" else 0)
    try:
        yield request.param
    finally:
        _lib.call("mbu_set_option", 3, 0)
