"""Shared test configuration: the `gpu` marker, golden-fixture loaders and
the max-norm relative error the reference uses as its parity metric
(prefixdec cli.py:125-128, tests/conftest.py:15-18)."""
from __future__ import annotations

import json
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")


def rel_err(out, ref) -> float:
    ref = np.asarray(ref, dtype=np.float64)
    scale = max(float(np.max(np.abs(ref))), 1e-300)
    return float(np.max(np.abs(np.asarray(out, dtype=np.float64) - ref)) / scale)


@lru_cache(maxsize=None)
def golden_json(name):
    return json.loads((GOLDEN / name).read_text(encoding="utf-8"))


@lru_cache(maxsize=None)
def golden_npz():
    return dict(np.load(GOLDEN / "forests.npz"))


def golden_table_text(name="a100_d128.csv"):
    return (GOLDEN / name).read_text(encoding="utf-8")


@pytest.fixture(scope="session")
def cuda_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return True
