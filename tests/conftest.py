"""Shared fixtures: golden fixtures, oracle import, GPU marker."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parent.parent
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))
sys.path.insert(0, str(REPO / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    class G:
        fpround = dict(np.load(GOLDEN / "fpround_golden.npz"))
        errors = json.loads((GOLDEN / "fpround_errors.json").read_text())
        roundlog = json.loads((GOLDEN / "roundlog_golden.json").read_text())
        roundlog_digits = dict(np.load(GOLDEN / "roundlog_digits.npz"))
        tau = json.loads((GOLDEN / "tau_golden.json").read_text())
        merkle = json.loads((GOLDEN / "merkle_golden.json").read_text())
        configs = json.loads((GOLDEN / "config_golden.json").read_text())
    return G


@pytest.fixture(scope="session")
def oracle():
    import vt_oracle
    return vt_oracle


def bits(a) -> np.ndarray:
    """Bit pattern view: parity is on bits, so -0.0 != 0.0."""
    a = np.ascontiguousarray(a)
    if a.dtype == np.float64:
        return a.view(np.uint64)
    if a.dtype == np.float32:
        return a.view(np.uint32)
    return a
