"""INTEGRATION.md §2's ctypes stub -- the binding a vtrain maintainer would
add -- executed as written (only the library path is filled in): the
documented signature and flag layout must produce the reference's
rnd_array bit for bit."""

from __future__ import annotations

import re

import numpy as np
import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _stub() -> str:
    text = (REPO / "INTEGRATION.md").read_text()
    m = re.search(r"```python\n(import ctypes as C\n.*?)```", text, re.S)
    assert m, "the ctypes stub block is missing from INTEGRATION.md"
    lib = REPO / "paper_2403_09603_b200" / "libvtrain_b200.so"
    return m.group(1).replace('C.CDLL("libvtrain_b200.so")', f'C.CDLL("{lib}")')


def test_documented_ctypes_stub_matches_the_reference(oracle):
    ns = {"np": np}
    exec(compile(_stub(), "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(3)
    for b_r in (32, 26, 10):
        x = rng.normal(0.0, 1.0, 10_007) * np.exp2(rng.integers(-30, 30, 10_007))
        got = ns["rnd_array"](x, b_r)
        assert np.array_equal(got.view(np.uint64), oracle.rnd_array(x, b_r).view(np.uint64))
    with pytest.raises(ValueError, match="non-finite value"):
        ns["rnd_array"](np.array([1.0, np.inf]), 32)
    with pytest.raises(ValueError, match="out of representable range"):
        ns["rnd_array"](np.array([1e300]), 10)
