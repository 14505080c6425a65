"""Drop-in end to end: the exact channel-call sequences of real
reference train + audit runs (tiny, logreg, and the prefix of trend that holds
all 77 of its auditor corrections; recorded in the build container by
tests/golden/make_golden.py) replayed through the GPU channels.
Outputs, directed / correction counts and the .vtrl file must match the
reference bit for bit."""

from __future__ import annotations

import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN, bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def traces():
    return dict(np.load(GOLDEN / "channel_traces.npz")), json.loads((GOLDEN / "channel_traces.json").read_text())


def _split(flat, shapes):
    out, off = [], 0
    for s in shapes:
        k = int(np.prod(s))
        out.append(flat[off:off + k].reshape(s))
        off += k
    assert off == flat.size
    return out


@pytest.mark.parametrize("name", ["tiny", "logreg", "trend"])
def test_reference_run_through_gpu_channels(traces, name, tmp_path):
    from paper_2403_09603_b200 import protocol, roundlog
    arr, meta = traces
    m = meta[name]
    shapes = m["shapes"]
    t_in = _split(arr[f"{name}_t_in"], shapes)
    t_out = _split(arr[f"{name}_t_out"], shapes)
    a_in = _split(arr[f"{name}_a_in"], shapes)
    a_out = _split(arr[f"{name}_a_out"], shapes)
    path = tmp_path / f"{name}.vtrl"
    w = roundlog.LogWriter(path, m["b_r"])
    ch = protocol.GpuTrainerChannel(w, m["b_r"])
    for i, (x, tau) in enumerate(zip(t_in, m["taus"])):
        y, directed, corr = ch.process(x, tau)
        assert y.shape == x.shape and y.dtype == np.float64
        assert np.array_equal(bits(y.astype(np.float32)), bits(t_out[i])), i
        assert np.array_equal(bits(y), bits(t_out[i].astype(np.float64))), i
        assert directed == m["directed"][i] and corr == 0
    w.close()
    assert hashlib.sha256(path.read_bytes()).hexdigest() == m["vtrl_sha"]
    r = roundlog.LogReader(path)
    au = protocol.GpuAuditorChannel(r, m["b_r"])
    for i, (x, tau) in enumerate(zip(a_in, m["taus"])):
        y, directed, corr = au.process(x, tau)
        assert np.array_equal(bits(y.astype(np.float32)), bits(a_out[i])), i
        assert corr == m["corrections"][i] and directed == 0
    assert r.remaining == 0
