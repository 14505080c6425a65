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


@pytest.mark.parametrize("b_r", [32, 26, 10])
def test_staged_channels_shapes_and_grids(oracle, b_r, tmp_path):
    """The host-array paths of the GPU channels (zero-copy for small arrays,
    one H2D + one D2H for large ones) over odd shapes -- 0-d, empty, non-contiguous, 3-D, sizes around the
    5-code packing phase -- at several grids: outputs and counts equal the
    oracle's channel arithmetic (protocol.py:198-216), the .vtrl file the
    reference writer's bytes, and a corrupt payload byte raises."""
    from paper_2403_09603_b200 import protocol, roundlog
    rng = np.random.default_rng(b_r)
    base = rng.normal(0, 3, size=(40, 30))
    tensors = [np.float64(1.0 + 0.6 * 2.0 ** -23), np.zeros(0), base[:, ::3], rng.normal(0, 1e-3, (2, 3, 7)),
               rng.normal(0, 1, 4), rng.normal(0, 1, 5), rng.normal(0, 1, 6), rng.normal(0, 50, 10_007),
               rng.normal(0, 2, 300_001)]  # the last above HostStage.ZERO_COPY_MAX: the staged-copy path
    tau = 2.0 ** -25
    path = tmp_path / "s.vtrl"
    w = roundlog.LogWriter(path, b_r)
    tc = protocol.GpuTrainerChannel(w, b_r)
    all_codes = []
    for t in tensors:
        y, directed, corr = tc.process(t, tau)
        codes = oracle.direction_array(t, b_r, tau)
        all_codes.append(np.asarray(codes).reshape(-1))
        want = oracle.rnd_array(t, b_r)
        assert y.shape == np.shape(want) and np.array_equal(bits(y), bits(want))
        assert directed == int(np.count_nonzero(codes != 1)) and corr == 0
    w.close()
    assert path.read_bytes() == oracle.vtrl_bytes(all_codes, b_r)
    ac = protocol.GpuAuditorChannel(roundlog.LogReader(path), b_r)
    for t, codes in zip(tensors, all_codes):
        noisy = np.nextafter(t, np.where(rng.random(np.shape(t)) < 0.5, np.inf, -np.inf))
        y, directed, corr = ac.process(noisy, tau)
        want = oracle.rev_array(noisy, b_r, codes.reshape(np.shape(noisy)) if np.shape(noisy) else codes)
        assert np.array_equal(bits(y), bits(want))
        assert corr == int(np.count_nonzero(want != oracle.rnd_array(noisy, b_r)))
    assert ac.reader.remaining == 0
    raw = bytearray(path.read_bytes())
    raw[roundlog.HEADER_LEN + 3] = 251
    path.write_bytes(bytes(raw))
    with pytest.raises(roundlog.LogFormatError, match="corrupt log byte"):
        roundlog.LogReader(path)
