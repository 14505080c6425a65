"""GPU parity: .vtrl codec, writer/reader and the drop-in channels."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def rl():
    from paper_2403_09603_b200 import roundlog
    return roundlog


def test_pack5_known_answers(rl):
    assert rl.pack5([0, 0, 0, 0, 0]) == 0
    assert rl.pack5([1, 1, 1, 1, 1]) == 121
    assert rl.pack5([2, 0, 0, 0, 1]) == 83
    assert rl.pack5([2, 2, 2, 2, 2]) == 242
    assert rl.unpack5(121) == [1, 1, 1, 1, 1]
    with pytest.raises(rl.LogFormatError, match="corrupt log byte"):
        rl.unpack5(243)


def test_writer_files_match_reference(golden, rl, tmp_path):
    for i, case in enumerate(golden.roundlog["cases"]):
        digits = golden.roundlog_digits[f"d{i}"]
        path = tmp_path / f"c{i}.vtrl"
        with rl.LogWriter(path, case["b_r"], compress=case["compress"]) as w:
            prev = 0
            for c in case["cuts"] + [case["n"]]:
                w.write_array(digits[prev:c])
                prev = c
        raw = path.read_bytes()
        assert hashlib.sha256(raw).hexdigest() == case["file_sha"], case["n"]
        r = rl.LogReader(path)
        assert r.entry_count == case["n"]
        assert r.histogram() == {int(k): v for k, v in case["histogram"].items()}
        assert np.array_equal(r.read_array(case["n"]), digits)
        assert r.remaining == 0


def test_scalar_writes_and_reads(rl, tmp_path):
    path = tmp_path / "b.vtrl"
    with rl.LogWriter(path, 32) as w:
        for d in (0, 0, 0, 0, 0, 2):
            w.write(d)
    assert list(path.read_bytes()[rl.HEADER_LEN:]) == [0, 122]
    r = rl.LogReader(path)
    assert [r.read() for _ in range(6)] == [0, 0, 0, 0, 0, 2]
    with pytest.raises(rl.LogExhaustedError, match="log exhausted"):
        r.read()


def test_reader_rejects_bad_files(rl, tmp_path):
    p = tmp_path / "e.bin"
    p.write_bytes(b"NOPE" + bytes(20))
    with pytest.raises(rl.LogFormatError, match="not a rounding log"):
        rl.LogReader(p)
    p = tmp_path / "c.vtrl"
    with rl.LogWriter(p, 32) as w:
        w.write_array(np.zeros(10, dtype=np.uint8))
    raw = bytearray(p.read_bytes())
    raw[rl.HEADER_LEN] = 250
    p.write_bytes(bytes(raw))
    with pytest.raises(rl.LogFormatError, match="corrupt log byte"):
        rl.LogReader(p)
    raw[rl.HEADER_LEN] = 0
    raw[4] = 9
    p.write_bytes(bytes(raw))
    with pytest.raises(rl.LogFormatError, match="version"):
        rl.LogReader(p)
    p2 = tmp_path / "t.vtrl"
    with rl.LogWriter(p2, 32) as w:
        w.write_array(np.ones(100, dtype=np.uint8))
    p2.write_bytes(p2.read_bytes()[:-3])
    with pytest.raises(rl.LogFormatError, match="truncated"):
        rl.LogReader(p2)
    with pytest.raises(ValueError):
        with rl.LogWriter(tmp_path / "x.vtrl", 32) as w:
            w.write_array(np.array([0, 3], dtype=np.uint8))


def test_empty_log(rl, tmp_path):
    p = tmp_path / "z.vtrl"
    rl.LogWriter(p, 26).close()
    assert rl.LogReader(p).entry_count == 0
    assert p.stat().st_size == rl.HEADER_LEN


@pytest.mark.parametrize("compress", [False, True])
def test_write_values_fused_matches_reference_stream(oracle, rl, tmp_path, compress):
    """Fused round+direction+pack over ragged tensors == reference LogWriter bytes."""
    rng = np.random.default_rng(11)
    tau = 0.25 * 2.0 ** -23
    sizes = [1, 3, 7, 5120, 5121, 4, 640 * 3 + 2, 99_999, 2, 0, 13, 70_001]
    tensors = [rng.normal(size=s) * np.exp2(rng.integers(-20, 20, size=s)) for s in sizes]
    path = tmp_path / "f.vtrl"
    directed_total = 0
    with rl.LogWriter(path, 32, compress=compress) as w:
        for x in tensors:
            y, directed = w.write_values(x, tau)
            assert np.array_equal(bits(y.cpu().numpy()), bits(oracle.rnd_array(x, 32) if x.size else x))
            directed_total += directed
    codes = [oracle.direction_array(x, 32, tau) if x.size else np.zeros(0, np.uint8) for x in tensors]
    want = oracle.vtrl_bytes(codes, 32, compress)
    assert path.read_bytes() == want
    assert directed_total == sum(int(np.count_nonzero(c != 1)) for c in codes)


def test_channels_end_to_end(oracle, tmp_path):
    """Trainer then auditor through the plug-in channels, reference semantics."""
    from paper_2403_09603_b200 import protocol, roundlog
    rng = np.random.default_rng(12)
    tau = 2.0 ** -25
    shapes = [(8, 12), (8, 12), (8, 2), (8, 2), (8, 12), (8, 8), (1,), (3, 5, 7)]
    xs = [rng.normal(size=s) for s in shapes]
    xas = [x + rng.uniform(-1, 1, size=x.shape) * np.abs(x) * 2.0 ** -40 for x in xs]
    path = tmp_path / "run.vtrl"
    w = roundlog.LogWriter(path, 32)
    tr = protocol.GpuTrainerChannel(w, 32)
    outs = []
    for x in xs:
        y, directed, corr = tr.process(x, tau)
        assert y.shape == x.shape and y.dtype == np.float64 and corr == 0
        assert np.array_equal(bits(y), bits(oracle.rnd_array(x, 32)))
        assert directed == int(np.count_nonzero(oracle.direction_array(x, 32, tau) != 1))
        outs.append(y)
    w.close()
    assert path.read_bytes() == oracle.vtrl_bytes([oracle.direction_array(x, 32, tau) for x in xs], 32)
    r = roundlog.LogReader(path)
    au = protocol.GpuAuditorChannel(r, 32)
    for x, xa, yt in zip(xs, xas, outs):
        ya, directed, corr = au.process(xa, tau)
        want = oracle.rev_array(xa, 32, oracle.direction_array(x, 32, tau))
        assert np.array_equal(bits(ya), bits(want))
        assert corr == int(np.count_nonzero(want != oracle.rnd_array(xa, 32)))
    assert r.remaining == 0
    with pytest.raises(roundlog.LogExhaustedError):
        au.process(xs[0], tau)
    pl = protocol.GpuPlainChannel(32)
    y, _, _ = pl.process(xs[2], tau)
    assert np.array_equal(bits(y), bits(oracle.rnd_array(xs[2], 32)))


def test_unpack_and_histogram_device(rl, oracle):
    import torch
    rng = np.random.default_rng(13)
    digits = rng.integers(0, 3, size=5 * 40_001).astype(np.uint8)
    packed = rl.pack_device(torch.from_numpy(digits).cuda())
    assert packed.cpu().numpy().tobytes() == oracle.pack_groups(digits)
    for pos, n in [(0, 17), (3, 1000), (7, 5 * 40_000 - 7)]:
        assert np.array_equal(rl.unpack_device(packed, pos, n).cpu().numpy(), digits[pos:pos + n])


def _packed_payload(codes_all):
    """Reference .vtrl payload bytes for a code stream (roundlog.py:67-70, pad with 1)."""
    c = np.asarray(codes_all, dtype=np.uint8)
    pad = (-c.size) % 5
    g = np.concatenate([c, np.ones(pad, np.uint8)]).reshape(-1, 5).astype(np.uint16)
    return (g * np.array([1, 3, 9, 27, 81], np.uint16)).sum(1).astype(np.uint8)


@pytest.mark.parametrize("b_r,out64", [(32, False), (32, True), (26, True)])
def test_fused_packed_replay_matches_oracle_and_tile_path(oracle, b_r, out64):
    """vt_replay with the .vtrl payload through the persistent TMA replay
    (rp_fused_kernel<PACKED>, a workspace given) == the per-tile
    replay_kernel<PACKED> (no workspace) == oracle rev_array, over ragged
    sizes and every stream phase; a corrupt byte and a short payload raise
    the error bit."""
    import torch
    from paper_2403_09603_b200 import _device as D
    from paper_2403_09603_b200 import _lib, workloads
    rng = np.random.default_rng(17)
    for n in (1, 4, 5, 2047, 2048, 2049, 8192 * 3 + 7, (1 << 18) + 3, (1 << 20) + 13):
        for pos in (0, 1, 3, 4, 12_345_679):
            x = workloads.config0_x(n, n % 97) * (1.0 if b_r == 32 else 3.0)
            codes = rng.integers(0, 3, size=n).astype(np.uint8)
            stream_pos = pos  # the tensor's first entry in the .vtrl stream
            lead = stream_pos % 5  # earlier entries sharing its first byte (code 1 here)
            payload = np.concatenate([np.zeros(stream_pos // 5, np.uint8),
                                      _packed_payload(np.concatenate([np.ones(lead, np.uint8), codes]))])
            want = oracle.rev_array(x, b_r, codes)
            want = want if out64 else want.astype(np.float32)
            corr_want = int(np.count_nonzero(oracle.rev_array(x, b_r, codes) != oracle.rnd_array(x, b_r)))
            xd = torch.from_numpy(x).cuda()
            pd = torch.from_numpy(payload).cuda()
            res = []
            for use_ws in (True, False):
                y = torch.empty(n, dtype=torch.float64 if out64 else torch.float32, device="cuda")
                f = D.Flags()
                ws = D.workspace(int(_lib.lib().vt_replay_workspace(n)), "t_packed") if use_ws else None
                _lib.call("vt_replay", D.ptr(xd), n, b_r, _lib.LOG_PACKED, D.ptr(pd), payload.size, stream_pos,
                          _lib.OUT_F64 if out64 else _lib.OUT_F32, D.ptr(y), f.cnt_ptr, f.err_ptr,
                          D.ptr(ws) if use_ws else None, ws.numel() if use_ws else 0, D.stream_ptr())
                err, cnt = f.read()
                assert err == 0, (n, pos, use_ws, err)
                assert cnt[0] == corr_want, (n, pos, use_ws)
                res.append(bits(y.cpu().numpy()))
            assert np.array_equal(res[0], bits(want)), (n, pos)
            assert np.array_equal(res[1], res[0])
    # a corrupt byte inside the tensor's range, and a payload cut short
    n = 300_001  # above the fused path's size threshold
    x = torch.from_numpy(workloads.config0_x(n, 5)).cuda()
    payload = _packed_payload(np.ones(n, np.uint8))
    for bad, length in ((payload.copy(), payload.size), (payload, payload.size - 3)):
        if length == payload.size:
            bad[54_321] = 250
        pd = torch.from_numpy(bad).cuda()
        y = torch.empty(n, dtype=torch.float32, device="cuda")
        f = D.Flags()
        ws = D.workspace(int(_lib.lib().vt_replay_workspace(n)), "t_packed")
        _lib.call("vt_replay", D.ptr(x), n, 32, _lib.LOG_PACKED, D.ptr(pd), length, 0, _lib.OUT_F32, D.ptr(y),
                  f.cnt_ptr, f.err_ptr, D.ptr(ws), ws.numel(), D.stream_ptr())
        assert f.read()[0] & _lib.ERR_BAD_LOG_BYTE
