"""CPU-side checks of the C ABI: the library loads and exports every symbol
``include/vtrain_b200.h`` declares; ctypes signatures cover all of them; no
compute is called (there is no GPU here)."""

from __future__ import annotations

import re

import pytest

from conftest import REPO

HEADER = REPO / "include" / "vtrain_b200.h"


def declared() -> set[str]:
    text = HEADER.read_text()
    body = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(vt_[a-z0-9_]+)\s*\(", body))


def test_header_declares_the_path():
    names = declared()
    for must in ("vt_round_log", "vt_replay", "vt_pack5", "vt_unpack5", "vt_tau_kth_key",
                 "vt_sha256_leaves", "vt_merkle_level", "vt_merkle_build"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2403_09603_b200 import _lib
    lib = _lib.lib()
    for name in declared():
        assert hasattr(lib, name), name
    assert set(_lib.EXPORTS) == declared()
    assert lib.vt_version().startswith(b"vtrain_b200")
    assert _lib.tile_elems() % 640 == 0


def test_host_only_entry_points():
    from paper_2403_09603_b200 import _lib
    lib = _lib.lib()
    assert lib.vt_merkle_node_count(1) == 1
    assert lib.vt_merkle_node_count(3) == 3 + 2 + 1
    assert lib.vt_merkle_node_count(1_464_844) > 2 * 1_464_844 - 1
    assert lib.vt_round_log_workspace(1 << 30) >= 8 * ((1 << 30) // _lib.tile_elems())


def test_sm100a_cubin_only():
    import subprocess
    so = REPO / "paper_2403_09603_b200" / "libvtrain_b200.so"
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(so)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if "ELF file" in line)


def test_operator_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2403_09603_b200 import fpround
    with pytest.raises(RuntimeError, match="CUDA"):
        fpround.rnd_array([1.0], 32)


# Every compute entry point rejects malformed arguments before touching the
# device (VT_EINVAL = -1, vt_last_error names the entry point), so these
# run without a GPU.  None = NULL pointer.
BAD_CALLS = [
    ("vt_round_log", (None, -1, 32, 0.0, 1, None, None, 0, 0, None, None, None, None, 0, None, None, None, None, 0,
                      None)),
    ("vt_replay", (None, 10, 9, 0, None, 0, 0, 1, None, None, None, None, 0, None)),
    ("vt_grid_neighbors", (None, -1, 32, None, None, None, None)),
    ("vt_exponent_scale", (None, -1, None, None, None)),
    ("vt_is_on_grid", (None, 4, 33, None, None)),
    ("vt_norm_distance", (None, 4, 9, None, None, None)),
    ("vt_pack5", (None, -1, None, None, None)),
    ("vt_unpack5", (None, -1, 5, None, None, None)),
    ("vt_log_validate", (None, -1, None, None)),
    ("vt_log_histogram", (None, -1, None, None, None)),
    ("vt_tau_kth_key", (None, -1, 32, 0, None, None, None, 0, None)),
    ("vt_tau_budget_key", (None, 10, 32, -1, 0.1, 0.2, None, None, None, None, 0, None)),
    ("vt_tau_budget", (None, 10, 32, -1, 30, None, None, None, None, 0, None)),
    ("vt_tau_shard_plan", (0, 32, 10, None, None)),
    ("vt_round_log_exchange", (None, 10, 32, 0.0, 1, None, None, 0, 0, None, None, None, 0, None, 1, 0, None)),
    ("vt_round_log_exchange", (None, 10, 32, 0.0, 1, None, None, 0, 0, None, None, None, 0, None, 1, 1, None)),
    ("vt_counts_wait", (None, 1, 0, None, None, None)),
    ("vt_merkle_level_exchange", (None, 2, None, None, 1, 0, 0, 1, None)),
    ("vt_merkle_level_exchange", (1 << 40, 4, 1 << 40, 1 << 40, 2, 0, 1, 2, None)),  # roots past n_total
    ("vt_digests_publish", (None, 1, 1 << 40, 1, 0, 0, 1, None)),
    ("vt_digests_publish", (1 << 40, 1, 1 << 40, 2, 2, 0, 1, None)),  # rank >= world
    ("vt_digests_wait", (1 << 40, 2, 0, 3, None, 1 << 40, None)),  # no out buffer for 3 roots
    ("vt_tau_shard_search_x", (None, 10, 32, 10, 1, 30, 1 << 40, 1 << 40, 1, 0, 16, 1 << 40, 1 << 40, 1 << 40,
                               None, 0, 7, None)),  # no workspace
    ("vt_tau_shard_search_x", (None, 0, 32, 10, 1, 30, 1 << 40, 1 << 40, 1, 0, 16, 1 << 40, 1 << 40, 1 << 40,
                               1 << 40, 1 << 40, 8, None)),  # phases out of range
    ("vt_tau_shard_candidates", (None, 10, 32, 5, 1, None, None, None, 0, None)),
    ("vt_tau_shard_digit_keys", (10, 32, 10, 1, 5000, None, 0, None, None, 0, None)),
    ("vt_round_log_adaptive", (None, 0, 32, 10, 30, 1, None, None, 0, 0, None, None, None, None, None, None, 0,
                               None)),
    ("vt_round_log_adaptive_batch", (None, 0, 32, 30, 1, None, 0, None)),
    ("vt_straddle_min", (None, None, -1, 32, None, None, None, None, None)),
    ("vt_min_f64", (None, -1, None, None, None)),
    ("vt_sha256_leaves", (None, 0, 4096, None, None)),
    ("vt_merkle_level", (None, 0, None, None)),
    ("vt_merkle_build", (None, 0, 4096, None, 0, None)),
    ("vt_sha256_peak_bench", (None, 0, 1, None)),
    ("vt_int_mix_peak_bench", (None, 0, 1, 0, None)),
    ("vt_serialize_f32", (None, -1, None, 0, None, None)),
    ("vt_tau_kth_begin", (-1, None, None, 0, None)),
    ("vt_tau_kth_hist", (None, 10, 32, 7, None, None, 0, None)),
    ("vt_tau_kth_select", (9, None, None, 0, None)),
]


@pytest.mark.parametrize("name,args", BAD_CALLS, ids=[c[0] for c in BAD_CALLS])
def test_entry_points_reject_bad_arguments(name, args):
    from paper_2403_09603_b200 import _lib
    lib = _lib.lib()
    assert getattr(lib, name)(*args) == _lib.VT_EINVAL
    assert lib.vt_last_error().decode().startswith(name)


def test_every_compute_entry_point_is_covered():
    host_only = {"vt_version", "vt_last_error", "vt_tile_elems", "vt_merkle_node_count", "vt_tau_kth_hist_offset",
                 "vt_tau_kth_hist_bins", "vt_int_mix_ops_per_thread_rep", "vt_exchange_words",
                 "vt_digest_exchange_words", "vt_stream_synchronize",
                 "vt_tau_shard_exchange_words"}
    covered = {c[0] for c in BAD_CALLS}
    assert declared() - host_only - covered == {n for n in declared() if n.endswith("_workspace")}


def test_adaptive_batch_validates_segments_on_the_host():
    """Segments are checked before any launch: empty, misaligned, in-place."""
    import ctypes as C
    from paper_2403_09603_b200 import _lib
    lib = _lib.lib()
    ns = (C.c_int64 * 3)(1000, 1 << 20, 7)
    total = lib.vt_round_log_adaptive_batch_workspace(ns, 3)
    assert total >= sum(lib.vt_round_log_adaptive_workspace(n) - lib.vt_round_log_workspace(n) for n in ns) > 0
    fake = 1 << 40  # never dereferenced: validation fails first

    def seg(**kw):
        d = dict(x=fake, n=1000, budget=5, out=fake + (1 << 30), log=fake + (2 << 30), log_cap=6, global_base=0,
                 tau_out=fake + (3 << 30), flags=fake + (4 << 30))
        d.update(kw)
        return _lib.AdaptiveSegment(**d)

    for bad, what in [(seg(n=0), "bad segment"), (seg(x=fake + 8), "bad segment"),
                      (seg(out=fake + 64, n=1000), "in-place")]:
        arr = (_lib.AdaptiveSegment * 1)(bad)
        assert lib.vt_round_log_adaptive_batch(C.cast(arr, C.c_void_p), 1, 32, 30, 1, fake, 1 << 40, None) == \
            _lib.VT_EINVAL
        assert what in lib.vt_last_error().decode()


def test_out_buffer_validation_host_logic():
    """Caller buffers reach the C ABI as raw pointers; check_out rejects a wrong
    dtype, a short or strided buffer and the wrong device before any call."""
    import torch
    from paper_2403_09603_b200 import _device as D
    cpu = torch.device("cpu")
    D.check_out(None, 10, torch.float32, cpu)
    D.check_out(torch.empty(10), 10, torch.float32, cpu)
    D.check_out(torch.empty(12), 10, torch.float32, cpu)
    for t, dev in ((torch.empty(10, dtype=torch.float64), cpu), (torch.empty(9), cpu),
                   (torch.empty(20)[::2], cpu), (torch.empty(10), torch.device("meta")), ([0.0] * 10, cpu)):
        with pytest.raises(ValueError):
            D.check_out(t, 10, torch.float32, dev)


def test_default_log_capacity_bound():
    from paper_2403_09603_b200 import ops
    assert ops.default_log_capacity(0) == 1
    assert ops.default_log_capacity(1000) == 1000
    assert ops.default_log_capacity(1 << 20) == 1 << 17
    assert ops.default_log_capacity(1 << 30) == 1 << 27  # 1 GiB of words at 2^30, not 8 GiB


def test_int_mix_peak_kernel_is_the_sha_op_mix():
    """The Merkle roofline's denominator kernel: its loop body is the SHA-256
    op mix (6 SHF : 4 LOP3 : 4 three-input adds per unit, 8 units per
    iteration) with no memory instructions; the adds are IADD3 on the ALU
    pipe, or two IMADs each on the FMA pipe in the FMA_ADDS variant."""
    import subprocess
    from paper_2403_09603_b200 import _lib
    so = REPO / "paper_2403_09603_b200" / "libvtrain_b200.so"
    for fma, name in ((False, "_ZN2vt19int_mix_peak_kernelILb0EEEvPjijj"),
                      (True, "_ZN2vt19int_mix_peak_kernelILb1EEEvPjijj")):
        sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", "-fun", name, str(so)],
                              capture_output=True, text=True).stdout
        lines = [ln for ln in sass.splitlines() if re.search(r"/\*[0-9a-f]{4}\*/", ln)]
        start = next(i for i, ln in enumerate(lines) if " SHF." in ln)
        end = next(i for i, ln in enumerate(lines) if i > start and "BRA" in ln)
        body = lines[start:end]
        count = lambda op: sum(1 for ln in body if re.search(rf"\b{op}\b", ln))  # noqa: E731
        assert count("SHF.R.W.U32") == 48 and count("LOP3.LUT") == 32, name
        if fma:
            assert count("IADD3") == 0 and count("IMAD") >= 64, name
        else:
            assert count("IADD3") == 32, name
        assert not any(re.search(r"\b(LDG|STG|LDS|STS)\b", ln) for ln in body)
    assert _lib.lib().vt_int_mix_ops_per_thread_rep() == 8 * 14
