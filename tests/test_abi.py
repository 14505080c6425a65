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
