"""The C ABI from plain C (examples/abi_roundtrip.c): the library links and
runs without Python or torch -- the boundary a non-Python caller binds."""

from __future__ import annotations

import subprocess

import pytest

from conftest import REPO

SRC = REPO / "examples" / "abi_roundtrip.c"


def _build(out) -> None:
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", str(REPO / "include"), "-I", "/usr/local/cuda/include",
           str(SRC), "-L", str(REPO / "paper_2403_09603_b200"), "-lvtrain_b200", "-L", "/usr/local/cuda/lib64",
           "-lcudart", "-lm", f"-Wl,-rpath,{REPO / 'paper_2403_09603_b200'}", "-o", str(out)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)


def test_c_example_compiles_and_links(tmp_path):
    _build(tmp_path / "abi_roundtrip")
    deps = subprocess.run(["ldd", str(REPO / "paper_2403_09603_b200" / "libvtrain_b200.so")], capture_output=True,
                          text=True).stdout
    assert "torch" not in deps and "python" not in deps  # the product library is plain CUDA C++


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 4099, (1 << 22) + 12345])
def test_c_example_runs(tmp_path, n, oracle):
    exe = tmp_path / "abi_roundtrip"
    _build(exe)
    ybin = tmp_path / "y.bin"
    r = subprocess.run([str(exe), str(n), str(ybin)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bad_y=0 bad_auditor=0 bad_log=0" in r.stdout and "replay_err=0" in r.stdout
    # the Merkle root the C caller got from vt_merkle_build == the oracle's
    # (hashlib SHA-256 of 4 KiB chunks, merkle.build's promotion rule)
    data = ybin.read_bytes()
    assert len(data) == 4 * n
    want = oracle.merkle_levels(oracle.chunk_leaves(data, 4096))[-1][0]
    assert f"root={want.hex()}" in r.stdout, r.stdout
