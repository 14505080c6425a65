"""Multi-GPU host logic on CPU: world-size-2 gloo processes.

The per-shard device work is stood in for by the oracle (test
infrastructure); what is tested is the sharding plan, the count all-gather
/ offset arithmetic and the Merkle block-root exchange of
paper_2403_09603_b200/dist.py -- the parts that differ between 1 and N GPUs.
"""

from __future__ import annotations

import hashlib
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = Path(__file__).resolve().parent.parent


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _sha_leaves(b: torch.Tensor, leaf_bytes: int) -> torch.Tensor:
    raw = b.numpy().tobytes()
    d = [hashlib.sha256(raw[i:i + leaf_bytes]).digest() for i in range(0, len(raw), leaf_bytes)]
    return torch.frombuffer(bytearray(b"".join(d)), dtype=torch.uint8).reshape(-1, 32)


def _sha_level(cur: torch.Tensor) -> torch.Tensor:
    rows = [bytes(r) for r in cur.numpy()]
    out = [hashlib.sha256(rows[i] + rows[i + 1]).digest() for i in range(0, len(rows) - 1, 2)]
    if len(rows) % 2:
        out.append(rows[-1])
    return torch.frombuffer(bytearray(b"".join(out)), dtype=torch.uint8).reshape(-1, 32)


def _worker(rank: int, world: int, port: int, q) -> None:
    sys.path.insert(0, str(REPO))
    sys.path.insert(0, str(REPO / "oracle"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import vt_oracle as O
        from paper_2403_09603_b200 import dist as vd
        from paper_2403_09603_b200 import workloads

        # --- round-and-log: shards with global indices + count all-gather
        n = 100_003
        x = workloads.config0_x(n, 3)
        lo, hi = vd.shard_range(n, rank, world)
        tau = workloads.TAU_CONFIG0
        words = O.sparse_from_codes(O.direction_array(x[lo:hi], 32, tau), base=lo)
        counts = vd.all_gather_counts(int(words.size))
        offs = vd.exclusive_offsets(counts)
        gathered = [None] * world
        dist.all_gather_object(gathered, (int(offs[rank]), words.tolist()))
        full = O.sparse_from_codes(O.direction_array(x, 32, tau))
        placed = np.zeros(int(counts.sum()), dtype=np.uint64)
        for off, w in gathered:
            placed[off:off + len(w)] = np.array(w, dtype=np.uint64)
        ok_log = bool(np.array_equal(placed, full)) and int(counts.sum()) == full.size

        # --- Merkle: whole 2^k-leaf blocks per rank, all-gathered block roots;
        # the assembled level list equals merkle.build's, level for level
        ok_tree = True
        for n_floats, k in ((123_457, 3), (100 * 1024, 12), (1024, 3), (9 * 1024 + 5, 3), (17 * 1024, 2)):
            w32 = np.random.default_rng(9).normal(0, 0.02, size=n_floats).astype(np.float32)
            data = w32.tobytes()
            leaf_bytes = 4096
            nl = (len(data) + leaf_bytes - 1) // leaf_bytes
            l0, l1 = vd.leaf_block_range(nl, rank, world, k)
            raw = data[l0 * leaf_bytes: min(len(data), l1 * leaf_bytes)]
            mine = torch.frombuffer(bytearray(raw), dtype=torch.uint8) if raw else torch.zeros(0, dtype=torch.uint8)
            lv, top = vd.merkle_sharded(mine, nl, leaf_bytes, k,
                                        hash_leaves=lambda b: _sha_leaves(b, leaf_bytes), hash_level=_sha_level)
            ref = O.merkle_levels(O.chunk_leaves(data, leaf_bytes))
            all_lv = [None] * world
            dist.all_gather_object(all_lv, [[bytes(r) for r in t.numpy()] for t in lv])
            tops = [[bytes(r) for r in t.numpy()] for t in top]
            ok_tree &= vd.assemble_levels(all_lv, tops) == ref
            ok_tree &= len(lv) == vd.local_depth(nl, k) + 1
        q.put((rank, ok_log, ok_tree, (lo, hi)))
    except Exception as e:  # surface the error instead of leaving the parent waiting
        q.put((rank, False, repr(e), (0, 0)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_log_and_merkle_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    res = sorted((q.get() for _ in range(world)), key=lambda r: r[0])
    for rank, ok_log, ok_tree, rng in res:
        assert ok_log, (rank, rng)
        assert ok_tree is True, (rank, ok_tree)
    assert res[0][3][1] == res[1][3][0] and res[0][3][0] == 0


def test_shard_range_plan():
    from paper_2403_09603_b200 import dist as vd
    for n in (0, 1, 639, 640, 641, 10_000, 1 << 26):
        for world in (1, 2, 3, 4, 8):
            rs = [vd.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
                assert a1 == b0 and a1 % vd.SHARD_ALIGN == 0 or a1 == n
    for nl in (1, 7, 4096, 4097, 100_000):
        for world in (1, 2, 8):
            rs = [vd.leaf_block_range(nl, r, world, 12) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == nl
            assert all(a1 == b0 for (_, a1), (b0, _) in zip(rs, rs[1:]))


def test_sharded_paths_without_a_process_group():
    """Single process (no torch.distributed init): the sharded functions are the
    one-rank case -- the gathers are copies and the levels equal merkle.build."""
    sys.path.insert(0, str(REPO / "oracle"))
    import vt_oracle as O
    from paper_2403_09603_b200 import dist as vd
    assert not dist.is_initialized()
    assert vd.all_gather_counts(7).tolist() == [7]
    data = np.random.default_rng(3).normal(0, 0.02, size=70_001).astype(np.float32).tobytes()
    nl = (len(data) + 4095) // 4096
    lv, top = vd.merkle_sharded(torch.frombuffer(bytearray(data), dtype=torch.uint8), nl, 4096, 3,
                                hash_leaves=lambda b: _sha_leaves(b, 4096), hash_level=_sha_level)
    got = vd.assemble_levels([[[bytes(r) for r in t.numpy()] for t in lv]], [[bytes(r) for r in t.numpy()] for t in top])
    assert got == O.merkle_levels(O.chunk_leaves(data, 4096))
