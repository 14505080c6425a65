"""bench.py's multi-rank code paths at N = 2 on a one-GPU box: two ranks on
GPU 0 with gloo host collectives (``--dist-backend gloo``; no kernel waits on
another rank's).  What is checked is the multi-rank logic the driver's
scaling runs execute -- shard ranges and global indices, the count exchange
and max-over-ranks timing, the e2e leg, and the strong-scaling legs: the
sharded Merkle root equals the single-GPU root, the LPT-split configs[2]
taus equal the single-GPU batch.  Its numbers are not measurements."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(900)
def test_bench_two_ranks_gloo_on_one_gpu():
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29517", str(REPO / "bench.py"),
                        "--dist-backend", "gloo", "--steps", "3", "--warmup", "3", "--log2n", "24", "--no-cpu"],
                       capture_output=True, text=True, timeout=840, env=env, cwd=str(REPO))
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["auditor_equals_trainer_bitwise"]
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 16 * (1 << 24)
    st = d["strong_scaling"]
    assert st["n_gpus"] == 2
    assert st["merkle_1.5B"]["root_equals_single_gpu"] is True
    assert st["configs[2]_lpt"]["taus_equal_single_gpu"] is True
    assert 0.0995 < st["round_log_replay_2^32"]["logged_fraction"] < 0.1023
