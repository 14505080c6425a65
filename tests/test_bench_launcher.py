"""bench.py's multi-rank launcher on CPU (``--gpus N`` must be
real).  ``--gpus 2`` without a launcher re-executes under
torch.distributed.run with 2 ranks; ``--harness-check`` runs the rank /
barrier / max-over-ranks / single-JSON-line path with gloo and no kernels."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO


def _run(*extra):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    p = subprocess.run([sys.executable, str(REPO / "bench.py"), "--harness-check", "--steps", "2", "--warmup", "1",
                        *extra], capture_output=True, text=True, timeout=240, env=env, cwd=str(REPO))
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [json.loads(ln) for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout  # rank 0 alone prints, once
    return lines[0]


@pytest.mark.timeout(300)
def test_bench_gpus_2_spawns_two_ranks():
    line = _run("--gpus", "2")
    assert line["n_gpus"] == 2 and line["ranks_reporting"] == 2 and line["harness_check"] is True


@pytest.mark.timeout(300)
def test_bench_gpus_1_is_a_single_process():
    line = _run("--gpus", "1")
    assert line["n_gpus"] == 1 and line["ranks_reporting"] == 1
