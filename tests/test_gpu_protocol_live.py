"""The drop-in, live: the reference's own training / audit loop
(``vtrain.protocol._run``, pkg/src/vtrain/protocol.py:239-307) runs
UNMODIFIED with the GPU channels in its channel seam (protocol.py:268, 278,
283) for every shipped config, and must reproduce what the reference produced
with its NumPy channels (frozen by
``tests/golden/make_golden.py`` ``golden_live_runs`` in the build container):
the Merkle roots of trainer and auditor, the ``.vtrl`` file byte for byte,
the entry count and direction histogram, and -- for ``trend`` -- the 77
auditor corrections.

The reference package is a TEST-ONLY dependency installed by
``tools/install_reference.sh`` into ``baseline/_ref`` (git-ignored, never
imported by the product); without it these tests skip.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time

import pytest

from conftest import GOLDEN, REPO

pytestmark = pytest.mark.gpu

REF = REPO / "baseline" / "_ref"
LIVE = json.loads((GOLDEN / "live_runs.json").read_text())


def _vtrain():
    if not (REF / "vtrain" / "protocol.py").exists():
        pytest.skip("reference not installed (tools/install_reference.sh)")
    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    from vtrain import cli, protocol
    return cli, protocol


@pytest.mark.timeout(600)
@pytest.mark.parametrize("name", ["tiny", "mlp", "logreg", "trend"])
def test_reference_loop_with_gpu_channels(name, tmp_path):
    cli, pr = _vtrain()
    from paper_2403_09603_b200 import protocol as gp
    from paper_2403_09603_b200 import roundlog
    want = LIVE[name]
    cfg = cli.load_config(REF / "vtrain_configs" / f"{name}.json")
    log = tmp_path / f"{name}.vtrl"
    t0 = time.perf_counter()
    writer = roundlog.LogWriter(log, cfg.b_r)
    try:
        tree_t, leaves_t, _, per_step_t, _, _ = pr._run(cfg, pr.get_profile(cfg.trainer_profile),
                                                         gp.GpuTrainerChannel(writer, cfg.b_r), False)
    finally:
        writer.close()
    t1 = time.perf_counter()
    reader = roundlog.LogReader(log)
    tree_a, _, _, per_step_a, _, _ = pr._run(cfg, pr.get_profile("pairwise"), gp.GpuAuditorChannel(reader, cfg.b_r),
                                             False)
    t2 = time.perf_counter()
    assert tree_t.root.hex() == want["root"]
    assert hashlib.sha256(log.read_bytes()).hexdigest() == want["vtrl_sha"]
    assert writer.entry_count == want["entries"]
    assert {str(k): v for k, v in roundlog.LogReader(log).histogram().items()} == want["histogram"]
    assert tree_a.root.hex() == want["audit_root"] == want["root"]
    assert reader.remaining == 0
    corr = sum(s.forward_corrections + s.backward_corrections for s in per_step_a)
    assert corr == want["corrections"]
    directed = sum(s.forward_directed + s.backward_directed for s in per_step_t)
    assert directed == want["histogram"]["0"] + want["histogram"]["2"]
    print(f"{name}: GPU channels train {t1 - t0:.2f}s audit {t2 - t1:.2f}s "
          f"(reference NumPy channels in the build container: {want['cpu_train_s_here']}s / "
          f"{want['cpu_audit_s_here']}s)")


@pytest.mark.timeout(300)
def test_reference_channels_against_gpu_channels_on_tensors():
    """The reference's _TrainerChannel / _AuditorChannel and the GPU channels
    on the same tensors produce identical outputs, counts and log bytes (the
    channel seam, call by call, on the reference's own writer / reader)."""
    _, pr = _vtrain()
    import numpy as np

    from vtrain import roundlog as rrl

    from paper_2403_09603_b200 import protocol as gp
    from paper_2403_09603_b200 import roundlog, workloads
    import tempfile
    from pathlib import Path
    rng = np.random.default_rng(5)
    tensors = [workloads.config0_x(m, s).reshape(-1, 8) * 10.0 ** rng.uniform(-3, 1) for s, m in
               ((1, 4096), (2, 8), (3, 40_000), (4, 1000))]
    tau = 2.0 ** -25
    with tempfile.TemporaryDirectory() as td:
        ref_log, gpu_log = Path(td) / "r.vtrl", Path(td) / "g.vtrl"
        rw, gw = rrl.LogWriter(ref_log, 32), roundlog.LogWriter(gpu_log, 32)
        rc, gc = pr._TrainerChannel(rw, 32), gp.GpuTrainerChannel(gw, 32)
        for t in tensors:
            ro, rd, _ = rc.process(t, tau)
            go, gd, _ = gc.process(t, tau)
            assert rd == gd and go.shape == ro.shape and np.array_equal(go.view(np.uint64), ro.view(np.uint64))
        rw.close()
        gw.close()
        assert ref_log.read_bytes() == gpu_log.read_bytes()
        ra, ga = pr._AuditorChannel(rrl.LogReader(ref_log), 32), gp.GpuAuditorChannel(roundlog.LogReader(gpu_log), 32)
        for t in tensors:
            noisy = np.nextafter(t, np.where(rng.random(t.shape) < 0.5, np.inf, -np.inf))
            ro, _, rcorr = ra.process(noisy, tau)
            go, _, gcorr = ga.process(noisy, tau)
            assert rcorr == gcorr and np.array_equal(go.view(np.uint64), ro.view(np.uint64))
