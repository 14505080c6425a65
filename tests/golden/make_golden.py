"""Freeze golden outputs of the REAL reference (vtrain 0.1.0) as fixtures.

Run in the build container, where the read-only reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports ``vtrain`` from ``/root/reference/pkg/src`` (never copied), runs
its functions on seeded inputs and writes small fixtures next to this
script.  The GPU box has no ``/root/reference``; tests there only read the
committed fixtures.  Everything is regenerated deterministically from the
seeds below.
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parent.parent))

from vtrain import fpround as fp  # noqa: E402
from vtrain import merkle as mk  # noqa: E402
from vtrain import protocol as pr  # noqa: E402
from vtrain import roundlog as rl  # noqa: E402

from paper_2403_09603_b200 import workloads  # noqa: E402

B_VALUES = (10, 26, 29, 32)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def fp_inputs(b_r: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    wide = rng.normal(size=2400) * np.exp2(rng.integers(-60, 38, size=2400))
    # exact ties and near-ties on this grid
    step = 2.0 ** (9 - b_r)
    k = rng.integers(0, 1 << min(20, b_r - 9), size=300)
    e = np.exp2(rng.integers(-20, 20, size=300).astype(np.float64))
    ties = (1.0 + (k + 0.5) * step) * e
    near = ties * (1.0 + rng.choice([-1.0, 1.0], size=300) * 2.0 ** -50)
    # FP32-subnormal region and the 2^-126 boundary
    tiny = rng.normal(size=300) * 1e-40
    q = 2.0 ** ((32 - b_r) - 149)
    tiny_ties = (rng.integers(0, 1 << 12, size=100) + 0.5) * q
    special = np.array([
        0.0, -0.0, 2.0 ** -126, -(2.0 ** -126), 2.0 ** -149, -(2.0 ** -149),
        2.0 ** -150, -(2.0 ** -150), 2.0 ** -151, -(2.0 ** -151),
        np.nextafter(2.0 ** -126, 0.0), -np.nextafter(2.0 ** -126, 0.0),
        fp.grid_max(b_r), -fp.grid_max(b_r), np.nextafter(fp.grid_max(b_r), 0.0),
        1.0, -1.0, 1.0 + 2.0 ** -24, 1.5, 0.2, 3.7, 2.0 ** 127, 1e-300, -1e-300,
        np.nextafter(2.0, 0.0), np.nextafter(1.0, 2.0), np.nextafter(1.0, 0.0),
    ])
    sgn = rng.choice([-1.0, 1.0], size=300 + 100)
    x = np.concatenate([wide, ties * sgn[:300], near, tiny, tiny_ties * sgn[300:], special])
    return x


def taus_for(b_r: int) -> list[float]:
    lo, hi = fp.tau_bounds(b_r)
    return [lo, (lo + hi) / 2.0, hi, 0.0, lo * 1.37, float(workloads.TAU_CONFIG0) if b_r == 32 else lo * 1.9]


def golden_fpround() -> None:
    out = {}
    for b_r in B_VALUES:
        x = fp_inputs(b_r, 100 + b_r)
        rng = np.random.default_rng(200 + b_r)
        codes = rng.integers(0, 3, size=x.size).astype(np.uint8)
        out[f"x_{b_r}"] = x
        out[f"rnd_{b_r}"] = fp.rnd_array(x, b_r)
        lo, hi = fp.grid_neighbors_array(x, b_r)
        out[f"below_{b_r}"] = lo
        out[f"above_{b_r}"] = hi
        out[f"scale_{b_r}"] = fp.exponent_scale_array(x)
        out[f"ongrid_{b_r}"] = fp.is_on_grid(x, b_r)
        out[f"codes_{b_r}"] = codes
        out[f"rev_{b_r}"] = fp.rev_array(x, b_r, codes)
        taus = taus_for(b_r)
        out[f"taus_{b_r}"] = np.array(taus)
        for i, t in enumerate(taus):
            d = fp.direction_array(x, b_r, t)
            out[f"dir_{b_r}_{i}"] = d
            out[f"revdir_{b_r}_{i}"] = fp.rev_array(x, b_r, d)
    np.savez_compressed(HERE / "fpround_golden.npz", **out)


def golden_errors() -> None:
    """(function, args, error message or None) straight from the reference."""
    cases = []
    gm = fp.grid_max(32)
    gm26 = fp.grid_max(26)
    spacing32 = 2.0 ** (127 - 23)
    probes = [
        ("rnd_array", [1e39], 32), ("rnd_array", [float("nan")], 32), ("rnd_array", [float("inf")], 32),
        ("rnd_array", [-float("inf")], 32), ("rnd_array", [gm + 0.4 * spacing32], 32),
        ("rnd_array", [gm + 0.5 * spacing32], 32), ("rnd_array", [1.0, float("nan"), 1e39], 32),
        ("rnd_array", [gm26 * (1 + 2.0 ** -20)], 26), ("rnd_array", [1.0], 9), ("rnd_array", [1.0], 33),
        ("grid_neighbors_array", [gm + 0.4 * spacing32], 32), ("grid_neighbors_array", [gm], 32),
        ("grid_neighbors_array", [float("nan")], 32), ("rev_array", [gm + 0.4 * spacing32], 32),
        ("direction_array", [gm + 0.4 * spacing32], 32), ("direction_array", [1e39], 32),
        ("direction_array", [float("inf")], 32), ("exponent_scale_array", [float("nan")], 32),
        ("rev_array_badcode", [1.5], 32), ("rev_array_badcode_nan", [float("nan")], 32),
        ("rev_array_shape", [1.0, 2.0], 32),
    ]
    for fn, xs, b_r in probes:
        x = np.array(xs, dtype=np.float64)
        try:
            if fn == "rnd_array":
                fp.rnd_array(x, b_r)
            elif fn == "grid_neighbors_array":
                fp.grid_neighbors_array(x, b_r)
            elif fn == "rev_array":
                fp.rev_array(x, b_r, np.ones(x.shape, np.uint8))
            elif fn == "direction_array":
                fp.direction_array(x, b_r, 2.0 ** -25)
            elif fn == "exponent_scale_array":
                fp.exponent_scale_array(x)
            elif fn in ("rev_array_badcode", "rev_array_badcode_nan"):
                fp.rev_array(x, b_r, np.full(x.shape, 3, np.uint8))
            elif fn == "rev_array_shape":
                fp.rev_array(x, b_r, np.ones(3, np.uint8))
            err = None
        except ValueError as e:
            err = str(e)
        cases.append({"fn": fn, "x": [v.hex() for v in x.tolist()], "b_r": b_r, "error": err})
    (HERE / "fpround_errors.json").write_text(json.dumps(cases, indent=1))


def golden_roundlog() -> None:
    rng = np.random.default_rng(21)
    cases = []
    all_digits = {}
    with tempfile.TemporaryDirectory() as td:
        for n, cuts, compress in [(0, [], False), (1, [], False), (4, [], False), (5, [], False),
                                  (6, [], False), (2003, [7, 1500], False), (12345, [3, 4, 999], True),
                                  (100000, [1, 2, 3, 77777], False)]:
            digits = rng.integers(0, 3, size=n).astype(np.uint8)
            if n == 100000:
                digits = np.where(rng.random(n) < 0.9, 1, digits).astype(np.uint8)
            path = Path(td) / f"r{n}.vtrl"
            with rl.LogWriter(path, 29, compress=compress) as w:
                prev = 0
                for c in cuts + [n]:
                    w.write_array(digits[prev:c])
                    prev = c
            raw = path.read_bytes()
            r = rl.LogReader(path)
            cases.append({
                "n": n, "cuts": cuts, "compress": compress, "b_r": 29,
                "digits_sha": sha(digits.tobytes()), "seed_index": len(cases),
                "file_sha": sha(raw), "file_len": len(raw),
                "payload_hex": raw[rl.HEADER_LEN:].hex() if (n <= 2003 and not compress) else None,
                "histogram": r.histogram(),
            })
            all_digits[f"d{len(cases) - 1}"] = digits
    known = {
        "pack5": [[[0, 0, 0, 0, 0], rl.pack5([0, 0, 0, 0, 0])], [[1, 1, 1, 1, 1], rl.pack5([1, 1, 1, 1, 1])],
                  [[2, 0, 0, 0, 1], rl.pack5([2, 0, 0, 0, 1])], [[2, 2, 2, 2, 2], rl.pack5([2, 2, 2, 2, 2])]],
        "unpack5": [[b, rl.unpack5(b)] for b in (0, 1, 83, 121, 122, 242)],
        "payload_bytes_for": [[n, rl.payload_bytes_for(n)] for n in (0, 1, 5, 6, 100000)],
        "file_bytes_for": [[n, rl.file_bytes_for(n)] for n in (0, 1, 5, 6, 100000)],
    }
    np.savez_compressed(HERE / "roundlog_digits.npz", **all_digits)
    (HERE / "roundlog_golden.json").write_text(json.dumps({"cases": cases, "known": known}, indent=1))


def golden_tau() -> None:
    rng = np.random.default_rng(31)
    cases = []
    for b_r in (26, 29, 32):
        lo, hi = fp.tau_bounds(b_r)
        for iters in (1, 10, 25, 30, 40):
            for size in (0, 1, 3, 17):
                s = rng.uniform(0, 2 * hi, size=size).tolist()
                cases.append({"b_r": b_r, "iters": iters, "samples": [v.hex() for v in s],
                              "tau": pr.search_tau(s, b_r, iters).hex()})
    # budget search restated from reference functions
    budget = []
    for seed, n, sigma_exp in [(41, 200003, -2.5), (42, 65536, 0.7), (43, 1000, -1.0), (44, 5120 * 3 + 7, 1.0)]:
        x = np.random.default_rng(seed).normal(0.0, 10.0 ** sigma_exp, size=n)
        r = fp.rnd_array(x, 32)
        p = np.abs(x - r) / np.maximum(fp.exponent_scale_array(x), fp.SCALE_FLOOR)
        B = int(0.005 * n)
        lo, hi = fp.tau_bounds(32)
        for _ in range(30):
            t = (lo + hi) / 2.0
            if int(np.count_nonzero(p > t)) <= B:
                hi = t
            else:
                lo = t
        logged = int(np.count_nonzero(fp.direction_array(x, 32, hi) != fp.IGNORE))
        budget.append({"seed": seed, "n": n, "sigma_exp": sigma_exp, "budget": B,
                       "tau": hi.hex(), "logged": logged})
    (HERE / "tau_golden.json").write_text(json.dumps({"search_tau": cases, "budget": budget}, indent=1))


def golden_merkle() -> None:
    cases = []
    for n in list(range(1, 41)) + [64, 100, 257]:
        leaves = [hashlib.sha256(f"leaf-{i}".encode()).digest() for i in range(n)]
        t = mk.build(leaves)
        cases.append({"n": n, "levels": [[d.hex() for d in lvl] for lvl in t.levels]})
    # chunked leaves over an FP32 weight vector, reference build
    w = np.random.default_rng(4).normal(0.0, 0.02, size=300_001).astype(np.float32)
    data = w.astype("<f4").tobytes()
    leaves = [hashlib.sha256(data[i:i + 4096]).digest() for i in range(0, len(data), 4096)]
    t = mk.build(leaves)
    chunked = {"seed": 4, "n_params": 300_001, "leaf_bytes": 4096,
               "levels": [[d.hex() for d in lvl] for lvl in t.levels]}
    hw = {"empty": mk.hash_weights([]).hex(),
          "arange": mk.hash_weights([np.arange(6, dtype=np.float64).reshape(2, 3)]).hex()}
    (HERE / "merkle_golden.json").write_text(json.dumps({"build": cases, "chunked": chunked,
                                                          "hash_weights": hw}))


def golden_merkle_game() -> None:
    """merkle.node / path / verify_path / first_divergence and hash_weights
    (merkle.py:75-166) on seeded inputs, for the device-level drop-ins."""
    rng = np.random.default_rng(17)
    trees = []
    for n in (1, 2, 3, 5, 8, 13, 40, 257):
        leaves = [hashlib.sha256(f"t{n}-{i}".encode()).digest() for i in range(n)]
        t = mk.build(leaves)
        nodes = []
        for lv in range(len(t.levels)):
            for ix in sorted({0, len(t.levels[lv]) - 1, len(t.levels[lv]) // 2}):
                nodes.append([lv, ix, mk.node(t, lv, ix).hex()])
        paths = []
        for li in sorted({0, n - 1, n // 2, (7 * n) // 11}):
            pth = mk.path(t, li)
            paths.append({"leaf_index": li, "leaf": pth.leaf.hex(),
                          "siblings": [[d.hex(), side] for d, side in pth.siblings],
                          "verifies": mk.verify_path(pth, t.root)})
        # a second tree diverging at planted leaves: reference first_divergence
        div = []
        for planted in sorted({0, n - 1, n // 3}):
            other = list(leaves)
            for j in range(planted, n, max(1, n // 4)):
                other[j] = hashlib.sha256(f"x{n}-{j}".encode()).digest()
            div.append({"planted": planted, "other": [d.hex() for d in other],
                        "first": mk.first_divergence(t, mk.build(other))})
        trees.append({"n": n, "seed_tag": f"t{n}", "nodes": nodes, "paths": paths, "divergence": div})
    errors = {}
    t3 = mk.build([hashlib.sha256(b"e%d" % i).digest() for i in range(3)])
    for name, fn in (("level", lambda: mk.node(t3, 5, 0)), ("index", lambda: mk.node(t3, 1, 2)),
                     ("path", lambda: mk.path(t3, 3))):
        try:
            fn()
        except IndexError as e:
            errors[name] = str(e)
    w1 = rng.normal(0.0, 0.02, size=(37, 41))
    w2 = rng.normal(0.0, 1.0, size=100_003)
    w3 = np.array([1e300, -1e300, 3.4028235e38, 1e-45, -0.0, 2.0 ** -149, 2.0 ** -150], dtype=np.float64)
    hw = {"pair": mk.hash_weights([w1, w2]).hex(), "specials": mk.hash_weights([w3]).hex(),
          "f32_input": mk.hash_weights([w1.astype(np.float32)]).hex(),
          "w1_sha": sha(w1.tobytes()), "w2_sha": sha(w2.tobytes())}
    bad = np.zeros(50, dtype=np.float64)
    bad[17] = np.inf
    bad[31] = np.nan
    try:
        mk.hash_weights([w1, bad])
    except ValueError as e:
        hw["nonfinite_error"] = str(e)
    try:
        mk.hash_weights([w1], b_m=16)
    except ValueError as e:
        hw["b_m_error"] = str(e)
    (HERE / "merkle_game_golden.json").write_text(json.dumps({"trees": trees, "errors": errors,
                                                               "hash_weights": hw}))


def golden_configs() -> None:
    """Config 0 / config 1 at 2^20 through the reference functions, as digests."""
    n = 1 << 20
    tau = workloads.TAU_CONFIG0
    x = workloads.config0_x(n, 0)
    r = fp.rnd_array(x, 32)
    d = fp.direction_array(x, 32, tau)
    idx = np.flatnonzero(d != fp.IGNORE).astype(np.uint64)
    words = (idx << np.uint64(1)) | (d[idx.astype(np.int64)] == fp.UP).astype(np.uint64)
    c0 = {"n": n, "seed": 0, "tau": tau.hex(), "x_sha": sha(x.tobytes()),
          "rnd_f32_sha": sha(r.astype(np.float32).tobytes()), "rnd_f64_sha": sha(r.tobytes()),
          "codes_sha": sha(d.tobytes()), "sparse_sha": sha(words.tobytes()),
          "logged": int(idx.size), "n_up": int(np.count_nonzero(d == fp.UP))}
    xt, xa = workloads.config1_pair(n, 1)
    rt = fp.rnd_array(xt, 32)
    dt = fp.direction_array(xt, 32, tau)
    ya = fp.rev_array(xa, 32, dt)
    ra = fp.rnd_array(xa, 32)
    c1 = {"n": n, "seed": 1, "tau": tau.hex(), "xt_sha": sha(xt.tobytes()), "xa_sha": sha(xa.tobytes()),
          "trainer_f32_sha": sha(rt.astype(np.float32).tobytes()),
          "auditor_f32_sha": sha(ya.astype(np.float32).tobytes()),
          "auditor_equals_trainer": bool(np.array_equal(ya.view(np.uint64), rt.view(np.uint64))),
          "corrections": int(np.count_nonzero(ya != ra)), "logged": int(np.count_nonzero(dt != 1)),
          "plain_mismatch": int(np.count_nonzero(ra != rt))}
    (HERE / "config_golden.json").write_text(json.dumps({"config0": c0, "config1": c1}, indent=1))


def golden_channel_traces() -> None:
    """Record every channel call of real reference train + audit runs.

    A recording wrapper sits in the channel seam of ``protocol._run``
    (protocol.py:239-307) around the reference ``_TrainerChannel`` /
    ``_AuditorChannel``; the fixture stores each call's input tensor, tau,
    output and counts, plus the .vtrl file digest.  On the GPU box the same
    inputs are replayed through the GPU channels (no reference needed)."""
    from vtrain.cli import load_config

    class Rec:
        def __init__(self, inner):
            self.inner, self.calls = inner, []

        def process(self, values, tau):
            out, directed, corr = self.inner.process(values, tau)
            self.calls.append((np.array(values, dtype=np.float64), float(tau), np.array(out), directed, corr))
            return out, directed, corr

    arrays = {}
    meta = {}
    # trend: only the prefix up to the last call with auditor corrections
    # (calls 18 and 20 hold all 77 of the run's corrections; 102,144 elements)
    prefix = {"tiny": None, "logreg": None, "trend": 21}
    with tempfile.TemporaryDirectory() as td:
        for name in ("tiny", "logreg", "trend"):
            cfg = load_config(Path("/root/reference/pkg/configs") / f"{name}.json")
            log = Path(td) / f"{name}.vtrl"
            w = rl.LogWriter(log, cfg.b_r)
            tr = Rec(pr._TrainerChannel(w, cfg.b_r))
            tree_t, *_ = pr._run(cfg, pr.get_profile(cfg.trainer_profile), tr, False)
            w.close()
            au = Rec(pr._AuditorChannel(rl.LogReader(log), cfg.b_r))
            tree_a, *_ = pr._run(cfg, pr.get_profile("pairwise"), au, False)
            k = prefix[name]
            vtrl_sha = sha(log.read_bytes())
            if k is not None:  # .vtrl of the prefix: the reference writer over the prefix's codes
                tr.calls, au.calls = tr.calls[:k], au.calls[:k]
                plog = Path(td) / f"{name}_prefix.vtrl"
                pw = rl.LogWriter(plog, cfg.b_r)
                for c in tr.calls:
                    pw.write_array(fp.direction_array(c[0], cfg.b_r, c[1]))
                pw.close()
                vtrl_sha = sha(plog.read_bytes())
            meta[name] = {"b_r": cfg.b_r, "vtrl_sha": vtrl_sha, "root": tree_t.root.hex(),
                          "prefix_calls": k, "total_corrections": int(sum(c[4] for c in au.calls)),
                          "audit_root": tree_a.root.hex(), "n_calls": len(tr.calls),
                          "directed": [c[3] for c in tr.calls], "corrections": [c[4] for c in au.calls],
                          "taus": [c[1] for c in tr.calls], "shapes": [list(c[0].shape) for c in tr.calls]}
            for role, rec in (("t", tr), ("a", au)):
                arrays[f"{name}_{role}_in"] = np.concatenate([c[0].reshape(-1) for c in rec.calls])
                # outputs are grid values (FP32-exact): stored as FP32, lossless
                arrays[f"{name}_{role}_out"] = np.concatenate([c[2].reshape(-1) for c in rec.calls]).astype(np.float32)
    np.savez_compressed(HERE / "channel_traces.npz", **arrays)
    (HERE / "channel_traces.json").write_text(json.dumps(meta))


def golden_live_runs() -> None:
    """Appendix C of SURVEY.md, frozen from the real reference here: full
    ``train`` + ``audit`` runs (trainer profile of the config, auditor
    ``pairwise``) of every shipped config -- root, audit root, .vtrl digest,
    entry count, direction histogram, total corrections.  The GPU test
    tests/test_gpu_protocol_live.py runs ``protocol._run`` unmodified with the
    GPU channels and must reproduce them."""
    from vtrain.cli import load_config

    out = {}
    with tempfile.TemporaryDirectory() as td:
        for name in ("tiny", "mlp", "logreg", "trend"):
            cfg = load_config(Path("/root/reference/pkg/configs") / f"{name}.json")
            log = Path(td) / f"{name}.vtrl"
            t = pr.train(cfg, log)
            a = pr.audit(cfg, "pairwise", log)
            r = rl.LogReader(log)
            out[name] = {"root": t.root.hex(), "audit_root": a.root.hex(), "vtrl_sha": sha(log.read_bytes()),
                         "entries": int(t.entries_logged), "histogram": {str(k): int(v) for k, v in r.histogram().items()},
                         "corrections": int(a.total_corrections), "steps": len(t.per_step),
                         "b_r": cfg.b_r, "trainer_profile": cfg.trainer_profile,
                         "cpu_train_s_here": round(t.seconds, 3), "cpu_audit_s_here": round(a.seconds, 3)}
    (HERE / "live_runs.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    import sys as _sys
    if "--live-only" in _sys.argv:
        golden_live_runs()
        raise SystemExit(0)
    golden_live_runs()
    golden_channel_traces()
    golden_fpround()
    golden_errors()
    golden_roundlog()
    golden_tau()
    golden_merkle()
    golden_merkle_game()
    golden_configs()
    print("golden fixtures written to", HERE)
