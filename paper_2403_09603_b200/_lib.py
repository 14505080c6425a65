"""ctypes binding of the in-tree C-ABI library ``libvtrain_b200.so``.

The library is the product: every operator in this package calls it, and
there is no CPU fallback.  If the shared object is missing the import of
any operator fails loudly (run ``python -c "import __graft_entry__ as g;
g.build()"`` or ``python paper_2403_09603_b200/build_lib.py``).

Signatures mirror ``include/vtrain_b200.h`` exactly; ``EXPORTS`` is the
single source of truth used both to set ``argtypes`` and by the symbol test.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import os

# VTRAIN_B200_LIB: an alternative build of the same library (A/B measurements)
LIB_PATH = Path(os.environ.get("VTRAIN_B200_LIB") or Path(__file__).resolve().with_name("libvtrain_b200.so"))

VT_OK, VT_EINVAL, VT_ECUDA = 0, -1, -2
ERR_NONFINITE = 1
ERR_RANGE = 2
ERR_RANGE_NEIGHBOR = 4
ERR_BAD_CODE = 8
ERR_BAD_LOG_BYTE = 16
ERR_BAD_SPARSE = 32
ERR_EXCHANGE = 64
OUT_NONE, OUT_F32, OUT_F64 = 0, 1, 2
LOG_SPARSE, LOG_CODES, LOG_PACKED = 0, 1, 2

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int
_dbl = C.c_double
_sz = C.c_size_t

EXPORTS: dict[str, tuple] = {
    "vt_version": (C.c_char_p, []),
    "vt_last_error": (C.c_char_p, []),
    "vt_tile_elems": (_i32, []),
    "vt_round_log_workspace": (_sz, [_i64]),
    "vt_round_log": (_i32, [_p, _i64, _i32, _dbl, _i32, _p, _p, _i64, _i64, _p, _p, _p, _p, _i64, _p,
                            _p, _p, _p, _sz, _p]),
    "vt_replay_workspace": (_sz, [_i64]),
    "vt_replay": (_i32, [_p, _i64, _i32, _i32, _p, _i64, _i64, _i32, _p, _p, _p, _p, _sz, _p]),
    "vt_grid_neighbors": (_i32, [_p, _i64, _i32, _p, _p, _p, _p]),
    "vt_exponent_scale": (_i32, [_p, _i64, _p, _p, _p]),
    "vt_is_on_grid": (_i32, [_p, _i64, _i32, _p, _p]),
    "vt_norm_distance": (_i32, [_p, _i64, _i32, _p, _p, _p]),
    "vt_pack5": (_i32, [_p, _i64, _p, _p, _p]),
    "vt_unpack5": (_i32, [_p, _i64, _i64, _p, _p, _p]),
    "vt_log_validate": (_i32, [_p, _i64, _p, _p]),
    "vt_log_histogram": (_i32, [_p, _i64, _p, _p, _p]),
    "vt_tau_workspace": (_sz, [_i64]),
    "vt_tau_kth_key": (_i32, [_p, _i64, _i32, _i64, _p, _p, _p, _sz, _p]),
    "vt_tau_kth_hist_offset": (_sz, [_i32]),
    "vt_tau_kth_hist_bins": (_i32, [_i32]),
    "vt_tau_kth_begin": (_i32, [_i64, _p, _p, _sz, _p]),
    "vt_tau_kth_hist": (_i32, [_p, _i64, _i32, _i32, _p, _p, _sz, _p]),
    "vt_tau_kth_select": (_i32, [_i32, _p, _p, _sz, _p]),
    "vt_tau_budget_key": (_i32, [_p, _i64, _i32, _i64, _dbl, _dbl, _p, _p, _p, _p, _sz, _p]),
    "vt_tau_budget_workspace": (_sz, [_i64]),
    "vt_tau_budget": (_i32, [_p, _i64, _i32, _i64, _i32, _p, _p, _p, _p, _sz, _p]),
    "vt_exchange_words": (_sz, [_i32]),
    "vt_stream_synchronize": (_i32, [_p]),
    "vt_tau_shard_exchange_words": (_sz, [_i32, _i64]),
    "vt_tau_shard_search_x_workspace": (_sz, [_i64]),
    "vt_tau_shard_search_x": (_i32, [_p, _i64, _i32, _i64, _i64, _i32, _p, _p, _i32, _i32, _i64, _p, _p, _p, _p,
                                     _sz, _i32, _p]),
    "vt_round_log_exchange": (_i32, [_p, _i64, _i32, _dbl, _i32, _p, _p, _i64, _i64, _p, _p, _p, _sz, _p, _i32, _i32,
                                     _p]),
    "vt_counts_wait": (_i32, [_p, _i32, _i32, _p, _p, _p]),
    "vt_digest_exchange_words": (_sz, [_i32, _i64]),
    "vt_merkle_level_exchange": (_i32, [_p, _i64, _p, _p, _i32, _i32, _i64, _i64, _p]),
    "vt_digests_publish": (_i32, [_p, _i64, _p, _i32, _i32, _i64, _i64, _p]),
    "vt_digests_wait": (_i32, [_p, _i32, _i32, _i64, _p, _p, _p]),
    "vt_tau_shard_workspace": (_sz, [_i64]),
    "vt_tau_shard_plan": (_i32, [_i64, _i32, _i64, _p, _p]),
    "vt_tau_shard_candidates": (_i32, [_p, _i64, _i32, _i64, _i64, _p, _p, _p, _sz, _p]),
    "vt_tau_shard_digit_keys": (_i32, [_i64, _i32, _i64, _i64, _i64, _p, _i64, _p, _p, _sz, _p]),
    "vt_round_log_adaptive_workspace": (_sz, [_i64]),
    "vt_round_log_adaptive": (_i32, [_p, _i64, _i32, _i64, _i32, _i32, _p, _p, _i64, _i64, _p, _p, _p, _p, _p,
                                     _p, _sz, _p]),
    "vt_round_log_adaptive_batch_workspace": (_sz, [_p, _i32]),
    "vt_round_log_adaptive_batch": (_i32, [_p, _i32, _i32, _i32, _i32, _p, _sz, _p]),
    "vt_straddle_min": (_i32, [_p, _p, _i64, _i32, _p, _p, _p, _p, _p]),
    "vt_min_f64": (_i32, [_p, _i64, _p, _p, _p]),
    "vt_sha256_leaves": (_i32, [_p, _i64, _i64, _p, _p]),
    "vt_merkle_level": (_i32, [_p, _i64, _p, _p]),
    "vt_merkle_node_count": (_i64, [_i64]),
    "vt_merkle_build": (_i32, [_p, _i64, _i64, _p, _i64, _p]),
    "vt_sha256_peak_bench": (_i32, [_p, _i64, _i32, _p]),
    "vt_int_mix_peak_bench": (_i32, [_p, _i64, _i32, _i32, _p]),
    "vt_int_mix_ops_per_thread_rep": (_i64, []),
    "vt_serialize_f32": (_i32, [_p, _i64, _p, _i64, _p, _p]),
}



class AdaptiveSegment(C.Structure):
    """``vt_adaptive_segment`` of include/vtrain_b200.h."""

    _fields_ = [("x", _p), ("n", _i64), ("budget", _i64), ("out", _p), ("log", _p), ("log_cap", _i64),
                ("global_base", _i64), ("tau_out", _p), ("flags", _p)]


_LIB: C.CDLL | None = None


class VtLibraryMissing(ImportError):
    pass


class VtCudaError(RuntimeError):
    pass


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        if not LIB_PATH.exists():
            raise VtLibraryMissing(
                f"{LIB_PATH} is not built; run paper_2403_09603_b200/build_lib.py (there is no CPU fallback)")
        handle = C.CDLL(str(LIB_PATH))
        for name, (res, args) in EXPORTS.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = handle
    return _LIB


def call(name: str, *args) -> None:
    """Call an entry point; raise on a non-zero status."""
    rc = getattr(lib(), name)(*args)
    if rc != VT_OK:
        msg = lib().vt_last_error().decode(errors="replace")
        if rc == VT_EINVAL:
            raise ValueError(f"{name}: {msg}")
        raise VtCudaError(f"{name}: {msg}")


def tile_elems() -> int:
    return int(lib().vt_tile_elems())
