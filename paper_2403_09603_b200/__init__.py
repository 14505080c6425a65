"""B200-native (sm_100a) hot path of the vtrain verifiable-training scheme
(arXiv 2403.09603): round-and-log, replay, adaptive threshold search and
SHA-256 Merkle commitments, behind the reference package's operator API.

Modules mirror the reference layout:
  fpround   -- vtrain.fpround   (grid arithmetic; GPU kernels)
  roundlog  -- vtrain.roundlog  (.vtrl writer/reader; device pack/unpack)
  merkle    -- vtrain.merkle    (build, game queries, hash_weights + the chunked commitment)
  protocol  -- channel plug-ins for vtrain.protocol._run, search_tau(+budget)
  ops       -- device-level north-star operators (sparse log)
  dist      -- contiguous sharding across GPUs (torch.distributed / NCCL)
All compute runs in the in-tree C-ABI library libvtrain_b200.so.
"""

from .fpround import DOWN, IGNORE, UP, RoundingParams, direction, rev, rnd  # noqa: F401
from .merkle import MerklePath, MerkleTree, build, hash_weights  # noqa: F401  (vtrain/__init__.py re-exports)

__version__ = "0.1.0"
