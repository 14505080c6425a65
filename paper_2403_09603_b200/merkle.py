"""SHA-256 Merkle commitments on the B200 -- drop-in for ``vtrain.merkle.build``.

* ``build(leaves)`` -- reference ``merkle.build`` (pkg/src/vtrain/merkle.py:55-72):
  node = SHA-256(left || right), an unpaired last node promoted unchanged,
  every level kept; levels are hashed on the device (``vt_merkle_level``).
* ``merkle_chunked(weights)`` -- the north-star checkpoint commitment
  (SURVEY.md Appendix A.5): leaf i = SHA-256 of bytes [4096 i, 4096 (i+1))
  of the FP32 little-endian weight serialization, then ``build``'s rule.
  The whole tree is computed in HBM (``vt_merkle_build``); levels stay
  device tensors until a caller asks for bytes.

``MerkleTree`` exposes ``.leaves`` / ``.levels`` (lists of 32-byte
``bytes``) and ``.root`` like the reference dataclass, so the reference's
``node`` / ``path`` / ``first_divergence`` / ``write_tree`` work on it.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as D
from . import _lib

DIGEST_LEN = 32


class MerkleTree:
    """Tree whose levels live on the device as uint8 [n_level, 32] tensors."""

    def __init__(self, levels_device: list[torch.Tensor]):
        self.levels_device = levels_device
        self._levels: list[list[bytes]] | None = None

    @property
    def levels(self) -> list[list[bytes]]:
        if self._levels is None:
            out = []
            for lvl in self.levels_device:
                raw = lvl.cpu().numpy().tobytes()
                out.append([raw[i:i + DIGEST_LEN] for i in range(0, len(raw), DIGEST_LEN)])
            self._levels = out
        return self._levels

    @property
    def leaves(self) -> list[bytes]:
        return self.levels[0]

    @property
    def root(self) -> bytes:
        return self.levels_device[-1][0].cpu().numpy().tobytes()

    @property
    def root_hex(self) -> str:
        return self.root.hex()

    def n_nodes(self) -> int:
        return sum(int(lvl.shape[0]) for lvl in self.levels_device)


def _levels_from(nodes: torch.Tensor, n_leaves: int) -> list[torch.Tensor]:
    levels, off, m = [], 0, n_leaves
    while True:
        levels.append(nodes[off:off + m])
        off += m
        if m == 1:
            break
        m = (m + 1) // 2
    return levels


def build_device(leaves: torch.Tensor) -> MerkleTree:
    """Levels above device leaves [n, 32] uint8."""
    n = int(leaves.shape[0])
    if n == 0:
        raise ValueError("cannot build a Merkle tree with no leaves")
    total = int(_lib.lib().vt_merkle_node_count(n))
    nodes = torch.empty((total, DIGEST_LEN), dtype=torch.uint8, device=leaves.device)
    nodes[:n] = leaves
    off, m = 0, n
    while m > 1:
        _lib.call("vt_merkle_level", D.ptr(nodes[off:]), m, D.ptr(nodes[off + m:]), D.stream_ptr())
        off += m
        m = (m + 1) // 2
    return MerkleTree(_levels_from(nodes, n))


def build(leaves: list[bytes]) -> MerkleTree:
    """Build a tree over ordered 32-byte leaf digests (merkle.py:55-72)."""
    if not leaves:
        raise ValueError("cannot build a Merkle tree with no leaves")
    for i, leaf in enumerate(leaves):
        if not isinstance(leaf, bytes) or len(leaf) != DIGEST_LEN:
            raise ValueError(f"leaf {i} is not a 32-byte digest")
    dev = D.require_cuda()
    host = torch.frombuffer(bytearray(b"".join(leaves)), dtype=torch.uint8).reshape(-1, DIGEST_LEN)
    return build_device(host.to(dev))


def _as_bytes_tensor(data) -> torch.Tensor:
    if isinstance(data, torch.Tensor):
        t = data if data.is_cuda else data.to(D.require_cuda())
        if t.dtype == torch.float64:
            raise TypeError("serialize FP64 weights to FP32 first (the commitment is over FP32 bytes)")
        return t.contiguous().reshape(-1).view(torch.uint8)
    if isinstance(data, (bytes, bytearray, memoryview)):
        arr = np.frombuffer(bytes(data), dtype=np.uint8)
    else:
        arr = np.ascontiguousarray(np.asarray(data, dtype="<f4")).reshape(-1).view(np.uint8)
    return torch.from_numpy(arr.copy()).to(D.require_cuda())


def sha256_leaves(data, leaf_bytes: int = 4096) -> torch.Tensor:
    """SHA-256 of each ``leaf_bytes`` chunk -> uint8 [n_leaves, 32] on the device."""
    b = _as_bytes_tensor(data)
    n = b.numel()
    if n == 0:
        raise ValueError("cannot hash an empty checkpoint")
    nl = (n + leaf_bytes - 1) // leaf_bytes
    out = torch.empty((nl, DIGEST_LEN), dtype=torch.uint8, device=b.device)
    _lib.call("vt_sha256_leaves", D.ptr(b), n, int(leaf_bytes), D.ptr(out), D.stream_ptr())
    return out


def merkle_chunked(weights, leaf_bytes: int = 4096) -> MerkleTree:
    """North-star checkpoint commitment over 4 KiB chunks of FP32 LE bytes."""
    b = _as_bytes_tensor(weights)
    n = b.numel()
    if n == 0:
        raise ValueError("cannot hash an empty checkpoint")
    nl = (n + leaf_bytes - 1) // leaf_bytes
    total = int(_lib.lib().vt_merkle_node_count(nl))
    nodes = torch.empty((total, DIGEST_LEN), dtype=torch.uint8, device=b.device)
    _lib.call("vt_merkle_build", D.ptr(b), n, int(leaf_bytes), D.ptr(nodes), total, D.stream_ptr())
    return MerkleTree(_levels_from(nodes, nl))
