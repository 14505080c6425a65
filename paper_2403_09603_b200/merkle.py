"""SHA-256 Merkle commitments on the B200 -- drop-in for ``vtrain.merkle.build``.

* ``build(leaves)`` -- reference ``merkle.build`` (pkg/src/vtrain/merkle.py:55-72):
  node = SHA-256(left || right), an unpaired last node promoted unchanged,
  every level kept; levels are hashed on the device (``vt_merkle_level``).
* ``merkle_chunked(weights)`` -- the north-star checkpoint commitment
  (SURVEY.md Appendix A.5): leaf i = SHA-256 of bytes [4096 i, 4096 (i+1))
  of the FP32 little-endian weight serialization, then ``build``'s rule.
  The whole tree is computed in HBM (``vt_merkle_build``); levels stay
  device tensors until a caller asks for bytes.

* ``node`` / ``path`` / ``verify_path`` / ``first_divergence`` -- the
  verification-game queries (merkle.py:75-152) answered from the device
  levels: only the digests a query needs cross PCIe.
* ``hash_weights(tensors)`` -- the canonical checkpoint digest
  (merkle.py:155-166): FP64 -> FP32 little-endian serialization and the
  finiteness check on the device (``vt_serialize_f32``), chunks copied to
  pinned host memory while the next one converts, and ONE sequential
  SHA-256 stream on the host (hashlib, the reference's own SHA-256): the
  digest is a single stream over all bytes, so it cannot be split.

``MerkleTree`` exposes ``.leaves`` / ``.levels`` (lists of 32-byte
``bytes``) and ``.root`` like the reference dataclass, so the reference's
own ``node`` / ``path`` / ``first_divergence`` / ``write_tree`` also work on
it (by materialising every level on the host).
"""

from __future__ import annotations

import hashlib
from dataclasses import dataclass

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


# ---------------------------------------------------------------------------
# verification-game queries from device levels (merkle.py:75-152)
# ---------------------------------------------------------------------------

@dataclass
class MerklePath:
    """Reference ``MerklePath`` (merkle.py:41-52): leaf digest + siblings to the root."""

    leaf_index: int
    leaf: bytes
    siblings: list[tuple[bytes, str]]


def _gather(tree: MerkleTree, refs: list[tuple[int, int]]) -> list[bytes]:
    """Digests at (level, index) pairs with one device gather and one copy."""
    if not refs:
        return []
    rows = torch.cat([tree.levels_device[lv][ix:ix + 1] for lv, ix in refs])
    raw = rows.cpu().numpy().tobytes()
    return [raw[i * DIGEST_LEN:(i + 1) * DIGEST_LEN] for i in range(len(refs))]


def node(tree: MerkleTree, level: int, index: int) -> bytes:
    """Digest at (level, index); level 0 is the leaves (merkle.py:75-83)."""
    if not 0 <= level < len(tree.levels_device):
        raise IndexError(f"level {level} out of range")
    if not 0 <= index < int(tree.levels_device[level].shape[0]):
        raise IndexError(f"index {index} out of range at level {level}")
    return _gather(tree, [(level, index)])[0]


def path(tree: MerkleTree, leaf_index: int) -> MerklePath:
    """Authentication path for one leaf (merkle.py:86-102): a promoted node
    contributes no sibling."""
    sizes = [int(lvl.shape[0]) for lvl in tree.levels_device]
    if not 0 <= leaf_index < sizes[0]:
        raise IndexError(f"leaf index {leaf_index} out of range")
    refs, sides = [(0, leaf_index)], []
    idx = leaf_index
    for level in range(len(sizes) - 1):
        if idx % 2 == 0:
            if idx + 1 < sizes[level]:
                refs.append((level, idx + 1))
                sides.append("right")
        else:
            refs.append((level, idx - 1))
            sides.append("left")
        idx //= 2
    got = _gather(tree, refs)
    return MerklePath(leaf_index=leaf_index, leaf=got[0], siblings=list(zip(got[1:], sides)))


def verify_path(p, root: bytes) -> bool:
    """Recompute the root from a path and compare (merkle.py:105-115)."""
    h = p.leaf
    for sibling, side in p.siblings:
        if side == "right":
            h = hashlib.sha256(h + sibling).digest()
        elif side == "left":
            h = hashlib.sha256(sibling + h).digest()
        else:
            return False
    return h == root


def first_divergence(a: MerkleTree, b: MerkleTree) -> int | None:
    """Smallest leaf index where the trees disagree, or None if the roots
    match (merkle.py:118-152): the same logarithmic descent as the
    reference, reading the two children of each mismatching node from the
    device."""
    na, nb = int(a.levels_device[0].shape[0]), int(b.levels_device[0].shape[0])
    if na != nb:
        raise ValueError("checkpoint schedule mismatch")
    if a.root == b.root:
        return None
    level, index = len(a.levels_device) - 1, 0
    while level > 0:
        child = level - 1
        li = 2 * index
        if li + 1 >= int(a.levels_device[child].shape[0]):
            index, level = li, child  # promoted single child carries the parent digest
            continue
        pair = torch.stack([a.levels_device[child][li], b.levels_device[child][li],
                            a.levels_device[child][li + 1], b.levels_device[child][li + 1]])
        d = pair.cpu().numpy()
        if not np.array_equal(d[0], d[1]):
            index = li
        else:
            if np.array_equal(d[2], d[3]):
                raise RuntimeError("parent digests differ but both children match")
            index = li + 1
        level = child
    return index


# ---------------------------------------------------------------------------
# canonical checkpoint digest (merkle.py:155-166)
# ---------------------------------------------------------------------------

_HW_CHUNK = 1 << 24  # elements per serialized chunk (64 MiB of FP32)


def hash_weights(tensors, b_m: int = 32, chunk: int = _HW_CHUNK) -> bytes:
    """SHA-256 over the canonical FP32 serialization of parameter tensors:
    tensors in order, row-major, each element cast to FP32 and written as
    four little-endian bytes.  Same errors as the reference."""
    if b_m != 32:
        raise ValueError("only FP32 target precision is supported")
    dev = D.require_cuda()
    h = hashlib.sha256()
    stream = torch.cuda.current_stream(dev)
    dbuf = [torch.empty(chunk, dtype=torch.float32, device=dev) for _ in range(2)]
    hbuf = [torch.empty(chunk, dtype=torch.float32).pin_memory() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    bad = torch.empty(1, dtype=torch.int64, device=dev)
    pending = None  # (slot, count) copied to host, not yet hashed
    slot = 0
    for i, t in enumerate(tensors):
        x = t if isinstance(t, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(t, dtype=np.float64))
        x = D.aligned_f64(x.to(dev, torch.float64).reshape(-1))
        n = x.numel()
        bad.fill_(np.iinfo(np.int64).max)
        for lo in range(0, n, chunk):
            m = min(chunk, n - lo)
            _lib.call("vt_serialize_f32", D.ptr(x[lo:]), m, D.ptr(dbuf[slot]), lo, D.ptr(bad), D.stream_ptr(dev))
            hbuf[slot][:m].copy_(dbuf[slot][:m], non_blocking=True)
            done[slot].record(stream)
            if pending is not None:  # hash the previous chunk while this one converts and copies
                ps, pm = pending
                done[ps].synchronize()
                h.update(memoryview(hbuf[ps][:pm].numpy()).cast("B"))
            first = int(bad.item()) if lo + m >= n else None
            if first is not None and first != np.iinfo(np.int64).max:
                raise ValueError(f"non-finite weight in tensor {i} at flat index {first}")
            pending = (slot, m)
            slot ^= 1
    if pending is not None:
        ps, pm = pending
        done[ps].synchronize()
        h.update(memoryview(hbuf[ps][:pm].numpy()).cast("B"))
    return h.digest()
