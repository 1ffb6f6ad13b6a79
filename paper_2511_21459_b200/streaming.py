"""Capacity tier: eviction of blocks to a host archive and stream-in on
allocation (reference streaming.py:1-156, integrate.py:122-140).

The active tier is the device table.  When its worst level fills up, blocks
that are spatially irrelevant to the current pose (outside the camera
frustum, or beyond a radius) move to a host-side archive, farthest first,
until occupancy falls to the low-water mark.  A coordinate is live or
archived, never both: the integrate functions stream archived blocks back in
(payload intact, at their archived level) before a frame that reaches them
is fused.

B200 design: the selection math runs on the host exactly as the reference
evaluates it (numpy, same op order), but the blocks move in bulk -- one
device gather + D2H per level for an eviction (HashTable.evict), one H2D +
scatter per level for a stream-in (HashTable.import_blocks) -- and the keys
a frame will touch come from a key-only pass of the device DDA
(tsdf_depth_keys / tsdf_scan_keys), checked against the archive with one
vectorized membership test.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import CapacityError, NotFoundError
from .geometry import Intrinsics, SensorPose, project
from .hashgrid import BlockPayload, HashTable


@dataclass
class EvictionStats:
    evicted: int = 0
    bytes_out: int = 0
    fill_before: float = 0.0
    fill_after: float = 0.0


def _pack(coords) -> np.ndarray:
    c = np.asarray(coords, dtype=np.int64).reshape(-1, 3) + (1 << 20)
    return ((c[:, 0].astype(np.uint64) << np.uint64(42)) | (c[:, 1].astype(np.uint64) << np.uint64(21))
            | c[:, 2].astype(np.uint64))


def _unpack(keys) -> np.ndarray:
    k = np.asarray(keys, dtype=np.uint64)
    m = np.uint64(0x1FFFFF)
    return np.stack([((k >> np.uint64(42)) & m).astype(np.int64), ((k >> np.uint64(21)) & m).astype(np.int64),
                     (k & m).astype(np.int64)], axis=1) - (1 << 20)


class ArchiveStore:
    """Host-side store of serialized blocks (reference block records),
    keyed by coordinate (streaming.py:28-70)."""

    def __init__(self):
        self._records: dict = {}
        self.nbytes = 0
        self._keys = None  # sorted packed keys, rebuilt lazily

    def __contains__(self, coord) -> bool:
        return tuple(int(c) for c in coord) in self._records

    def __len__(self) -> int:
        return len(self._records)

    def coords(self) -> list:
        return sorted(self._records.keys())

    def record(self, coord) -> bytes:
        return self._records[tuple(int(c) for c in coord)]

    def put_record(self, coord, record: bytes) -> int:
        coord = tuple(int(c) for c in coord)
        old = self._records.get(coord)
        if old is not None:
            self.nbytes -= len(old)
        self._records[coord] = bytes(record)
        self.nbytes += len(record)
        self._keys = None
        return len(record)

    def store(self, payload: BlockPayload) -> int:
        from .formats import pack_block_record
        return self.put_record(payload.coord, pack_block_record(payload, archived=True))

    def store_level(self, level: int, coords, tsdf, weight, s2, color) -> int:
        """Archive n blocks of one level at once; returns the bytes stored."""
        from .formats import pack_records
        recs = pack_records(level, coords, tsdf, weight, s2, color, archived=True)
        raw = recs.tobytes()
        size = recs.dtype.itemsize
        total = 0
        for i, c in enumerate(np.asarray(coords, dtype=np.int64).reshape(-1, 3).tolist()):
            total += self.put_record(c, raw[i * size:(i + 1) * size])
        return total

    def take(self, coord) -> BlockPayload:
        from .formats import unpack_block_record
        coord = tuple(int(c) for c in coord)
        rec = self._records.pop(coord, None)
        if rec is None:
            raise NotFoundError(f"block {coord} is not archived")
        self.nbytes -= len(rec)
        self._keys = None
        return unpack_block_record(rec, 0)[0]

    def peek(self, coord) -> BlockPayload:
        from .formats import unpack_block_record
        coord = tuple(int(c) for c in coord)
        rec = self._records.get(coord)
        if rec is None:
            raise NotFoundError(f"block {coord} is not archived")
        return unpack_block_record(rec, 0)[0]

    def archived_among(self, keys) -> np.ndarray:
        """The packed keys (uint64) of `keys` that are archived."""
        if not self._records:
            return np.zeros(0, dtype=np.uint64)
        if self._keys is None:
            self._keys = np.sort(_pack(list(self._records.keys())))
        keys = np.asarray(keys, dtype=np.uint64)
        return keys[np.isin(keys, self._keys, assume_unique=False)]


def active_fill_fraction(table: HashTable) -> float:
    """Worst-case occupancy across the per-level heaps, in [0, 1]."""
    return max(table.fill_fractions())


def _live(table: HashTable):
    coords, levels = [], []
    for level in range(table.num_levels):
        c, _ = table.live_blocks(level, sort=True)
        if len(c):
            coords.append(c)
            levels.append(np.full(len(c), level, dtype=np.int64))
    if not coords:
        return np.zeros((0, 3), dtype=np.int64), np.zeros(0, dtype=np.int64)
    return np.concatenate(coords), np.concatenate(levels)


def _evictable(table: HashTable, coords, mode: str, pose: SensorPose,
               intrinsics: Intrinsics | None, image_size, radius: float):
    """Indices of evictable blocks, farthest first (streaming.py:80-119)."""
    if len(coords) == 0:
        return np.zeros(0, dtype=np.int64)
    centers = (coords.astype(np.float64) + 0.5) * table.block_edge
    dist = np.linalg.norm(centers - pose.translation, axis=1)
    if mode == "radius":
        ok = dist > radius
    elif mode == "frustum":
        if intrinsics is None or image_size is None:
            raise ValueError("frustum mode needs intrinsics and image_size")
        width, height = image_size
        cube = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 0], [1, 0, 1],
                         [0, 1, 1], [1, 1, 1]], dtype=np.float64)
        corners = (coords[:, None, :].astype(np.float64) + cube[None]) * table.block_edge
        cam = pose.to_sensor(corners.reshape(-1, 3)).reshape(len(coords), 8, 3)
        u, v, z = project(cam, intrinsics)
        out = (z <= 0) | (u < -0.5) | (u > width - 0.5) | (v < -0.5) | (v > height - 0.5)
        ok = out.all(axis=1)
    else:
        raise ValueError(f"unknown eviction mode {mode!r}")
    idx = np.nonzero(ok)[0]
    return idx[np.argsort(-dist[idx], kind="stable")]


def select_evictable(table: HashTable, mode: str, pose: SensorPose,
                     intrinsics: Intrinsics | None = None, image_size=None,
                     radius: float = 50.0) -> list:
    """Blocks safe to evict, ordered by decreasing distance from the sensor:
    frustum mode drops a block only when all 8 corners project outside the
    image or behind the camera; radius mode when its centre is beyond the
    radius."""
    coords, _ = _live(table)
    idx = _evictable(table, coords, mode, pose, intrinsics, image_size, radius)
    return [tuple(int(c) for c in coords[i]) for i in idx]


def stream_out(table: HashTable, archive: ArchiveStore, pose: SensorPose, mode: str,
               fill_threshold: float = 0.85, low_water: float = 0.70,
               intrinsics: Intrinsics | None = None, image_size=None,
               radius: float = 50.0) -> EvictionStats:
    """Evict irrelevant blocks once occupancy reaches the threshold
    (streaming.py:122-145): candidates farthest first until the worst level
    is at or below the low-water mark; CapacityError if that is not reached
    while still at or above the threshold."""
    occ = np.array([h.occupied for h in table.heaps], dtype=np.int64)
    cap = np.array([h.capacity for h in table.heaps], dtype=np.float64)
    fill = lambda: float(max(o / c if c else 0.0 for o, c in zip(occ, cap)))
    st = EvictionStats(fill_before=fill())
    st.fill_after = st.fill_before
    if st.fill_before < fill_threshold:
        return st
    coords, levels = _live(table)
    order = _evictable(table, coords, mode, pose, intrinsics, image_size, radius)
    take = []
    for i in order:  # the reference's stopping rule, evaluated on counts
        if fill() <= low_water:
            break
        take.append(i)
        occ[levels[i]] -= 1
    take = np.asarray(take, dtype=np.int64)
    for level in range(table.num_levels):
        sel = take[levels[take] == level] if len(take) else take
        if len(sel):
            t, w, s2, col = table.evict(level, coords[sel])
            st.bytes_out += archive.store_level(level, coords[sel], t, w, s2, col)
    st.evicted = int(len(take))
    st.fill_after = active_fill_fraction(table)
    if st.fill_after >= fill_threshold:
        raise CapacityError(
            f"occupancy {st.fill_after:.2f} still at/above threshold {fill_threshold:.2f} "
            f"after evicting {st.evicted} of {len(order)} candidates; "
            "no spatially irrelevant blocks left to stream out")
    return st


def stream_in(table: HashTable, archive: ArchiveStore, coord):
    """Restore one archived block into the active tier, payload intact
    (streaming.py:148-156).  Returns (handle, level)."""
    coord = tuple(int(c) for c in coord)
    if table.find(coord) is not None:
        raise ValueError(f"block {coord} is already live")
    p = archive.peek(coord)
    table.import_blocks(p.level, [coord], p.tsdf[None], p.weight[None], p.s2[None], p.color[None])
    archive.take(coord)
    return table.find(coord)


def stream_in_keys(table: HashTable, archive: ArchiveStore, keys) -> int:
    """Stream back every archived block among `keys` (packed block keys of
    the coordinates a frame will touch), in bulk per level -- the archive
    branch of _ensure_blocks (integrate.py:122-140).  Returns the count."""
    hit = archive.archived_among(keys)
    if len(hit) == 0:
        return 0
    coords = _unpack(np.sort(hit))
    by_level = {}
    for c in coords.tolist():
        p = archive.peek(c)
        by_level.setdefault(p.level, []).append(p)
    for level, ps in by_level.items():
        # all or nothing per level; a block leaves the archive only once live
        table.import_blocks(level, [p.coord for p in ps], np.stack([p.tsdf for p in ps]),
                            np.stack([p.weight for p in ps]), np.stack([p.s2 for p in ps]),
                            np.stack([p.color for p in ps]))
        for p in ps:
            archive.take(p.coord)
    return int(len(coords))
