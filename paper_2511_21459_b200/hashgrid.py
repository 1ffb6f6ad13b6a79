"""Device-resident flat spatial hash over voxel blocks of several resolutions.

Drop-in for the reference's ``HashTable`` (hashgrid.py:139-354): the same
constructor, find / insert / remove / find_batch / insert_batch /
live_blocks, per-level heaps and capacity semantics (level heaps plus the
bucket + overflow-chain limit per Teschner slot, emulated with per-slot
occupancy counters).  The index itself is an open-addressing table of
64-bit packed keys in HBM with lock-free atomicCAS insertion
(csrc/tsdf_common.cuh); voxel payloads live in per-level SoA slabs on the
device.  ``heaps[level].tsdf`` etc. are read-only host snapshots indexed by
heap handle, like the reference's arrays; write voxel data with
``write_payload``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import CapacityError, NotFoundError

HASH_PRIMES = (73856093, 19349669, 83492791)
FINE_SIDE = 8
_M64 = 1 << 64


def hash_key(coord, n_hash: int) -> int:
    """Reference slot index (hashgrid.py:30-46): 64-bit wrapped Teschner hash,
    Euclidean mod."""
    if n_hash <= 0:
        raise ValueError("n_hash must be positive")
    x, y, z = (int(c) for c in coord)
    h = ((x * HASH_PRIMES[0]) ^ (y * HASH_PRIMES[1]) ^ (z * HASH_PRIMES[2])) & (_M64 - 1)
    if h >= 1 << 63:
        h -= _M64
    return h % n_hash


def hash_key_batch(coords, n_hash: int) -> np.ndarray:
    c = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
    with np.errstate(over="ignore"):
        h = (c[:, 0] * np.int64(HASH_PRIMES[0])) ^ (c[:, 1] * np.int64(HASH_PRIMES[1])) \
            ^ (c[:, 2] * np.int64(HASH_PRIMES[2]))
    return h % np.int64(n_hash)


def voxel_side(level: int) -> int:
    return FINE_SIDE >> level


def voxel_count(level: int) -> int:
    return voxel_side(level) ** 3


def voxel_index(world_point, block_coord, level: int, block_edge: float) -> int:
    """Row-major (x slowest, z fastest) voxel offset of a point in a block
    (hashgrid.py:357-367)."""
    p = np.asarray(world_point, dtype=np.float64)
    local = p - np.asarray(block_coord, dtype=np.float64) * block_edge
    if np.any(local < 0) or np.any(local >= block_edge):
        raise ValueError(f"point {tuple(p)} lies outside block {tuple(block_coord)}")
    side = voxel_side(level)
    ijk = np.minimum((local / (block_edge / side)).astype(np.int64), side - 1)
    return int((ijk[0] * side + ijk[1]) * side + ijk[2])


@dataclass
class BlockPayload:
    """Full copy of one block's voxel data, detached from the table."""

    coord: tuple
    level: int
    tsdf: np.ndarray
    weight: np.ndarray
    s2: np.ndarray
    color: np.ndarray


class BlockHeap:
    """Per-level view: sizes, occupancy and the level's voxel arrays by
    handle (snapshots of the device heap; item assignment writes through)."""

    def __init__(self, table: "HashTable", level: int, capacity: int):
        self._table = table
        self.level = level
        self.side = voxel_side(level)
        self.nvox = self.side ** 3
        self.capacity = int(capacity)

    @property
    def occupied(self) -> int:
        n = C.c_int64()
        N.check(N.lib().tsdf_live_count(self._table._h, self.level, C.byref(n)), "live_count")
        return int(n.value)

    def fill_fraction(self) -> float:
        return self.occupied / self.capacity if self.capacity else 0.0

    def _snapshot(self):
        # one export per map change (tsdf_table_version), not per attribute read
        ver = self._table.version
        cached = self.__dict__.get("_snap")
        if cached is not None and cached[0] == ver:
            return cached[1]
        out = self._export()
        self.__dict__["_snap"] = (ver, out)
        return out

    def _export(self):
        coords, handles, t, w, s2, c = self._table.export_level(self.level)
        n = self.capacity * self.nvox
        out = {"tsdf": np.zeros(n), "weight": np.zeros(n), "s2": np.zeros(n),
               "color": np.zeros((n, 3), dtype=np.float32),
               "coords": np.zeros((self.capacity, 3), dtype=np.int64),
               "live": np.zeros(self.capacity, dtype=bool)}
        if len(handles):
            idx = (handles[:, None] * self.nvox + np.arange(self.nvox)).ravel()
            out["tsdf"][idx] = t.ravel()
            out["weight"][idx] = w.ravel()
            out["s2"][idx] = s2.ravel()
            out["color"][idx] = c.reshape(-1, 3)
            out["coords"][handles] = coords
            out["live"][handles] = True
        for a in out.values():
            a.setflags(write=False)
        return out

    def __getattr__(self, name):
        if name in _VOXEL_FIELDS:
            return HeapField._over(self, name, self._snapshot())
        if name in ("coords", "live"):
            return self._snapshot()[name]
        raise AttributeError(name)

    def payload(self, handle: int) -> BlockPayload:
        """Copy of the block stored at `handle` (hashgrid.py:115-125).  A
        live block is read from the device; a free handle reads as the
        zeros the slab holds."""
        snap = self._snapshot()
        h = int(handle)
        if snap["live"][h]:
            coord = tuple(int(v) for v in snap["coords"][h])
            return self._table.payload(coord)
        lo, hi = h * self.nvox, (h + 1) * self.nvox
        return BlockPayload(coord=tuple(int(v) for v in snap["coords"][h]), level=self.level,
                            tsdf=snap["tsdf"][lo:hi].copy(), weight=snap["weight"][lo:hi].copy(),
                            s2=snap["s2"][lo:hi].copy(), color=snap["color"][lo:hi].copy())

    def write_payload(self, handle: int, payload: BlockPayload) -> None:
        """Overwrite the voxels of the live block at `handle`
        (hashgrid.py:127-133); its key and level stay."""
        snap = self._snapshot()
        h = int(handle)
        if not snap["live"][h]:
            raise ValueError(f"heap slot {h} of level {self.level} holds no live block")
        coord = tuple(int(v) for v in snap["coords"][h])
        self._table.write_payload(coord, payload)

    def _write_back(self, snap: dict, name: str, before: np.ndarray) -> None:
        """Push the blocks whose `name` values changed in `snap` to the
        device.  The other fields of each block are read back from the device
        first, so a stale snapshot never overwrites them."""
        after = snap[name]
        diff = (before != after) & ~(np.isnan(before) & np.isnan(after))
        rows = np.nonzero(diff.any(axis=1) if diff.ndim == 2 else diff)[0]
        handles = np.unique(rows // self.nvox)
        dead = [int(h) for h in handles if not snap["live"][h]]
        if dead:
            after[...] = before
            raise ValueError(f"heap slot(s) {dead[:8]} of level {self.level} hold no live block; "
                             "only live blocks can be written")
        for h in handles:
            coord = tuple(int(v) for v in snap["coords"][h])
            pay = self._table.payload(coord)
            setattr(pay, name, np.array(after[h * self.nvox:(h + 1) * self.nvox]))
            self._table.write_payload(coord, pay)


_VOXEL_FIELDS = ("tsdf", "weight", "s2", "color")


class HeapField(np.ndarray):
    """A level's flat voxel array in the reference's heap layout
    (hashgrid.py:95-140: handle * nvox + voxel index).  Reading it is a
    snapshot of the device heap; item assignment on the array itself writes
    the changed blocks through to the device, which is what the reference's
    own tests do to craft fields (tests/test_meshing.py:22-39).  Views derived
    from it are read-only; copies are ordinary arrays."""

    _owner = None

    def __array_finalize__(self, obj):
        self._owner = None          # slices / views of a field do not write through

    @classmethod
    def _over(cls, heap: "BlockHeap", name: str, snap: dict) -> "HeapField":
        out = snap[name].view(cls)
        out._owner = (heap, name, snap)
        return out

    def __setitem__(self, index, value):
        if self._owner is None:
            # a copy writes normally; a view of the snapshot is read-only and
            # numpy says so
            np.ndarray.__setitem__(self, index, value)
            return
        heap, name, snap = self._owner
        base = snap[name]
        before = base.copy()
        base.setflags(write=True)
        try:
            np.ndarray.__setitem__(base, index, value)
        finally:
            base.setflags(write=False)
        heap._write_back(snap, name, before)


class HashTable:
    """Index from integer block coordinates to (heap handle, level)."""

    def __init__(self, n_hash: int, bucket_capacity: int, overflow_capacity: int,
                 block_edge: float, heap_capacities=(16384, 8192), stream=None):
        if n_hash <= 0 or bucket_capacity <= 0 or overflow_capacity <= 0:
            raise ValueError("table sizes must be positive")
        self.n_hash = int(n_hash)
        self.bucket_capacity = int(bucket_capacity)
        self.overflow_capacity = int(overflow_capacity)
        self.block_edge = float(block_edge)
        caps = np.ascontiguousarray([int(c) for c in heap_capacities], dtype=np.int64)
        h = C.c_void_p()
        stream_ptr = None if stream is None else int(getattr(stream, "cuda_stream", stream))
        N.check(N.lib().tsdf_table_create(self.n_hash, self.bucket_capacity,
                                          self.overflow_capacity, self.block_edge, len(caps),
                                          caps, stream_ptr, C.byref(h)), "HashTable")
        self._h = h
        self.heaps = [BlockHeap(self, l, c) for l, c in enumerate(caps.tolist())]
        self.num_levels = len(self.heaps)

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            N.lib().tsdf_table_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- sizes -----------------------------------------------------------
    def voxel_size(self, level: int) -> float:
        return self.block_edge / voxel_side(level)

    def live_count(self) -> int:
        n = C.c_int64()
        N.check(N.lib().tsdf_live_count(self._h, -1, C.byref(n)), "live_count")
        return int(n.value)

    def fill_fractions(self) -> list:
        return [h.fill_fraction() for h in self.heaps]

    def set_shard(self, rank: int, world: int) -> None:
        """Own only blocks whose key hashes to ``rank`` of ``world`` GPUs."""
        N.check(N.lib().tsdf_table_set_shard(self._h, int(rank), int(world)), "set_shard")

    def set_depth_scale(self, depth_scale: float) -> None:
        """Raw uint16 depth units per metre for the following depth calls
        (z = raw / depth_scale in f64, datasets.py:108-113)."""
        depth_scale = float(depth_scale)
        if getattr(self, "_depth_scale", 1.0) != depth_scale:
            N.check(N.lib().tsdf_table_set_depth_scale(self._h, depth_scale), "set_depth_scale")
            self._depth_scale = depth_scale

    @property
    def version(self) -> int:
        """Bumped by every call that can change the map."""
        out = C.c_uint64()
        N.check(N.lib().tsdf_table_version(self._h, C.byref(out)), "version")
        return int(out.value)

    @property
    def cuda_stream(self) -> int:
        """The cudaStream_t (as an int) every call of this table is ordered on."""
        out = C.c_void_p()
        N.check(N.lib().tsdf_table_stream(self._h, C.byref(out)), "cuda_stream")
        return int(out.value or 0)

    def set_lidar_mode(self, mode: str) -> None:
        """LiDAR hot-block update order: "ordered" (default; bit-identical to
        the reference's ray-order Welford chain) or "chunked" (observations
        folded in 512-ray groups and merged by Chan's formula -- TSDF /
        variance within rounding, exact weights, keys and audited levels;
        include/tsdf_b200.h)."""
        modes = {"ordered": 0, "chunked": 1}
        if mode not in modes:
            raise ValueError(f"lidar mode must be one of {sorted(modes)}")
        N.check(N.lib().tsdf_table_set_lidar_mode(self._h, modes[mode]), "set_lidar_mode")
        self._lidar_mode = mode

    def merge_audit(self) -> int:
        """Level decisions so far within 1e-6 relative of sigma (0: every
        level is robust to the chunked mode's rounding)."""
        out = C.c_int64(0)
        N.check(N.lib().tsdf_table_merge_audit(self._h, C.byref(out)), "merge_audit")
        return int(out.value)

    def reset(self) -> None:
        N.check(N.lib().tsdf_table_reset(self._h), "reset")

    def profile(self, on: bool = True) -> None:
        """Bracket every kernel launch with CUDA events on the table's stream."""
        N.check(N.lib().tsdf_profile_enable(self._h, int(bool(on))), "profile")

    def kernel_times(self, reset: bool = True) -> dict:
        """{kernel: (total ms, launches)} accumulated while profiling."""
        cap, stride = 64, 64
        names = C.create_string_buffer(cap * stride)
        ms = np.zeros(cap)
        cnt = np.zeros(cap, dtype=np.int64)
        n = C.c_int32()
        N.check(N.lib().tsdf_profile_read(self._h, int(reset), cap, names, stride, ms, cnt,
                                          C.byref(n)), "kernel_times")
        raw = names.raw
        out = {}
        for i in range(min(n.value, cap)):
            nm = raw[i * stride:(i + 1) * stride].split(b"\0", 1)[0].decode()
            out[nm] = (float(ms[i]), int(cnt[i]))
        return out

    def work_totals(self, reset: bool = True) -> dict:
        """Diagnostics: frames, touched blocks, near-filter / band-cull survivors
        (blocks, 2x2x2 micro-bricks), voxels screened in FP32 and run on the
        exact FP64 path, LiDAR near pairs, DDA cap sum."""
        out = np.zeros(16, dtype=np.int64)
        N.check(N.lib().tsdf_work_totals(self._h, out, int(bool(reset))), "work_totals")
        return {"frames": int(out[0]), "touched": int(out[1]), "block_pass": int(out[2]),
                "pairs": int(out[3]), "dda_cap_sum": int(out[4]), "near_pass": int(out[6]),
                "micro_pass": int(out[7]), "voxels_screened": int(out[8]),
                "voxels_exact": int(out[9]), "subbrick_pass": int(out[10]),
                "dda_steps": int(out[11])}

    @property
    def slots(self) -> int:
        """Device hash-table slots (the bound on distinct blocks one call can touch)."""
        return int(N.lib().tsdf_table_slots(self._h))

    def probe_stats(self) -> dict:
        """Block-index health: live entries, tombstones left by erased
        blocks, the longest / mean probe sequence of a live key and the
        number of tombstone rebuilds so far."""
        out = np.zeros(4, np.int64)
        mean = C.c_double()
        N.check(N.lib().tsdf_table_probe_stats(self._h, out, C.byref(mean)), "probe_stats")
        return {"live": int(out[0]), "tombstones": int(out[1]), "max_probe": int(out[2]),
                "rehashes": int(out[3]), "mean_probe": float(mean.value)}

    def compact(self) -> None:
        """Rebuild the block index without tombstones (done automatically
        once they pass a quarter of the slots)."""
        N.check(N.lib().tsdf_table_compact(self._h), "compact")

    @property
    def kernel_launches(self) -> int:
        return int(N.lib().tsdf_kernel_launches(self._h))

    # -- core operations ---------------------------------------------------
    def find(self, coord):
        h, l, f = self.find_batch(np.asarray(coord, dtype=np.int64).reshape(1, 3))
        return (int(h[0]), int(l[0])) if f[0] else None

    def insert(self, coord, level: int) -> int:
        out = C.c_int64()
        N.check(N.lib().tsdf_insert(self._h, np.asarray(coord, dtype=np.int64).reshape(3),
                                    int(level), C.byref(out)), "insert")
        return int(out.value)

    def _payload_call(self, fn, coord, what):
        # one library call: buffers sized for the finest level, trimmed to
        # the level the call reports (two device round trips, no find first)
        c = np.ascontiguousarray(np.asarray(coord, dtype=np.int64).reshape(3))
        nmax = self.heaps[0].nvox
        t, w, s2 = np.zeros(nmax), np.zeros(nmax), np.zeros(nmax)
        col = np.zeros((nmax, 3), dtype=np.float32)
        lv = C.c_int32()
        try:
            N.check(fn(self._h, c, C.byref(lv), t.ctypes.data, w.ctypes.data, s2.ctypes.data,
                       col.ctypes.data), what)
        except NotFoundError:
            raise NotFoundError(f"block {tuple(int(v) for v in c)} is not live") from None
        n = self.heaps[int(lv.value)].nvox
        return BlockPayload(coord=tuple(int(v) for v in c), level=int(lv.value), tsdf=t[:n].copy(),
                            weight=w[:n].copy(), s2=s2[:n].copy(), color=col[:n].copy())

    def remove(self, coord) -> BlockPayload:
        return self._payload_call(N.lib().tsdf_remove, coord, "remove")

    def payload(self, coord) -> BlockPayload:
        return self._payload_call(N.lib().tsdf_read_block, coord, "payload")

    def write_payload(self, coord, payload: BlockPayload) -> None:
        c = np.asarray(coord, dtype=np.int64).reshape(3)
        t = np.ascontiguousarray(payload.tsdf, dtype=np.float64)
        w = np.ascontiguousarray(payload.weight, dtype=np.float64)
        s2 = np.ascontiguousarray(payload.s2, dtype=np.float64)
        col = np.ascontiguousarray(payload.color, dtype=np.float32)
        N.check(N.lib().tsdf_write_block(self._h, c, t.ctypes.data, w.ctypes.data,
                                         s2.ctypes.data, col.ctypes.data), "write_payload")

    def probe_length(self, coord) -> int:
        """Index slots examined before a find of `coord` resolves (1 = at its
        home slot; diagnostics, hashgrid.py:194-212 -- there the count is of
        bucket and chain entries)."""
        return int(self.probe_lengths([coord])[0])

    def probe_lengths(self, coords) -> np.ndarray:
        c = np.ascontiguousarray(np.asarray(coords, dtype=np.int64).reshape(-1, 3))
        out = np.zeros(len(c), dtype=np.int32)
        if len(c):
            N.check(N.lib().tsdf_probe_length(self._h, c, len(c), out.ctypes.data), "probe_length")
        return out

    # -- batch operations ------------------------------------------------------
    def find_batch(self, coords):
        c = np.ascontiguousarray(np.asarray(coords, dtype=np.int64).reshape(-1, 3))
        n = len(c)
        handles = np.full(n, -1, dtype=np.int64)
        levels = np.zeros(n, dtype=np.int32)
        found = np.zeros(n, dtype=np.uint8)
        if n:
            N.check(N.lib().tsdf_find_batch(self._h, c, n, handles, levels, found), "find_batch")
        return handles, levels.astype(np.int64), found.astype(bool)

    def insert_batch(self, coords, level: int):
        c = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
        handles, levels, found = self.find_batch(c)
        created = ~found
        for j in np.nonzero(created)[0]:
            handles[j] = self.insert(c[j], level)
            levels[j] = level
        return handles, levels, created

    # -- iteration ---------------------------------------------------------
    def export_level(self, level: int):
        """(coords, handles, tsdf, weight, s2, color) of every live block of a
        level in canonical (x, y, z) order."""
        n = C.c_int64()
        N.check(N.lib().tsdf_export_level(self._h, int(level), 0, None, None, None, None, None,
                                          None, C.byref(n)), "export_level")
        nb, nvox = int(n.value), self.heaps[level].nvox
        coords = np.zeros((nb, 3), dtype=np.int64)
        handles = np.zeros(nb, dtype=np.int64)
        t, w, s2 = (np.zeros((nb, nvox)) for _ in range(3))
        col = np.zeros((nb, nvox, 3), dtype=np.float32)
        if nb:
            N.check(N.lib().tsdf_export_level(self._h, int(level), nb, coords.ctypes.data,
                                              handles.ctypes.data, t.ctypes.data, w.ctypes.data,
                                              s2.ctypes.data, col.ctypes.data, C.byref(n)),
                    "export_level")
        return coords, handles, t, w, s2, col

    def live_blocks(self, level: int, sort: bool = True):
        """(coords, handles) of a level's live blocks in canonical (x, y, z)
        order (hashgrid.py:345-354); no voxel payloads are moved."""
        n = C.c_int64()
        N.check(N.lib().tsdf_export_level(self._h, int(level), 0, None, None, None, None, None,
                                          None, C.byref(n)), "live_blocks")
        nb = int(n.value)
        coords = np.zeros((nb, 3), dtype=np.int64)
        handles = np.zeros(nb, dtype=np.int64)
        if nb:
            N.check(N.lib().tsdf_export_level(self._h, int(level), nb, coords.ctypes.data,
                                              handles.ctypes.data, None, None, None, None,
                                              C.byref(n)), "live_blocks")
        return coords, handles

    # -- capacity tier: bulk block transfer ----------------------------------
    def evict(self, level: int, coords):
        """Remove live blocks of one level and return their payloads
        (tsdf, weight, s2 f64 [n, nvox]; color f32 [n, nvox, 3]).  All or
        nothing: NotFoundError if any block is not live at that level."""
        c = np.ascontiguousarray(np.asarray(coords, dtype=np.int64).reshape(-1, 3))
        n, nvox = len(c), self.heaps[level].nvox
        t, w, s2 = (np.zeros((n, nvox)) for _ in range(3))
        col = np.zeros((n, nvox, 3), dtype=np.float32)
        if n:
            N.check(N.lib().tsdf_evict_level(self._h, int(level), c, n, t.ctypes.data,
                                             w.ctypes.data, s2.ctypes.data, col.ctypes.data),
                    "evict")
        return t, w, s2, col

    def read_blocks(self, level: int, keys):
        """Payloads (tsdf, weight, s2 f64 [n, nvox]; color f32 [n, nvox, 3])
        of live blocks of one level given as packed keys; the table is
        unchanged (NotFoundError if one is not live at that level)."""
        k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64).reshape(-1))
        n, nvox = len(k), self.heaps[level].nvox
        t, w, s2 = (np.zeros((n, nvox)) for _ in range(3))
        col = np.zeros((n, nvox, 3), dtype=np.float32)
        if n:
            N.check(N.lib().tsdf_read_level_blocks(self._h, int(level), k.ctypes.data, n, t.ctypes.data,
                                                   w.ctypes.data, s2.ctypes.data, col.ctypes.data),
                    "read_blocks")
        return t, w, s2, col

    def import_blocks(self, level: int, coords, tsdf, weight, s2, color) -> None:
        """Insert blocks at `level` with their payloads (the inverse of
        evict).  All or nothing: ValueError if one is already live,
        CapacityError on heap / bucket-chain exhaustion."""
        c = np.ascontiguousarray(np.asarray(coords, dtype=np.int64).reshape(-1, 3))
        n, nvox = len(c), self.heaps[level].nvox
        if n == 0:
            return
        t = np.ascontiguousarray(np.asarray(tsdf, dtype=np.float64).reshape(n, nvox))
        w = np.ascontiguousarray(np.asarray(weight, dtype=np.float64).reshape(n, nvox))
        s = np.ascontiguousarray(np.asarray(s2, dtype=np.float64).reshape(n, nvox))
        col = np.ascontiguousarray(np.asarray(color, dtype=np.float32).reshape(n, nvox, 3))
        N.check(N.lib().tsdf_import_level(self._h, int(level), c, n, t.ctypes.data, w.ctypes.data,
                                          s.ctypes.data, col.ctypes.data), "import_blocks")

    def key_levels(self) -> dict:
        """{coord: level} of every live block (the parity key set)."""
        out = {}
        for l in range(self.num_levels):
            for c in map(tuple, self.live_blocks(l)[0].tolist()):
                out[c] = l
        return out
