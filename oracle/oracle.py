"""ctypes binding of the C oracle (oracle/tsdf_oracle.c).

TEST INFRASTRUCTURE ONLY -- the checker and the CPU baseline, never the
product path.  The API mirrors the reference's table / operator surface
(reference hashgrid.py:139-354, integrate.py:143-342, adapt.py:119-136,
meshing.py:412-552) so parity tests read like the reference's own tests.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

STATUS = {0: None, 3: "DatasetError", 4: "CapacityError", 5: "NotFoundError",
          8: "ValueError", 9: "MemoryError"}


class OracleError(Exception):
    def __init__(self, code, what):
        super().__init__(f"oracle {what}: {STATUS.get(code, code)}")
        self.code = code
        self.kind = STATUS.get(code, str(code))


def build_oracle(force: bool = False) -> Path:
    so = _HERE / "liboracle.so"
    src = _HERE / "tsdf_oracle.c"
    if force or not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE), "liboracle.so"], check=True)
    return so


def oracle_lib():
    global _LIB
    if _LIB is not None:
        return _LIB
    so = _HERE / "liboracle.so"
    if not so.exists():
        build_oracle()
    lib = C.CDLL(str(so))
    vp = C.c_void_p
    lib.ot_create.restype = vp
    lib.ot_create.argtypes = [C.c_int64, C.c_int, C.c_int, C.c_double, C.c_int, _i64p]
    lib.ot_destroy.argtypes = [vp]
    lib.ot_hash_key.restype = C.c_int64
    lib.ot_hash_key.argtypes = [C.c_int64] * 4
    lib.ot_insert.argtypes = [vp, _i64p, C.c_int, C.POINTER(C.c_int64)]
    lib.ot_find.argtypes = [vp, _i64p, C.POINTER(C.c_int64), C.POINTER(C.c_int32)]
    lib.ot_remove.argtypes = [vp, _i64p, C.POINTER(C.c_int32), vp, vp, vp, vp]
    for name, rt in [("ot_heap_tsdf", C.POINTER(C.c_double)), ("ot_heap_weight", C.POINTER(C.c_double)),
                     ("ot_heap_s2", C.POINTER(C.c_double)), ("ot_heap_color", C.POINTER(C.c_float)),
                     ("ot_heap_coords", C.POINTER(C.c_int64)), ("ot_heap_live", C.POINTER(C.c_uint8))]:
        getattr(lib, name).restype = rt
        getattr(lib, name).argtypes = [vp, C.c_int]
    lib.ot_heap_occupied.restype = C.c_int64
    lib.ot_heap_occupied.argtypes = [vp, C.c_int]
    lib.ot_live_blocks.restype = C.c_int64
    lib.ot_live_blocks.argtypes = [vp, C.c_int, C.POINTER(C.POINTER(C.c_int64))]
    lib.ot_free.argtypes = [vp]
    lib.ot_dda_blocks.restype = C.c_int64
    lib.ot_dda_blocks.argtypes = [_f64p, _f64p, C.c_double, vp, C.c_int64]
    lib.ot_dda_blocks_batch.restype = C.c_int64
    lib.ot_dda_blocks_batch.argtypes = [_f64p, _f64p, C.c_int64, C.c_double,
                                        C.POINTER(C.POINTER(C.c_int64))]
    lib.ot_integrate_depth.argtypes = [vp, _f64p, vp, C.c_int, C.c_int, _f64p, _f64p, _f64p,
                                       C.c_double, C.c_double, _i64p]
    lib.ot_integrate_points.argtypes = [vp, _f64p, vp, C.c_int64, _f64p, _f64p,
                                        C.c_double, C.c_double, _i64p]
    lib.ot_allocate_for_measurement.argtypes = [vp, _f64p, _f64p, C.c_double, _i64p, C.c_int64,
                                                C.POINTER(C.c_int64)]
    lib.ot_apply_merges.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_int, _i64p]
    lib.ot_block_stats.restype = C.c_int64
    lib.ot_block_stats.argtypes = [vp, C.c_int, C.c_double, C.POINTER(C.POINTER(C.c_int64)),
                                   C.POINTER(C.POINTER(C.c_double))]
    dpp = C.POINTER(C.POINTER(C.c_double))
    ipp = C.POINTER(C.POINTER(C.c_int64))
    lib.ot_extract_mesh.argtypes = [vp, C.c_double, C.c_double, dpp, dpp, dpp,
                                    C.POINTER(C.c_int64), ipp, C.POINTER(C.c_int64)]
    lib.ot_collapse_vertices.argtypes = [_f64p, _f64p, _f64p, C.c_int64, _i64p, C.c_int64,
                                         C.c_double, dpp, dpp, dpp, C.POINTER(C.c_int64), ipp,
                                         C.POINTER(C.c_int64)]
    _LIB = lib
    return lib


def _check(code, what):
    if code:
        raise OracleError(code, what)


def _take(ptr, n, dtype, cols=None):
    lib = oracle_lib()
    if n == 0 or not ptr:
        arr = np.zeros((0, cols) if cols else 0, dtype=dtype)
    else:
        ct = {np.float64: C.c_double, np.int64: C.c_int64}[dtype]
        count = n * (cols or 1)
        buf = C.cast(ptr, C.POINTER(ct * count)).contents
        arr = np.frombuffer(buf, dtype=dtype).copy()
        if cols:
            arr = arr.reshape(n, cols)
    if ptr:
        lib.ot_free(ptr)
    return arr


STAT_FIELDS = ("measurements", "skipped_invalid", "blocks_allocated", "blocks_touched",
               "voxels_updated", "observations")


def _stats_dict(st):
    d = {k: int(v) for k, v in zip(STAT_FIELDS, st[:6])}
    d["warnings"] = ["frame has no valid depth pixels"] if st[6] else []
    return d


def _rot(pose_R, pose_t):
    return (np.ascontiguousarray(pose_R, dtype=np.float64).reshape(9),
            np.ascontiguousarray(pose_t, dtype=np.float64).reshape(3))


class _HeapView:
    """numpy views onto one oracle heap (reference BlockHeap field names)."""

    def __init__(self, tbl, level, cap):
        lib = oracle_lib()
        self.level = level
        self.side = 8 >> level
        self.nvox = self.side ** 3
        self.capacity = cap
        n = cap * self.nvox
        h = tbl._h
        self.tsdf = np.ctypeslib.as_array(lib.ot_heap_tsdf(h, level), shape=(n,))
        self.weight = np.ctypeslib.as_array(lib.ot_heap_weight(h, level), shape=(n,))
        self.s2 = np.ctypeslib.as_array(lib.ot_heap_s2(h, level), shape=(n,))
        self.color = np.ctypeslib.as_array(lib.ot_heap_color(h, level), shape=(n, 3))
        self.coords = np.ctypeslib.as_array(lib.ot_heap_coords(h, level), shape=(cap, 3))
        self.live = np.ctypeslib.as_array(lib.ot_heap_live(h, level), shape=(cap,)).view(bool)
        self._tbl = tbl

    @property
    def occupied(self):
        return int(oracle_lib().ot_heap_occupied(self._tbl._h, self.level))


class OracleTable:
    """Reference-shaped table backed by the C oracle."""

    def __init__(self, n_hash, bucket_capacity, overflow_capacity, block_edge,
                 heap_capacities=(16384, 8192)):
        lib = oracle_lib()
        caps = np.ascontiguousarray(heap_capacities, dtype=np.int64)
        self._h = lib.ot_create(int(n_hash), int(bucket_capacity), int(overflow_capacity),
                                float(block_edge), len(caps), caps)
        if not self._h:
            raise OracleError(9, "create")
        self.n_hash = int(n_hash)
        self.block_edge = float(block_edge)
        self.num_levels = len(caps)
        self.heaps = [_HeapView(self, l, int(c)) for l, c in enumerate(caps)]

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            oracle_lib().ot_destroy(h)
            self._h = None

    def voxel_size(self, level):
        return self.block_edge / (8 >> level)

    def live_count(self):
        return sum(h.occupied for h in self.heaps)

    def insert(self, coord, level):
        out = C.c_int64()
        _check(oracle_lib().ot_insert(self._h, np.asarray(coord, dtype=np.int64).reshape(3),
                                      int(level), C.byref(out)), "insert")
        return int(out.value)

    def find(self, coord):
        hd, lv = C.c_int64(), C.c_int32()
        rc = oracle_lib().ot_find(self._h, np.asarray(coord, dtype=np.int64).reshape(3),
                                  C.byref(hd), C.byref(lv))
        return None if rc else (int(hd.value), int(lv.value))

    def remove(self, coord):
        lv = C.c_int32()
        _check(oracle_lib().ot_remove(self._h, np.asarray(coord, dtype=np.int64).reshape(3),
                                      C.byref(lv), None, None, None, None), "remove")
        return int(lv.value)

    def live_blocks(self, level):
        p = C.POINTER(C.c_int64)()
        n = oracle_lib().ot_live_blocks(self._h, level, C.byref(p))
        rows = _take(p, n, np.int64, 4)
        return rows[:, :3].copy(), rows[:, 3].copy()

    def key_levels(self):
        """{coord: level} over all live blocks (the parity key set)."""
        out = {}
        for l in range(self.num_levels):
            coords, _ = self.live_blocks(l)
            for c in map(tuple, coords.tolist()):
                out[c] = l
        return out

    def block_arrays(self, level):
        """(coords sorted, tsdf, weight, s2, color) per live block of a level."""
        coords, handles = self.live_blocks(level)
        h = self.heaps[level]
        nv = h.nvox
        idx = (handles[:, None] * nv + np.arange(nv)[None, :])
        return (coords, h.tsdf[idx], h.weight[idx], h.s2[idx], h.color[idx])

    # -- operators ----------------------------------------------------------

    def integrate_depth(self, depth, K, R, t, tau, color=None, weight_cap=0.0):
        depth = np.ascontiguousarray(depth, dtype=np.float64)
        H, W = depth.shape
        col = None if color is None else np.ascontiguousarray(color, dtype=np.float64)
        st = np.zeros(8, dtype=np.int64)
        Rf, tf = _rot(R, t)
        rc = oracle_lib().ot_integrate_depth(
            self._h, depth, None if col is None else col.ctypes.data, H, W,
            np.ascontiguousarray(K, dtype=np.float64), Rf, tf, float(tau), float(weight_cap), st)
        _check(rc, "integrate_depth")
        return _stats_dict(st)

    def integrate_points(self, pts, R, t, tau, colors=None, weight_cap=0.0):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        col = None if colors is None else np.ascontiguousarray(colors, dtype=np.float64)
        st = np.zeros(8, dtype=np.int64)
        Rf, tf = _rot(R, t)
        rc = oracle_lib().ot_integrate_points(
            self._h, pts, None if col is None else col.ctypes.data, len(pts), Rf, tf,
            float(tau), float(weight_cap), st)
        _check(rc, "integrate_points")
        return _stats_dict(st)

    def allocate_for_measurement(self, origin, p, tau):
        cap = 1 << 16
        out = np.zeros(cap, dtype=np.int64)
        n = C.c_int64()
        _check(oracle_lib().ot_allocate_for_measurement(
            self._h, np.asarray(origin, dtype=np.float64).reshape(3),
            np.asarray(p, dtype=np.float64).reshape(3), float(tau), out, cap, C.byref(n)),
            "allocate_for_measurement")
        return out[:n.value].tolist()

    def apply_merges(self, sigma, min_frac=0.05, min_w=3.0, all_levels=False):
        st = np.zeros(2, dtype=np.int64)
        _check(oracle_lib().ot_apply_merges(self._h, float(sigma), float(min_frac), float(min_w),
                                            int(bool(all_levels)), st), "apply_merges")
        return {"candidates": int(st[0]), "merged": int(st[1])}

    def block_stats(self, level, min_frac=0.05):
        cp, vp = C.POINTER(C.c_int64)(), C.POINTER(C.c_double)()
        n = oracle_lib().ot_block_stats(self._h, level, float(min_frac), C.byref(cp), C.byref(vp))
        return _take(cp, n, np.int64, 3), _take(vp, n, np.float64, 2)

    def extract_mesh(self, iso=0.0, collapse_epsilon=None):
        eps = 0.25 * self.voxel_size(0) if collapse_epsilon is None else float(collapse_epsilon)
        dp = [C.POINTER(C.c_double)() for _ in range(3)]
        tp = C.POINTER(C.c_int64)()
        nv, nt = C.c_int64(), C.c_int64()
        _check(oracle_lib().ot_extract_mesh(self._h, float(iso), eps, C.byref(dp[0]),
                                            C.byref(dp[1]), C.byref(dp[2]), C.byref(nv),
                                            C.byref(tp), C.byref(nt)), "extract_mesh")
        v = _take(dp[0], nv.value, np.float64, 3)
        n = _take(dp[1], nv.value, np.float64, 3)
        c = _take(dp[2], nv.value, np.float64, 3)
        tr = _take(tp, nt.value, np.int64, 3)
        return v, n, c, tr


def oracle_hash_key(coord, n_hash):
    x, y, z = (int(c) for c in coord)
    return int(oracle_lib().ot_hash_key(x, y, z, int(n_hash)))


def oracle_dda_blocks(origin, endpoint, edge):
    lib = oracle_lib()
    o = np.asarray(origin, dtype=np.float64).reshape(3)
    e = np.asarray(endpoint, dtype=np.float64).reshape(3)
    n = lib.ot_dda_blocks(o, e, float(edge), None, 0)
    buf = np.zeros((n, 3), dtype=np.int64)
    lib.ot_dda_blocks(o, e, float(edge), buf.ctypes.data, n)
    return [tuple(r) for r in buf.tolist()]


def oracle_dda_blocks_batch(origins, endpoints, edge):
    lib = oracle_lib()
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    e = np.ascontiguousarray(endpoints, dtype=np.float64).reshape(-1, 3)
    p = C.POINTER(C.c_int64)()
    n = lib.ot_dda_blocks_batch(o, e, len(o), float(edge), C.byref(p))
    rows = _take(p, n, np.int64, 4)
    return rows[:, 0].copy(), rows[:, 1:].copy()
