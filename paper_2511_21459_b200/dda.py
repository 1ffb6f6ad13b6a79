"""Amanatides-Woo traversal of the block grid (reference dda.py:8-86), run
on the device through the same FP64 stepping code the allocation kernel
uses (csrc/fusion.cu: dda_setup / k_trace)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N


def _trace(origins, endpoints, edge, batch):
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    e = np.ascontiguousarray(endpoints, dtype=np.float64).reshape(-1, 3)
    ids = C.POINTER(C.c_int64)()
    co = C.POINTER(C.c_int64)()
    n = C.c_int64()
    L = N.lib()
    N.check(L.tsdf_dda_blocks(o.ctypes.data, e.ctypes.data, C.c_int64(len(o)), C.c_double(edge),
                              C.c_int32(int(batch)), C.byref(ids), C.byref(co), C.byref(n)),
            "dda_blocks")
    rows = int(n.value)
    try:
        if rows == 0:
            return np.zeros(0, dtype=np.int64), np.zeros((0, 3), dtype=np.int64)
        r = np.frombuffer(C.cast(ids, C.POINTER(C.c_int64 * rows)).contents, dtype=np.int64).copy()
        c = np.frombuffer(C.cast(co, C.POINTER(C.c_int64 * (3 * rows))).contents,
                          dtype=np.int64).reshape(rows, 3).copy()
        return r, c
    finally:
        L.tsdf_free(C.cast(ids, C.c_void_p))
        L.tsdf_free(C.cast(co, C.c_void_p))


def dda_blocks(origin, endpoint, block_edge: float) -> list:
    """Blocks the segment [origin, endpoint] crosses, in traversal order."""
    if block_edge <= 0:
        raise ValueError("block_edge must be positive")
    o = np.asarray(origin, dtype=np.float64).reshape(3)
    e = np.asarray(endpoint, dtype=np.float64).reshape(3)
    if not np.any(e - o):
        raise ValueError("origin and endpoint coincide")
    _, c = _trace(o, e, block_edge, batch=False)
    return [tuple(int(v) for v in row) for row in c]


def dda_blocks_batch(origins, endpoints, block_edge: float):
    """Lock-step traversal of many segments: (ray_ids, coords) grouped by ray."""
    if block_edge <= 0:
        raise ValueError("block_edge must be positive")
    return _trace(origins, endpoints, block_edge, batch=True)
