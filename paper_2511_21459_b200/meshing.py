"""Mixed-resolution Marching Cubes over the device-resident grid.

``extract_mesh`` keeps the reference signature and output (meshing.py:412-487)
and runs on the GPU (csrc/mesh.cu): observed-range cull over the
27-neighbourhood, cross-level corner blending, transition truncation,
per-cut-edge vertices in the reference's canonical emission order, exact
vertex dedup, winding fix and epsilon collapse.  The result is bit-identical
to the reference (pinned by the reference's golden digests).
``effective_cell_extent`` / ``cell_triangles`` / ``sample_corner`` are the
reference's single-cell helpers, kept for API parity.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .hashgrid import HashTable, voxel_side

HALF_UNITS = 16


@dataclass
class Mesh:
    vertices: np.ndarray
    normals: np.ndarray
    colors: np.ndarray
    triangles: np.ndarray

    @classmethod
    def empty(cls) -> "Mesh":
        return cls(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)),
                   np.zeros((0, 3), dtype=np.int64))

    @property
    def num_vertices(self) -> int:
        return len(self.vertices)

    @property
    def num_triangles(self) -> int:
        return len(self.triangles)


@dataclass
class CornerSample:
    sdf: float
    valid: bool
    source_level: int


def _take(ptr, n, ctype, dtype, cols=3):
    if n == 0:
        return np.zeros((0, cols), dtype=dtype)
    buf = C.cast(ptr, C.POINTER(ctype * (n * cols))).contents
    return np.frombuffer(buf, dtype=dtype).reshape(n, cols).copy()


def _mesh_from_c(m: N.MeshC) -> Mesh:
    try:
        nv, nt = int(m.num_vertices), int(m.num_triangles)
        if nt == 0 and nv == 0:
            return Mesh.empty()
        return Mesh(vertices=_take(m.vertices, nv, C.c_double, np.float64),
                    normals=_take(m.normals, nv, C.c_double, np.float64),
                    colors=_take(m.colors, nv, C.c_double, np.float64),
                    triangles=_take(m.triangles, nt, C.c_int64, np.int64))
    finally:
        N.lib().tsdf_mesh_free(C.byref(m))


def extract_mesh(table: HashTable, iso: float = 0.0, collapse_epsilon=None) -> Mesh:
    """Triangulate the iso-surface of the whole grid (meshing.py:412-487)."""
    eps = -1.0 if collapse_epsilon is None else float(collapse_epsilon)
    if collapse_epsilon is not None and eps < 0:
        raise ValueError("epsilon must be non-negative")
    nv, nt = C.c_int64(), C.c_int64()
    L = N.lib()
    N.check(L.tsdf_extract_mesh_begin(table._h, float(iso), eps, C.byref(nv), C.byref(nt)), "extract_mesh")
    nv, nt = int(nv.value), int(nt.value)
    if nv == 0 and nt == 0:
        return Mesh.empty()
    v, n, c = (np.empty((nv, 3), dtype=np.float64) for _ in range(3))
    tri = np.empty((nt, 3), dtype=np.int64)
    N.check(L.tsdf_extract_mesh_read(table._h, v.ctypes.data, n.ctypes.data, c.ctypes.data,
                                     tri.ctypes.data), "extract_mesh")
    return Mesh(vertices=v, normals=n, colors=c, triangles=tri)


def collapse_vertices(mesh: Mesh, epsilon: float) -> Mesh:
    """Merge vertices by epsilon buckets to their centroid (meshing.py:502-552), on the GPU."""
    if epsilon < 0:
        raise ValueError("epsilon must be non-negative")
    if mesh.num_vertices == 0:
        return mesh
    v = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
    n = np.ascontiguousarray(mesh.normals, dtype=np.float64)
    c = np.ascontiguousarray(mesh.colors, dtype=np.float64)
    t = np.ascontiguousarray(mesh.triangles, dtype=np.int64).reshape(-1, 3)
    m = N.MeshC()
    N.check(N.lib().tsdf_collapse_vertices(v.ctypes.data, n.ctypes.data, c.ctypes.data, len(v),
                                           t.ctypes.data, len(t), C.c_double(float(epsilon)),
                                           C.byref(m)), "collapse_vertices")
    return _mesh_from_c(m)


# ---- staged extraction (sharding.extract_mesh_halo) -------------------------

def block_summary(table: HashTable) -> dict:
    """Every live block of the table: packed key (u64, 21 bits per axis),
    level, observed flag and observed tsdf range -- the inputs of the
    reference's kept-block test (meshing.py:428-456)."""
    cap = max(1, table.live_count())
    out = {"keys": np.empty(cap, np.uint64), "levels": np.empty(cap, np.int32),
           "obs": np.empty(cap, np.uint8), "lo": np.empty(cap, np.float64),
           "hi": np.empty(cap, np.float64)}
    n = C.c_int64()
    N.check(N.lib().tsdf_mesh_block_summary(table._h, out["keys"].ctypes.data, out["levels"].ctypes.data,
                                            out["obs"].ctypes.data, out["lo"].ctypes.data,
                                            out["hi"].ctypes.data, cap, C.byref(n)), "mesh_block_summary")
    return {k: v[:n.value].copy() for k, v in out.items()}


def emit_raw(table: HashTable, keys, level_counts, iso: float = 0.0) -> Mesh:
    """Marching Cubes output before the vertex dedup (lattice-unit positions,
    unnormalised normals, triangles into the raw vertex list) for a kept list
    in canonical order (include/tsdf_b200.h tsdf_mesh_emit_keys)."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    lc = np.zeros(4, dtype=np.int64)
    lc[:len(level_counts)] = level_counts
    m = N.MeshC()
    N.check(N.lib().tsdf_mesh_emit_keys(table._h, k.ctypes.data, lc.ctypes.data, float(iso), C.byref(m)),
            "mesh_emit_keys")
    return _mesh_from_c(m)


def finish_raw(raws, block_edge: float, collapse_epsilon=None) -> Mesh:
    """Concatenate raw emissions (in emission order) and run the exact vertex
    dedup, winding fix and epsilon collapse: the extract_mesh result."""
    raws = [r for r in raws if r.num_triangles]
    if not raws:
        return Mesh.empty()
    offs = np.cumsum([0] + [r.num_vertices for r in raws[:-1]])
    v = np.ascontiguousarray(np.concatenate([r.vertices for r in raws]))
    n = np.ascontiguousarray(np.concatenate([r.normals for r in raws]))
    c = np.ascontiguousarray(np.concatenate([r.colors for r in raws]))
    t = np.ascontiguousarray(np.concatenate([r.triangles + o for r, o in zip(raws, offs)]), dtype=np.int64)
    eps = -1.0 if collapse_epsilon is None else float(collapse_epsilon)
    m = N.MeshC()
    N.check(N.lib().tsdf_mesh_finish(v.ctypes.data, n.ctypes.data, c.ctypes.data, len(v), t.ctypes.data,
                                     len(t), float(block_edge), eps, C.byref(m)), "mesh_finish")
    return _mesh_from_c(m)


def effective_cell_extent(level: int, finer_faces, block_edge: float):
    """Per-axis corner planes (metres, block-local) after transition
    truncation (meshing.py:69-88)."""
    side = voxel_side(level)
    step = HALF_UNITS // side
    out = []
    for axis in range(3):
        h = np.arange(side + 1, dtype=np.float64) * step
        if level > 0:
            if finer_faces[2 * axis]:
                h[0] += step / 2
            if finer_faces[2 * axis + 1]:
                h[-1] -= step / 2
        out.append(h * (block_edge / HALF_UNITS))
    return out[0], out[1], out[2]


def sample_corner(table: HashTable, corner_pos, home_level: int) -> CornerSample:
    """Cross-level blend of the voxels meeting one lattice corner (meshing.py:161-202)."""
    unit = table.block_edge / HALF_UNITS
    h = np.round(np.asarray(corner_pos, dtype=np.float64) / unit).astype(np.int64)
    num = den = 0.0
    best = home_level
    seen = set()
    for sx in (-1, 1):
        for sy in (-1, 1):
            for sz in (-1, 1):
                probe = h + (sx, sy, sz)
                b = probe // HALF_UNITS
                hit = table.find(tuple(b))
                if hit is None:
                    continue
                handle, level = hit
                cs = 2 << level
                side = HALF_UNITS // cs
                v3 = (probe - b * HALF_UNITS) // cs
                vid = int((v3[0] * side + v3[1]) * side + v3[2])
                if (level, handle, vid) in seen:
                    continue
                seen.add((level, handle, vid))
                pl = table.payload(tuple(b))
                if pl.weight[vid] <= 0:
                    continue
                center = b * HALF_UNITS + (v3 + 0.5) * cs
                coeff = float(np.prod(np.maximum(0.0, 1.0 - np.abs(h - center) / cs)))
                w = coeff * (2.0 / cs)
                if w > 0:
                    num += w * pl.tsdf[vid]
                    den += w
                    best = min(best, level)
    if den == 0.0:
        return CornerSample(sdf=0.0, valid=False, source_level=home_level)
    return CornerSample(sdf=num / den, valid=True, source_level=best)


def cell_triangles(corners, corner_positions, iso: float = 0.0) -> list:
    """Triangulate one cell from its 8 corner samples (meshing.py:208-237)."""
    from ._mc_tables import CORNER_PAIRS, EDGE_TABLE, TRI_TABLE
    pos = np.asarray(corner_positions, dtype=np.float64).reshape(8, 3)
    if not all(c.valid for c in corners):
        return []
    vals = np.array([c.sdf for c in corners], dtype=np.float64)
    case = int(sum(1 << i for i in range(8) if vals[i] < iso))
    if EDGE_TABLE[case] == 0:
        return []
    ev = {}
    for e in range(12):
        if EDGE_TABLE[case] & (1 << e):
            a, b = CORNER_PAIRS[e]
            t = (iso - vals[a]) / (vals[b] - vals[a])
            ev[e] = pos[a] + t * (pos[b] - pos[a])
    row = TRI_TABLE[case]
    return [np.stack([ev[int(row[k + j])] for j in range(3)]) for k in range(0, 16, 3) if row[k] >= 0]
