"""Block records and the `.tsdfmap` container (reference formats.py:182-292).

The byte layout is the reference's, so maps written here load in the
reference and vice versa:

* block record: ``<BBqqq`` (archived flag, level, coord x y z), then tsdf,
  weight and s2 as little-endian f64 [nvox] and colour as f32 [nvox, 3];
* map file: header ``<8sIIdddQIIQQQQ`` (magic, version, sensor mode, fine
  voxel size, block edge, tau, n_hash, bucket / overflow capacity, heap
  capacities of levels 0 and 1, live and archived record counts), its CRC-32
  (u32), then the live records (level 0 then 1, canonical coordinate order)
  and the archived records (sorted coordinates).

Records are built and parsed a level at a time through numpy structured
arrays whose packed layout is exactly the record, so saving or loading a map
moves each level's voxels in one bulk device transfer (HashTable.export_level
/ import_blocks) instead of one call per block.
"""
from __future__ import annotations

import struct
import zlib
from pathlib import Path

import numpy as np

from .errors import FormatError
from .hashgrid import BlockPayload, HashTable, voxel_count

MAP_MAGIC = b"TSDFMAP\x00"
MAP_VERSION = 1
_HEAD = struct.Struct("<BBqqq")
_MAP_HEADER = struct.Struct("<8sIIdddQIIQQQQ")
_SENSOR_CODE = {"depth": 0, "pointcloud": 1}


def record_dtype(level: int) -> np.dtype:
    """Packed numpy dtype of one block record of `level` (no padding)."""
    nv = voxel_count(level)
    return np.dtype([("archived", "u1"), ("level", "u1"), ("coord", "<i8", (3,)),
                     ("tsdf", "<f8", (nv,)), ("weight", "<f8", (nv,)), ("s2", "<f8", (nv,)),
                     ("color", "<f4", (nv, 3))], align=False)


def pack_records(level: int, coords, tsdf, weight, s2, color, archived: bool = False) -> np.ndarray:
    """Structured array of n records of one level (its .tobytes() is the
    concatenation of the n reference records)."""
    coords = np.asarray(coords, dtype=np.int64).reshape(-1, 3)
    rec = np.zeros(len(coords), dtype=record_dtype(level))
    rec["archived"] = 1 if archived else 0
    rec["level"] = level
    rec["coord"] = coords
    nv = voxel_count(level)
    rec["tsdf"] = np.asarray(tsdf, dtype=np.float64).reshape(-1, nv)
    rec["weight"] = np.asarray(weight, dtype=np.float64).reshape(-1, nv)
    rec["s2"] = np.asarray(s2, dtype=np.float64).reshape(-1, nv)
    rec["color"] = np.asarray(color, dtype=np.float32).reshape(-1, nv, 3)
    return rec


def pack_block_record(payload: BlockPayload, archived: bool = False) -> bytes:
    """One reference block record (formats.py:185-193)."""
    return pack_records(payload.level, [payload.coord], payload.tsdf, payload.weight, payload.s2,
                        payload.color, archived).tobytes()


def unpack_block_record(buf, offset: int):
    """(payload, archived, next offset) of the record at `offset`."""
    if len(buf) < offset + _HEAD.size:
        raise FormatError("truncated block record")
    _, level = struct.unpack_from("<BB", buf, offset)
    if level > 3:
        raise FormatError(f"block record with level {level}")
    dt = record_dtype(level)
    if len(buf) < offset + dt.itemsize:
        raise FormatError("truncated block record")
    r = np.frombuffer(buf, dtype=dt, count=1, offset=offset)[0]
    payload = BlockPayload(coord=tuple(int(c) for c in r["coord"]), level=int(level),
                           tsdf=r["tsdf"].copy(), weight=r["weight"].copy(), s2=r["s2"].copy(),
                           color=r["color"].copy())
    return payload, bool(r["archived"]), offset + dt.itemsize


def _table_records(table: HashTable):
    out = []
    for level in range(table.num_levels):
        coords, _, t, w, s2, col = table.export_level(level)
        if len(coords):
            out.append(pack_records(level, coords, t, w, s2, col))
    return out


def save_map(table: HashTable, path, archive=None, sensor_mode: str = "depth",
             tau: float = 0.0) -> None:
    """Serialize the live table plus the archive (formats.py:223-253)."""
    caps = [h.capacity for h in table.heaps]
    if table.num_levels > 2 and any(table.heaps[l].occupied for l in range(2, table.num_levels)):
        raise FormatError("the .tsdfmap v1 container holds two resolution levels")
    live = _table_records(table)
    n_live = sum(len(r) for r in live)
    archived = [] if archive is None else [archive.record(c) for c in archive.coords()]
    header = _MAP_HEADER.pack(MAP_MAGIC, MAP_VERSION, _SENSOR_CODE.get(sensor_mode, 0),
                              table.voxel_size(0), table.block_edge, tau, table.n_hash,
                              table.bucket_capacity, table.overflow_capacity, caps[0],
                              caps[1] if len(caps) > 1 else 0, n_live, len(archived))
    with open(Path(path), "wb") as f:
        f.write(header)
        f.write(struct.pack("<I", zlib.crc32(header)))
        for r in live:
            f.write(r.tobytes())
        for rec in archived:
            f.write(rec)


def load_map(path, stream=None):
    """Rebuild (table, archive, info) from a map file (formats.py:256-292).
    A bad magic, an unsupported version or a header whose CRC does not match
    is a FormatError."""
    from .streaming import ArchiveStore
    path = Path(path)
    try:
        blob = path.read_bytes()
    except OSError as exc:
        raise FormatError(f"cannot read map {path}: {exc}") from exc
    if len(blob) < _MAP_HEADER.size + 4:
        raise FormatError(f"{path}: truncated map file")
    (magic, version, sensor_code, nu_fine, block_edge, tau, n_hash, bucket, overflow, cap0, cap1,
     n_live, n_archived) = _MAP_HEADER.unpack_from(blob, 0)
    if magic != MAP_MAGIC:
        raise FormatError(f"{path}: not a map file (bad magic)")
    if version != MAP_VERSION:
        raise FormatError(f"{path}: map version {version} is not supported (supported: {MAP_VERSION})")
    (crc,) = struct.unpack_from("<I", blob, _MAP_HEADER.size)
    if zlib.crc32(blob[:_MAP_HEADER.size]) != crc:
        raise FormatError(f"{path}: header checksum mismatch; file edited or corrupt")
    table = HashTable(n_hash=n_hash, bucket_capacity=bucket, overflow_capacity=overflow,
                      block_edge=block_edge, heap_capacities=(cap0, cap1), stream=stream)
    archive = ArchiveStore()
    off = _MAP_HEADER.size + 4
    pending = {}  # level -> list of structured records, imported in bulk
    for _ in range(n_live + n_archived):
        if len(blob) < off + _HEAD.size:
            raise FormatError(f"{path}: truncated block records")
        flag, level = struct.unpack_from("<BB", blob, off)
        if level > 1:
            raise FormatError(f"{path}: block record with level {level}")
        dt = record_dtype(level)
        if len(blob) < off + dt.itemsize:
            raise FormatError(f"{path}: truncated block records")
        if flag:
            archive.put_record(tuple(int(c) for c in np.frombuffer(blob, "<i8", 3, off + 2)),
                               blob[off:off + dt.itemsize])
        else:
            pending.setdefault(level, []).append(np.frombuffer(blob, dt, 1, off))
        off += dt.itemsize
    for level, recs in pending.items():
        r = np.concatenate(recs)
        table.import_blocks(level, r["coord"], r["tsdf"], r["weight"], r["s2"], r["color"])
    info = {"sensor_mode": {v: k for k, v in _SENSOR_CODE.items()}.get(sensor_code, "depth"),
            "nu_fine": nu_fine, "block_edge": block_edge, "tau": tau}
    return table, archive, info


def read_points(path) -> np.ndarray:
    """Points of a PLY (its vertices) or a whitespace-separated xyz text file
    (formats.py:145-154)."""
    path = Path(path)
    if path.suffix.lower() == ".ply":
        return read_mesh(path).vertices
    try:
        data = np.loadtxt(path, dtype=np.float64, ndmin=2)
    except (OSError, ValueError) as exc:
        raise FormatError(f"cannot read points from {path}: {exc}") from exc
    return data[:, :3]


# -- meshes (binary little-endian PLY, formats.py:33-120) -----------------------

_PLY_VERTEX = np.dtype([("xyz", "<f4", (3,)), ("n", "<f4", (3,)), ("rgb", "u1", (3,))], align=False)
_PLY_FACE = np.dtype([("k", "u1"), ("idx", "<i4", (3,))], align=False)


def write_mesh(mesh, path) -> None:
    """Mesh -> PLY: f32 position and normal, u8 colour (round(c * 255)
    clipped), triangles as u8 count + 3 i32 indices."""
    nv, nt = int(len(mesh.vertices)), int(len(mesh.triangles))
    head = ("ply\nformat binary_little_endian 1.0\n"
            f"element vertex {nv}\n"
            "property float x\nproperty float y\nproperty float z\n"
            "property float nx\nproperty float ny\nproperty float nz\n"
            "property uchar red\nproperty uchar green\nproperty uchar blue\n"
            f"element face {nt}\n"
            "property list uchar int vertex_indices\nend_header\n")
    v = np.zeros(nv, dtype=_PLY_VERTEX)
    v["xyz"] = np.asarray(mesh.vertices, dtype=np.float32)
    v["n"] = np.asarray(mesh.normals, dtype=np.float32)
    v["rgb"] = np.clip(np.round(np.asarray(mesh.colors) * 255.0), 0, 255).astype(np.uint8)
    f = np.zeros(nt, dtype=_PLY_FACE)
    f["k"] = 3
    f["idx"] = np.asarray(mesh.triangles, dtype=np.int32)
    try:
        with open(Path(path), "wb") as fh:
            fh.write(head.encode("ascii"))
            fh.write(v.tobytes())
            fh.write(f.tobytes())
    except OSError as exc:
        raise FormatError(f"cannot write mesh to {path}: {exc}") from exc


def _vertex_layout(props: list) -> np.dtype:
    """Vertex record of the PLYs this package writes: xyz, then optional
    normals, rgb and scale, in that order (formats.py:64-116)."""
    names = {p.split()[-1] for p in props}
    fields = [("xyz", "<f4", (3,))]
    if "nx" in names:
        fields.append(("n", "<f4", (3,)))
    if "red" in names:
        fields.append(("rgb", "u1", (3,)))
    if "scale" in names:
        fields.append(("scale", "<f4"))
    return np.dtype(fields)


def read_mesh(path):
    """A binary little-endian PLY written by write_mesh / write_point_cloud /
    write_seeds -> Mesh (f64 positions; normals 0 and colours 0.5 when the
    file has none; no faces for a point cloud)."""
    from .meshing import Mesh
    try:
        blob = Path(path).read_bytes()
    except OSError as exc:
        raise FormatError(f"cannot read {path}: {exc}") from exc
    end = blob.find(b"end_header\n")
    if not blob.startswith(b"ply") or end < 0:
        raise FormatError(f"{path} is not a PLY file")
    lines = blob[:end].decode("ascii", errors="replace").splitlines()
    if "format binary_little_endian 1.0" not in lines:
        raise FormatError(f"{path}: only binary little-endian PLY is supported")
    counts, props, elem = {}, {}, None
    for line in lines:
        parts = line.split()
        if parts[:1] == ["element"]:
            elem = parts[1]
            counts[elem], props[elem] = int(parts[2]), []
        elif parts[:1] == ["property"] and elem is not None:
            props[elem].append(line)
    body = blob[end + len(b"end_header\n"):]
    vdt = _vertex_layout(props.get("vertex", []))
    nv, nt = counts.get("vertex", 0), counts.get("face", 0)
    if len(body) < nv * vdt.itemsize + nt * _PLY_FACE.itemsize:
        raise FormatError(f"{path}: truncated PLY body")
    v = np.frombuffer(body, dtype=vdt, count=nv)
    tris = np.zeros((0, 3), dtype=np.int64)
    if nt:
        f = np.frombuffer(body, dtype=_PLY_FACE, count=nt, offset=nv * vdt.itemsize)
        if not (f["k"] == 3).all():
            raise FormatError(f"{path}: only triangle faces are supported")
        tris = f["idx"].astype(np.int64)
    names = vdt.names
    normals = v["n"].astype(np.float64) if "n" in names else np.zeros((nv, 3))
    colors = v["rgb"].astype(np.float64) / 255.0 if "rgb" in names else np.full((nv, 3), 0.5)
    return Mesh(vertices=v["xyz"].astype(np.float64), normals=normals, colors=colors,
                triangles=tris)


# -- point clouds and splat seeds (binary little-endian PLY, formats.py:119-180)

def _u8_color(c) -> np.ndarray:
    return np.clip(np.round(np.asarray(c) * 255.0), 0, 255).astype(np.uint8)


def _write_vertex_ply(path, props: str, rec: np.ndarray) -> None:
    head = ("ply\nformat binary_little_endian 1.0\n"
            f"element vertex {len(rec)}\n{props}end_header\n")
    with open(Path(path), "wb") as fh:
        fh.write(head.encode("ascii"))
        fh.write(rec.tobytes())


_XYZ_PROPS = "property float x\nproperty float y\nproperty float z\n"
_RGB_PROPS = "property uchar red\nproperty uchar green\nproperty uchar blue\n"


def write_point_cloud(points, path, colors=None) -> None:
    """Points (and optional colours in [0, 1]) -> PLY vertices: f32 xyz,
    u8 rgb (round(c * 255) clipped)."""
    xyz = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    layout = [("xyz", "<f4", (3,))] + ([("rgb", "u1", (3,))] if colors is not None else [])
    rec = np.zeros(len(xyz), dtype=np.dtype(layout))
    rec["xyz"] = xyz.astype(np.float32)
    if colors is not None:
        rec["rgb"] = _u8_color(colors)
    _write_vertex_ply(path, _XYZ_PROPS + (_RGB_PROPS if colors is not None else ""), rec)


def write_seeds(seeds, path) -> None:
    """Splat seeds (position, colour, scale) -> PLY vertices with a float
    `scale` property after the colour."""
    seeds = list(seeds)
    rec = np.zeros(len(seeds), dtype=np.dtype([("xyz", "<f4", (3,)), ("rgb", "u1", (3,)),
                                               ("scale", "<f4")]))
    if seeds:
        rec["xyz"] = np.array([s.position for s in seeds], dtype=np.float64)
        rec["rgb"] = np.clip(np.round(np.array([np.asarray(s.color, dtype=np.float64)
                                                for s in seeds]) * 255.0), 0, 255)
        rec["scale"] = np.array([s.scale for s in seeds], dtype=np.float64)
    _write_vertex_ply(path, _XYZ_PROPS + _RGB_PROPS + "property float scale\n", rec)
