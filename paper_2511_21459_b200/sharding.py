"""Block-key-hash sharding across the GPUs of one node.

owner(key) = (splitmix64(packed key) >> 32) mod G, decorrelated from the
table's slot hash.  Every rank receives the whole frame (NCCL broadcast over
NVLink from rank 0) and allocates / updates only the blocks it owns; merges
are rank-local (a block's merge depends only on its own voxels), so the union
over ranks equals the single-GPU table bit-for-bit.  Counters that partition
by block are summed with one all-reduce; per-frame counters (measurements,
skipped) are rank-invariant.

Depth frames use ray-sharded allocation: rank r walks 1/G of the rays
(integrate_depth_walk), the per-owner key buckets go through one
all-to-all, and each rank inserts and updates the keys it owns
(integrate_depth_keys) -- the full-ray DDA is split G ways instead of
replicated.  LiDAR scans walk every ray on every rank and keep the blocks
they own (the (block, ray) pairs would need the ray data exchanged too).
"""
from __future__ import annotations

import numpy as np

_BIAS = 1 << 20
_M = (1 << 64) - 1


def pack_keys(coords) -> np.ndarray:
    """21 bits per axis, the device layout (csrc/tsdf_common.cuh pack_key)."""
    c = np.asarray(coords, dtype=np.int64).reshape(-1, 3) + _BIAS
    return ((c[:, 0].astype(np.uint64) << np.uint64(42)) | (c[:, 1].astype(np.uint64) << np.uint64(21))
            | c[:, 2].astype(np.uint64))


def owner_of_keys(keys, world: int) -> np.ndarray:
    """Host mirror of the device owner_of()."""
    with np.errstate(over="ignore"):
        z = np.asarray(keys, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    return ((z >> np.uint64(32)) % np.uint64(world)).astype(np.int64)


def owner_of_coords(coords, world: int) -> np.ndarray:
    return owner_of_keys(pack_keys(coords), world)


PARTITIONED = ("blocks_allocated", "blocks_touched", "voxels_updated", "observations")
INVARIANT = ("measurements", "skipped_invalid")


class ShardedFusion:
    """One process per GPU; wraps a FusionEngine whose table owns one shard."""

    def __init__(self, config, group=None, device=None):
        import torch
        import torch.distributed as dist
        from .pipeline import FusionEngine
        self.dist, self.torch, self.group = dist, torch, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device
        self.engine = FusionEngine(config, shard=(self.rank, self.world) if self.world > 1 else None)

    def broadcast_frame(self, frame):
        """Rank 0's frame -> every rank (device tensors over NCCL)."""
        return broadcast_frame(frame, self.dist, self.torch, self.group, self.device)

    def integrate_frame(self, frame):
        from .geometry import DepthFrame
        f = self.broadcast_frame(frame) if self.world > 1 else frame
        if self.world > 1 and isinstance(f, DepthFrame):
            cfg = self.engine.config
            st = integrate_depth_raysharded(self.engine.table, f, cfg.tau, self.dist, self.torch,
                                            self.group, self.device, cfg.weight_cap)
            self.engine.frame_index += 1
            return st
        st = self.engine.integrate_frame(f)
        return combine_stats(st, self.dist, self.torch, self.group, self.device)

    def integrate_window(self, frames, merge: bool = True):
        """A merge window of depth frames (rank 0's frames; every rank passes
        a list of the same length) through the ray-sharded window protocol:
        the frames, then (merge) the merge pass, with three collectives and
        one host synchronisation per window.  Returns (per-frame stats,
        merged blocks), summed over ranks."""
        frames = [self.broadcast_frame(f) if self.world > 1 else f for f in frames]
        cfg = self.engine.config
        st, ms = integrate_depth_window_sharded(
            self.engine.table, frames, cfg.tau, self.dist, self.torch, self.group, self.device,
            sigma_threshold=cfg.sigma_threshold if merge else 0.0,
            min_eligible_fraction=cfg.merge_min_eligible_fraction,
            min_mean_weight=cfg.merge_min_mean_weight, all_levels=cfg.merge_all_levels,
            weight_cap=cfg.weight_cap)
        self.engine.frame_index += len(frames)
        return st, ms.merged

    def extract(self, iso: float = 0.0, dst: int = 0):
        """FusionEngine.extract over the whole map: the mesh on rank `dst`
        (None elsewhere)."""
        if self.world == 1:
            return self.engine.extract(iso=iso)
        cfg = self.engine.config
        return extract_mesh_halo(self.engine.table, self.dist, self.torch, self.group,
                                 self.device, iso, cfg.collapse_epsilon_factor * cfg.nu_fine, dst)

    def maybe_merge(self):
        n = self.engine.maybe_merge()
        t = self.torch.tensor([n], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())


_DTYPES = ("<f8", "<f4", "|u1", "<u2")


class _DeviceView:
    """A received device array: the broadcast byte tensor seen with the
    sender's element type and shape (through __cuda_array_interface__, so
    the kernels read it in place)."""

    def __init__(self, raw, typestr, shape):
        self._raw = raw
        self.shape = tuple(shape)
        self.__cuda_array_interface__ = {"data": (raw.data_ptr(), False), "shape": self.shape,
                                         "typestr": typestr, "strides": None, "version": 2}


def _bytes_of(a, torch, device):
    """(uint8 tensor on `device`, typestr, shape) of a host or device array."""
    if isinstance(a, torch.Tensor):
        t = a.contiguous()
        typestr = np.dtype(str(t.dtype).replace("torch.", "")).str
        return t.reshape(-1).view(torch.uint8).to(device), typestr, tuple(t.shape)
    cai = getattr(a, "__cuda_array_interface__", None)
    if cai is not None:
        t = torch.as_tensor(a, device=device).contiguous()
        return t.reshape(-1).view(torch.uint8), np.dtype(cai["typestr"]).str, tuple(cai["shape"])
    h = np.ascontiguousarray(a)
    return torch.from_numpy(h.reshape(-1).view(np.uint8)).to(device), h.dtype.str, h.shape


def stream_ready(t, torch):
    """Make a tensor a collective just wrote safe to hand to the library.
    NCCL collectives only order torch's current stream; the library runs on
    its own stream, so the host waits for torch's stream before passing the
    buffer on (tsdf_b200.h: TSDF_MEM_DEVICE buffers must be ready at the
    call)."""
    if t is not None and getattr(t, "is_cuda", False):
        torch.cuda.current_stream(t.device).synchronize()
    return t


def _bcast_array(a, rank, dist, torch, group, device):
    """Broadcast one array from rank 0 bit-for-bit in its own element type
    (f64 / f32 / u8 / u16): a header of (type, rank, shape), then the bytes."""
    head = torch.zeros(5, dtype=torch.int64, device=device)
    raw = None
    if rank == 0:
        raw, typestr, shape = _bytes_of(a, torch, device)
        if typestr not in _DTYPES:
            raise ValueError(f"cannot broadcast arrays of type {typestr}")
        head.copy_(torch.tensor([_DTYPES.index(typestr), len(shape)] + list(shape)
                                + [0] * (3 - len(shape)), dtype=torch.int64))
    dist.broadcast(head, 0, group=group)
    code, nd, *dims = (int(x) for x in head.tolist())
    shape, typestr = tuple(dims[:nd]), _DTYPES[code]
    if rank != 0:
        raw = torch.empty(int(np.prod(shape)) * np.dtype(typestr).itemsize, dtype=torch.uint8,
                          device=device)
    dist.broadcast(raw, 0, group=group)
    if raw.is_cuda:
        return _DeviceView(stream_ready(raw, torch), typestr, shape)
    return raw.numpy().view(np.dtype(typestr)).reshape(shape)


def broadcast_frame(frame, dist, torch, group=None, device=None):
    """Rank 0's frame on every rank: pose, intrinsics and depth scale, then
    the depth (or points) and colour arrays in their own element types, so
    every rank fuses exactly the values rank 0 was given."""
    from .geometry import DepthFrame, Intrinsics, PointCloudFrame, SensorPose
    rank = dist.get_rank(group)
    flags = torch.zeros(2, dtype=torch.int64, device=device)
    meta = torch.zeros(17, dtype=torch.float64, device=device)
    if rank == 0:
        is_depth = isinstance(frame, DepthFrame)
        col = frame.color if is_depth else frame.colors
        flags.copy_(torch.tensor([int(is_depth), int(col is not None)], dtype=torch.int64))
        k = frame.intrinsics.as_array() if is_depth else np.zeros(4)
        scale = frame.depth_scale if is_depth else 1.0
        meta.copy_(torch.from_numpy(np.concatenate([frame.pose.rotation.reshape(9),
                                                    frame.pose.translation, k, [scale]])))
    dist.broadcast(flags, 0, group=group)
    dist.broadcast(meta, 0, group=group)
    is_depth, has_col = (bool(x) for x in flags.tolist())
    data = (frame.depth if is_depth else frame.points) if rank == 0 else None
    arr = _bcast_array(data, rank, dist, torch, group, device)
    carr = None
    if has_col:
        carr = _bcast_array((frame.color if is_depth else frame.colors) if rank == 0 else None,
                            rank, dist, torch, group, device)
    m = meta.cpu().numpy()
    pose = SensorPose(m[:9].reshape(3, 3), m[9:12])
    if is_depth:
        return DepthFrame(depth=arr, intrinsics=Intrinsics(*m[12:16]), pose=pose, color=carr,
                          depth_scale=float(m[16]))
    return PointCloudFrame(points=arr, pose=pose, colors=carr)


def combine_stats(st, dist, torch, group=None, device=None):
    """Sum the block-partitioned counters over ranks (one all-reduce)."""
    from .integrate import IntegrationStats
    host = dist.get_backend(group) == "gloo"
    v = torch.tensor([getattr(st, k) for k in PARTITIONED], dtype=torch.int64,
                     device="cpu" if host else device)
    dist.all_reduce(v, group=group)
    out = IntegrationStats(**{k: getattr(st, k) for k in INVARIANT})
    for k, x in zip(PARTITIONED, v.tolist()):
        setattr(out, k, int(x))
    out.warnings = list(st.warnings)
    return out


def exchange_keys(buckets, counts, dist, torch, group=None, device=None):
    """All-to-all of per-owner key buckets: bucket o of this rank goes to rank
    o; returns the concatenation of every rank's bucket for this rank."""
    world = dist.get_world_size(group)
    # gloo (CPU tests, or several ranks sharing one GPU) exchanges host copies
    host = dist.get_backend(group) == "gloo"
    cdev = "cpu" if host else device
    send_counts = torch.as_tensor(np.asarray(counts, dtype=np.int64), device=cdev)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    sc = [int(x) for x in np.asarray(counts)]
    rc = [int(x) for x in recv_counts.tolist()]
    send = torch.cat([buckets[o, :sc[o]] for o in range(world)])
    out_dev = send.device
    if host:
        send = send.cpu()
    recv = torch.empty(sum(rc), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send, output_split_sizes=rc, input_split_sizes=sc, group=group)
    return stream_ready(recv.to(out_dev), torch)


def integrate_depth_raysharded(table, frame, tau, dist, torch, group=None, device=None,
                               weight_cap: float = 0.0):
    """One depth frame on a block-key-hash shard with the rays split across
    ranks: walk this rank's rays -> all-to-all of the owned keys -> insert,
    commit and update this rank's blocks -> one all-reduce of the
    block-partitioned counters."""
    from .integrate import integrate_depth_keys, integrate_depth_walk
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    buckets = torch.empty((world, table.slots), dtype=torch.int64, device=device)
    st1, counts = integrate_depth_walk(table, frame, tau, rank, world, buckets, weight_cap)
    recv = exchange_keys(buckets, counts, dist, torch, group, device)
    st2 = integrate_depth_keys(table, recv)
    for k in INVARIANT:
        setattr(st2, k, getattr(st1, k))
    st2.warnings = list(st1.warnings)
    return combine_stats(st2, dist, torch, group, device)


# -- mesh extraction over shards ------------------------
#
# Corner sampling reads the 26 lattice neighbours of a block (meshing.py:
# 94-158, 306-310), and with hash ownership nearly every neighbour of a block
# lives on another rank.  Two paths:
#   * extract_mesh_sharded gathers every shard's blocks (bulk level exports,
#     packed in the reference's block-record layout) onto one GPU, which
#     rebuilds the map in a scratch table and extracts it there (simple; the
#     whole map on one device);
#   * extract_mesh_halo (below; what ShardedFusion.extract uses) re-partitions
#     the map spatially: each rank meshes a slab from the slab plus a
#     one-block halo and only the raw output meets on one rank.
# The mesh depends only on map content (never on heap handles), so both are
# bit-identical to extracting the single-GPU table.

def shard_records(table) -> bytes:
    """This shard's live blocks: a header of per-level block counts (u64),
    then the blocks as reference block records, level by level (canonical
    order within a level)."""
    from .formats import pack_records
    counts, out = [], []
    for level in range(table.num_levels):
        coords, _, t, w, s2, col = table.export_level(level)
        counts.append(len(coords))
        if len(coords):
            out.append(pack_records(level, coords, t, w, s2, col).tobytes())
    return np.asarray([table.num_levels] + counts, dtype="<u8").tobytes() + b"".join(out)


def table_from_records(blobs, like):
    """A table with the hash geometry of `like` holding every block of the
    shard_records blobs."""
    from .formats import record_dtype
    from .hashgrid import HashTable
    per_level = {}
    for blob in blobs:
        nl = int(np.frombuffer(blob, "<u8", 1, 0)[0])
        counts = np.frombuffer(blob, "<u8", nl, 8).astype(np.int64)
        off = 8 * (nl + 1)
        for level, n in enumerate(counts.tolist()):
            if n:
                dt = record_dtype(level)
                per_level.setdefault(level, []).append(np.frombuffer(blob, dt, n, off))
                off += n * dt.itemsize
    caps = [max(1, sum(len(r) for r in per_level.get(l, []))) for l in range(like.num_levels)]
    t = HashTable(like.n_hash, like.bucket_capacity, like.overflow_capacity, like.block_edge,
                  heap_capacities=tuple(caps))
    for level, recs in sorted(per_level.items()):
        r = np.concatenate(recs)
        t.import_blocks(level, r["coord"], r["tsdf"], r["weight"], r["s2"], r["color"])
    return t


def _gather_bytes(blob: bytes, dst: int, dist, torch, group=None, device=None):
    """Every rank's byte string on rank `dst` (None elsewhere): lengths,
    then one padded all-gather (NCCL has no variable-size gather)."""
    world = dist.get_world_size(group)
    device = "cpu" if dist.get_backend(group) == "gloo" else device
    n = torch.tensor([len(blob)], dtype=torch.int64, device=device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(1, max(sizes))
    buf = torch.zeros(cap, dtype=torch.uint8, device=device)
    if blob:
        buf[:len(blob)] = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(device)
    parts = [torch.empty(cap, dtype=torch.uint8, device=device) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    if dist.get_rank(group) != dst:
        return None
    return [bytes(p[:s].cpu().numpy().tobytes()) for p, s in zip(parts, sizes)]


def extract_mesh_sharded(table, dist, torch, group=None, device=None, iso: float = 0.0,
                         collapse_epsilon=None, dst: int = 0):
    """extract_mesh over the union of the shards' tables: the Mesh on rank
    `dst`, None on the other ranks."""
    from .meshing import extract_mesh
    blobs = _gather_bytes(shard_records(table), dst, dist, torch, group, device)
    if blobs is None:
        return None
    return extract_mesh(table_from_records(blobs, table), iso=iso, collapse_epsilon=collapse_epsilon)


# ---------------------------------------------------------------------------
# Sharded extraction with a one-block halo (meshing.py:412-487)
# ---------------------------------------------------------------------------
# Hash ownership scatters a block's 26 neighbours over every rank, so meshing
# re-partitions the map spatially instead:
#   1. every rank summarises its live blocks (key, level, observed flag and
#      tsdf range: the inputs of the 27-neighbourhood kept test,
#      meshing.py:428-456) and the summaries are all-gathered (~25 B/block);
#   2. every rank computes the same plan: the global kept list in canonical
#      order (packed keys ascending per level), cut into the reference's
#      256-block chunks (meshing.py:457-459), and a contiguous run of chunks
#      per rank -- an x-major slab of the map -- plus the live 26-neighbours
#      of that run (the halo);
#   3. one all-to-all moves each owner's blocks of every rank's run + halo to
#      that rank as reference block records;
#   4. each rank rebuilds its slab + halo in a scratch table and runs the
#      Marching Cubes passes for its chunks only (raw, pre-dedup output in
#      the reference's emission order);
#   5. the raw outputs are gathered in rank (= emission) order and one rank
#      runs the exact vertex dedup, winding fix and epsilon collapse.
# Chunk runs start on chunk boundaries and every kept block sees the same 26
# neighbours as in the full map, so the concatenated raw output equals the
# single-GPU one and the mesh is bit-identical.

_NBR = np.array([(i // 9 - 1, (i // 3) % 3 - 1, i % 3 - 1) for i in range(27)], dtype=np.int64)


def unpack_keys(keys) -> np.ndarray:
    k = np.asarray(keys, dtype=np.uint64)
    m = np.uint64((1 << 21) - 1)
    return np.stack([(k >> np.uint64(42)) & m, (k >> np.uint64(21)) & m, k & m], axis=1).astype(np.int64) - _BIAS


class _BlockIndex:
    """coordinate -> index into a sorted key array: a dense grid over the
    blocks' bounding box (plus a one-block margin) when it is small enough,
    else binary search on the packed keys."""

    def __init__(self, sorted_keys):
        self.keys = sorted_keys
        self.grid = None
        if len(sorted_keys):
            c = unpack_keys(sorted_keys)
            self.lo = c.min(axis=0) - 1
            ext = c.max(axis=0) + 2 - self.lo
            if int(np.prod(ext)) <= 64 << 20:
                self.ext = ext
                self.grid = np.full(tuple(ext.tolist()), -1, dtype=np.int64)
                g = c - self.lo
                self.grid[g[:, 0], g[:, 1], g[:, 2]] = np.arange(len(c))

    def __call__(self, coords):
        c = np.asarray(coords, dtype=np.int64)
        if len(self.keys) == 0:
            return np.full(len(c), -1, dtype=np.int64)
        if self.grid is not None:
            g = c - self.lo
            ok = np.all((g >= 0) & (g < self.ext), axis=1)
            g = np.where(ok[:, None], g, 0)
            return np.where(ok, self.grid[g[:, 0], g[:, 1], g[:, 2]], -1)
        ok = np.all((c >= -_BIAS) & (c < _BIAS), axis=1)
        k = pack_keys(np.where(ok[:, None], c, 0))
        i = np.minimum(np.searchsorted(self.keys, k), len(self.keys) - 1)
        return np.where(ok & (self.keys[i] == k), i, -1)


def mesh_plan(summaries, world: int, iso: float = 0.0, n_levels: int = 2) -> dict:
    """The extraction plan every rank derives from the all-gathered block
    summaries: canonical kept list per level, each rank's run of whole
    256-block chunks ('emit': keys + per-level counts) and the blocks each
    rank needs (its run + live 26-neighbours, 'need': sorted packed keys)."""
    keys = np.concatenate([s["keys"] for s in summaries]).astype(np.uint64)
    levels = np.concatenate([s["levels"] for s in summaries]).astype(np.int32)
    obs = np.concatenate([s["obs"] for s in summaries]).astype(bool)
    lo = np.concatenate([s["lo"] for s in summaries])
    hi = np.concatenate([s["hi"] for s in summaries])
    order = np.argsort(keys, kind="stable")
    keys, levels, obs, lo, hi = keys[order], levels[order], obs[order], lo[order], hi[order]
    coords = unpack_keys(keys)
    lookup = _BlockIndex(keys)
    # every block's 27 neighbours (indices into keys, -1 absent), once; on
    # the dense grid (one-block margin) no bounds checks are needed
    if lookup.grid is not None and len(keys):
        g = coords - lookup.lo
        nbr = np.stack([lookup.grid[g[:, 0] + d[0], g[:, 1] + d[1], g[:, 2] + d[2]] for d in _NBR])
    else:
        nbr = np.stack([lookup(coords + d) for d in _NBR]) if len(keys) else np.zeros((27, 0), np.int64)
    # 27-neighbourhood straddle test (meshing.py:440-456; k_keep)
    use = (nbr >= 0) & obs[np.maximum(nbr, 0)]
    nlo = np.where(use, lo[np.maximum(nbr, 0)], np.inf).min(axis=0)
    nhi = np.where(use, hi[np.maximum(nbr, 0)], -np.inf).max(axis=0)
    kept = obs & (nlo <= iso) & (iso <= nhi)
    per_level = [np.nonzero(kept & (levels == l))[0] for l in range(n_levels)]  # indices, canonical
    # chunks of 256 per level, levels concatenated; contiguous runs per rank
    chunks = []  # (level, start, stop)
    for l, kl in enumerate(per_level):
        chunks += [(l, s0, min(s0 + 256, len(kl))) for s0 in range(0, len(kl), 256)]
    total = sum(len(k) for k in per_level)
    bounds, acc, r = [0], 0, 1
    for ci, (l, a, b) in enumerate(chunks):
        acc += b - a
        if r < world and acc >= total * r / world:
            bounds.append(ci + 1)
            r += 1
    bounds += [len(chunks)] * (world + 1 - len(bounds))
    emit, need = [], []
    for rk in range(world):
        parts = [[] for _ in range(n_levels)]
        for l, a, b in chunks[bounds[rk]:bounds[rk + 1]]:
            parts[l].append(per_level[l][a:b])
        idx = [np.concatenate(p) if p else np.zeros(0, np.int64) for p in parts]
        allidx = np.concatenate(idx)
        emit.append({"keys": keys[allidx], "level_counts": [len(x) for x in idx]})
        j = nbr[:, allidx].ravel()
        need.append(keys[np.unique(j[j >= 0])])
    return {"emit": emit, "need": need, "kept": int(total), "chunks": len(chunks), "bounds": bounds}


def _records_for(table, keys, levels) -> bytes:
    """shard_records restricted to the given packed keys (with their levels):
    one device gather per level, the table unchanged."""
    from .formats import pack_records
    counts, out = [], []
    keys = np.asarray(keys, dtype=np.uint64)
    levels = np.asarray(levels)
    for level in range(table.num_levels):
        k = np.sort(keys[levels == level])
        counts.append(len(k))
        if len(k):
            t, w, s2, col = table.read_blocks(level, k)
            out.append(pack_records(level, unpack_keys(k), t, w, s2, col).tobytes())
    return np.asarray([table.num_levels] + counts, dtype="<u8").tobytes() + b"".join(out)


def _owned_need(summary, need):
    """(keys, levels) of this rank's blocks among `need` (sorted packed keys)."""
    k = np.asarray(summary["keys"], dtype=np.uint64)
    sel = np.isin(k, need)
    return k[sel], np.asarray(summary["levels"])[sel]


def _raw_bytes(m) -> bytes:
    hdr = np.asarray([m.num_vertices, m.num_triangles], dtype="<i8").tobytes()
    if not m.num_triangles:
        return np.asarray([0, 0], dtype="<i8").tobytes()
    return hdr + b"".join(np.ascontiguousarray(a).tobytes()
                          for a in (m.vertices, m.normals, m.colors, m.triangles))


def _raw_from_bytes(b: bytes):
    from .meshing import Mesh
    nv, nt = (int(x) for x in np.frombuffer(b, "<i8", 2, 0))
    if nt == 0:
        return Mesh.empty()
    off = 16
    arrs = []
    for n, dt in ((nv, np.float64), (nv, np.float64), (nv, np.float64), (nt, np.int64)):
        arrs.append(np.frombuffer(b, dt, 3 * n, off).reshape(n, 3))
        off += 24 * n
    return Mesh(vertices=arrs[0], normals=arrs[1], colors=arrs[2], triangles=arrs[3])


def _mesh_slab(table, plan, rank, blobs, iso):
    """Step 4 on one rank: its slab + halo in a scratch table, raw emission."""
    from .meshing import emit_raw
    e = plan["emit"][rank]
    if not len(e["keys"]):
        return _raw_bytes(type("M", (), {"num_triangles": 0})())
    scratch = table_from_records(blobs, table)
    try:
        return _raw_bytes(emit_raw(scratch, e["keys"], e["level_counts"], iso))
    finally:
        scratch.close()


def _comm_device(dist, group, device):
    """Where byte payloads travel: host tensors on gloo (CPU tests, ranks
    sharing one GPU), the rank's device on NCCL."""
    return "cpu" if dist.get_backend(group) == "gloo" else device


def _all_gather_bytes(blob: bytes, dist, torch, group=None, device=None):
    world = dist.get_world_size(group)
    device = _comm_device(dist, group, device)
    n = torch.tensor([len(blob)], dtype=torch.int64, device=device)
    sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    cap = max(1, max(sizes))
    buf = torch.zeros(cap, dtype=torch.uint8, device=device)
    if blob:
        buf[:len(blob)] = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(device)
    parts = [torch.empty(cap, dtype=torch.uint8, device=device) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return [bytes(p[:s].cpu().numpy().tobytes()) for p, s in zip(parts, sizes)]


def all_to_all_bytes(blobs, dist, torch, group=None, device=None):
    """blobs[d] goes to rank d; returns what every rank sent here (by source)."""
    world = dist.get_world_size(group)
    device = _comm_device(dist, group, device)
    send = torch.tensor([len(b) for b in blobs], dtype=torch.int64, device=device)
    recv = torch.empty(world, dtype=torch.int64, device=device)
    dist.all_to_all_single(recv, send, group=group)
    rs = [int(x) for x in recv.cpu().tolist()]
    out_t = torch.empty(max(1, sum(rs)), dtype=torch.uint8, device=device)
    flat = b"".join(blobs)
    in_t = torch.zeros(max(1, len(flat)), dtype=torch.uint8, device=device)
    if flat:
        in_t[:len(flat)] = torch.frombuffer(bytearray(flat), dtype=torch.uint8).to(device)
    dist.all_to_all_single(out_t[:sum(rs)] if sum(rs) else out_t[:0], in_t[:len(flat)] if flat else in_t[:0],
                           output_split_sizes=rs, input_split_sizes=[len(b) for b in blobs], group=group)
    host = out_t[:sum(rs)].cpu().numpy().tobytes()
    offs = np.cumsum([0] + rs)
    return [host[offs[i]:offs[i + 1]] for i in range(world)]


def _summary_bytes(s) -> bytes:
    n = len(s["keys"])
    return (np.asarray([n], "<i8").tobytes() + s["keys"].astype("<u8").tobytes()
            + s["levels"].astype("<i4").tobytes() + s["obs"].astype("u1").tobytes()
            + s["lo"].astype("<f8").tobytes() + s["hi"].astype("<f8").tobytes())


def _summary_from_bytes(b: bytes) -> dict:
    n = int(np.frombuffer(b, "<i8", 1, 0)[0])
    off = 8
    out = {}
    for name, dt, sz in (("keys", "<u8", 8), ("levels", "<i4", 4), ("obs", "u1", 1), ("lo", "<f8", 8),
                         ("hi", "<f8", 8)):
        out[name] = np.frombuffer(b, dt, n, off)
        off += sz * n
    return out


def extract_mesh_halo(table, dist, torch, group=None, device=None, iso: float = 0.0,
                      collapse_epsilon=None, dst: int = 0):
    """extract_mesh over the union of the shards with spatially partitioned
    work and a one-block halo (see above): the Mesh on rank `dst`, None
    elsewhere.  Bit-identical to extract_mesh of the single-GPU map."""
    from .meshing import block_summary, finish_raw
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    summ = [_summary_from_bytes(b) for b in
            _all_gather_bytes(_summary_bytes(block_summary(table)), dist, torch, group, device)]
    plan = mesh_plan(summ, world, iso, table.num_levels)
    sends = [_records_for(table, *_owned_need(summ[rank], plan["need"][d])) for d in range(world)]
    blobs = all_to_all_bytes(sends, dist, torch, group, device)
    raw = _mesh_slab(table, plan, rank, blobs, iso)
    raws = _gather_bytes(raw, dst, dist, torch, group, device)
    if raws is None:
        return None
    return finish_raw([_raw_from_bytes(b) for b in raws], table.block_edge, collapse_epsilon)


def extract_mesh_halo_local(tables, iso: float = 0.0, collapse_epsilon=None):
    """The same protocol over shard tables living in one process (every
    collective replaced by list plumbing): the single-GPU test of
    extract_mesh_halo, step for step."""
    from .meshing import block_summary, finish_raw
    world = len(tables)
    summ = [block_summary(t) for t in tables]
    plan = mesh_plan(summ, world, iso, tables[0].num_levels)
    sends = [[_records_for(tables[o], *_owned_need(summ[o], plan["need"][d])) for d in range(world)]
             for o in range(world)]
    raws = [_mesh_slab(tables[r], plan, r, [sends[o][r] for o in range(world)], iso) for r in range(world)]
    return finish_raw([_raw_from_bytes(b) for b in raws], tables[0].block_edge, collapse_epsilon), plan


# ---------------------------------------------------------------------------
# Ray-sharded merge windows (the multi-GPU split of a window of
# pipeline.py:88-137).  Per window of B frames: the pixel passes (span for
# the lock-step cap split by tile) -> all-reduce MAX of B caps -> the walks of
# this rank's rays of all B frames -> one all-to-all of the per-(owner,
# frame) key buckets -> inserts, commits and voxel updates frame by frame ->
# one merge pass -> one all-reduce of the per-frame counters.  The library
# and the collectives are ordered through CUDA events (no host wait) except
# for one small read of the bucket counts per window (sizes the exchange) and
# the final counters.  Frame order per block is unchanged, so the union of
# the shards equals the single-GPU window bit for bit.
# ---------------------------------------------------------------------------

def _torch_waits_for_table(table, torch):
    s = table.cuda_stream
    if s:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.ExternalStream(s))
        torch.cuda.current_stream().wait_event(ev)


def _table_waits_for_torch(table, torch):
    s = table.cuda_stream
    if s:
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        torch.cuda.ExternalStream(s).wait_event(ev)


def _window_cap(table, counts_max: int) -> int:
    return max(4096, -(-int(counts_max * 5 // 4 + 64) // 1024) * 1024)


def integrate_depth_window_sharded(table, frames, tau, dist, torch, group=None, device=None,
                                   sigma_threshold: float = 0.0, min_eligible_fraction: float = 0.05,
                                   min_mean_weight: float = 3.0, all_levels: bool = False,
                                   weight_cap: float = 0.0):
    """One merge window on this rank's shard (see above).  Returns (per-frame
    IntegrationStats summed over ranks, MergeStats summed over ranks)."""
    from .adapt import MergeStats
    from .integrate import (IntegrationStats, depth_window_frames, depth_window_update,
                            depth_window_walk)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    gloo = dist.get_backend(group) == "gloo"
    frames = list(frames)
    B = len(frames)
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    caps = torch.zeros(B, dtype=torch.int64, device=dev)
    depth_window_frames(table, frames, tau, rank, world, caps, weight_cap)
    _torch_waits_for_table(table, torch)
    if gloo:
        hc = caps.cpu()
        dist.all_reduce(hc, op=dist.ReduceOp.MAX, group=group)
        caps.copy_(hc)
    else:
        dist.all_reduce(caps, op=dist.ReduceOp.MAX, group=group)
    _table_waits_for_torch(table, torch)
    cap = getattr(table, "_win_cap", 8192)
    for _ in range(3):
        stride = B * (cap + 1)
        exch = torch.zeros(world * stride, dtype=torch.int64, device=dev)
        depth_window_walk(table, caps, exch, cap)
        _torch_waits_for_table(table, torch)
        # the largest bucket of the window, over every rank (one small read)
        mx = exch.view(world, stride)[:, :B].max().reshape(1)
        mx = mx.cpu() if gloo else mx
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=group)
        need = int(mx.item())
        table._win_cap = _window_cap(table, need)
        if need <= cap:
            break
        cap = table._win_cap  # re-walk with room (the walk changes nothing)
        table._win_rewalks = getattr(table, "_win_rewalks", 0) + 1
    if gloo:
        send = exch.cpu()
        recv = torch.empty_like(send)
        dist.all_to_all_single(recv, send, group=group)
        recv = recv.to(dev)
        torch.cuda.current_stream().synchronize()
    else:
        recv = torch.empty_like(exch)
        dist.all_to_all_single(recv, exch, group=group)
    _table_waits_for_torch(table, torch)
    st, ms = depth_window_update(table, recv, world, cap, B, sigma_threshold, min_eligible_fraction,
                                 min_mean_weight, all_levels)
    v = torch.tensor([[getattr(s, k) for k in PARTITIONED] for s in st] + [[ms.candidates, ms.merged, 0, 0]],
                     dtype=torch.int64, device="cpu" if gloo else dev)
    dist.all_reduce(v, group=group)
    v = v.cpu().tolist()
    out = []
    for s, row in zip(st, v[:B]):
        o = IntegrationStats(**{k: getattr(s, k) for k in INVARIANT})
        for k, x in zip(PARTITIONED, row):
            setattr(o, k, int(x))
        o.warnings = list(s.warnings)
        out.append(o)
    return out, MergeStats(int(v[B][0]), int(v[B][1]))


def integrate_depth_window_local(tables, frames, tau, sigma_threshold: float = 0.0,
                                 all_levels: bool = False, weight_cap: float = 0.0, bucket_cap=None):
    """The same window protocol over shard tables living in one process (the
    collectives replaced by tensor plumbing): the single-GPU test of
    integrate_depth_window_sharded, step for step."""
    import torch
    from .adapt import MergeStats
    from .integrate import (IntegrationStats, depth_window_frames, depth_window_update,
                            depth_window_walk)
    world, B = len(tables), len(frames)
    dev = torch.device("cuda", torch.cuda.current_device())
    caps = [torch.zeros(B, dtype=torch.int64, device=dev) for _ in range(world)]
    for r, t in enumerate(tables):
        depth_window_frames(t, frames, tau, r, world, caps[r], weight_cap)
    torch.cuda.synchronize()
    cap_all = torch.stack(caps).max(0).values.contiguous()
    cap = bucket_cap or 8192
    stride = B * (cap + 1)
    exch = [torch.zeros(world * stride, dtype=torch.int64, device=dev) for _ in range(world)]
    for r, t in enumerate(tables):
        depth_window_walk(t, cap_all, exch[r], cap)
    torch.cuda.synchronize()
    need = max(int(e.view(world, stride)[:, :B].max()) for e in exch)
    recv = [torch.cat([exch[s].view(world, stride)[r] for s in range(world)]).contiguous()
            for r in range(world)]
    res = [depth_window_update(t, recv[r], world, cap, B, sigma_threshold, all_levels=all_levels)
           for r, t in enumerate(tables)]
    out = []
    for i in range(B):
        o = IntegrationStats(**{k: getattr(res[0][0][i], k) for k in INVARIANT})
        for k in PARTITIONED:
            setattr(o, k, sum(getattr(r[0][i], k) for r in res))
        out.append(o)
    return out, MergeStats(sum(r[1].candidates for r in res), sum(r[1].merged for r in res)), need
