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

    def extract(self, iso: float = 0.0, dst: int = 0):
        """FusionEngine.extract over the whole map: the mesh on rank `dst`
        (None elsewhere)."""
        if self.world == 1:
            return self.engine.extract(iso=iso)
        cfg = self.engine.config
        return extract_mesh_sharded(self.engine.table, self.dist, self.torch, self.group,
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
# lives on another rank, so a per-rank halo would be most of the map anyway.
# The shards therefore gather their blocks (bulk level exports, packed in the
# reference's block-record layout) onto one GPU, which rebuilds the map in a
# scratch table and extracts it there.  The mesh depends only on map content
# (never on heap handles), so it is bit-identical to extracting the
# single-GPU table.  A large-room map is ~5 GB: one NVLink all-gather.

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
