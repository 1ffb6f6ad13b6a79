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

    def maybe_merge(self):
        n = self.engine.maybe_merge()
        t = self.torch.tensor([n], dtype=self.torch.int64, device=self.device)
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())


def broadcast_frame(frame, dist, torch, group=None, device=None):
    from .geometry import DepthFrame, Intrinsics, PointCloudFrame, SensorPose
    rank = dist.get_rank(group)
    is_depth = torch.tensor([1 if isinstance(frame, DepthFrame) else 0] if rank == 0 else [0],
                            dtype=torch.int64, device=device)
    dist.broadcast(is_depth, 0, group=group)
    data = frame.depth if (rank == 0 and is_depth.item()) else (frame.points if rank == 0 else None)
    meta = torch.zeros(16, dtype=torch.float64, device=device)
    shape = torch.zeros(3, dtype=torch.int64, device=device)
    has_col = torch.zeros(1, dtype=torch.int64, device=device)
    if rank == 0:
        R, t = frame.pose.rotation.reshape(9), frame.pose.translation
        k = frame.intrinsics.as_array() if is_depth.item() else np.zeros(4)
        meta.copy_(torch.from_numpy(np.concatenate([R, t, k])))
        shape.copy_(torch.tensor(list(np.asarray(data).shape) + [0] * (3 - np.asarray(data).ndim)))
        col = frame.color if is_depth.item() else frame.colors
        has_col[0] = 0 if col is None else 1
    for x in (meta, shape, has_col):
        dist.broadcast(x, 0, group=group)
    shp = [int(s) for s in shape.tolist() if s]
    buf = (torch.as_tensor(np.ascontiguousarray(data, dtype=np.float32), device=device) if rank == 0
           else torch.empty(shp, dtype=torch.float32, device=device))
    dist.broadcast(buf, 0, group=group)
    col_t = None
    if has_col.item():
        csh = shp + [3] if is_depth.item() else [shp[0], 3]
        col_t = (torch.as_tensor(np.ascontiguousarray(frame.color if is_depth.item() else frame.colors,
                                                      dtype=np.float32), device=device)
                 if rank == 0 else torch.empty(csh, dtype=torch.float32, device=device))
        dist.broadcast(col_t, 0, group=group)
    m = meta.cpu().numpy()
    pose = SensorPose(m[:9].reshape(3, 3), m[9:12])
    arr = buf if buf.is_cuda else buf.numpy()
    carr = None if col_t is None else (col_t if col_t.is_cuda else col_t.numpy())
    if is_depth.item():
        return DepthFrame(depth=arr, intrinsics=Intrinsics(*m[12:16]), pose=pose, color=carr)
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
    return recv.to(out_dev)


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
