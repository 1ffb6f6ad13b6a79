"""Block-key-hash sharding across the GPUs of one node.

owner(key) = (splitmix64(packed key) >> 32) mod G, decorrelated from the
table's slot hash.  Every rank receives the whole frame (NCCL broadcast over
NVLink from rank 0), traverses all rays, and allocates / updates only the
blocks it owns; merges are rank-local (a block's merge depends only on its
own voxels), so the union over ranks equals the single-GPU table
bit-for-bit.  Counters that partition by block are summed with one
all-reduce; per-frame counters (measurements, skipped) are rank-invariant.
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
        f = self.broadcast_frame(frame) if self.world > 1 else frame
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
    v = torch.tensor([getattr(st, k) for k in PARTITIONED], dtype=torch.int64, device=device)
    dist.all_reduce(v, group=group)
    out = IntegrationStats(**{k: getattr(st, k) for k in INVARIANT})
    for k, x in zip(PARTITIONED, v.tolist()):
        setattr(out, k, int(x))
    out.warnings = list(st.warnings)
    return out
