"""Fusion of depth frames and point clouds into the device-resident grid.

``integrate_depth`` / ``integrate_pointcloud`` / ``allocate_for_measurement``
keep the reference signatures (integrate.py:143-342) and run entirely on
the GPU: frame prep, full-ray FP64 DDA with lock-free block allocation,
touched-block compaction and the per-voxel Welford update
(csrc/fusion.cu).  The scalar helpers (``sdf_ray``, ``sdf_projective``,
``update_voxel``, ``Voxel``) are the reference's single-value formulas,
kept for API parity; they are not on the integration path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .geometry import DepthFrame, PointCloudFrame
from .hashgrid import HashTable


@dataclass
class Voxel:
    tsdf: float = 0.0
    weight: float = 0.0
    color: tuple = (0.0, 0.0, 0.0)
    s2: float = 0.0

    def variance(self) -> float:
        return self.s2 / self.weight if self.weight >= 1 else 0.0


@dataclass
class IntegrationStats:
    measurements: int = 0
    skipped_invalid: int = 0
    blocks_allocated: int = 0
    blocks_touched: int = 0
    voxels_updated: int = 0
    observations: int = 0
    warnings: list = field(default_factory=list)


def sdf_ray(p, x, o, tau: float) -> float:
    """Along-ray signed distance of x to surface point p, clipped (integrate.py:53-65)."""
    p, x, o = (np.asarray(v, dtype=np.float64) for v in (p, x, o))
    ray = p - o
    n = np.linalg.norm(ray)
    if n == 0.0:
        raise ValueError("surface point coincides with the sensor origin")
    return float(np.clip(np.dot(p - x, ray / n), -tau, tau))


def sdf_projective(d: float, x, tau: float) -> float:
    """Measured ray distance minus voxel range, clipped (integrate.py:68-71)."""
    return float(np.clip(d - np.linalg.norm(np.asarray(x, dtype=np.float64)), -tau, tau))


def update_voxel(v: Voxel, d_k: float, rgb=None, weight_cap: float = 0.0) -> Voxel:
    """One unit-weight running-mean + Welford step (integrate.py:74-89)."""
    w0 = v.weight
    mean = (w0 * v.tsdf + d_k) / (w0 + 1.0)
    s2 = v.s2 + (d_k - v.tsdf) * (d_k - mean)
    w1 = w0 + 1.0
    if weight_cap > 0.0:
        w1 = min(w1, weight_cap)
    color = v.color
    if rgb is not None:
        color = tuple((w0 * np.asarray(v.color) + np.asarray(rgb)) / (w0 + 1.0))
    return Voxel(tsdf=mean, weight=w1, color=color, s2=s2)


def _has_archive(archive) -> bool:
    return archive is not None and len(archive) != 0


def _stream_in_for(table: HashTable, frame, tau: float, archive) -> None:
    """The archive branch of _ensure_blocks (integrate.py:122-140): archived
    blocks the frame reaches come back, payload intact, before it is fused."""
    if not _has_archive(archive):
        return
    from .streaming import stream_in_keys
    keys = _frame_keys_tau(table, frame, tau)
    stream_in_keys(table, archive, keys)


def _frame_keys_tau(table: HashTable, frame, tau: float) -> np.ndarray:
    """Distinct packed block keys the frame's allocation will touch (the
    reference's np.unique of the DDA rows, integrate.py:203, :289), from a
    key-only pass of the device DDA; the table is not changed."""
    cap = max(1024, 2 * table.slots)
    out = np.zeros(cap, dtype=np.uint64)
    n = C.c_int64()
    R, t = _pose(frame.pose)
    if isinstance(frame, DepthFrame):
        dptr, ddt, dmem, _keep = _depth_buffer(table, frame)
        rc = N.lib().tsdf_depth_keys(table._h, dptr, ddt, frame.height, frame.width, dmem,
                                     frame.intrinsics.as_array(), R, t, float(tau),
                                     out.ctypes.data, cap, C.byref(n))
    else:
        pptr, pdt, pmem, _keep = N.as_buffer(frame.points, (N.F64, N.F32))
        rc = N.lib().tsdf_scan_keys(table._h, pptr, pdt, int(frame.points.shape[0]), pmem, R, t,
                                    float(tau), out.ctypes.data, cap, C.byref(n))
    N.check(rc, "frame_keys")
    return out[:n.value]


def _depth_buffer(table: HashTable, frame, scale=None):
    """as_buffer of the frame's depth.  Raw uint16 depth is scaled on the
    device (z = raw / depth_scale in f64, datasets.py:108-113): the table's
    depth scale is set to the frame's before the call."""
    p, dt, m, k = N.as_buffer(frame.depth, (N.F64, N.F32, N.U16))
    if dt == N.U16:
        if scale is not None and frame.depth_scale != scale:
            raise ValueError("frames of one window must share depth_scale")
        table.set_depth_scale(frame.depth_scale)
    return p, dt, m, k


def _stats(st) -> IntegrationStats:
    out = IntegrationStats(st.measurements, st.skipped_invalid, st.blocks_allocated,
                           st.blocks_touched, st.voxels_updated, st.observations)
    if st.no_valid_warning:
        out.warnings.append("frame has no valid depth pixels")
    return out


def _pose(pose):
    return (np.ascontiguousarray(pose.rotation, dtype=np.float64).reshape(9),
            np.ascontiguousarray(pose.translation, dtype=np.float64).reshape(3))


def integrate_depth(table: HashTable, frame: DepthFrame, tau: float, archive=None,
                    weight_cap: float = 0.0) -> IntegrationStats:
    """Projective fusion of one depth image (integrate.py:255-342).  With a
    non-empty `archive` (streaming.ArchiveStore), archived blocks the frame
    reaches are streamed back in first."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    _stream_in_for(table, frame, tau, archive)
    dptr, ddt, dmem, _keep_d = _depth_buffer(table, frame)
    cptr, cdt, cmem, _keep_c = (None, 0, dmem, None)
    if frame.color is not None:
        cptr, cdt, cmem, _keep_c = N.as_buffer(frame.color, (N.F64, N.F32, N.U8))
        if cmem != dmem:
            raise ValueError("depth and colour must both live on the host or both on the device")
    R, t = _pose(frame.pose)
    st = N.IntegrationStatsC()
    N.check(N.lib().tsdf_integrate_depth(table._h, dptr, ddt, cptr, cdt, frame.height,
                                         frame.width, dmem, frame.intrinsics.as_array(), R, t,
                                         float(tau), float(weight_cap), C.byref(st)),
            "integrate_depth")
    return _stats(st)


def integrate_depth_walk(table: HashTable, frame: DepthFrame, tau: float, ray_rank: int,
                         ray_world: int, buckets, weight_cap: float = 0.0):
    """Step 1 of ray-sharded depth integration (multi-GPU).

    Walks this rank's share of the rays (16x16-pixel tiles t with
    t % ray_world == ray_rank) with the reference's full-ray DDA
    (integrate.py:282-290) and writes each block key it meets once into the
    bucket of the shard that owns it.  `buckets` is a CUDA int64 array of
    shape (shard_world, cap).  Returns (stats with the rank-invariant fields,
    per-owner key counts).  The frame must stay alive until
    integrate_depth_keys returns."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    dptr, ddt, dmem, _keep_d = _depth_buffer(table, frame)
    cptr, cdt, cmem, _keep_c = (None, 0, dmem, None)
    if frame.color is not None:
        cptr, cdt, cmem, _keep_c = N.as_buffer(frame.color, (N.F64, N.F32, N.U8))
        if cmem != dmem:
            raise ValueError("depth and colour must both live on the host or both on the device")
    cai = getattr(buckets, "__cuda_array_interface__", None)
    if cai is None or len(cai["shape"]) != 2 or np.dtype(cai["typestr"]).itemsize != 8:
        raise ValueError("buckets must be a 2-D 64-bit CUDA array (shard_world, cap)")
    world, cap = (int(x) for x in cai["shape"])
    counts = np.zeros(max(world, 1), dtype=np.int64)
    R, t = _pose(frame.pose)
    st = N.IntegrationStatsC()
    N.check(N.lib().tsdf_integrate_depth_walk(table._h, dptr, ddt, cptr, cdt, frame.height,
                                              frame.width, dmem, frame.intrinsics.as_array(), R, t,
                                              float(tau), float(weight_cap), int(ray_rank),
                                              int(ray_world), cai["data"][0], cap, counts,
                                              C.byref(st)),
            "integrate_depth_walk")
    return _stats(st), counts[:world]


def integrate_depth_keys(table: HashTable, keys, n: int = None) -> IntegrationStats:
    """Step 2 of ray-sharded depth integration: insert the block keys this
    shard owns (a CUDA int64 array gathered from every rank; duplicates are
    fine), commit the new blocks and run the voxel update of the frame given
    to the preceding integrate_depth_walk.  Returns the block-partitioned
    stats (blocks_allocated, blocks_touched, voxels_updated, observations)."""
    cai = getattr(keys, "__cuda_array_interface__", None)
    if cai is None or np.dtype(cai["typestr"]).itemsize != 8:
        raise ValueError("keys must be a 64-bit CUDA array")
    n = int(np.prod(cai["shape"])) if n is None else int(n)
    st = N.IntegrationStatsC()
    N.check(N.lib().tsdf_integrate_depth_keys(table._h, cai["data"][0] if n else None, n,
                                              C.byref(st)), "integrate_depth_keys")
    return _stats(st)


def integrate_depth_batch(table: HashTable, frames, tau: float, archive=None,
                          weight_cap: float = 0.0) -> list:
    """Fuse a merge window of depth frames with one host synchronisation
    (the same results as integrate_depth per frame).  On an error at frame i
    the later frames are not applied and the error is raised.  All frames
    must share size and dtypes."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    frames = list(frames)
    if not frames:
        return []
    if _has_archive(archive):
        # stream-in depends on the table after the previous frame: per frame
        return [integrate_depth(table, f, tau, archive, weight_cap) for f in frames]
    return _depth_window(table, frames, tau, weight_cap, None)[0]


def integrate_depth_window(table: HashTable, frames, tau: float, sigma_threshold: float,
                           min_eligible_fraction: float = 0.05, min_mean_weight: float = 3.0,
                           all_levels: bool = False, weight_cap: float = 0.0):
    """One merge window of the reference's engine loop (pipeline.py:88-137):
    the frames, then one apply_merges pass, enqueued back to back on the
    device with a single host synchronisation.  Returns (per-frame stats,
    MergeStats).  If a frame fails, the later frames and the merge are not
    applied and the error is raised."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    if not sigma_threshold > 0:
        raise ValueError("sigma_threshold must be positive")
    frames = list(frames)
    if not frames:
        from .adapt import apply_merges
        return [], apply_merges(table, sigma_threshold, min_eligible_fraction, min_mean_weight,
                                all_levels=all_levels)
    st, ms, _ = _depth_window(table, frames, tau, weight_cap,
                              (sigma_threshold, min_eligible_fraction, min_mean_weight, all_levels))
    return st, ms


def _window_args(table, frames):
    """The C-ABI view of a window of depth frames: (keep-alive list, depth
    pointer array, depth dtype, colour pointer array or None, colour dtype,
    memory kind, H, W, K, R, t)."""
    n = len(frames)
    keep, dptrs, cptrs = [], [], []
    ddt = cdt = mem = None
    H, W = frames[0].height, frames[0].width
    scale0 = frames[0].depth_scale
    for f in frames:
        p, dt, m, k = _depth_buffer(table, f, scale0)
        keep.append(k)
        if ddt is None:
            ddt, mem = dt, m
        if dt != ddt or m != mem or tuple(f.depth.shape) != (H, W):
            raise ValueError("integrate_depth_batch: frames must share size, dtype and memory kind")
        dptrs.append(p)
        if f.color is not None:
            cp, ct, cm, ck = N.as_buffer(f.color, (N.F64, N.F32, N.U8))
            keep.append(ck)
            if cdt is None:
                cdt = ct
            if ct != cdt or cm != mem:
                raise ValueError("integrate_depth_batch: colours must share dtype and memory kind")
            cptrs.append(cp)
    if cptrs and len(cptrs) != n:
        raise ValueError("integrate_depth_batch: either every frame has colour or none")
    K = np.array([(f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx, f.intrinsics.cy) for f in frames],
                 dtype=np.float64).reshape(-1)
    R = np.concatenate([f.pose.rotation.reshape(9) for f in frames])  # f64, C-contiguous (SensorPose)
    T = np.concatenate([f.pose.translation for f in frames])
    darr = (C.c_void_p * n)(*dptrs)
    carr = (C.c_void_p * n)(*cptrs) if cptrs else None
    return keep, darr, ddt, carr, cdt or 0, mem, H, W, K, R, T


def _depth_window(table, frames, tau, weight_cap, merge, fill_limit=0.0, partial=False):
    """-> (stats of the frames applied, MergeStats, frames applied); with
    partial=True a failing frame does not raise: its error is returned as a
    fourth element (None if every frame was applied or the fill mark stopped
    the window)."""
    n = len(frames)
    keep, darr, ddt, carr, cdt, mem, H, W, K, R, T = _window_args(table, frames)
    st = (N.IntegrationStatsC * n)()
    done = C.c_int32()
    ms = N.MergeStatsC()
    sig, frac, minw, alll = merge if merge is not None else (0.0, 0.0, 0.0, False)
    rc = N.lib().tsdf_integrate_depth_window(table._h, n, darr, ddt, carr, cdt,
                                             H, W, mem, K, R, T,
                                             float(tau), float(weight_cap), st, C.byref(done),
                                             float(sig), float(frac), float(minw), int(bool(alll)),
                                             float(fill_limit),
                                             C.byref(ms) if merge is not None else None)
    from .adapt import MergeStats
    k = int(done.value)
    if rc and partial:
        # frames before the failing one are applied: report them with the error
        try:
            N.check(rc, "integrate_depth_window")
        except Exception as exc:
            return [_stats(s) for s in st[:k]], MergeStats(), k, exc
    N.check(rc, "integrate_depth_batch" if merge is None else "integrate_depth_window")
    out = [_stats(s) for s in st[:k]], MergeStats(int(ms.candidates), int(ms.merged)), k
    return out + (None,) if partial else out




# ---- ray-sharded merge windows (sharding.integrate_depth_window_sharded) ----

def _cuda_ptr(a, what, n_min=1):
    cai = getattr(a, "__cuda_array_interface__", None)
    if cai is None or np.dtype(cai["typestr"]).itemsize != 8 or int(np.prod(cai["shape"])) < n_min:
        raise ValueError(f"{what} must be a 64-bit CUDA array of at least {n_min} elements")
    return cai["data"][0]


def depth_window_frames(table: HashTable, frames, tau: float, ray_rank: int, ray_world: int, caps,
                        weight_cap: float = 0.0):
    """Window step 1 (include/tsdf_b200.h tsdf_depth_window_frames): the
    frames' pixel passes, this rank's partial lock-step caps into `caps`
    (CUDA u64/i64 [B]).  The frames must stay alive until the update step."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    frames = list(frames)
    keep, darr, ddt, carr, cdt, mem, H, W, K, R, T = _window_args(table, frames)
    table._win_keep = (frames, keep, darr, carr)
    N.check(N.lib().tsdf_depth_window_frames(table._h, len(frames), darr, ddt, carr, cdt, H, W, mem, K, R, T,
                                             float(tau), float(weight_cap), int(ray_rank), int(ray_world),
                                             _cuda_ptr(caps, "caps", len(frames))),
            "depth_window_frames")


def depth_window_walk(table: HashTable, caps, exchange, bucket_cap: int):
    """Window step 2: walk this rank's rays with the all-reduced caps and fill
    the exchange buffer (CUDA 64-bit, shard_world * B * (bucket_cap + 1))."""
    N.check(N.lib().tsdf_depth_window_walk(table._h, _cuda_ptr(caps, "caps"), _cuda_ptr(exchange, "exchange"),
                                           int(bucket_cap)), "depth_window_walk")


def depth_window_update(table: HashTable, received, world: int, bucket_cap: int, n_frames: int,
                        sigma_threshold: float = 0.0, min_eligible_fraction: float = 0.05,
                        min_mean_weight: float = 3.0, all_levels: bool = False):
    """Window step 3: insert / commit / update every frame from the exchanged
    keys, then one merge pass (sigma_threshold > 0).  Returns (this shard's
    per-frame stats, MergeStats)."""
    from .adapt import MergeStats
    st = (N.IntegrationStatsC * n_frames)()
    ms = N.MergeStatsC()
    try:
        N.check(N.lib().tsdf_depth_window_update(table._h, _cuda_ptr(received, "received"), int(world),
                                                 int(bucket_cap), float(sigma_threshold),
                                                 float(min_eligible_fraction), float(min_mean_weight),
                                                 int(bool(all_levels)), st, C.byref(ms)),
                "depth_window_update")
    finally:
        table._win_keep = None
    return [_stats(x) for x in st], MergeStats(int(ms.candidates), int(ms.merged))


def integrate_pointcloud(table: HashTable, frame: PointCloudFrame, tau: float, archive=None,
                         weight_cap: float = 0.0) -> IntegrationStats:
    """Ray-based fusion of one point cloud (integrate.py:175-252); archived
    blocks the scan reaches are streamed back in first."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    n = int(frame.points.shape[0])
    if n == 0:
        return IntegrationStats()
    _stream_in_for(table, frame, tau, archive)
    pptr, pdt, pmem, _keep_p = N.as_buffer(frame.points, (N.F64, N.F32))
    cptr, cdt, _keep_c = None, 0, None
    if frame.colors is not None:
        cptr, cdt, cmem, _keep_c = N.as_buffer(frame.colors, (N.F64, N.F32, N.U8))
        if cmem != pmem:
            raise ValueError("points and colours must both live on the host or both on the device")
    R, t = _pose(frame.pose)
    st = N.IntegrationStatsC()
    N.check(N.lib().tsdf_integrate_points(table._h, pptr, pdt, cptr, cdt, n, pmem, R, t,
                                          float(tau), float(weight_cap), C.byref(st)),
            "integrate_pointcloud")
    return _stats(st)


def allocate_for_measurement(table: HashTable, origin, p, tau: float, archive=None) -> list:
    """Allocate every block the segment origin -> p (+tau) crosses
    (integrate.py:143-161); handles in traversal order."""
    if tau <= 0:
        raise ValueError("tau must be positive")
    o = np.ascontiguousarray(origin, dtype=np.float64).reshape(3)
    q = np.ascontiguousarray(p, dtype=np.float64).reshape(3)
    if _has_archive(archive):
        from .dda import dda_blocks
        from .streaming import _pack, stream_in_keys
        ray = q - o
        n_ = np.linalg.norm(ray)
        if n_ == 0.0:
            raise ValueError("measurement coincides with the sensor origin")
        end = q + tau * ray / n_  # integrate.py:157, same evaluation order
        coords = np.asarray(dda_blocks(o, end, table.block_edge), dtype=np.int64).reshape(-1, 3)
        stream_in_keys(table, archive, np.unique(_pack(coords)))
    cap = 1 << 16
    out = np.zeros(cap, dtype=np.int64)
    n = C.c_int64()
    N.check(N.lib().tsdf_allocate_for_measurement(table._h, o, q, float(tau), out, cap,
                                                  C.byref(n)), "allocate_for_measurement")
    if n.value > cap:
        out = np.zeros(n.value, dtype=np.int64)
        N.check(N.lib().tsdf_allocate_for_measurement(table._h, o, q, float(tau), out, n.value,
                                                      C.byref(n)), "allocate_for_measurement")
    return [int(h) for h in out[:n.value]]
