"""Variance-driven resolution adaptation (reference adapt.py:1-136).

``apply_merges`` runs on the GPU: one warp per live block reproduces
NumPy's pairwise block-variance sum bit-for-bit, so the level decision
equals the reference's; candidates are re-homed one level coarser in place
(2x2x2 pooled downsample, Chan k-way S2).  ``all_levels=True`` enables the
labelled multi-level extension (L -> L+1 for every L < top level).
``block_mean_variance`` / ``downsample_block`` are the reference's
payload-level helpers, kept for API parity.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .hashgrid import BlockPayload, HashTable, voxel_side

MERGE_MIN_ELIGIBLE_FRACTION = 0.05
MERGE_MIN_MEAN_WEIGHT = 3.0


@dataclass
class MergeStats:
    candidates: int = 0
    merged: int = 0


def block_mean_variance(weight, s2, min_eligible_fraction: float = MERGE_MIN_ELIGIBLE_FRACTION) -> float:
    """Mean S2/W over voxels with W >= 2; +inf when too few qualify (adapt.py:26-38)."""
    w = np.asarray(weight, dtype=np.float64).ravel()
    s = np.asarray(s2, dtype=np.float64).ravel()
    ok = w >= 2.0
    if ok.sum() < min_eligible_fraction * w.size:
        return float("inf")
    return float(np.mean(s[ok] / w[ok]))


def downsample_block(fine: BlockPayload) -> BlockPayload:
    """2x2x2 pooled statistics of a block payload one level down (adapt.py:75-116)."""
    if fine.level != 0:
        raise ValueError(f"downsample_block expects a level-0 block, got level {fine.level}")
    s = voxel_side(fine.level)
    h = s // 2

    def children(a):
        tail = a.shape[1:]
        return (a.reshape(h, 2, h, 2, h, 2, *tail).transpose(0, 2, 4, 1, 3, 5, *range(6, 6 + len(tail)))
                .reshape(h ** 3, 8, *tail))

    w = children(np.asarray(fine.weight, dtype=np.float64))
    d = children(np.asarray(fine.tsdf, dtype=np.float64))
    q = children(np.asarray(fine.s2, dtype=np.float64))
    c = children(np.asarray(fine.color, dtype=np.float64))
    wsum = w.sum(axis=1)
    seen = wsum > 0
    den = np.where(seen, wsum, 1.0)
    mean = (w * d).sum(axis=1) / den
    pooled = q.sum(axis=1) + (w * (d - mean[:, None]) ** 2).sum(axis=1)
    col = (w[..., None] * c).sum(axis=1) / den[:, None]
    mean[~seen] = 0.0
    pooled[~seen] = 0.0
    col[~seen] = 0.0
    return BlockPayload(coord=fine.coord, level=fine.level + 1, tsdf=mean, weight=wsum,
                        s2=pooled, color=col.astype(np.float32))


def apply_merges(table: HashTable, sigma_threshold: float,
                 min_eligible_fraction: float = MERGE_MIN_ELIGIBLE_FRACTION,
                 min_mean_weight: float = MERGE_MIN_MEAN_WEIGHT,
                 all_levels: bool = False) -> MergeStats:
    """Re-home every quiet, well-observed block one level coarser (adapt.py:119-136)."""
    st = N.MergeStatsC()
    N.check(N.lib().tsdf_apply_merges(table._h, float(sigma_threshold),
                                      float(min_eligible_fraction), float(min_mean_weight),
                                      int(bool(all_levels)), C.byref(st)), "apply_merges")
    return MergeStats(candidates=int(st.candidates), merged=int(st.merged))


def select_merge_candidates(table: HashTable, sigma_threshold: float,
                            min_eligible_fraction: float = MERGE_MIN_ELIGIBLE_FRACTION,
                            min_mean_weight: float = MERGE_MIN_MEAN_WEIGHT) -> list:
    """Level-0 blocks apply_merges would re-home (adapt.py:61-72), canonical
    order; evaluated by the same device kernel apply_merges uses."""
    if sigma_threshold <= 0:
        raise ValueError("sigma_threshold must be positive")
    co = C.POINTER(C.c_int64)()
    n = C.c_int64()
    L = N.lib()
    N.check(L.tsdf_merge_candidates(table._h, float(sigma_threshold), float(min_eligible_fraction),
                                    float(min_mean_weight), C.byref(co), C.byref(n)),
            "select_merge_candidates")
    try:
        k = int(n.value)
        if k == 0:
            return []
        arr = np.frombuffer(C.cast(co, C.POINTER(C.c_int64 * (3 * k))).contents, dtype=np.int64)
        return [tuple(int(v) for v in row) for row in arr.reshape(k, 3)]
    finally:
        L.tsdf_free(C.cast(co, C.c_void_p))
