"""Contrast-driven image quadtree and depth-seeded splats (reference
quadtree.py:1-148; the paper's splat-seeding stage).

build_quadtree and seed_splats run on the GPU (csrc/quadtree.cu): integral
images by sequential running sums (numpy's cumsum order), a level-synchronous
breadth-first build whose leaves come out in the reference's order, and one
thread per leaf for seeding.  Results are bit-identical to the reference's
(tests/test_gpu_quadtree.py against tests/golden/quadtree.json).
region_contrast is the reference's direct per-node formula (host numpy; a
helper, not the build path).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .geometry import DepthFrame

LUMA_WEIGHTS = np.array([0.2989, 0.5870, 0.1140])


@dataclass
class QuadNode:
    x0: int
    y0: int
    w: int
    h: int
    contrast: float = 0.0
    is_leaf: bool = False

    def key(self) -> tuple:
        return (self.x0, self.y0, self.w, self.h)


@dataclass
class SplatSeed:
    position: np.ndarray  # (3,) world metres
    scale: float          # isotropic extent, metres
    color: np.ndarray     # (3,) in [0, 1]


def region_contrast(image: np.ndarray, node: QuadNode) -> float:
    """Luma-weighted mean squared deviation of the node's pixels
    (quadtree.py:42-47)."""
    region = np.asarray(image, dtype=np.float64)[node.y0:node.y0 + node.h, node.x0:node.x0 + node.w]
    mean = region.reshape(-1, 3).mean(axis=0)
    sq = (region.reshape(-1, 3) - mean) ** 2
    return float(LUMA_WEIGHTS @ (sq.sum(axis=0) / sq.shape[0]))


def build_quadtree(image, contrast_threshold: float = 0.1, min_pixel: int = 1) -> list:
    """Breadth-first, level-synchronous subdivision of the whole image
    (quadtree.py:94-109): a node splits when its contrast exceeds the
    threshold and min(w, h) exceeds min_pixel; the leaves tile the image."""
    image = np.asarray(image, dtype=np.float64)
    if image.ndim == 2:
        image = np.repeat(image[:, :, None], 3, axis=2)
    if image.size == 0:
        raise ValueError("image is empty")
    image = np.ascontiguousarray(image)
    h, w = image.shape[:2]
    leaves = np.empty((h * w, 4), dtype=np.int32)
    con = np.empty(h * w, dtype=np.float64)
    n = C.c_int64()
    N.check(N.lib().tsdf_quadtree_build(image.ctypes.data, h, w, N.MEM_HOST, float(contrast_threshold),
                                        int(min_pixel), leaves.ctypes.data, con.ctypes.data,
                                        C.byref(n), None), "build_quadtree")
    k = int(n.value)
    return [QuadNode(int(a), int(b), int(c), int(d), contrast=float(x), is_leaf=True)
            for (a, b, c, d), x in zip(leaves[:k].tolist(), con[:k].tolist())]


def seed_splats(leaves: list, depth: DepthFrame) -> list:
    """One splat per leaf with valid depth at its centre (quadtree.py:112-148):
    the centre back-projected to world, scale = leaf width * depth / fx,
    colour = the leaf's mean RGB (grey 0.5 without colour)."""
    if not leaves:
        return []
    lv = np.ascontiguousarray([[q.x0, q.y0, q.w, q.h] for q in leaves], dtype=np.int32)
    dptr, ddt, dmem, _kd = N.as_buffer(depth.depth, (N.F64, N.F32, N.U16))
    cptr, cdt, _kc = None, 0, None
    if depth.color is not None:
        cptr, cdt, cmem, _kc = N.as_buffer(depth.color, (N.F64, N.F32, N.U8))
        if cmem != dmem:
            raise ValueError("depth and colour must both live on the host or both on the device")
    n = len(lv)
    pos = np.empty((n, 3), dtype=np.float64)
    sc = np.empty(n, dtype=np.float64)
    col = np.empty((n, 3), dtype=np.float64)
    ok = np.empty(n, dtype=np.uint8)
    R = np.ascontiguousarray(depth.pose.rotation, dtype=np.float64).reshape(9)
    t = np.ascontiguousarray(depth.pose.translation, dtype=np.float64).reshape(3)
    N.check(N.lib().tsdf_seed_splats(lv.ctypes.data, n, dptr, ddt, float(depth.depth_scale), cptr, cdt,
                                     depth.height, depth.width, dmem, depth.intrinsics.as_array(), R, t,
                                     pos.ctypes.data, sc.ctypes.data, col.ctypes.data, ok.ctypes.data,
                                     None), "seed_splats")
    return [SplatSeed(position=pos[i].copy(), scale=float(sc[i]), color=col[i].copy())
            for i in np.nonzero(ok)[0]]
