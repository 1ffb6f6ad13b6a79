"""Inputs of the quadtree golden tests (scripts/make_golden_quadtree.py runs
the reference on them; tests/test_gpu_quadtree.py replays them on the GPU).
Everything is deterministic: the synthetic room renderer and numpy's
default_rng."""
from __future__ import annotations

import numpy as np


def _room(w, h, n=3, **kw):
    from paper_2511_21459_b200 import synth
    return synth.render_frames("room", n, w, h, **kw)


def image_cases():
    rng = np.random.default_rng(21)
    room = _room(160, 120)[1]
    smooth = np.clip(np.cumsum(rng.normal(0, 0.02, (48, 64, 3)), axis=1), -1, 1) * 0.5 + 0.5
    return {
        "room_160x120_t0.001": (np.asarray(room.color), 0.001, 1),
        "room_160x120_t0.01_mp4": (np.asarray(room.color), 0.01, 4),
        "random_37x23_t0.02": (rng.uniform(0, 1, (23, 37, 3)), 0.02, 1),
        "random_37x23_t0.02_mp3": (rng.uniform(0, 1, (23, 37, 3)), 0.02, 3),
        "gray_50x40_t0.005": (rng.uniform(0, 1, (40, 50)), 0.005, 1),
        "smooth_64x48_t0.0005": (smooth, 0.0005, 1),
        "constant_30x20": (np.full((20, 30, 3), 0.25), 0.1, 1),
        "single_pixel": (np.array([[[0.1, 0.9, 0.3]]]), 0.0, 0),
        "column_1x17_mp0": (rng.uniform(0, 1, (17, 1, 3)), 1e-6, 0),
    }


def seed_cases():
    from paper_2511_21459_b200 import DepthFrame
    f64 = _room(160, 120)[2]
    f32 = _room(160, 120, depth_dtype=np.float32, color_dtype=np.uint8)[2]
    raw = np.clip(np.round(np.nan_to_num(np.asarray(f32.depth, dtype=np.float64)) * 5000.0), 0, 65535)
    u16 = DepthFrame(raw.astype(np.uint16), f32.intrinsics, f32.pose, color=f32.color, depth_scale=5000.0)
    grey = DepthFrame(f64.depth, f64.intrinsics, f64.pose)
    return {
        "f64_rgbf64": (np.asarray(f64.color), 2e-4, 1, f64),
        "f32_rgbu8": (np.asarray(f32.color, dtype=np.float64) / 255.0, 1e-4, 2, f32),
        "u16_rgbu8": (np.asarray(f32.color, dtype=np.float64) / 255.0, 5e-5, 1, u16),
        "f64_no_colour": (np.asarray(f64.color), 2e-4, 1, grey),
    }
