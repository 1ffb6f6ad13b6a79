"""Shared inputs of the capacity-tier golden tests (scripts/make_golden_capacity.py
generates tests/golden/capacity.json from the reference with these; the
tests replay them on the product)."""
from __future__ import annotations

import numpy as np

# map file of the depth_room scenario (two levels, merges every 10 frames)
MAP_SPEC = dict(scene="room", frames=20, width=64, height=48, edge=0.08, tau=0.03,
                caps=(20000, 10000), n_hash=100003, sigma=2.5e-5)

# FusionEngine run whose heaps overflow the 0.85 high-water mark: maybe_stream
# parks out-of-frustum blocks in the archive; the last frames look back at
# the start of the sweep, so archived blocks stream back in
STREAM_SPEC = dict(config=dict(sensor_mode="depth", nu_fine=0.01, block_edge=0.08, tau=0.04,
                               n_hash=100003, heap_capacity_fine=1400, heap_capacity_coarse=1000,
                               merge_cadence=10, fill_threshold=0.85, low_water=0.70),
                   frames=30, revisit=8, width=64, height=48)


# forced path: no periodic streaming; a frame that overflows the level-0
# heap evicts down to low_water and is retried (pipeline.py:101-128)
FORCED = dict(heap_capacity_fine=1501, fill_threshold=0.99, low_water=0.7)


def stream_frames():
    from paper_2511_21459_b200 import synth
    s = STREAM_SPEC
    f = synth.render_frames("room", s["frames"], s["width"], s["height"],
                            depth_dtype=np.float32, color_dtype=np.uint8)
    return list(f) + list(f[:s["revisit"]])


def record_payloads():
    rng = np.random.default_rng(11)
    out = {}
    for level, coord in ((0, (-3, 5, 7)), (1, (1024, -77, 0))):
        nv = (8 >> level) ** 3
        t = rng.uniform(-0.04, 0.04, nv)
        w = rng.integers(0, 9, nv).astype(np.float64)
        s2 = rng.uniform(0, 1e-4, nv) * (w > 0)
        col = rng.uniform(0, 1, (nv, 3)).astype(np.float32)
        out[f"L{level}"] = (coord, level, t, w, s2, col)
    return out


def small_mesh():
    rng = np.random.default_rng(5)
    v = rng.uniform(-1, 1, (40, 3))
    n = rng.normal(size=(40, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    c = rng.uniform(0, 1, (40, 3))
    tri = rng.integers(0, 40, (30, 3)).astype(np.int64)
    return v, n, c, tri
