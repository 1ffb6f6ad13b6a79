"""Backend adapters + digests for the parity harness.

Three interchangeable backends run the same scenarios:
  * "reference" -- the reference package imported from /root/reference (only
    in the build container; used to generate tests/golden and to pin the
    oracle),
  * "oracle"    -- the C oracle (oracle/, test infrastructure),
  * "gpu"       -- the product (paper_2511_21459_b200 over the sm_100a library).
Every backend exposes the same calls and a canonical state export, so one
scenario function produces comparable stats, key sets and digests.
"""
from __future__ import annotations

import hashlib
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
REF_SRC = Path("/root/reference/pkg/src")
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

STAT_KEYS = ("measurements", "skipped_invalid", "blocks_allocated", "blocks_touched",
             "voxels_updated", "observations")


def have_reference() -> bool:
    return (REF_SRC / "tsdfusion" / "__init__.py").exists()


def import_reference():
    if str(REF_SRC) not in sys.path:
        sys.path.insert(0, str(REF_SRC))
    import tsdfusion  # noqa: F401
    from tsdfusion import adapt, hashgrid, integrate, meshing
    return hashgrid, integrate, adapt, meshing


# ---------------------------------------------------------------------------
# digests
# ---------------------------------------------------------------------------

def state_digest(state) -> str:
    """sha256 over every level's canonical-order coords, tsdf, weight, s2, colour."""
    h = hashlib.sha256()
    for level in sorted(state):
        coords, tsdf, w, s2, col = state[level]
        h.update(f"L{level}:{len(coords)}".encode())
        h.update(np.ascontiguousarray(coords, dtype=np.int64).tobytes())
        h.update(np.ascontiguousarray(tsdf, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(w, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(s2, dtype=np.float64).tobytes())
        h.update(np.ascontiguousarray(col, dtype=np.float32).tobytes())
    return h.hexdigest()


def keys_digest(state) -> str:
    """sha256 of the (coord, level) set only -- the bit-exact allocation contract."""
    h = hashlib.sha256()
    for level in sorted(state):
        h.update(f"L{level}:".encode())
        h.update(np.ascontiguousarray(state[level][0], dtype=np.int64).tobytes())
    return h.hexdigest()


def mesh_digest(v, t) -> str:
    """The reference's golden-mesh digest (tests/test_meshing.py:427-431)."""
    h = hashlib.sha256()
    h.update(np.round(v, 9).tobytes())
    h.update(np.asarray(t).astype(np.int64).tobytes())
    return h.hexdigest()


def array_digest(*arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------------------
# backends
# ---------------------------------------------------------------------------

def _metres(frame):
    """f64 depth in metres as the reference frame holds it (raw uint16 depth
    divided by its scale, datasets.py:113)."""
    d = np.asarray(frame.depth, dtype=np.float64)
    return d / frame.depth_scale if np.asarray(frame.depth).dtype == np.uint16 else d


class RefBackend:
    name = "reference"

    def __init__(self, n_hash, edge, caps, bucket=10, overflow=7):
        hg, self.I, self.A, self.M = import_reference()
        self.t = hg.HashTable(n_hash, bucket, overflow, edge, tuple(caps))

    def depth(self, frame, tau, weight_cap=0.0):
        from tsdfusion.geometry import DepthFrame, Intrinsics, SensorPose
        f = DepthFrame(depth=_metres(frame),
                       intrinsics=Intrinsics(frame.intrinsics.fx, frame.intrinsics.fy,
                                             frame.intrinsics.cx, frame.intrinsics.cy),
                       pose=SensorPose(frame.pose.rotation, frame.pose.translation),
                       color=None if frame.color is None else _color_f64(frame.color))
        s = self.I.integrate_depth(self.t, f, tau, weight_cap=weight_cap)
        return {k: getattr(s, k) for k in STAT_KEYS}

    def points(self, frame, tau, weight_cap=0.0):
        from tsdfusion.geometry import PointCloudFrame, SensorPose
        f = PointCloudFrame(points=np.asarray(frame.points, dtype=np.float64),
                            pose=SensorPose(frame.pose.rotation, frame.pose.translation),
                            colors=None if frame.colors is None else _color_f64(frame.colors))
        s = self.I.integrate_pointcloud(self.t, f, tau, weight_cap=weight_cap)
        return {k: getattr(s, k) for k in STAT_KEYS}

    def merge(self, sigma, all_levels=False):
        assert not all_levels, "the reference only merges level 0 -> 1"
        s = self.A.apply_merges(self.t, sigma)
        return {"candidates": s.candidates, "merged": s.merged}

    def state(self):
        out = {}
        for l in range(self.t.num_levels):
            coords, handles = self.t.live_blocks(l)
            h = self.t.heaps[l]
            idx = handles[:, None] * h.nvox + np.arange(h.nvox)[None, :]
            out[l] = (coords, h.tsdf[idx], h.weight[idx], h.s2[idx], h.color[idx])
        return out

    def mesh(self, iso=0.0, eps=None):
        m = self.M.extract_mesh(self.t, iso=iso, collapse_epsilon=eps)
        return m.vertices, m.normals, m.colors, m.triangles

    def insert(self, c, level):
        return self.t.insert(c, level)

    def write(self, c, tsdf, weight, s2=None):
        hd, lv = self.t.find(c)
        h = self.t.heaps[lv]
        sl = slice(hd * h.nvox, (hd + 1) * h.nvox)
        h.tsdf[sl] = tsdf
        h.weight[sl] = weight
        if s2 is not None:
            h.s2[sl] = s2


class OracleBackend:
    name = "oracle"

    def __init__(self, n_hash, edge, caps, bucket=10, overflow=7):
        from oracle.oracle import OracleTable
        self.t = OracleTable(n_hash, bucket, overflow, edge, tuple(caps))

    def depth(self, frame, tau, weight_cap=0.0):
        i = frame.intrinsics
        s = self.t.integrate_depth(_metres(frame),
                                   [i.fx, i.fy, i.cx, i.cy], frame.pose.rotation,
                                   frame.pose.translation, tau,
                                   color=None if frame.color is None else _color_f64(frame.color),
                                   weight_cap=weight_cap)
        return {k: s[k] for k in STAT_KEYS}

    def points(self, frame, tau, weight_cap=0.0):
        s = self.t.integrate_points(np.asarray(frame.points, dtype=np.float64), frame.pose.rotation,
                                    frame.pose.translation, tau,
                                    colors=None if frame.colors is None else _color_f64(frame.colors),
                                    weight_cap=weight_cap)
        return {k: s[k] for k in STAT_KEYS}

    def merge(self, sigma, all_levels=False):
        return self.t.apply_merges(sigma, all_levels=all_levels)

    def state(self):
        return {l: self.t.block_arrays(l) for l in range(self.t.num_levels)}

    def mesh(self, iso=0.0, eps=None):
        return self.t.extract_mesh(iso=iso, collapse_epsilon=eps)

    def insert(self, c, level):
        return self.t.insert(c, level)

    def write(self, c, tsdf, weight, s2=None):
        hd, lv = self.t.find(c)
        h = self.t.heaps[lv]
        sl = slice(hd * h.nvox, (hd + 1) * h.nvox)
        h.tsdf[sl] = tsdf
        h.weight[sl] = weight
        if s2 is not None:
            h.s2[sl] = s2


class GpuBackend:
    name = "gpu"

    def __init__(self, n_hash, edge, caps, bucket=10, overflow=7):
        import paper_2511_21459_b200 as P
        self.P = P
        self.t = P.HashTable(n_hash, bucket, overflow, edge, tuple(caps))

    def depth(self, frame, tau, weight_cap=0.0):
        s = self.P.integrate_depth(self.t, frame, tau, weight_cap=weight_cap)
        return {k: getattr(s, k) for k in STAT_KEYS}

    def points(self, frame, tau, weight_cap=0.0):
        s = self.P.integrate_pointcloud(self.t, frame, tau, weight_cap=weight_cap)
        return {k: getattr(s, k) for k in STAT_KEYS}

    def merge(self, sigma, all_levels=False):
        s = self.P.apply_merges(self.t, sigma, all_levels=all_levels)
        return {"candidates": s.candidates, "merged": s.merged}

    def state(self):
        out = {}
        for l in range(self.t.num_levels):
            coords, _, tsdf, w, s2, col = self.t.export_level(l)
            out[l] = (coords, tsdf, w, s2, col)
        return out

    def mesh(self, iso=0.0, eps=None):
        m = self.P.extract_mesh(self.t, iso=iso, collapse_epsilon=eps)
        return m.vertices, m.normals, m.colors, m.triangles

    def insert(self, c, level):
        return self.t.insert(c, level)

    def write(self, c, tsdf, weight, s2=None):
        from paper_2511_21459_b200.hashgrid import BlockPayload
        pl = self.t.payload(c)
        pl.tsdf = np.asarray(tsdf, dtype=np.float64) * np.ones(len(pl.tsdf))
        pl.weight = np.asarray(weight, dtype=np.float64) * np.ones(len(pl.tsdf))
        if s2 is not None:
            pl.s2 = np.asarray(s2, dtype=np.float64) * np.ones(len(pl.tsdf))
        self.t.write_payload(c, pl)

    def close(self):
        self.t.close()


def _color_f64(c):
    c = np.asarray(c)
    return c.astype(np.float64) / 255.0 if c.dtype == np.uint8 else c.astype(np.float64)


BACKENDS = {"reference": RefBackend, "oracle": OracleBackend, "gpu": GpuBackend}


# ---------------------------------------------------------------------------
# scenarios (shared by make_golden.py and the tests)
# ---------------------------------------------------------------------------

def run_depth_scenario(backend, scene, frames, width, height, edge, tau, caps, n_hash,
                       sigma=None, cadence=10, all_levels=False, color=True, weight_cap=0.0,
                       depth_dtype=np.float64, color_dtype=np.float64, sweep=None):
    from paper_2511_21459_b200 import synth
    b = BACKENDS[backend](n_hash, edge, caps)
    seq = synth.render_frames(scene, frames, width, height, depth_dtype=depth_dtype,
                              color_dtype=color_dtype, sweep=sweep)
    stats, merges = [], []
    for i, f in enumerate(seq):
        if not color:
            f.color = None
        stats.append(b.depth(f, tau, weight_cap=weight_cap))
        if sigma is not None and (i + 1) % cadence == 0:
            merges.append(b.merge(sigma, all_levels=all_levels))
    return b, stats, merges, seq


def run_lidar_scenario(backend, scans, beams, columns, edge, tau, caps, n_hash, sigma=None,
                       cadence=2, color=False, step=0.5):
    from paper_2511_21459_b200 import synth
    b = BACKENDS[backend](n_hash, edge, caps)
    seq = synth.lidar_frames(scans, beams, columns, step=step)
    rng = np.random.default_rng(5)
    stats, merges = [], []
    for i, f in enumerate(seq):
        if color:
            f.colors = rng.integers(0, 256, size=(len(f.points), 3)).astype(np.uint8)
        stats.append(b.points(f, tau))
        if sigma is not None and (i + 1) % cadence == 0:
            merges.append(b.merge(sigma))
    return b, stats, merges, seq


def level_summary(state):
    return {int(l): int(len(v[0])) for l, v in state.items()}


# ---------------------------------------------------------------------------
# full-scale scenarios (tests/golden/golden_full.json, scripts/make_golden_full.py)
# ---------------------------------------------------------------------------

FULL_SCENARIOS = {
    # BASELINE config 1 at its real size
    "c1_full": dict(kind="depth", scene="room", frames=30, width=320, height=240, edge=0.08,
                    tau=0.03, caps=(200000, 100000), n_hash=1000003, sigma=2.5e-5, cadence=10),
    # BASELINE config 2 geometry: large room, 640x480 @ 5 mm, bench input format;
    # the first two frames of the bench's 500-frame sweep
    "c2_large_frame": dict(kind="depth", scene="large_room", frames=2, width=640, height=480,
                           edge=0.04, tau=0.015, caps=(160000, 20000), n_hash=4000037,
                           sigma=2.5e-5, cadence=2, depth_dtype="float32", color_dtype="uint8",
                           sweep=500),
    # BASELINE config 3: one full 128-beam scan
    "c3_scan": dict(kind="lidar", scans=1, beams=128, columns=2048, edge=1.6, tau=0.8,
                    caps=(160000, 40000), n_hash=4000037, sigma=1e-2, cadence=1),
}


def run_full_scenario(backend, name, mesh=False):
    """Run one FULL_SCENARIOS entry on a backend; returns the golden record
    (stats, merges, levels, digests; mesh digests for depth when asked)."""
    spec = dict(FULL_SCENARIOS[name])
    kind = spec.pop("kind")
    if kind == "depth":
        spec["depth_dtype"] = np.dtype(spec.get("depth_dtype", "float64")).type
        spec["color_dtype"] = np.dtype(spec.get("color_dtype", "float64")).type
        b, stats, merges, seq = run_depth_scenario(backend, **spec)
        inp = array_digest(*[np.asarray(f.depth) for f in seq],
                           *[np.asarray(f.color) for f in seq if f.color is not None])
    else:
        b, stats, merges, seq = run_lidar_scenario(backend, **spec)
        inp = array_digest(*[np.asarray(f.points) for f in seq])
    st = b.state()
    out = {"stats": stats, "merges": merges, "levels": level_summary(st),
           "keys_digest": keys_digest(st), "state_digest": state_digest(st),
           "input_digest": inp}
    if mesh and kind == "depth" and name == "c1_full":
        v, n, c, t = b.mesh()
        out["mesh"] = {"nv": int(len(v)), "nt": int(len(t)), "digest": mesh_digest(v, t),
                       "full_digest": array_digest(v, n, c, t)}
    if hasattr(b, "close"):
        b.close()
    return out
