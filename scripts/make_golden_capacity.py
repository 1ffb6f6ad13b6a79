"""Generate tests/golden/capacity.json by running the REFERENCE package:
block-record and PLY bytes, the .tsdfmap of a scenario, and a streaming
run (FusionEngine with heaps small enough that maybe_stream evicts and
later frames stream blocks back in).

Run in the build container only (needs /root/reference):
    python scripts/make_golden_capacity.py
"""
from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import parity_utils as PU  # noqa: E402
from capacity_scenarios import (FORCED, STREAM_SPEC, MAP_SPEC, record_payloads,  # noqa: E402
                                small_mesh, stream_frames)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def ref_state(table):
    out = {}
    for l in range(table.num_levels):
        coords, handles = table.live_blocks(l)
        h = table.heaps[l]
        idx = handles[:, None] * h.nvox + np.arange(h.nvox)[None, :]
        out[l] = (coords, h.tsdf[idx], h.weight[idx], h.s2[idx], h.color[idx])
    return out


def main():
    assert PU.have_reference(), "needs /root/reference"
    PU.import_reference()
    from tsdfusion import formats, hashgrid
    from tsdfusion.config import PipelineConfig
    from tsdfusion.geometry import DepthFrame, Intrinsics, SensorPose
    from tsdfusion.meshing import Mesh
    from tsdfusion.pipeline import FusionEngine
    gold = {"generator": "scripts/make_golden_capacity.py"}
    # block records (formats.py:185-193)
    recs = {}
    for name, (coord, level, t, w, s2, col) in record_payloads().items():
        p = hashgrid.BlockPayload(coord=coord, level=level, tsdf=t, weight=w, s2=s2, color=col)
        for arch in (False, True):
            b = formats.pack_block_record(p, archived=arch)
            recs[f"{name}_{int(arch)}"] = {"len": len(b), "sha": sha(b)}
    gold["records"] = recs
    # PLY (formats.py:33-60)
    v, n, c, tri = small_mesh()
    with tempfile.TemporaryDirectory() as d:
        formats.write_mesh(Mesh(vertices=v, normals=n, colors=c, triangles=tri), Path(d) / "m.ply")
        gold["ply"] = {"sha": sha((Path(d) / "m.ply").read_bytes())}
    # map of a scenario (formats.py:223-253)
    spec = dict(MAP_SPEC)
    b, stats, merges, seq = PU.run_depth_scenario("reference", **spec)
    with tempfile.TemporaryDirectory() as d:
        formats.save_map(b.t, Path(d) / "x.tsdfmap", sensor_mode="depth", tau=spec["tau"])
        blob = (Path(d) / "x.tsdfmap").read_bytes()
    gold["map"] = {"spec": {k: (list(x) if isinstance(x, tuple) else x) for k, x in spec.items()},
                   "len": len(blob), "sha": sha(blob), "state_digest": PU.state_digest(ref_state(b.t))}
    # streaming run (pipeline.py:88-160, streaming.py)
    cfg = PipelineConfig(**STREAM_SPEC["config"])
    eng = FusionEngine(cfg)
    per = []
    for f in stream_frames():
        rf = DepthFrame(depth=np.asarray(f.depth, dtype=np.float64),
                        intrinsics=Intrinsics(f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx,
                                              f.intrinsics.cy),
                        pose=SensorPose(f.pose.rotation, f.pose.translation),
                        color=None if f.color is None else PU._color_f64(f.color))
        st = eng.integrate_frame(rf)
        merged = eng.maybe_merge()
        evicted = eng.maybe_stream()
        per.append({**{k: getattr(st, k) for k in PU.STAT_KEYS}, "merged": merged,
                    "evicted": evicted, "archived": len(eng.archive),
                    "live": [h.occupied for h in eng.table.heaps]})
    with tempfile.TemporaryDirectory() as d:
        eng.save(Path(d) / "s.tsdfmap")
        sblob = (Path(d) / "s.tsdfmap").read_bytes()
    gold["stream"] = {"per_frame": per, "state_digest": PU.state_digest(ref_state(eng.table)),
                      "archive_coords": [list(c) for c in eng.archive.coords()],
                      "map_len": len(sblob), "map_sha": sha(sblob),
                      "evicted_blocks": eng.evicted_blocks}
    # forced path: CapacityError mid-frame -> evict to low_water -> retry
    eng = FusionEngine(PipelineConfig(**{**STREAM_SPEC["config"], **FORCED}))
    per = []
    for f in stream_frames()[:20]:
        rf = DepthFrame(depth=np.asarray(f.depth, dtype=np.float64),
                        intrinsics=Intrinsics(f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx,
                                              f.intrinsics.cy),
                        pose=SensorPose(f.pose.rotation, f.pose.translation),
                        color=None if f.color is None else PU._color_f64(f.color))
        st = eng.integrate_frame(rf)
        eng.maybe_merge()
        eng.maybe_stream()
        per.append({**{k: getattr(st, k) for k in PU.STAT_KEYS}, "archived": len(eng.archive),
                    "live": [h.occupied for h in eng.table.heaps]})
    gold["forced"] = {"per_frame": per, "state_digest": PU.state_digest(ref_state(eng.table)),
                      "evicted_blocks": eng.evicted_blocks}
    out = ROOT / "tests" / "golden" / "capacity.json"
    out.write_text(json.dumps(gold, indent=1, sort_keys=True))
    print("wrote", out, {k: (v if k != "stream" else {"evicted": v["evicted_blocks"]}) for k, v in gold.items()
                         if k in ("map", "stream")})


if __name__ == "__main__":
    main()
