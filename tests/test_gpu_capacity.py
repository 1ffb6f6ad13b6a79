"""Capacity tier on the GPU: .tsdfmap bytes, bulk evict /
import, and a FusionEngine run whose heaps overflow so blocks are streamed
out to the host archive and back in -- all against the reference's own run
(tests/golden/capacity.json from scripts/make_golden_capacity.py)."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import parity_utils as PU
from capacity_scenarios import FORCED, MAP_SPEC, STREAM_SPEC, stream_frames

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).parent / "golden" / "capacity.json").read_text())


def _state(table):
    return PU.GpuBackend.state(type("x", (), {"t": table})())


def test_save_map_matches_reference_bytes_and_round_trips(tmp_path):
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.formats import load_map, save_map
    b, _, _, _ = PU.run_depth_scenario("gpu", **MAP_SPEC)
    save_map(b.t, tmp_path / "a.tsdfmap", sensor_mode="depth", tau=MAP_SPEC["tau"])
    blob = (tmp_path / "a.tsdfmap").read_bytes()
    assert len(blob) == GOLD["map"]["len"]
    assert hashlib.sha256(blob).hexdigest() == GOLD["map"]["sha"]
    t2, arch, info = load_map(tmp_path / "a.tsdfmap")
    assert len(arch) == 0 and info["tau"] == MAP_SPEC["tau"] and info["sensor_mode"] == "depth"
    assert PU.state_digest(_state(t2)) == GOLD["map"]["state_digest"]
    save_map(t2, tmp_path / "b.tsdfmap", sensor_mode="depth", tau=MAP_SPEC["tau"])
    assert (tmp_path / "b.tsdfmap").read_bytes() == blob
    # the reloaded table keeps integrating identically
    f = P.synth.render_frames("room", 21, 64, 48, depth_dtype=np.float32, color_dtype=np.uint8)[20]
    s1 = P.integrate_depth(b.t, f, MAP_SPEC["tau"])
    s2 = P.integrate_depth(t2, f, MAP_SPEC["tau"])
    assert {k: getattr(s1, k) for k in PU.STAT_KEYS} == {k: getattr(s2, k) for k in PU.STAT_KEYS}
    assert PU.state_digest(_state(b.t)) == PU.state_digest(_state(t2))


def test_bulk_evict_import_round_trip():
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.errors import CapacityError, NotFoundError
    b, _, _, _ = PU.run_depth_scenario("gpu", **MAP_SPEC)
    t = b.t
    before = PU.state_digest(_state(t))
    occ = [h.occupied for h in t.heaps]
    coords, _ = t.live_blocks(0)
    sel = coords[::3]
    out = t.evict(0, sel)
    assert t.heaps[0].occupied == occ[0] - len(sel)
    assert not any(t.find(c) for c in sel[:20])
    with pytest.raises(NotFoundError):
        t.evict(0, sel[:1])                   # no longer live: table unchanged
    t.import_blocks(0, sel, *out)
    assert PU.state_digest(_state(t)) == before
    with pytest.raises(ValueError):
        t.import_blocks(0, sel[:2], *(a[:2] for a in out))  # already live
    small = P.HashTable(100003, 10, 7, 0.08, (4, 4))
    with pytest.raises(CapacityError):
        small.import_blocks(0, sel[:5], *(a[:5] for a in out))
    assert small.heaps[0].occupied == 0       # all or nothing


def test_streaming_engine_matches_reference(tmp_path):
    import paper_2511_21459_b200 as P
    cfg = P.PipelineConfig(**STREAM_SPEC["config"])
    eng = P.FusionEngine(cfg)
    per = []
    for f in stream_frames():
        st = eng.integrate_frame(f)
        merged = eng.maybe_merge()
        evicted = eng.maybe_stream()
        per.append({**{k: getattr(st, k) for k in PU.STAT_KEYS}, "merged": merged,
                    "evicted": evicted, "archived": len(eng.archive),
                    "live": [h.occupied for h in eng.table.heaps]})
    g = GOLD["stream"]
    for i, (a, b) in enumerate(zip(per, g["per_frame"])):
        assert a == b, (i, a, b)
    assert eng.evicted_blocks == g["evicted_blocks"]
    assert [list(c) for c in eng.archive.coords()] == g["archive_coords"]
    assert PU.state_digest(_state(eng.table)) == g["state_digest"]
    eng.save(tmp_path / "s.tsdfmap")
    blob = (tmp_path / "s.tsdfmap").read_bytes()
    assert len(blob) == g["map_len"] and hashlib.sha256(blob).hexdigest() == g["map_sha"]
    live = set(map(tuple, eng.table.key_levels()))
    assert not live & set(eng.archive.coords())   # live xor archived


def test_capacity_error_evicts_and_retries():
    """A frame that overflows the level-0 heap triggers the engine's forced
    stream-out to low_water and one retry (pipeline.py:101-108).  (As in the
    reference, a capacity with low_water * capacity integral would stop
    exactly at low_water and raise.)  Matched against the reference's run."""
    import paper_2511_21459_b200 as P
    cfg = P.PipelineConfig(**{**STREAM_SPEC["config"], **FORCED})
    eng = P.FusionEngine(cfg)
    per = []
    for f in stream_frames()[:20]:
        st = eng.integrate_frame(f)
        eng.maybe_merge()
        eng.maybe_stream()
        per.append({**{k: getattr(st, k) for k in PU.STAT_KEYS}, "archived": len(eng.archive),
                    "live": [h.occupied for h in eng.table.heaps]})
    g = GOLD["forced"]
    for i, (a, b) in enumerate(zip(per, g["per_frame"])):
        assert a == b, (i, a, b)
    assert eng.evicted_blocks == g["evicted_blocks"] > 0
    assert PU.state_digest(_state(eng.table)) == g["state_digest"]
    assert not set(map(tuple, eng.table.key_levels())) & set(eng.archive.coords())


@pytest.mark.parametrize("which", ["stream", "forced"])
def test_engine_windows_match_reference(which):
    """FusionEngine.integrate_frames (device windows up to each merge
    boundary, stopping at the stream-out mark or a heap overflow) gives the
    reference's per-frame results: stats, evictions, archive and state."""
    import paper_2511_21459_b200 as P
    cfg = P.PipelineConfig(**STREAM_SPEC["config"]) if which == "stream" else \
        P.PipelineConfig(**{**STREAM_SPEC["config"], **FORCED})
    frames = stream_frames() if which == "stream" else stream_frames()[:20]
    eng = P.FusionEngine(cfg)
    st = eng.integrate_frames(frames)
    g = GOLD[which]
    assert [{k: getattr(s, k) for k in PU.STAT_KEYS} for s in st] == \
        [{k: r[k] for k in PU.STAT_KEYS} for r in g["per_frame"]]
    assert eng.evicted_blocks == g["evicted_blocks"]
    assert PU.state_digest(_state(eng.table)) == g["state_digest"]
    if which == "stream":
        assert [list(c) for c in eng.archive.coords()] == g["archive_coords"]


def test_run_pipeline_batched_equals_per_frame():
    import paper_2511_21459_b200 as P
    frames = P.synth.render_frames("room", 25, 64, 48, depth_dtype=np.float32, color_dtype=np.uint8)
    cfg = P.PipelineConfig(sensor_mode="depth", nu_fine=0.01, block_edge=0.08, tau=0.04,
                           n_hash=100003, heap_capacity_fine=20000, heap_capacity_coarse=10000)
    ra, ma = P.run_pipeline(cfg, frames, batched=True)
    rb, mb = P.run_pipeline(cfg, frames, batched=False)
    assert ra.frames == rb.frames == 25 and ra.merged_blocks == rb.merged_blocks > 0
    assert ra.live_blocks == rb.live_blocks
    assert np.array_equal(ma.vertices, mb.vertices) and np.array_equal(ma.triangles, mb.triangles)
