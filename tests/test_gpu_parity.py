"""GPU parity: the product (sm_100a kernels through the C ABI) against the
reference's golden vectors and against the C oracle on the same inputs.

Contract: allocated block-key set and per-key levels
bit-exact; integration/merge counters equal; TSDF / weight / variance /
colour bit-identical (stronger than the stated 1e-4 relative tolerance,
which the tolerance test below also checks explicitly).
"""
import numpy as np
import pytest

import parity_utils as PU

pytestmark = pytest.mark.gpu

TOL_REL = 1e-4  # north-star float tolerance for TSDF / S2


def _spec(golden, name):
    return {k: (tuple(v) if isinstance(v, list) else v)
            for k, v in golden["scenarios"][name]["spec"].items() if k != "kind"}


def assert_states_match(a, b, exact=True):
    assert set(a) == set(b)
    for level in a:
        ca, ta, wa, sa, cola = a[level]
        cb, tb, wb, sb, colb = b[level]
        assert np.array_equal(ca, cb), f"level {level}: block-key sets differ"
        assert np.array_equal(wa, wb), f"level {level}: weights differ"
        if exact:
            assert np.array_equal(ta, tb) and np.array_equal(sa, sb) and np.array_equal(cola, colb)
        else:
            assert np.all(np.abs(ta - tb) <= TOL_REL * np.abs(tb) + 1e-7)
            assert np.all(np.abs(sa - sb) <= TOL_REL * np.abs(sb) + 1e-12)


def test_device_is_b200_class():
    from paper_2511_21459_b200._native import device_info
    major, minor, sms = device_info()
    assert (major, minor) == (10, 0), (major, minor)
    assert sms >= 132


@pytest.mark.parametrize("name", ["depth_room", "depth_sphere", "depth_room_5mm",
                                  "depth_room_wcap", "lidar_small"])
def test_scenario_goldens(golden, name):
    g = golden["scenarios"][name]
    spec = _spec(golden, name)
    if name.startswith("lidar"):
        b, stats, merges, _ = PU.run_lidar_scenario("gpu", **spec)
    else:
        b, stats, merges, _ = PU.run_depth_scenario("gpu", **spec)
    assert stats == g["stats"]
    assert merges == g["merges"]
    st = b.state()
    assert PU.level_summary(st) == {int(k): v for k, v in g["levels"].items()}
    assert PU.keys_digest(st) == g["keys_digest"]
    assert PU.state_digest(st) == g["state_digest"]
    b.close()


def test_dda_goldens(golden):
    import paper_2511_21459_b200 as P
    for o, e, edge, want in golden["dda_scalar"]:
        assert [list(c) for c in P.dda_blocks(o, e, edge)] == want
    g = golden["dda_batch"]
    ids, co = P.dda_blocks_batch(np.array(g["origins"]), np.array(g["endpoints"]), g["edge"])
    assert PU.array_digest(ids.astype(np.int64), co.astype(np.int64)) == g["rows_digest"]


def _pair(spec_fn, *args, **kw):
    g = spec_fn("gpu", *args, **kw)
    o = spec_fn("oracle", *args, **kw)
    return g, o


def test_c1_room_320x240_vs_oracle():
    """Config 1 (reference room, 320x240, 30 frames, 2 levels, merges every 10)."""
    (bg, sg, mg, _), (bo, so, mo, _) = _pair(
        PU.run_depth_scenario, "room", 30, 320, 240, 0.08, 0.03, (60000, 20000), 1000003,
        sigma=2.5e-5)
    assert sg == so and mg == mo
    assert sum(m["merged"] for m in mg) > 0
    assert_states_match(bg.state(), bo.state())


def test_c2_room_640x480_5mm_vs_oracle():
    """Config 2 geometry at full resolution (640x480, 5 mm voxels), f32 depth + u8 RGB."""
    (bg, sg, _, _), (bo, so, _, _) = _pair(
        PU.run_depth_scenario, "room", 2, 640, 480, 0.04, 0.015, (200000, 20000), 1000003,
        depth_dtype=np.float32, color_dtype=np.uint8)
    assert sg == so
    assert_states_match(bg.state(), bo.state())


def test_c2_three_level_extension_vs_oracle():
    """3 levels (extension oracle): merges L0->L1->L2 with the same rule."""
    (bg, sg, mg, _), (bo, so, mo, _) = _pair(
        PU.run_depth_scenario, "sphere", 40, 64, 48, 0.08, 0.03, (30000, 10000, 4000), 100003,
        sigma=2.5e-4, all_levels=True)
    assert sg == so and mg == mo
    sg_ = bg.state()
    assert PU.level_summary(sg_)[2] > 0
    assert_states_match(sg_, bo.state())


def test_c3_lidar_full_scan_vs_oracle():
    """Config 3: one full 128-beam x 2048-column scan, 100 m range, 20 cm voxels."""
    (bg, sg, _, _), (bo, so, _, _) = _pair(
        PU.run_lidar_scenario, 1, 128, 2048, 1.6, 0.8, (400000, 50000), 4000037)
    assert sg == so
    assert sg[0]["measurements"] > 200000
    assert_states_match(bg.state(), bo.state())


def test_lidar_colour_and_merges_vs_oracle():
    (bg, sg, mg, _), (bo, so, mo, _) = _pair(
        PU.run_lidar_scenario, 4, 32, 512, 1.6, 0.8, (200000, 50000), 1000003, sigma=1e-2,
        color=True)
    assert sg == so and mg == mo
    assert_states_match(bg.state(), bo.state())


def _frame(P, depth, color=None, pose=None, intr=None):
    intr = intr or P.Intrinsics(60.0, 60.0, (depth.shape[1] - 1) / 2, (depth.shape[0] - 1) / 2)
    return P.DepthFrame(depth=depth, intrinsics=intr, pose=pose or P.SensorPose.identity(),
                        color=color)


def test_edge_cases_vs_oracle():
    import paper_2511_21459_b200 as P
    cases = []
    d = np.zeros((48, 64))
    cases.append(("all-invalid", d.copy()))
    d = np.full((48, 64), 1.0)
    d[10:20, 10:20] = np.nan
    d[0, :] = np.inf
    d[1, :] = -1.0
    cases.append(("nan-inf-negative", d))
    d = np.zeros((48, 64))
    d[17, 33] = 0.9
    cases.append(("single-valid-pixel", d))  # exercises the N == 1 gemv order
    d = np.full((1, 1), 0.5)
    cases.append(("1x1", d))
    R = P.synth.look_at(np.array([0.1, -0.2, 0.05]), np.array([1.0, 0.3, 0.2])).rotation
    for name, depth in cases:
        g = PU.GpuBackend(8209, 0.08, (4096, 256))
        o = PU.OracleBackend(8209, 0.08, (4096, 256))
        f = _frame(P, depth, pose=P.SensorPose(R, [0.1, -0.2, 0.05]))
        sg, so = g.depth(f, 0.04), o.depth(f, 0.04)
        assert sg == so, name
        assert_states_match(g.state(), o.state())
        g.close()


def test_point_cloud_edge_cases_vs_oracle():
    import paper_2511_21459_b200 as P
    rng = np.random.default_rng(3)
    for pts in [np.array([[0.51, 0.0, 0.0]]), np.zeros((0, 3)),
                np.array([[0.5, 0, 0], [np.nan, 0, 0], [np.inf, 1, 1], [0, 0, 0]]),
                rng.uniform(0.2, 0.7, size=(100, 3)), rng.normal(0, 1.5, (2000, 3))]:
        g = PU.GpuBackend(1000003, 0.08, (400000, 256))
        o = PU.OracleBackend(1000003, 0.08, (400000, 256))
        f = P.PointCloudFrame(points=pts, pose=P.SensorPose.identity())
        assert g.points(f, 0.04) == o.points(f, 0.04)
        assert g.points(f, 0.04) == o.points(f, 0.04)  # same frame twice
        assert_states_match(g.state(), o.state())
        g.close()


def test_same_frame_twice_weight_two_zero_variance():
    """reference tests/test_integrate.py:142-155"""
    import paper_2511_21459_b200 as P
    pts = np.array([[0.5, 0, 0], [0, 0.5, 0], [0, 0, 0.5], [0.4, 0.4, 0], [0, 0.4, 0.4]])
    t = P.HashTable(97, 10, 7, 0.08, (512, 16))
    f = P.PointCloudFrame(points=pts, pose=P.SensorPose.identity())
    P.integrate_pointcloud(t, f, tau=0.04)
    P.integrate_pointcloud(t, f, tau=0.04)
    _, _, _, w, s2, _ = t.export_level(0)
    touched = w > 0
    assert touched.any() and np.all(w[touched] == 2) and np.all(s2[touched] == 0.0)


def test_allocate_for_measurement_vs_oracle():
    import paper_2511_21459_b200 as P
    from oracle.oracle import OracleTable
    t = P.HashTable(97, 10, 7, 0.16, (128, 16))
    o = OracleTable(97, 10, 7, 0.16, (128, 16))
    for (org, p) in [((0, 0, 0), (0.5, 0, 0)), ((0.01, 0.02, 0.03), (0.5, -0.3, 0.2)),
                     ((0, 0, 0), (0.5, 0, 0))]:
        hg = P.allocate_for_measurement(t, org, p, tau=0.1)
        ho = o.allocate_for_measurement(org, p, 0.1)
        assert len(hg) == len(ho)
    assert t.key_levels() == o.key_levels()
    t.insert((1, 0, 0), 1) if t.find((1, 0, 0)) is None else None
    with pytest.raises(ValueError):
        P.allocate_for_measurement(t, (1, 1, 1), (1, 1, 1), tau=0.1)


def test_table_ops_and_capacity_semantics():
    """reference tests/test_hashgrid.py:58-140 on the device table."""
    import paper_2511_21459_b200 as P
    t = P.HashTable(97, 10, 7, 0.08, (512, 256))
    h = t.insert((1, 2, 3), 0)
    assert t.find((1, 2, 3)) == (h, 0)
    assert t.find((0, 0, 0)) is None
    assert t.insert((1, 2, 3), 0) == h and t.live_count() == 1
    t.insert((4, 5, 6), 1)
    t.remove((4, 5, 6))
    assert t.find((4, 5, 6)) is None
    with pytest.raises(P.NotFoundError):
        t.remove((4, 5, 6))
    # zero-initialised after remove + insert
    pl = t.payload((1, 2, 3))
    pl.tsdf[:] = 3.0
    pl.weight[:] = 1.0
    t.write_payload((1, 2, 3), pl)
    t.remove((1, 2, 3))
    t.insert((1, 2, 3), 0)
    assert np.all(t.payload((1, 2, 3)).tsdf == 0.0)
    # n_hash = 1: bucket 10 + chain 7 per slot, then CapacityError, no leak
    one = P.HashTable(1, 10, 7, 0.08, (64, 32))
    for i in range(17):
        one.insert((i, 0, 0), 0)
    with pytest.raises(P.CapacityError):
        one.insert((17, 0, 0), 0)
    assert one.heaps[0].occupied == 17
    one.remove((4, 0, 0))
    one.remove((13, 0, 0))
    one.insert((20, 0, 0), 0)
    one.insert((21, 0, 0), 0)
    with pytest.raises(P.CapacityError):
        one.insert((22, 0, 0), 0)
    # heap exhaustion
    small = P.HashTable(97, 10, 7, 0.08, (2, 1))
    small.insert((0, 0, 0), 0)
    small.insert((1, 0, 0), 0)
    with pytest.raises(P.CapacityError):
        small.insert((2, 0, 0), 0)


def test_capacity_error_parity_with_oracle():
    """A scan that overflows the reference's bucket+chain limit raises
    CapacityError on both sides (the reference raises on the 18th entry of a
    Teschner slot, hashgrid.py:232-244)."""
    import paper_2511_21459_b200 as P
    from oracle.oracle import OracleError
    pts = np.random.default_rng(3).normal(0, 8, (2000, 3))
    f = P.PointCloudFrame(points=pts, pose=P.SensorPose.identity())
    g = PU.GpuBackend(8209, 0.08, (400000, 256))
    o = PU.OracleBackend(8209, 0.08, (400000, 256))
    with pytest.raises(P.CapacityError):
        g.points(f, 0.04)
    with pytest.raises(OracleError) as e:
        o.points(f, 0.04)
    assert e.value.kind == "CapacityError"
    assert g.t.live_count() == 0  # GPU rolls the whole frame back


def test_frame_capacity_error_rolls_back():
    import paper_2511_21459_b200 as P
    f = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 1, 64, 48)[0]
    t = P.HashTable(100003, 10, 7, 0.08, (50, 10))
    with pytest.raises(P.CapacityError):
        P.integrate_depth(t, f, 0.03)
    assert t.live_count() == 0  # whole-frame rollback


def test_deterministic_rerun_bit_identical():
    digests = []
    for _ in range(2):
        b, _, _, _ = PU.run_depth_scenario("gpu", "sphere", 12, 48, 36, 0.08, 0.04,
                                           (20000, 4096), 100003, sigma=2.5e-4, cadence=6)
        digests.append(PU.state_digest(b.state()))
        b.close()
    assert digests[0] == digests[1]


def test_device_resident_inputs_match_host_inputs():
    torch = pytest.importorskip("torch")
    import paper_2511_21459_b200 as P
    frames = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 3, 160, 120, depth_dtype=np.float32,
                                   color_dtype=np.uint8)
    a = P.HashTable(1000003, 10, 7, 0.04, (60000, 1000))
    b = P.HashTable(1000003, 10, 7, 0.04, (60000, 1000))
    for f in frames:
        sa = P.integrate_depth(a, f, 0.015)
        fd = P.DepthFrame(depth=torch.from_numpy(f.depth).cuda(), intrinsics=f.intrinsics,
                          pose=f.pose, color=torch.from_numpy(f.color).cuda())
        sb = P.integrate_depth(b, fd, 0.015)
        assert sa == sb
    torch.cuda.synchronize()
    sa, sb = PU.GpuBackend.state(type("x", (), {"t": a})()), PU.GpuBackend.state(type("x", (), {"t": b})())
    assert PU.state_digest(sa) == PU.state_digest(sb)


def test_select_merge_candidates_matches_apply():
    import paper_2511_21459_b200 as P
    b, _, _, _ = PU.run_depth_scenario("gpu", "sphere", 20, 48, 36, 0.08, 0.03, (20000, 10000),
                                       100003)
    cands = P.select_merge_candidates(b.t, 2.5e-4)
    st = P.apply_merges(b.t, 2.5e-4)
    assert st.merged == len(cands) > 0
    assert all(b.t.find(c)[1] == 1 for c in cands)


@pytest.mark.parametrize("world", [2, 3])
def test_block_key_sharding_union_equals_single_gpu(world):
    """Multi-GPU path on one device: `world` shard tables (owner(key) == rank)
    integrate the same frames + merges; the union of shards is the single
    table bit-for-bit and the partitioned counters sum to its counters."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.sharding import INVARIANT, PARTITIONED, owner_of_coords
    frames = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 20, 160, 120, depth_dtype=np.float32,
                                   color_dtype=np.uint8)
    full = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000))
    shards = []
    for r in range(world):
        t = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000))
        t.set_shard(r, world)
        shards.append(t)
    for i, f in enumerate(frames):
        s_full = P.integrate_depth(full, f, 0.015)
        parts = [P.integrate_depth(t, f, 0.015) for t in shards]
        for k in PARTITIONED:
            assert sum(getattr(p, k) for p in parts) == getattr(s_full, k), k
        for k in INVARIANT:
            assert all(getattr(p, k) == getattr(s_full, k) for p in parts), k
        if (i + 1) % 10 == 0:
            m = P.apply_merges(full, 2.5e-5).merged
            assert sum(P.apply_merges(t, 2.5e-5).merged for t in shards) == m
    for level in range(2):
        co, _, ts, w, s2, col = full.export_level(level)
        rows = {}
        for r, t in enumerate(shards):
            c2, _, t2, w2, s22, col2 = t.export_level(level)
            assert np.all(owner_of_coords(c2, world) == r)
            for j, c in enumerate(map(tuple, c2.tolist())):
                rows[c] = (t2[j], w2[j], s22[j], col2[j])
        assert set(rows) == set(map(tuple, co.tolist()))
        for j, c in enumerate(map(tuple, co.tolist())):
            a = rows[c]
            assert np.array_equal(a[0], ts[j]) and np.array_equal(a[1], w[j])
            assert np.array_equal(a[2], s2[j]) and np.array_equal(a[3], col[j])


@pytest.mark.parametrize("world", [1, 2, 3])
def test_ray_sharded_allocation_union_equals_single_gpu(world):
    """Ray-sharded multi-GPU allocation on one device: `world`
    shard tables each walk 1/world of the rays, emit the keys they see into
    per-owner buckets, the buckets are exchanged (concatenated per owner, as
    all-to-all does), and each shard inserts + updates its own keys.  The
    union of shards equals the single table bit-for-bit, the partitioned
    counters sum to its counters, and the invariant ones agree."""
    import torch
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.sharding import INVARIANT, PARTITIONED, owner_of_coords
    frames = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 20, 160, 120, depth_dtype=np.float32,
                                   color_dtype=np.uint8)
    full = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000))
    shards = []
    for r in range(world):
        t = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000))
        if world > 1:
            t.set_shard(r, world)
        shards.append(t)
    dev = torch.device("cuda", 0)
    buckets = [torch.zeros((world, t.slots), dtype=torch.int64, device=dev) for t in shards]
    for i, f in enumerate(frames):
        s_full = P.integrate_depth(full, f, 0.015)
        walks = []
        for r, t in enumerate(shards):
            walks.append(P.integrate_depth_walk(t, f, 0.015, r, world, buckets[r]))
        parts = []
        for o, t in enumerate(shards):
            keys = torch.cat([buckets[r][o, :int(walks[r][1][o])] for r in range(world)])
            # the key call completes each shard's frame; the walk state is per table
            parts.append(P.integrate_depth_keys(t, keys))
        for k in PARTITIONED:
            assert sum(getattr(p, k) for p in parts) == getattr(s_full, k), (i, k)
        for k in INVARIANT:
            assert all(getattr(w[0], k) == getattr(s_full, k) for w in walks), (i, k)
        if (i + 1) % 10 == 0:
            m = P.apply_merges(full, 2.5e-5).merged
            assert sum(P.apply_merges(t, 2.5e-5).merged for t in shards) == m
    for level in range(2):
        co, _, ts, w, s2, col = full.export_level(level)
        rows = {}
        for r, t in enumerate(shards):
            c2, _, t2, w2, s22, col2 = t.export_level(level)
            assert np.all(owner_of_coords(c2, world) == r)
            for j, c in enumerate(map(tuple, c2.tolist())):
                rows[c] = (t2[j], w2[j], s22[j], col2[j])
        assert set(rows) == set(map(tuple, co.tolist()))
        for j, c in enumerate(map(tuple, co.tolist())):
            a = rows[c]
            assert np.array_equal(a[0], ts[j]) and np.array_equal(a[1], w[j])
            assert np.array_equal(a[2], s2[j]) and np.array_equal(a[3], col[j])


def test_ray_sharded_keys_need_walk_and_routing():
    """integrate_depth_keys without a preceding walk is an error, and a key
    routed to a shard that does not own it is rejected."""
    import torch
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.sharding import owner_of_keys, pack_keys
    t = P.HashTable(100003, 10, 7, 0.04, (10000, 1000))
    t.set_shard(0, 2)
    dev = torch.device("cuda", 0)
    with pytest.raises(ValueError):
        P.integrate_depth_keys(t, torch.zeros(1, dtype=torch.int64, device=dev))
    f = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 1, 64, 48, depth_dtype=np.float32)[0]
    b = torch.zeros((2, t.slots), dtype=torch.int64, device=dev)
    P.integrate_depth_walk(t, f, 0.015, 0, 1, b)
    coords = np.array([[i, 0, 0] for i in range(64)])
    keys = pack_keys(coords)
    foreign = keys[owner_of_keys(keys, 2) == 1][:1].astype(np.int64)
    with pytest.raises(ValueError):
        P.integrate_depth_keys(t, torch.as_tensor(foreign, device=dev))


@pytest.mark.parametrize("all_levels", [False, True])
def test_depth_window_equals_batch_then_merge(all_levels):
    """integrate_depth_window (frames + merge pass, one host sync) ==
    integrate_depth_batch followed by apply_merges, window after window."""
    import paper_2511_21459_b200 as P
    frames = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 30, 160, 120, depth_dtype=np.float32,
                                   color_dtype=np.uint8)
    caps = (100000, 20000, 5000)
    a = P.HashTable(1000003, 10, 7, 0.04, caps)
    b = P.HashTable(1000003, 10, 7, 0.04, caps)
    for w in range(3):
        win = frames[10 * w:10 * (w + 1)]
        sa, ma = P.integrate_depth_window(a, win, 0.015, 2.5e-5, all_levels=all_levels)
        sb = P.integrate_depth_batch(b, win, 0.015)
        mb = P.apply_merges(b, 2.5e-5, all_levels=all_levels)
        assert [vars(x) for x in sa] == [vars(x) for x in sb]
        assert (ma.candidates, ma.merged) == (mb.candidates, mb.merged)
    assert PU.state_digest(PU.GpuBackend.state(type("x", (), {"t": a})())) == \
        PU.state_digest(PU.GpuBackend.state(type("x", (), {"t": b})()))


def test_merge_heap_exhaustion_changes_nothing():
    """A merge pass whose candidates do not fit the coarse heap raises
    CapacityError and moves nothing (adapt.py / the device check)."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.errors import CapacityError
    b, _, _, _ = PU.run_depth_scenario("gpu", "sphere", 20, 48, 36, 0.08, 0.03, (20000, 3), 100003)
    t = b.t
    before = PU.state_digest(PU.GpuBackend.state(type("x", (), {"t": t})()))
    assert len(P.select_merge_candidates(t, 2.5e-4)) > 3
    with pytest.raises(CapacityError):
        P.apply_merges(t, 2.5e-4)
    assert PU.state_digest(PU.GpuBackend.state(type("x", (), {"t": t})())) == before


def test_depth_batch_equals_per_frame_and_oracle():
    """integrate_depth_batch (one host sync per merge window) == per-frame calls == oracle."""
    import paper_2511_21459_b200 as P
    frames = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 20, 160, 120, depth_dtype=np.float32,
                                   color_dtype=np.uint8)
    a = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000, 5000))
    b = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000, 5000))
    o = PU.OracleBackend(1000003, 0.04, (100000, 20000, 5000))
    for w in range(2):
        win = frames[10 * w:10 * (w + 1)]
        sa = P.integrate_depth_batch(a, win, 0.015)
        sb = [P.integrate_depth(b, f, 0.015) for f in win]
        so = [o.depth(f, 0.015) for f in win]
        assert [x.__dict__ for x in sa] == [x.__dict__ for x in sb]
        assert [{k: getattr(x, k) for k in PU.STAT_KEYS} for x in sa] == so
        ma = P.apply_merges(a, 2.5e-5, all_levels=True)
        mb = P.apply_merges(b, 2.5e-5, all_levels=True)
        mo = o.merge(2.5e-5, all_levels=True)
        assert (ma.candidates, ma.merged) == (mb.candidates, mb.merged) == (mo["candidates"], mo["merged"])
    ga = PU.GpuBackend.state(type("x", (), {"t": a})())
    assert PU.state_digest(ga) == PU.state_digest(o.state())


def test_depth_batch_capacity_error_stops_at_failing_frame():
    import paper_2511_21459_b200 as P
    frames = __import__("paper_2511_21459_b200.synth", fromlist=["x"]).render_frames("room", 4, 64, 48)
    t = P.HashTable(100003, 10, 7, 0.08, (700, 10))
    single = P.HashTable(100003, 10, 7, 0.08, (700, 10))
    n_ok = 0
    for f in frames:
        try:
            P.integrate_depth(single, f, 0.03)
            n_ok += 1
        except P.CapacityError:
            break
    assert n_ok < len(frames)
    with pytest.raises(P.CapacityError):
        P.integrate_depth_batch(t, frames, 0.03)
    assert t.key_levels() == single.key_levels()


def test_merge_memo_respects_parameter_changes():
    """Dirty-block merge passes must equal full evaluation, including when the
    parameters change between passes (then every block is re-evaluated)."""
    spec = ("sphere", 30, 48, 36, 0.08, 0.03, (20000, 10000, 4000), 100003)
    schedule = [(1e-6, False), (2.5e-4, False), (2.5e-4, True), (2.5e-3, True), (2.5e-3, True)]
    results = {}
    for name in ("gpu", "oracle"):
        from paper_2511_21459_b200 import synth
        b = PU.BACKENDS[name](spec[7], spec[4], spec[6])
        seq = synth.render_frames(spec[0], spec[1], spec[2], spec[3])
        out = []
        for i, f in enumerate(seq):
            b.depth(f, spec[5])
            if (i + 1) % 6 == 0:
                sigma, al = schedule[(i + 1) // 6 - 1]
                out.append(b.merge(sigma, all_levels=al))
        results[name] = (out, PU.state_digest(b.state()))
    assert results["gpu"] == results["oracle"]


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_extraction_equals_single_gpu(world):
    """Mesh extraction over block-key shards: the shards'
    blocks gathered as reference block records into one table extract the
    single-GPU mesh bit for bit (with and without vertex collapse)."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    from paper_2511_21459_b200.sharding import shard_records, table_from_records
    frames = synth.render_frames("room", 20, 128, 96, depth_dtype=np.float32, color_dtype=np.uint8)
    full = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000, 5000))
    shards = []
    for r in range(world):
        t = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000, 5000))
        t.set_shard(r, world)
        shards.append(t)
    for i, f in enumerate(frames):
        for t in [full] + shards:
            P.integrate_depth(t, f, 0.015)
        if (i + 1) % 10 == 0:
            for t in [full] + shards:
                P.apply_merges(t, 2.5e-5, all_levels=True)
    assert full.heaps[1].occupied > 0
    g = table_from_records([shard_records(t) for t in shards], full)
    for eps in (None, 0.0025):
        a, b = P.extract_mesh(full, collapse_epsilon=eps), P.extract_mesh(g, collapse_epsilon=eps)
        assert a.num_triangles > 1000
        for x, y in ((a.vertices, b.vertices), (a.normals, b.normals), (a.colors, b.colors),
                     (a.triangles, b.triangles)):
            assert np.array_equal(x, y)


def test_coordinates_beyond_the_packed_key_range_fail_cleanly():
    """Block coordinates are packed 21 bits per axis (+-2^20 blocks, +-84 km
    at 8 cm blocks); a measurement beyond that is a ValueError and leaves
    the table as it was (the reference's int64 keys have no such limit,
    DESIGN.md §3)."""
    import paper_2511_21459_b200 as P
    t = P.HashTable(100003, 10, 7, 0.08, (20000, 1000))
    near = P.PointCloudFrame(points=np.array([[0.5, 0.1, 0.2], [1.0, -0.4, 0.3]]), pose=P.SensorPose.identity())
    P.integrate_pointcloud(t, near, 0.04)
    before = PU.state_digest(PU.GpuBackend.state(type("x", (), {"t": t})()))
    far = P.PointCloudFrame(points=np.array([[0.5, 0.1, 0.2], [9.0e4, 0.0, 0.0]]), pose=P.SensorPose.identity())
    with pytest.raises(ValueError, match="21-bit"):
        P.integrate_pointcloud(t, far, 0.04)
    assert PU.state_digest(PU.GpuBackend.state(type("x", (), {"t": t})())) == before
    frame = _frame(P, np.full((8, 8), 1.0), pose=P.SensorPose(np.eye(3), [9.0e4, 0.0, 0.0]))
    with pytest.raises(ValueError, match="21-bit"):
        P.integrate_depth(t, frame, 0.04)
    assert PU.state_digest(PU.GpuBackend.state(type("x", (), {"t": t})())) == before


@pytest.mark.parametrize("weight_cap,color", [(3.0, False), (2.5, True)])
def test_lidar_weight_cap_hot_segments_vs_oracle(weight_cap, color):
    """A dense scan (hot segments of > 1024 rays near the sensor take the
    ray-parallel path) with an integral and a non-integral weight cap, with
    and without colour: every compile-time variant of the hot apply against
    the oracle (integrate.py:113-116)."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    scan = synth.lidar_frames(1, 96, 1536)[0]
    if color:
        scan.colors = np.random.default_rng(7).integers(0, 256, (len(scan.points), 3)).astype(np.uint8)
    g = PU.GpuBackend(2000003, 1.6, (300000, 20000))
    o = PU.OracleBackend(2000003, 1.6, (300000, 20000))
    for _ in range(2):  # twice: the cap binds on the second pass
        assert g.points(scan, 0.8, weight_cap=weight_cap) == o.points(scan, 0.8, weight_cap=weight_cap)
    assert_states_match(g.state(), o.state())
    w = g.state()[0][2]
    assert w.max() == weight_cap


def test_lidar_chunked_mode_within_tolerance_vs_oracle():
    """TSDF_LIDAR_CHUNKED (hot blocks folded in 512-ray groups, merged by
    Chan's formula) against the ORDERED oracle over 4 full config-3 scans with
    colour and two merge passes: counters, block keys, levels and weights
    exact; TSDF / variance within the north star's 1e-4 relative; colour
    within 1e-4; the level audit empty (integrate.py:92-119, adapt.py:41-72)."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    scans = synth.lidar_frames(4, 128, 2048)
    rng = np.random.default_rng(11)
    for s in scans:
        s.colors = rng.integers(0, 256, (len(s.points), 3)).astype(np.uint8)
    caps, nh = (500000, 60000), 4000037
    g = PU.GpuBackend(nh, 1.6, caps)
    g.t.set_lidar_mode("chunked")
    o = PU.OracleBackend(nh, 1.6, caps)
    for i, s in enumerate(scans):
        assert g.points(s, 0.8) == o.points(s, 0.8)
        if i % 2 == 1:
            assert g.merge(1e-2) == o.merge(1e-2)
    a, b = g.state(), o.state()
    assert set(a) == set(b)
    diff = 0
    for level in a:
        ca, ta, wa, sa, cola = a[level]
        cb, tb, wb, sb, colb = b[level]
        assert np.array_equal(ca, cb), f"level {level}: block keys differ"
        assert np.array_equal(wa, wb), f"level {level}: weights differ"
        assert np.all(np.abs(ta - tb) <= TOL_REL * np.abs(tb) + 1e-7 * 0.8)
        assert np.all(np.abs(sa - sb) <= TOL_REL * np.abs(sb) + 1e-10 * 0.64 * wb)
        assert np.all(np.abs(cola - colb) <= 1e-4)
        diff += int(np.count_nonzero(ta != tb))
    assert diff > 0, "chunked mode did not engage (no hot block differs from the ordered chain)"
    assert g.t.merge_audit() == 0
    g.close()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_halo_extraction_equals_single_gpu(world):
    """Sharded extraction with a one-block halo (
    sharding.extract_mesh_halo): each shard meshes a contiguous run of the
    kept list's 256-block chunks from its slab + halo, one rank dedups and
    collapses the concatenated raw output -- the single-GPU mesh bit for bit
    on a three-level map (with and without vertex collapse)."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    from paper_2511_21459_b200.sharding import extract_mesh_halo_local
    frames = synth.render_frames("room", 20, 128, 96, depth_dtype=np.float32, color_dtype=np.uint8)
    caps = (100000, 20000, 5000)
    full = P.HashTable(1000003, 10, 7, 0.04, caps)
    shards = []
    for r in range(world):
        t = P.HashTable(1000003, 10, 7, 0.04, caps)
        t.set_shard(r, world)
        shards.append(t)
    for i, f in enumerate(frames):
        for t in [full] + shards:
            P.integrate_depth(t, f, 0.015)
        if (i + 1) % 10 == 0:
            for t in [full] + shards:
                P.apply_merges(t, 2.5e-5, all_levels=True)
    assert full.heaps[1].occupied > 0 and full.heaps[2].occupied > 0
    for eps in (None, 0.0025):
        a = P.extract_mesh(full, collapse_epsilon=eps)
        b, plan = extract_mesh_halo_local(shards, collapse_epsilon=eps)
        assert a.num_triangles > 1000
        assert sum(1 for e in plan["emit"] if len(e["keys"])) == min(world, plan["chunks"])
        for x, y in ((a.vertices, b.vertices), (a.normals, b.normals), (a.colors, b.colors),
                     (a.triangles, b.triangles)):
            assert np.array_equal(x, y)
    # each rank moved its slab + halo, not the map
    need = sum(len(n) for n in plan["need"])
    assert need < 2.0 * full.live_count()


@pytest.mark.parametrize("world", [1, 2, 3])
def test_sharded_window_union_equals_single_gpu(world):
    """Ray-sharded merge windows (integrate_depth_window_sharded
    with its collectives as tensor plumbing): the pixel passes split the
    lock-step span by tile, the caps are max-reduced, every shard walks its
    rays of all frames, one exchange routes the keys, each shard inserts and
    updates frame by frame and merges -- the union equals the single-GPU
    window bit for bit, with identical per-frame stats and merge counts."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    from paper_2511_21459_b200.sharding import integrate_depth_window_local
    frames = synth.render_frames("room", 20, 128, 96, depth_dtype=np.float32, color_dtype=np.uint8)
    caps = (100000, 20000, 5000)
    full = P.HashTable(1000003, 10, 7, 0.04, caps)
    shards = []
    for r in range(world):
        t = P.HashTable(1000003, 10, 7, 0.04, caps)
        t.set_shard(r, world)
        shards.append(t)
    for w0 in (0, 10):
        win = frames[w0:w0 + 10]
        sf, mf = P.integrate_depth_window(full, win, 0.015, 2.5e-5, all_levels=True)
        ss, ms, need = integrate_depth_window_local(shards, win, 0.015, 2.5e-5, all_levels=True,
                                                    bucket_cap=200000)
        assert need <= 200000
        keys = PU.STAT_KEYS
        assert [{k: getattr(s, k) for k in keys} for s in ss] == [{k: getattr(s, k) for k in keys} for s in sf]
        assert (ms.candidates, ms.merged) == (mf.candidates, mf.merged)
    assert full.heaps[1].occupied > 0
    for l in range(full.num_levels):
        ref = full.export_level(l)
        parts = [s.export_level(l) for s in shards]
        uc = np.concatenate([p[0] for p in parts])
        order = np.lexsort((uc[:, 2], uc[:, 1], uc[:, 0]))
        assert np.array_equal(uc[order], ref[0])
        for i in (2, 3, 4, 5):
            assert np.array_equal(np.concatenate([p[i] for p in parts])[order], ref[i])


def test_heap_snapshots_are_cached_per_map_version():
    """heaps[l].tsdf & co. (read-only host snapshots) are exported once per
    map change (tsdf_table_version), not on every attribute read."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    f = synth.render_frames("room", 2, 64, 48)
    t = P.HashTable(100003, 10, 7, 0.08, (20000, 1000))
    P.integrate_depth(t, f[0], 0.03)
    v0 = t.version
    a, b = t.heaps[0].tsdf, t.heaps[0].weight
    # the same export each time (fresh write-through views over one buffer)
    assert np.shares_memory(t.heaps[0].tsdf, a) and np.shares_memory(t.heaps[0].weight, b)
    assert t.version == v0
    P.integrate_depth(t, f[1], 0.03)
    assert t.version > v0
    a2 = t.heaps[0].tsdf
    assert not np.shares_memory(a2, a) and not np.array_equal(a2, a)
    t.remove(tuple(t.heaps[0].coords[np.nonzero(t.heaps[0].live)[0][0]]))
    assert t.heaps[0].occupied == int(t.heaps[0].live.sum())


def _handles(backend):
    if backend.name == "oracle":
        return {l: backend.t.live_blocks(l) for l in range(backend.t.num_levels)}
    out = {}
    for l in range(backend.t.num_levels):
        coords, handles = backend.t.export_level(l)[:2]
        out[l] = (coords, handles)
    return out


@pytest.mark.parametrize("kind", ["depth", "lidar"])
def test_heap_handles_follow_the_references_allocation_order(kind):
    """New blocks take heap handles in ascending (x, y, z) order (the
    reference's np.unique + _ensure_blocks, integrate.py:203 / :289) and a
    merge pass re-homes candidates in the same order (adapt.py:130-135), so
    the heap layout -- not just the canonical state -- equals the oracle's,
    and two runs give the same layout (the reference's deterministic rerun,
    tests/test_integrate.py:273-288)."""
    if kind == "depth":
        spec = dict(scene="sphere", frames=20, width=64, height=48, edge=0.08, tau=0.03,
                    caps=(30000, 10000), n_hash=100003, sigma=2.5e-4, cadence=10)
        runs = [PU.run_depth_scenario(b, **spec) for b in ("gpu", "gpu", "oracle")]
    else:
        spec = dict(scans=3, beams=32, columns=256, edge=1.6, tau=0.8, caps=(200000, 20000),
                    n_hash=1000003, sigma=1e-2, cadence=2)
        runs = [PU.run_lidar_scenario(b, **spec) for b in ("gpu", "gpu", "oracle")]
    assert runs[0][1] == runs[2][1] and runs[0][2] == runs[2][2]
    assert sum(m["merged"] for m in runs[2][2]) > 0
    h = [_handles(r[0]) for r in runs]
    for l in h[2]:
        for a, b in ((h[0], h[2]), (h[1], h[2])):
            assert np.array_equal(a[l][0], b[l][0]), f"level {l} coords"
            assert np.array_equal(a[l][1], b[l][1]), f"level {l} handles"


def test_heap_voxel_arrays_write_through_like_the_reference():
    """heaps[l].tsdf[a:b] = x (how the reference's own tests craft fields,
    tests/test_meshing.py:22-39) writes the touched live blocks to the
    device; the other fields of those blocks are untouched; writing a slot
    that holds no live block is refused; derived views are read-only."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    f = synth.render_frames("room", 1, 64, 48)[0]
    t = P.HashTable(100003, 10, 7, 0.08, (20000, 1000))
    P.integrate_depth(t, f, 0.03)
    heap = t.heaps[0]
    h = int(np.nonzero(heap.live)[0][3])
    coord = tuple(int(v) for v in heap.coords[h])
    before = t.payload(coord)
    lo, n = h * heap.nvox, heap.nvox
    vals = np.linspace(-0.02, 0.02, n)
    heap.tsdf[lo:lo + n] = vals
    after = t.payload(coord)
    assert np.array_equal(after.tsdf, vals)
    assert np.array_equal(after.weight, before.weight) and np.array_equal(after.s2, before.s2)
    assert np.array_equal(t.heaps[0].tsdf[lo:lo + n], vals)
    heap.weight[lo + 5] = 7.0
    assert t.payload(coord).weight[5] == 7.0 and np.array_equal(t.payload(coord).tsdf, vals)
    heap.color[lo:lo + n] = 0.5
    assert np.all(t.payload(coord).color == 0.5)
    dead = int(np.nonzero(~t.heaps[0].live)[0][0])
    with pytest.raises(ValueError):
        t.heaps[0].tsdf[dead * n] = 1.0
    with pytest.raises(ValueError):
        t.heaps[0].tsdf[lo:lo + n][0] = 1.0
    cp = t.heaps[0].tsdf.copy()
    cp[0] = 3.0  # a copy is an ordinary array


def test_heap_payload_by_handle_and_probe_length():
    """BlockHeap.payload / write_payload by handle (hashgrid.py:115-133) and
    HashTable.probe_length (hashgrid.py:194-212): a handle addresses the
    same block as its coordinate; a free handle reads as zeros and cannot be
    written; n_hash >= 4x live blocks keeps mean probes <= 2 (the
    reference's own bound, tests/test_hashgrid.py:220-230)."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.hashgrid import BlockPayload
    rng = np.random.default_rng(100)
    t = P.HashTable(4099, 10, 7, 0.08, (600, 8))
    seen, coords = set(), []
    while len(coords) < 600:
        c = tuple(int(v) for v in rng.integers(-1000, 1000, size=3))
        if c not in seen:
            seen.add(c)
            coords.append(c)
    for c in coords:
        t.insert(c, 0)
    probes = t.probe_lengths(coords)
    assert probes.min() >= 1 and probes.mean() <= 2.0
    assert t.probe_length(coords[7]) == probes[7]
    heap = t.heaps[0]
    h, lv = t.find(coords[5])
    assert lv == 0
    p = heap.payload(h)
    assert p.coord == coords[5] and p.level == 0 and not p.tsdf.any()
    new = BlockPayload(coord=coords[5], level=0, tsdf=np.full(heap.nvox, 0.01),
                       weight=np.full(heap.nvox, 2.0), s2=np.zeros(heap.nvox),
                       color=np.full((heap.nvox, 3), 0.25, dtype=np.float32))
    heap.write_payload(h, new)
    back = t.payload(coords[5])
    assert np.array_equal(back.tsdf, new.tsdf) and np.array_equal(back.weight, new.weight)
    t.remove(coords[9])
    free_h = int(np.nonzero(~t.heaps[0].live)[0][0])
    assert not t.heaps[0].payload(free_h).tsdf.any()
    with pytest.raises(ValueError):
        t.heaps[0].write_payload(free_h, new)


def test_c5_two_million_point_scan_vs_oracle():
    """BASELINE config 5's LiDAR part: one 128 x 16384-column scan (~2 M
    returns, 100 m range, 1.6 m blocks) against the oracle -- stats and the
    full state bit-identical in the ordered mode, and the chunked mode
    within the north star's tolerance with exact keys and weights."""
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    scan = synth.lidar_frames(1, 128, 16384)[0]
    assert len(scan.points) > 1_800_000
    caps, nh = (600000, 20000), 8000009
    o = PU.OracleBackend(nh, 1.6, caps)
    so = o.points(scan, 0.8)
    ref = o.state()
    g = PU.GpuBackend(nh, 1.6, caps)
    assert g.points(scan, 0.8) == so
    assert_states_match(g.state(), ref)
    g.close()
    c = PU.GpuBackend(nh, 1.6, caps)
    c.t.set_lidar_mode("chunked")
    assert c.points(scan, 0.8) == so
    assert_states_match(c.state(), ref, exact=False)
    c.close()


def test_c5_1024x768_depth_frames_vs_oracle():
    """BASELINE config 5's depth part: the first frames of the large-room
    sweep at 1024 x 768, 5 mm voxels, f32 depth + u8 colour, a merge pass at
    all levels -- bit-identical to the oracle."""
    from paper_2511_21459_b200 import synth
    frames = synth.render_frames("large_room", 2, 1024, 768, depth_dtype=np.float32,
                                 color_dtype=np.uint8, sweep=500)
    caps, nh = (300000, 30000, 5000), 8000009
    res = []
    for b in (PU.GpuBackend(nh, 0.04, caps), PU.OracleBackend(nh, 0.04, caps)):
        st = [b.depth(f, 0.015) for f in frames]
        ms = b.merge(2.5e-5, all_levels=True)
        res.append((st, ms, b.state()))
    assert res[0][0] == res[1][0] and res[0][1] == res[1][1]
    assert res[0][0][0]["measurements"] > 700000
    assert_states_match(res[0][2], res[1][2])


def test_walk_cluster_dsmem_filter_matches_oracle():
    """The depth walk launched as 4-CTA thread-block clusters
    (TSDF_WALK_CLUSTER=4): the cluster-wide first-sighting filter in
    distributed shared memory leaves the allocation bit-identical (a fresh
    process, since the launch shape is read once)."""
    import os
    import subprocess
    import sys
    code = (
        "import sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "import numpy as np, parity_utils as PU\n"
        "spec = dict(scene='large_room', frames=3, width=160, height=120, edge=0.04, tau=0.015,\n"
        "            caps=(400000, 10000, 4000), n_hash=1000003, sigma=2.5e-5, cadence=3, all_levels=True,\n"
        "            depth_dtype=np.float32, color_dtype=np.uint8)\n"
        "g, sg, mg, _ = PU.run_depth_scenario('gpu', **spec)\n"
        "o, so, mo, _ = PU.run_depth_scenario('oracle', **spec)\n"
        "assert sg == so and mg == mo\n"
        "assert PU.state_digest(g.state()) == PU.state_digest(o.state())\n"
        "print('ok', sg[0]['blocks_allocated'])\n") % (str(PU.ROOT), str(PU.ROOT / "tests"))
    env = dict(os.environ, TSDF_WALK_CLUSTER="4")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
