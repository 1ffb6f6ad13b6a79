"""world_size-2 gloo test of the multi-GPU host logic on CPU: frame broadcast,
block-key ownership partition and the stats all-reduce.  Each rank plays a
shard by filtering the oracle's per-block results through owner_of (the
device kernel applies the same predicate); the reduced counters and the
union of shard key sets must equal the single-process run."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_21459_b200 import synth
    from paper_2511_21459_b200.sharding import broadcast_frame, combine_stats, owner_of_coords
    from paper_2511_21459_b200.integrate import IntegrationStats
    import parity_utils as PU
    frames = synth.render_frames("room", 3, 64, 48, depth_dtype=np.float32) if rank == 0 else [None] * 3
    oracle = PU.OracleBackend(100003, 0.08, (20000, 1000))
    out = []
    prev = {}
    for f in frames:
        g = broadcast_frame(f, dist, torch)
        st = oracle.depth(g, 0.03)
        state = oracle.state()
        coords, tsdf, w, s2, col = state[0]
        mine = owner_of_coords(coords, world) == rank
        # per-shard partitioned counters: voxels whose weight changed this frame
        cur = {tuple(c): wb for c, wb in zip(coords.tolist(), w)}
        upd = sum(int(np.sum(cur[c] != prev.get(c, np.zeros_like(cur[c]))))
                  for c, m in zip(map(tuple, coords.tolist()), mine) if m)
        part = IntegrationStats(measurements=st["measurements"], skipped_invalid=st["skipped_invalid"],
                                voxels_updated=upd, observations=upd,
                                blocks_touched=int(mine.sum()), blocks_allocated=0)
        red = combine_stats(part, dist, torch)
        out.append((st, red.voxels_updated, red.measurements, red.blocks_touched, int(len(coords))))
        prev = cur
    q.put((rank, out))
    dist.destroy_process_group()


def test_two_rank_partition_and_reduce():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for (st0, vox0, meas0, touched0, live0), (st1, vox1, _, touched1, _) in zip(res[0], res[1]):
        assert st0 == st1                      # both ranks saw the same broadcast frame
        assert vox0 == vox1 == st0["voxels_updated"]   # shard sums == whole frame
        assert meas0 == st0["measurements"]
        assert touched0 == touched1 == live0   # every live block owned exactly once


def _exchange_worker(rank, world, port, q):
    """Ray-sharded key exchange (sharding.exchange_keys) with the oracle as
    the walk: rank r takes the tiles t % world == r of a frame, emits the
    blocks its rays cross (the oracle's DDA rows) into per-owner buckets,
    and after the all-to-all every rank must hold exactly the frame's keys
    that it owns."""
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_21459_b200 import synth
    from paper_2511_21459_b200.sharding import exchange_keys, owner_of_keys, pack_keys
    from oracle.oracle import oracle_dda_blocks_batch
    f = synth.render_frames("room", 1, 48, 32, depth_dtype=np.float32)[0]
    H, W = f.depth.shape
    # back-project + segment ends as integrate.py:278-286 (host numpy, small case)
    v, u = np.mgrid[0:H, 0:W]
    z = f.depth.astype(np.float64)
    ok = np.isfinite(z) & (z > 0)
    k = f.intrinsics
    pc = np.stack([(u - k.cx) / k.fx * z, (v - k.cy) / k.fy * z, z], -1)[ok]
    tile = ((v // 16) * ((W + 15) // 16) + (u // 16))[ok]
    pw = pc @ f.pose.rotation.T + f.pose.translation
    ray = pw - f.pose.translation
    e = pw + 0.015 * ray / np.linalg.norm(ray, axis=1)[:, None]
    mine = tile % world == rank
    o = np.repeat(f.pose.translation[None], len(e), 0)
    # one lock-step batch over the whole frame (its global cap), then this
    # rank's rays' rows
    ids, rows_all = oracle_dda_blocks_batch(o, e, 0.04)
    rows_mine = rows_all[mine[ids]]
    keys = np.unique(pack_keys(rows_mine))
    own = owner_of_keys(keys, world)
    cap = max(1, len(keys))
    buckets = torch.zeros((world, cap), dtype=torch.int64)
    counts = np.zeros(world, dtype=np.int64)
    for r in range(world):
        sel = keys[own == r].astype(np.int64)
        buckets[r, :len(sel)] = torch.from_numpy(sel)
        counts[r] = len(sel)
    recv = exchange_keys(buckets, counts, dist, torch)
    got = set(np.unique(recv.numpy().astype(np.uint64)).tolist())
    allk = np.unique(pack_keys(rows_all))
    want = set(allk[owner_of_keys(allk, world) == rank].tolist())
    q.put((rank, got == want, len(want)))
    dist.destroy_process_group()


def test_two_rank_ray_sharded_key_exchange():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (ok, n)) for r, ok, n in (q.get(timeout=300) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok and n > 0 for ok, n in res.values())


def _broadcast_worker(rank, world, port, q):
    """broadcast_frame keeps every array's element type and bits: f64 and
    f32 depth, raw u16 depth with its scale, u8 / f64 colour, f32 points."""
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_21459_b200 import DepthFrame, synth
    from paper_2511_21459_b200.sharding import broadcast_frame
    from dataset_utils import SCALE, raw_depth
    d64 = synth.render_frames("room", 1, 40, 30)[0]
    d32 = synth.render_frames("room", 1, 40, 30, depth_dtype=np.float32, color_dtype=np.uint8)[0]
    raw = DepthFrame(raw_depth(d32.depth), d32.intrinsics, d32.pose, color=d32.color,
                     depth_scale=SCALE)
    pts = synth.lidar_frames(1, 8, 64)[0]
    pts.colors = np.arange(3 * len(pts.points), dtype=np.int64).reshape(-1, 3).astype(np.uint8)
    ok = []
    for f in (d64, d32, raw, pts):
        g = broadcast_frame(f if rank == 0 else None, dist, torch)
        a, b = (f.points, g.points) if hasattr(f, "points") else (f.depth, g.depth)
        ca, cb = (f.colors, g.colors) if hasattr(f, "points") else (f.color, g.color)
        same = (a.dtype == b.dtype and np.array_equal(a, b, equal_nan=True)
                and ca.dtype == cb.dtype and np.array_equal(ca, cb)
                and np.array_equal(f.pose.rotation, g.pose.rotation)
                and np.array_equal(f.pose.translation, g.pose.translation))
        if hasattr(f, "depth"):
            same = same and g.depth_scale == f.depth_scale and g.intrinsics == f.intrinsics
        ok.append(bool(same))
    q.put((rank, ok))
    dist.destroy_process_group()


def test_two_rank_frame_broadcast_keeps_types():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_broadcast_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1] == [True] * 4


def _gather_worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_21459_b200.sharding import _gather_bytes
    blob = bytes(range(rank * 7 % 256)) * (rank + 1)  # rank 0 sends nothing
    got = _gather_bytes(blob, 1, dist, torch)
    q.put((rank, got))
    dist.destroy_process_group()


def test_three_rank_variable_size_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] is None and res[2] is None
    assert res[1] == [bytes(range(r * 7 % 256)) * (r + 1) for r in range(3)]


def _bytes_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2511_21459_b200.sharding import _all_gather_bytes, all_to_all_bytes
    sends = [bytes([rank, d]) * (3 * d + rank + 1) for d in range(world)]
    got = all_to_all_bytes(sends, dist, torch)
    allg = _all_gather_bytes(bytes([rank]) * (rank + 2), dist, torch)
    q.put((rank, got, allg))
    dist.destroy_process_group()


def test_halo_extraction_byte_collectives_gloo():
    """The two variable-size collectives of extract_mesh_halo (all-to-all of
    block records, all-gather of block summaries) on world 3 over gloo."""
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 3
    ps = [ctx.Process(target=_bytes_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, got, allg = q.get(timeout=120)
        res[r] = (got, allg)
    for p in ps:
        p.join(timeout=60)
    for r in range(world):
        got, allg = res[r]
        assert got == [bytes([o, r]) * (3 * r + o + 1) for o in range(world)]
        assert allg == [bytes([o]) * (o + 2) for o in range(world)]


def test_mesh_plan_partitions_the_kept_list():
    """mesh_plan (pure host logic): the 27-neighbourhood kept test against a
    direct evaluation, chunk runs that tile the kept list on 256-block
    boundaries, and halos that hold every live neighbour of a rank's run."""
    import numpy as np
    from paper_2511_21459_b200.sharding import mesh_plan, pack_keys, unpack_keys
    rng = np.random.default_rng(3)
    coords = np.unique(rng.integers(-12, 12, size=(6000, 3)), axis=0)
    keys = pack_keys(coords)
    n = len(keys)
    summ = {"keys": keys, "levels": rng.integers(0, 2, n).astype(np.int32),
            "obs": (rng.random(n) < 0.9).astype(np.uint8),
            "lo": rng.uniform(-0.05, 0.02, n), "hi": rng.uniform(-0.02, 0.05, n)}
    parts = [{k: v[i::3] for k, v in summ.items()} for i in range(3)]
    plan = mesh_plan(parts, 4, 0.0, 2)
    # direct kept test
    idx = {tuple(c): i for i, c in enumerate(coords.tolist())}
    kept = set()
    for i, c in enumerate(coords.tolist()):
        if not summ["obs"][i]:
            continue
        lo, hi = np.inf, -np.inf
        for d in np.ndindex(3, 3, 3):
            j = idx.get((c[0] + d[0] - 1, c[1] + d[1] - 1, c[2] + d[2] - 1))
            if j is not None and summ["obs"][j]:
                lo, hi = min(lo, summ["lo"][j]), max(hi, summ["hi"][j])
        if lo <= 0.0 <= hi:
            kept.add(int(keys[i]))
    emitted = np.concatenate([e["keys"] for e in plan["emit"]])
    assert set(emitted.tolist()) == kept and len(emitted) == len(kept) == plan["kept"]
    level_of = dict(zip(keys.tolist(), summ["levels"].tolist()))
    for l in range(2):
        lvl = np.sort(np.array([k for k in kept if level_of[k] == l], dtype=np.uint64))
        got = np.concatenate([e["keys"][sum(e["level_counts"][:l]):sum(e["level_counts"][:l + 1])]
                              for e in plan["emit"]])
        assert np.array_equal(got, lvl)
        starts = np.cumsum([0] + [e["level_counts"][l] for e in plan["emit"]])[:-1]
        assert all(s % 256 == 0 or s == len(lvl) for s in starts)
    live = set(keys.tolist())
    for e, need in zip(plan["emit"], plan["need"]):
        nd = set(need.tolist())
        for c in unpack_keys(e["keys"]):
            for d in np.ndindex(3, 3, 3):
                k = int(pack_keys((c + np.array(d) - 1)[None])[0])
                if k in live:
                    assert k in nd


def test_mesh_plan_empty_and_sparse_maps():
    """mesh_plan on an empty map and on a map whose bounding box is too large
    for the dense index grid (binary-search fallback): same plan shape."""
    import numpy as np
    from paper_2511_21459_b200.sharding import mesh_plan, pack_keys
    empty = {"keys": np.zeros(0, np.uint64), "levels": np.zeros(0, np.int32), "obs": np.zeros(0, np.uint8),
             "lo": np.zeros(0), "hi": np.zeros(0)}
    p = mesh_plan([empty, empty], 3, 0.0, 2)
    assert p["kept"] == 0 and all(len(e["keys"]) == 0 for e in p["emit"]) and all(len(n) == 0 for n in p["need"])
    # two clusters of blocks ~1e6 blocks apart: the grid would be too large
    c = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [900000, 5, 5], [900001, 5, 5]], dtype=np.int64)
    s = {"keys": pack_keys(c), "levels": np.zeros(5, np.int32), "obs": np.ones(5, np.uint8),
         "lo": np.full(5, -0.01), "hi": np.full(5, 0.01)}
    p = mesh_plan([s], 2, 0.0, 2)
    assert p["kept"] == 5
    got = set(np.concatenate([e["keys"] for e in p["emit"]]).tolist())
    assert got == set(pack_keys(c).tolist())
    assert set(np.concatenate(p["need"]).tolist()) == got
