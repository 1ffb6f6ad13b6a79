"""ShardedFusion end to end in real processes: two
ranks over gloo sharing cuda:0 -- frame broadcast, ray-sharded allocation
with the key all-to-all, the stats all-reduce, merges and the halo mesh
extraction -- against a single-process FusionEngine on the same frames.
The union of the shards' block keys, levels and voxel state and the mesh
must be bit-identical."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import os
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import parity_utils as PU
        from paper_2511_21459_b200 import PipelineConfig, synth
        from paper_2511_21459_b200.sharding import ShardedFusion
        cfg = PipelineConfig(nu_fine=0.005, block_edge=0.04, tau=0.015, n_hash=1000003,
                             heap_capacity_fine=100000, heap_capacity_coarse=20000,
                             heap_capacity_extra=(5000,), merge_all_levels=True, merge_cadence=10)
        torch.cuda.set_device(0)
        sf = ShardedFusion(cfg, device=torch.device("cuda", 0))
        frames = synth.render_frames("room", 20, 128, 96, depth_dtype=np.float32, color_dtype=np.uint8)
        stats, merged = [], 0
        for f in frames:
            st = sf.integrate_frame(f if rank == 0 else None)
            stats.append({k: getattr(st, k) for k in PU.STAT_KEYS})
            merged += sf.maybe_merge()
        mesh = sf.extract()
        state = {l: tuple(sf.engine.table.export_level(l)[i] for i in (0, 2, 3, 4, 5))
                 for l in range(sf.engine.table.num_levels)}
        q.put((rank, stats, merged, state,
               None if mesh is None else (mesh.vertices, mesh.normals, mesh.colors, mesh.triangles)))
    except Exception as e:  # surface the error in the parent
        import traceback
        q.put((rank, "error", traceback.format_exc(), None, None))
    finally:
        dist.destroy_process_group()


def test_sharded_engine_two_ranks_equals_single_gpu():
    import multiprocessing as mp
    import socket
    import parity_utils as PU
    from paper_2511_21459_b200 import FusionEngine, PipelineConfig, synth
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
    for r in res.values():
        assert r[1] != "error", r[2]
    # single-process reference run of the same engine configuration
    cfg = PipelineConfig(nu_fine=0.005, block_edge=0.04, tau=0.015, n_hash=1000003,
                         heap_capacity_fine=100000, heap_capacity_coarse=20000,
                         heap_capacity_extra=(5000,), merge_all_levels=True, merge_cadence=10)
    eng = FusionEngine(cfg)
    frames = synth.render_frames("room", 20, 128, 96, depth_dtype=np.float32, color_dtype=np.uint8)
    stats, merged = [], 0
    for f in frames:
        st = eng.integrate_frame(f)
        stats.append({k: getattr(st, k) for k in PU.STAT_KEYS})
        merged += eng.maybe_merge()
    assert merged > 0
    for r in range(world):
        assert res[r][1] == stats, f"rank {r} stats"
        assert res[r][2] == merged
    # union of the shards == the single table, level by level
    for l in range(eng.table.num_levels):
        coords, _, t, w, s2, col = eng.table.export_level(l)
        parts = [res[r][3][l] for r in range(world)]
        uc = np.concatenate([p[0] for p in parts])
        order = np.lexsort((uc[:, 2], uc[:, 1], uc[:, 0]))
        assert np.array_equal(uc[order], coords)
        for i, ref in zip(range(1, 5), (t, w, s2, col)):
            assert np.array_equal(np.concatenate([p[i] for p in parts])[order], ref)
    m = eng.extract()
    got = res[0][4]
    assert res[1][4] is None and m.num_triangles > 100
    for x, y in zip(got, (m.vertices, m.normals, m.colors, m.triangles)):
        assert np.array_equal(x, y)


def _window_worker(rank, world, port, q):
    import os
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import parity_utils as PU
        import paper_2511_21459_b200 as P
        from paper_2511_21459_b200 import synth
        from paper_2511_21459_b200.sharding import integrate_depth_window_sharded
        torch.cuda.set_device(0)
        t = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000, 5000))
        t.set_shard(rank, world)
        t._win_cap = 256  # start small: the first window must re-walk with room
        frames = synth.render_frames("room", 20, 128, 96, depth_dtype=np.float32, color_dtype=np.uint8)
        out = []
        for w0 in (0, 10):
            st, ms = integrate_depth_window_sharded(t, frames[w0:w0 + 10], 0.015, dist, torch,
                                                    device=torch.device("cuda", 0),
                                                    sigma_threshold=2.5e-5, all_levels=True)
            out.append(([{k: getattr(s, k) for k in PU.STAT_KEYS} for s in st], (ms.candidates, ms.merged)))
        state = {l: tuple(t.export_level(l)[i] for i in (0, 2, 3, 4, 5)) for l in range(t.num_levels)}
        q.put((rank, out, state, getattr(t, "_win_rewalks", 0)))
    except Exception:
        import traceback
        q.put((rank, "error", traceback.format_exc(), None))
    finally:
        dist.destroy_process_group()


def test_sharded_windows_two_ranks_equal_single_gpu():
    """integrate_depth_window_sharded over real collectives (gloo, two ranks
    sharing cuda:0): capped-span pixel passes + MAX all-reduce, bucket sizing
    with a re-walk, the all-to-all, per-frame inserts/updates, merges and the
    counter all-reduce -- equal to the single-GPU windows bit for bit."""
    import multiprocessing as mp
    import socket
    import parity_utils as PU
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    ps = [ctx.Process(target=_window_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for p in ps:
        p.join(timeout=60)
    for r in res.values():
        assert r[1] != "error", r[2]
    full = P.HashTable(1000003, 10, 7, 0.04, (100000, 20000, 5000))
    frames = synth.render_frames("room", 20, 128, 96, depth_dtype=np.float32, color_dtype=np.uint8)
    ref = []
    for w0 in (0, 10):
        st, ms = P.integrate_depth_window(full, frames[w0:w0 + 10], 0.015, 2.5e-5, all_levels=True)
        ref.append(([{k: getattr(s, k) for k in PU.STAT_KEYS} for s in st], (ms.candidates, ms.merged)))
    for r in range(world):
        assert res[r][1] == ref
        assert res[r][3] == 1  # the first window re-walked once with room, the second fit
    for l in range(full.num_levels):
        coords, _, t, w, s2, col = full.export_level(l)
        parts = [res[r][2][l] for r in range(world)]
        uc = np.concatenate([p[0] for p in parts])
        order = np.lexsort((uc[:, 2], uc[:, 1], uc[:, 0]))
        assert np.array_equal(uc[order], coords)
        for i, a in zip(range(1, 5), (t, w, s2, col)):
            assert np.array_equal(np.concatenate([p[i] for p in parts])[order], a)
