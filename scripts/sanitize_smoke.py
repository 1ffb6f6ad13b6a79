"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): depth window with merges (3 levels), the ray-sharded walk/keys
split, a LiDAR scan, the capacity tier (evict / import / key pass), and mesh
extraction, u16 depth, the NN metrics and the quadtree -- every kernel
family of the library, at sizes the sanitizer
finishes in minutes.

    compute-sanitizer --tool memcheck python scripts/sanitize_smoke.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_21459_b200 as P  # noqa: E402
from paper_2511_21459_b200 import synth  # noqa: E402,F401


def main():
    frames = P.synth.render_frames("room", 12, 64, 48, depth_dtype=np.float32, color_dtype=np.uint8)
    t = P.HashTable(100003, 10, 7, 0.08, (20000, 10000, 4000))
    st, ms = P.integrate_depth_window(t, frames[:6], 0.03, 2.5e-4, all_levels=True)
    st2, ms2 = P.integrate_depth_window(t, frames[6:], 0.03, 2.5e-4, all_levels=True)
    print("depth window", sum(s.voxels_updated for s in st + st2), ms.merged + ms2.merged)
    m = P.extract_mesh(t, 0.0, 0.0025)
    print("mesh", m.num_vertices, m.num_triangles)
    # ray-sharded split on 2 shard tables of one device
    import torch
    shards = []
    for r in range(2):
        s = P.HashTable(100003, 10, 7, 0.08, (20000, 10000))
        s.set_shard(r, 2)
        shards.append(s)
    dev = torch.device("cuda", 0)
    b = [torch.zeros((2, s.slots), dtype=torch.int64, device=dev) for s in shards]
    w = [P.integrate_depth_walk(s, frames[0], 0.03, r, 2, b[r]) for r, s in enumerate(shards)]
    for o, s in enumerate(shards):
        keys = torch.cat([b[r][o, :int(w[r][1][o])] for r in range(2)])
        P.integrate_depth_keys(s, keys)
    print("sharded ok")
    # LiDAR
    pts = P.synth.lidar_frames(1, 16, 128)[0]
    tl = P.HashTable(1000003, 10, 7, 1.6, (40000, 1000))
    print("lidar", P.integrate_pointcloud(tl, pts, 0.8).observations)
    # raw uint16 depth scaled on the device
    raw = [P.DepthFrame(np.clip(np.round(np.nan_to_num(f.depth.astype(np.float64)) * 5000), 0, 65535)
                        .astype(np.uint16), f.intrinsics, f.pose, color=f.color, depth_scale=5000.0)
           for f in frames[:3]]
    tu = P.HashTable(100003, 10, 7, 0.08, (20000, 10000))
    print("u16", sum(s.voxels_updated for s in P.integrate_depth_batch(tu, raw, 0.03)))
    # nearest-neighbour metrics and the quadtree / splat seeding
    from paper_2511_21459_b200.metrics import eval_reconstruction
    ref = np.random.default_rng(0).uniform(-2, 2, (5000, 3))
    print("metrics", round(eval_reconstruction(m, ref, 0.1, samples_per_m2=2000)["fscore"], 4))
    leaves = P.build_quadtree(np.asarray(frames[0].color, dtype=np.float64) / 255.0, 1e-5, 1)
    print("quadtree", len(leaves), len(P.seed_splats(leaves, frames[0])))
    if "--no-engine" in sys.argv:
        return
    # capacity tier
    cfg = P.PipelineConfig(sensor_mode="depth", nu_fine=0.01, block_edge=0.08, tau=0.04,
                           n_hash=100003, heap_capacity_fine=1501, heap_capacity_coarse=1001,
                           fill_threshold=0.85, low_water=0.7)
    eng = P.FusionEngine(cfg)
    for f in frames:
        eng.integrate_frame(f)
        eng.maybe_merge()
        eng.maybe_stream()
    print("engine evicted", eng.evicted_blocks, "archived", len(eng.archive))


if __name__ == "__main__":
    main()
