"""compute-sanitizer workload for the kernels added in round 2: the LiDAR
chunked mode (hot mask with FP32-certain gating, partial states, Chan
combine, the reciprocal table), the ray-sharded merge window (pixel passes
with split spans, cap plumbing, bucket walk, window inserts and updates),
the halo mesh extraction (block summary, slot lookup, raw emission, the
dedup/collapse finish, the non-destructive block gather) and the ordered
LiDAR update with integral-weight quotients.

    compute-sanitizer --tool memcheck python scripts/sanitize_round2.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_21459_b200 as P  # noqa: E402
from paper_2511_21459_b200 import synth  # noqa: E402
from paper_2511_21459_b200.sharding import (extract_mesh_halo_local,  # noqa: E402
                                            integrate_depth_window_local)


def main():
    # LiDAR, both modes, colour, a merge
    scans = synth.lidar_frames(2, 32, 512)
    rng = np.random.default_rng(1)
    for s in scans:
        s.colors = rng.integers(0, 256, (len(s.points), 3)).astype(np.uint8)
    for mode in ("ordered", "chunked"):
        t = P.HashTable(1000003, 10, 7, 1.6, (200000, 20000))
        t.set_lidar_mode(mode)
        obs = sum(P.integrate_pointcloud(t, s, 0.8).observations for s in scans)
        ms = P.apply_merges(t, 1e-2)
        print("lidar", mode, obs, ms.merged, t.merge_audit())
        t.close()
    # sharded merge windows (world 2) and the halo extraction
    frames = synth.render_frames("room", 10, 64, 48, depth_dtype=np.float32, color_dtype=np.uint8)
    shards = []
    for r in range(2):
        t = P.HashTable(100003, 10, 7, 0.08, (20000, 10000, 4000))
        t.set_shard(r, 2)
        shards.append(t)
    st, ms, need = integrate_depth_window_local(shards, frames, 0.03, 2.5e-4, all_levels=True,
                                                bucket_cap=20000)
    print("window", sum(s.voxels_updated for s in st), ms.merged, need)
    mesh, plan = extract_mesh_halo_local(shards, collapse_epsilon=0.0025)
    print("halo mesh", mesh.num_vertices, mesh.num_triangles, plan["chunks"])
    from paper_2511_21459_b200.meshing import block_summary
    summ = block_summary(shards[0])
    own0 = summ["keys"][summ["levels"] == 0][:4]
    blk = shards[0].read_blocks(0, own0) if len(own0) else None
    print("read_blocks", None if blk is None else blk[0].shape)


if __name__ == "__main__":
    main()
