"""compute-sanitizer workload for the kernels added late in round 2: the
mirrored-key walk with its min(L1, cap) budget, canonical heap-handle order
(k_new_canonical for new blocks, k_rank_keys + k_permute_by_rank for merge
candidates), the single-block fast path (k_locate, k_block_gather /
k_block_scatter, small-find read-back), k_probe_length, and the write-through
heap arrays.

    compute-sanitizer --tool memcheck python scripts/sanitize_session3.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2511_21459_b200 as P  # noqa: E402
from paper_2511_21459_b200 import synth  # noqa: E402


def main():
    # depth: single calls, then a window, then merges (3 levels)
    frames = synth.render_frames("sphere", 20, 64, 48, depth_dtype=np.float32, color_dtype=np.uint8)
    t = P.HashTable(100003, 10, 7, 0.08, (30000, 10000, 4000))
    for f in frames[:10]:
        P.integrate_depth(t, f, 0.03)
    ms0 = P.apply_merges(t, 2.5e-4, all_levels=True)
    from paper_2511_21459_b200.integrate import integrate_depth_window
    _, ms = integrate_depth_window(t, frames[10:], 0.03, 2.5e-4, all_levels=True)
    print("depth", t.live_count(), ms0.merged, ms.merged)
    assert ms0.merged > 0 and ms.merged > 0
    # LiDAR (walk with near pairs; 64-bit keys)
    scan = synth.lidar_frames(1, 16, 256)[0]
    tl = P.HashTable(1000003, 10, 7, 1.6, (100000, 10000))
    st = P.integrate_pointcloud(tl, scan, 0.8)
    print("lidar", st.blocks_allocated, st.observations)
    # single-block API
    coords = [(i, -2 * i, 3) for i in range(40)]
    for c in coords:
        t.insert(c, 0)
    print("probes", t.probe_lengths(coords).max(), t.probe_length((999, 999, 999)))
    h, lv = t.find(coords[3])
    pay = t.heaps[lv].payload(h)
    pay.tsdf[:] = 0.01
    pay.weight[:] = 1.0
    t.heaps[lv].write_payload(h, pay)
    back = t.payload(coords[3])
    assert np.all(back.tsdf == 0.01)
    removed = t.remove(coords[4])
    assert removed.coord == coords[4]
    heap = t.heaps[0]
    h5 = t.find(coords[5])[0]
    heap.tsdf[h5 * heap.nvox:(h5 + 1) * heap.nvox] = 0.02
    assert np.all(t.payload(coords[5]).tsdf == 0.02)
    print("single-block ok", t.live_count())
    t.close()
    tl.close()


if __name__ == "__main__":
    main()
