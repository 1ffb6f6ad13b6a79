"""Time eval_reconstruction (GPU nearest-neighbour queries) against the
reference's cKDTree path on the same inputs: the room map's mesh sampled at
the reference's default density (1e5 / m^2, capped at 1 M) against 1 M
reference points back-projected from the frames.  Prints one JSON line.

    python scripts/bench_metrics.py [--frames 20]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=20)
    args = ap.parse_args()
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    from paper_2511_21459_b200.metrics import eval_reconstruction, nn_distance, sample_mesh_points
    frames = synth.render_frames("room", args.frames, 640, 480, depth_dtype=np.float32,
                                 color_dtype=np.uint8)
    t = P.HashTable(1000003, 10, 7, 0.04, (400000, 100000))
    for f in frames:
        P.integrate_depth(t, f, 0.015)
    mesh = P.extract_mesh(t)
    uu, vv = np.meshgrid(np.arange(640.0), np.arange(480.0))
    ref = []
    for f in frames:
        d = np.asarray(f.depth, dtype=np.float64)
        ok = np.isfinite(d) & (d > 0)
        ref.append(f.pose.to_world(P.backproject(uu[ok], vv[ok], d[ok], f.intrinsics)))
    ref = np.concatenate(ref)
    ref = ref[np.random.default_rng(0).choice(len(ref), min(len(ref), 1_000_000), replace=False)]
    samples = sample_mesh_points(mesh)
    nn_distance(ref[:1000], samples[:1000])  # warm-up (context, pool)
    t0 = time.perf_counter()
    d_sr = nn_distance(ref, samples)
    d_rs = nn_distance(samples, ref)
    gpu_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    got = eval_reconstruction(mesh, ref, 0.1)
    total_s = time.perf_counter() - t0
    out = {"n_samples": len(samples), "n_reference": len(ref), "gpu_nn_both_ways_s": round(gpu_s, 4),
           "eval_reconstruction_s": round(total_s, 4), "fscore": got["fscore"],
           "chamfer_l1": got["chamfer_l1"]}
    try:
        from scipy.spatial import cKDTree
        t0 = time.perf_counter()
        c_sr = cKDTree(ref).query(samples, k=1)[0]
        c_rs = cKDTree(samples).query(ref, k=1)[0]
        out["ckdtree_both_ways_s"] = round(time.perf_counter() - t0, 4)
        out["bit_identical_to_ckdtree"] = bool(np.array_equal(c_sr, d_sr) and np.array_equal(c_rs, d_rs))
    except ImportError:
        out["ckdtree_both_ways_s"] = None
    print(json.dumps(out))


if __name__ == "__main__":
    main()
