"""Where a merge window's time goes on the host: Python preparation before
the C call, the C call (enqueue + the single sync), and the device time of
the window (CUDA events), on the bench's room workload.  Prints JSON.

    python scripts/probe_window_overhead.py
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import _native as N
    wl = bench.WORKLOADS["room"]
    frames = bench.make_frames(wl, 80)
    dev = [(torch.as_tensor(f[0]).cuda(), torch.as_tensor(f[1]).cuda()) for f in frames]
    stream = torch.cuda.current_stream()
    t = bench.make_table(P, wl, stream=stream.cuda_stream)
    L = N.lib()
    orig = L.tsdf_integrate_depth_window
    marks = {}

    def wrapped(*a):
        marks["c_in"] = time.perf_counter()
        r = orig(*a)
        marks["c_out"] = time.perf_counter()
        return r
    L.tsdf_integrate_depth_window = wrapped
    rows = []
    torch.cuda.synchronize()
    for w in range(8):
        frs = frames[10 * w:10 * (w + 1)]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        bench.window_and_merge(P, t, wl, frs, dev[10 * w:10 * (w + 1)])
        h1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        rows.append({"py_prep_us": (marks["c_in"] - h0) * 1e6, "c_call_us": (marks["c_out"] - marks["c_in"]) * 1e6,
                     "py_post_us": (h1 - marks["c_out"]) * 1e6, "device_us": e0.elapsed_time(e1) * 1e3})
    L.tsdf_integrate_depth_window = orig
    med = {k: float(np.median([r[k] for r in rows[2:]])) for k in rows[0]}
    print(json.dumps({"median": med, "rows": rows}))




def profile_prep():
    """cProfile of the host side of 20 windows (python scripts/probe_window_overhead.py prof)."""
    import cProfile
    import pstats
    import torch
    import bench
    import paper_2511_21459_b200 as P
    wl = bench.WORKLOADS["room"]
    frames = bench.make_frames(wl, 40)
    dev = [(torch.as_tensor(f[0]).cuda(), torch.as_tensor(f[1]).cuda()) for f in frames]
    t = bench.make_table(P, wl, stream=torch.cuda.current_stream().cuda_stream)
    for w in range(2):
        bench.window_and_merge(P, t, wl, frames[10 * w:10 * w + 10], dev[10 * w:10 * w + 10])
    pr = cProfile.Profile()
    pr.enable()
    for w in range(20):
        k = w % 4
        bench.window_and_merge(P, t, wl, frames[10 * k:10 * k + 10], dev[10 * k:10 * k + 10])
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)


if __name__ == "__main__" and sys.argv[1:] == ["prof"]:
    profile_prep()
    sys.exit(0)


if __name__ == "__main__":
    main()
