import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import bench
import paper_2511_21459_b200 as P
wl = bench.WORKLOADS["lidar"]
frames = bench.make_frames(wl, 3)
t = bench.make_table(P, wl)
t.profile(True); t.kernel_times(reset=True)
d, c, pose, intr = frames[0]
s = P.integrate_pointcloud(t, P.PointCloudFrame(points=d, pose=pose), wl["tau"])
kt = t.kernel_times(reset=True)
w = np.concatenate([t.export_level(l)[3].reshape(-1) for l in range(t.num_levels)])
print("obs", s.observations, "max W", w.max(), "p99.99", np.percentile(w[w>0], 99.99), "voxels", (w>0).sum())
print({k: round(v[0], 3) for k, v in kt.items()})
# chain bound: max W * ~5 dependent FP64 ops * ~8 cycles at 1.965 GHz
print("chain bound ms (40 cyc/obs):", w.max() * 40 / 1.965e9 * 1e3)
