"""Where an extract_mesh call's wall time goes on the room map: the device
pass (tsdf_extract_mesh_begin) vs the D2H into the caller's arrays."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2511_21459_b200 as P  # noqa: E402
from paper_2511_21459_b200 import _native as N  # noqa: E402

wl = bench.WORKLOADS["room"]
frames = bench.gen_frames("room", 30)
t = bench.make_table(P, wl)
for w in range(3):
    bench.window_and_merge(P, t, wl, frames[10 * w:10 * w + 10])
L = N.lib()
for rep in range(3):
    nv, nt = C.c_int64(), C.c_int64()
    t0 = time.perf_counter()
    N.check(L.tsdf_extract_mesh_begin(t._h, 0.0, 0.00125, C.byref(nv), C.byref(nt)), "begin")
    t1 = time.perf_counter()
    v, n, c = (np.empty((nv.value, 3)) for _ in range(3))
    tri = np.empty((nt.value, 3), dtype=np.int64)
    t2 = time.perf_counter()
    N.check(L.tsdf_extract_mesh_read(t._h, v.ctypes.data, n.ctypes.data, c.ctypes.data, tri.ctypes.data), "read")
    t3 = time.perf_counter()
    print(f"begin {1e3*(t1-t0):.2f} ms  alloc {1e3*(t2-t1):.2f} ms  read {1e3*(t3-t2):.2f} ms  "
          f"({nv.value} v, {nt.value} t)")
t.profile(True)
t.kernel_times(reset=True)
N.check(L.tsdf_extract_mesh_begin(t._h, 0.0, 0.00125, C.byref(nv), C.byref(nt)), "begin")
kt = t.kernel_times(reset=True)
print({k: round(v[0], 3) for k, v in sorted(kt.items(), key=lambda kv: -kv[1][0])})
print("sum", round(sum(v[0] for v in kt.values()), 3))
