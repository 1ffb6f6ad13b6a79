"""Time mesh extraction of the bench's room map: wall clock, per-kernel
CUDA-event times and the host copy-out.  python scripts/probe_extract.py"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    import bench
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import _native as N, meshing
    wl = bench.WORKLOADS["room"]
    frames = bench.make_frames(wl, 60)
    t = bench.make_table(P, wl, stream=torch.cuda.current_stream().cuda_stream)
    for w in range(6):
        bench.window_and_merge(P, t, wl, frames[10 * w:10 * w + 10])
    eps = 0.25 * wl["edge"] / 8
    P.extract_mesh(t, 0.0, eps)
    torch.cuda.synchronize()
    t.profile(True)
    t.kernel_times(reset=True)
    t0 = time.perf_counter()
    m = N.MeshC()
    N.check(N.lib().tsdf_extract_mesh(t._h, 0.0, eps, __import__("ctypes").byref(m)), "x")
    t1 = time.perf_counter()
    mesh = meshing._mesh_from_c(m)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    mesh2 = P.extract_mesh(t, 0.0, eps)
    t4 = time.perf_counter()
    assert mesh2.num_triangles == mesh.num_triangles
    print(f"public extract_mesh (two-phase): {1e3 * (t4 - t3):.2f} ms")
    kt = t.kernel_times(reset=True)
    print(f"c call {1e3 * (t1 - t0):.2f} ms, copy-out {1e3 * (t2 - t1):.2f} ms, "
          f"{mesh.num_vertices} v {mesh.num_triangles} t, blocks {[h.occupied for h in t.heaps]}")
    for k, (ms, n) in sorted(kt.items(), key=lambda kv: -kv[1][0]):
        print(f"  {k:28s} {ms:8.3f} ms x{n}")


if __name__ == "__main__":
    main()
