"""Benchmark of the B200 TSDF-fusion hot path (BASELINE.json metric).

Workload (N=1): BASELINE config 2 -- synthetic indoor room, 640x480 RGB-D
(f32 depth + u8 RGB, 7 B/px), 3 resolution levels 5/10/20 mm (labelled
multi-level merge extension), the SURVEY §8d "large room" (6 x 5 x 3 m,
12 spheres) swept by the reference's yaw/pitch trajectory over 500 frames.
One step = one merge window: 10 frames integrated + one merge pass
(merge_cadence = 10).  value = integrated Mpoints/s (valid depth pixels /
device time), inputs resident in HBM; e2e = the same through the public
API from pinned host buffers (H2D inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload room|lidar]

Multi-GPU (torchrun, one rank per GPU): block-key-hash sharding -- every
rank sees the same frames and owns 1/N of the blocks; depth frames split
the full-ray DDA across ranks and route the keys to their owners with one
all-to-all per frame (strong scaling of a fixed frame stream); time = max
over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "room": dict(kind="depth", scene="large_room", width=640, height=480, edge=0.04, tau=0.015,
                 sigma=2.5e-5, caps=(1_500_000, 300_000, 100_000), n_hash=4_000_037,
                 cadence=10, frames_total=500,
                 name="large room 6x5x3 m, 640x480 RGB-D (f32 depth + u8 RGB), 3 levels 5/10/20 mm, "
                      "500-frame sweep, merge every 10 frames"),
    # BASELINE config 4: fixed 5 mm, single level (no merges), large hash
    # table and a ~100 GB level-0 heap (the hash-capacity / memory stress)
    "room_fixed5mm": dict(kind="depth", scene="large_room", width=640, height=480, edge=0.04,
                          tau=0.015, sigma=5e-324, caps=(6_000_000,), n_hash=16_000_057,
                          cadence=10, frames_total=500,
                          name="large room 6x5x3 m, 640x480 RGB-D, fixed 5 mm single level "
                               "(merges off), 6M-block (98 GB) heap, 16M-slot hash"),
    # BASELINE config 5 (depth part): 1024x768 frames of the large room
    "room1024": dict(kind="depth", scene="large_room", width=1024, height=768, edge=0.04,
                     tau=0.015, sigma=2.5e-5, caps=(2_500_000, 500_000, 150_000),
                     n_hash=8_000_009, cadence=10, frames_total=500,
                     name="large room 6x5x3 m, 1024x768 RGB-D, 3 levels 5/10/20 mm, "
                          "merge every 10 frames"),
    "lidar": dict(kind="lidar", beams=128, columns=2048, edge=1.6, tau=0.8, sigma=1e-2,
                  caps=(1_500_000, 200_000, 50_000), n_hash=4_000_037, cadence=10, step_m=0.5,
                  lidar_mode="chunked",
                  name="128-beam x 2048-column LiDAR, 100 m range, 0.2/0.4/0.8 m levels, "
                       "sensor advancing 0.5 m/scan, merge every 10 scans; hot blocks in chunked "
                       "mode (Chan-merged 512-ray partial states, TSDF/variance within 1e-4)"),
}
# the same stream with every voxel's observations applied in ray order
# (bit-identical to the reference); reported inside the lidar line
WORKLOADS["lidar_ordered"] = dict(WORKLOADS["lidar"], lidar_mode="ordered",
                                  name="128-beam x 2048-column LiDAR as `lidar`, every voxel "
                                       "applying its observations in ray order (bit-identical)")
ORACLE_OF = {"lidar_ordered": "lidar"}  # workloads sharing an oracle run
METRIC = {"room": "integrated Mpoints/s (640x480 RGB-D room, 3 levels)",
          "room_fixed5mm": "integrated Mpoints/s (640x480 RGB-D room, fixed 5 mm)",
          "room1024": "integrated Mpoints/s (1024x768 RGB-D room, 3 levels)",
          "lidar": "integrated Mpoints/s (128-beam LiDAR)",
          "lidar_ordered": "integrated Mpoints/s (128-beam LiDAR, ray-ordered hot blocks)"}
FRAMES_PER_STEP = int(os.environ.get("TSDF_BENCH_WINDOW", "10"))  # = merge cadence
# in-process parity sample per workload: (frames, merge cadence).  Room: two
# full merge windows (20 frames, 2 passes at 3 levels); LiDAR: 4 scans with a
# merge pass every 2 (the oracle needs ~12 s per 128x2048 scan)
PARITY = {"room": (20, 10), "room1024": (20, 10), "room_fixed5mm": (20, 10), "lidar": (4, 2),
          "lidar_ordered": (4, 2)}
TOL_REL = 1e-4  # north-star TSDF / variance tolerance (chunked LiDAR parity)
LIDAR_STEPS = 5  # timed windows of the N=1 LiDAR sub-run (10 scans each)
S_IN = {"depth": 7, "lidar": 12}  # algorithmic input bytes per measurement


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    every ~2 ms (the timed region is tens of ms), nvidia-smi as fallback."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        self.index = index
        self.rows = []  # (sm_mhz, max_mhz, [4 reason flags])
        self._stop = threading.Event()
        self._ready = threading.Event()  # set once the first sample is in

    def _run_nvml(self, nv):
        h = nv.nvmlDeviceGetHandleByIndex(self.index)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        while not self._stop.is_set():
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append((float(sm), float(mx), [bool(r & b) for b in bits]))
            self._ready.set()
            self._stop.wait(0.002)

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                r = [x.strip() for x in out.split(",")]
                if len(r) >= 6 and r[0].replace(".", "").isdigit():
                    self.rows.append((float(r[0]), float(r[1]), [x == "Active" for x in r[2:6]]))
                    self._ready.set()
            except Exception:
                pass
            self._stop.wait(0.2)

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            try:
                self.source = "nvml"
                self._run_nvml(nv)
            finally:
                nv.nvmlShutdown()
        except Exception:
            self.source = "nvidia-smi"
            self._run_smi()

    def __enter__(self):
        # NVML initialisation can take longer than a short timed region: the
        # region starts only after the sampler has its first reading
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        self._ready.wait(timeout=10.0)
        return self

    def __exit__(self, *a):
        self._stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(r[0] for r in self.rows),
                "sm_max_mhz": max(r[1] for r in self.rows),
                "reasons": sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2][i]}),
                "samples": len(self.rows), "source": getattr(self, "source", "?")}


def make_frames(wl, n, start=0):
    from paper_2511_21459_b200 import synth
    if wl["kind"] == "depth":
        scene = synth.make_scene(wl["scene"])
        intr = synth.default_intrinsics("room", wl["width"], wl["height"])
        poses = synth.trajectory(synth.Scene("room"), wl["frames_total"])
        out = []
        for i in range(start, start + n):
            d, c = synth.render_depth(scene, poses[i % len(poses)], intr, wl["width"], wl["height"])
            out.append((d.astype(np.float32), np.round(c * 255.0).astype(np.uint8),
                        poses[i % len(poses)], intr))
        return out
    scene = synth.make_lidar_scene()
    dirs = synth.lidar_directions(wl["beams"], wl["columns"])
    from paper_2511_21459_b200.geometry import SensorPose
    out = []
    for i in range(start, start + n):
        org = np.array([wl["step_m"] * i, 0.0, 0.0])
        out.append((synth.lidar_scan(scene, org, dirs), None, SensorPose(np.eye(3), org), None))
    return out


def _gen_one(a):
    name, i = a
    return make_frames(WORKLOADS[name], 1, i)[0]


def gen_frames(name, n, start=0):
    """make_frames on a process pool (rendering is per-frame independent)."""
    import multiprocessing as mp
    procs = max(1, min(n, 32, (os.cpu_count() or 1) - 2))
    if n <= 4 or procs == 1:
        return make_frames(WORKLOADS[name], n, start)
    with mp.get_context("fork").Pool(procs) as pool:
        return pool.map(_gen_one, [(name, i) for i in range(start, start + n)],
                        chunksize=max(1, n // (4 * procs)))


def n_meas(fr):
    d = fr[0]
    return int(np.count_nonzero(np.isfinite(d) & (d > 0))) if d.ndim == 2 else int(len(d))


def make_table(P, wl, stream=None, shard=None):
    t = P.HashTable(wl["n_hash"], 10, 7, wl["edge"], wl["caps"], stream=stream)
    if shard:
        t.set_shard(*shard)
    if wl.get("lidar_mode"):
        t.set_lidar_mode(wl["lidar_mode"])
    return t


def integrate(P, t, wl, fr, device=None):
    d, c, pose, intr = fr
    if wl["kind"] == "depth":
        f = P.DepthFrame(depth=d if device is None else device[0], intrinsics=intr, pose=pose,
                         color=c if device is None else device[1])
        return P.integrate_depth(t, f, wl["tau"])
    f = P.PointCloudFrame(points=d if device is None else device[0], pose=pose)
    return P.integrate_pointcloud(t, f, wl["tau"])


_MULTI = {}  # set under torchrun: {"dist", "torch", "device"} for ray-sharded depth frames


def window(P, t, wl, frs, dev=None):
    """One merge window through the public API: depth frames go through
    integrate_depth_batch (one host sync per window), scans per scan.  On
    N > 1 GPUs depth frames use ray-sharded allocation: each rank walks 1/N
    of the rays, one all-to-all routes the block keys to their owners, and
    each rank updates the blocks it owns (sharding.integrate_depth_raysharded)."""
    if wl["kind"] == "depth" and _MULTI:
        from paper_2511_21459_b200.sharding import integrate_depth_raysharded
        out = []
        for i, fr in enumerate(frs):
            f = P.DepthFrame(depth=fr[0] if dev is None else dev[i][0], intrinsics=fr[3], pose=fr[2],
                             color=fr[1] if dev is None else dev[i][1])
            out.append(integrate_depth_raysharded(t, f, wl["tau"], _MULTI["dist"], _MULTI["torch"],
                                                  device=_MULTI["device"]))
        return out
    if wl["kind"] == "depth":
        fs = [P.DepthFrame(depth=fr[0] if dev is None else dev[i][0], intrinsics=fr[3], pose=fr[2],
                           color=fr[1] if dev is None else dev[i][1]) for i, fr in enumerate(frs)]
        return P.integrate_depth_batch(t, fs, wl["tau"])
    return [integrate(P, t, wl, fr, None if dev is None else dev[i]) for i, fr in enumerate(frs)]


def window_and_merge(P, t, wl, frs, dev=None):
    """One step: a merge window plus its merge pass.  Depth windows go
    through integrate_depth_window (frames + merge pass enqueued together,
    one host synchronisation) or, on N GPUs, integrate_depth_window_sharded;
    scans through window() + apply_merges."""
    if wl["kind"] == "depth":
        fs = [P.DepthFrame(depth=fr[0] if dev is None else dev[i][0], intrinsics=fr[3], pose=fr[2],
                           color=fr[1] if dev is None else dev[i][1]) for i, fr in enumerate(frs)]
        if _MULTI:
            # ray-sharded merge window: 3 collectives per window, no per-frame host sync
            from paper_2511_21459_b200.sharding import integrate_depth_window_sharded
            stats, ms = integrate_depth_window_sharded(t, fs, wl["tau"], _MULTI["dist"], _MULTI["torch"],
                                                       device=_MULTI["device"], sigma_threshold=wl["sigma"],
                                                       all_levels=True)
            return stats, ms.merged
        stats, ms = P.integrate_depth_window(t, fs, wl["tau"], wl["sigma"], all_levels=True)
        return stats, ms.merged
    stats = window(P, t, wl, frs, dev)
    return stats, P.apply_merges(t, wl["sigma"], all_levels=True).merged


def kernel_bytes(stats_list, wl):
    """Algorithmic bytes: B = s_in*P + 16*T + 16*A + 48*U per frame."""
    s_in = S_IN[wl["kind"]]
    P_ = sum(s.measurements for s in stats_list)
    T_ = sum(s.blocks_touched for s in stats_list)
    A_ = sum(s.blocks_allocated for s in stats_list)
    U_ = sum(s.voxels_updated for s in stats_list)
    return {"path": s_in * P_ + 16 * T_ + 16 * A_ + 48 * U_,
            "update": 48 * U_ + 16 * T_,          # voxel RMW + hash-entry reads
            "alloc": s_in * P_ + 16 * T_ + 16 * A_,  # frame read + entry probes/writes
            "P": P_, "T": T_, "A": A_, "U": U_}


KERNEL_ROLE = {"k_depth_update": "update", "k_lidar_update": "update", "k_dda_walk": "alloc"}


def run_b200(name, W, K, rank, world, dist, torch, frames=None):
    """The B200 arm on workload `name`: W warm-up windows, K timed windows
    (inputs resident in HBM), K profiled windows, then the e2e run."""
    import paper_2511_21459_b200 as P
    wl = WORKLOADS[name]
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1))
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    shard = (rank, world) if world > 1 else None
    if world > 1:
        _MULTI.update(dist=dist, torch=torch, device=dev)
    nfr = FRAMES_PER_STEP * (W + 2 * K)  # warm-up, timed, then profiled windows
    if frames is None or len(frames) < nfr:
        t0 = time.time()
        frames = gen_frames(name, nfr)
        log(f"[bench] generated {nfr} {name} frames in {time.time() - t0:.1f}s")
    # device-resident inputs
    dframes = []
    for d, c, _, _ in frames:
        dframes.append((torch.from_numpy(d).to(dev), None if c is None else torch.from_numpy(c).to(dev)))
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # 256 MB > 126 MB L2

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- value: inputs resident in HBM -----------------------------------
    with torch.cuda.stream(stream):
        table = make_table(P, wl, stream=stream, shard=shard)
    all_stats, step_ms, merged = [], [], 0
    fi = 0
    for s in range(W):
        window_and_merge(P, table, wl, frames[fi:fi + FRAMES_PER_STEP],
                         dframes[fi:fi + FRAMES_PER_STEP])
        fi += FRAMES_PER_STEP
    launches0 = table.kernel_launches
    barrier()
    sampler = ClockSampler(dev.index)
    with sampler:
        for s in range(K):
            flush.fill_(s & 0xFF)  # L2 flush between timed steps (outside the events)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            st_, m_ = window_and_merge(P, table, wl, frames[fi:fi + FRAMES_PER_STEP],
                                       dframes[fi:fi + FRAMES_PER_STEP])
            all_stats += st_
            merged += m_
            fi += FRAMES_PER_STEP
            e1.record(stream)
            e1.synchronize()
            step_ms.append(e0.elapsed_time(e1))
    barrier()
    launches = table.kernel_launches - launches0
    # per-kernel CUDA-event breakdown on the next K windows (outside the
    # timed region: the events themselves perturb the step time)
    table.profile(True)
    table.kernel_times(reset=True)
    table.work_totals(reset=True)
    prof_stats = []
    for s in range(K):
        flush.fill_(s & 0xFF)
        torch.cuda.synchronize()
        prof_stats += window_and_merge(P, table, wl, frames[fi:fi + FRAMES_PER_STEP],
                                       dframes[fi:fi + FRAMES_PER_STEP])[0]
        fi += FRAMES_PER_STEP
    torch.cuda.synchronize()
    ktimes = table.kernel_times(reset=True)
    work = table.work_totals(reset=True)
    table.profile(False)
    occ = [h.occupied for h in table.heaps]
    # mesh extraction of the final map (reported separately):
    # one warm-up, then one timed call through the public API (device
    # kernels + D2H of the mesh), eps = 0.25 * nu_fine as FusionEngine uses
    extract = None
    if wl["kind"] == "depth":
        eps = 0.25 * wl["edge"] / 8
        if world > 1:
            # the whole map's mesh from the shards: spatial chunk runs + halo
            from paper_2511_21459_b200.sharding import extract_mesh_halo
            run = lambda: extract_mesh_halo(table, dist, torch, device=dev, collapse_epsilon=eps)  # noqa: E731
            how = "sharding.extract_mesh_halo over the shards (mesh on rank 0), wall clock"
        else:
            run = lambda: P.extract_mesh(table, 0.0, eps)  # noqa: E731
            how = "public extract_mesh on the final map, wall clock incl. D2H of the mesh"
        run()
        table.kernel_times(reset=True)
        table.profile(True)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        mesh = run()
        ex_s = time.perf_counter() - t0
        mk = table.kernel_times(reset=True)
        table.profile(False)
        if mesh is not None:
            extract = {"ms": round(ex_s * 1e3, 3), "vertices": int(mesh.num_vertices),
                       "triangles": int(mesh.num_triangles),
                       "mtriangles_per_s": round(mesh.num_triangles / ex_s / 1e6, 3),
                       "kernels_ms": {k: round(v[0], 3) for k, v in sorted(mk.items(), key=lambda kv: -kv[1][0])[:6]},
                       "note": how}
    dev_ms = float(sum(step_ms))
    if world > 1:
        tt = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_ms = float(tt.item())
    points = sum(s.measurements for s in all_stats)  # invariant across ranks
    nframes = K * FRAMES_PER_STEP
    value = points / (dev_ms * 1e-3) / 1e6
    fps = nframes / (dev_ms * 1e-3)
    table.close()
    del table

    # ---- e2e: public API from pinned host buffers ----------------------------
    with torch.cuda.stream(stream):
        t2 = make_table(P, wl, stream=stream, shard=shard)
    pinned = []
    for d, c, pose, intr in frames:
        pd = torch.from_numpy(d).pin_memory().numpy()
        pc = None if c is None else torch.from_numpy(c).pin_memory().numpy()
        pinned.append((pd, pc, pose, intr))
    h2d = d2h = 0
    fi = 0
    pinned = pinned[:FRAMES_PER_STEP * (W + K)]
    for s in range(W):
        window_and_merge(P, t2, wl, pinned[fi:fi + FRAMES_PER_STEP])
        fi += FRAMES_PER_STEP
    barrier()
    e2e_t0 = time.perf_counter()
    e2e_pts = 0
    for s in range(K):
        win = pinned[fi:fi + FRAMES_PER_STEP]
        sts, _ = window_and_merge(P, t2, wl, win)
        e2e_pts += sum(st.measurements for st in sts)
        for fr in win:
            h2d += fr[0].nbytes + (0 if fr[1] is None else fr[1].nbytes)
            d2h += 192  # per-frame counters block (stats) read back
        fi += FRAMES_PER_STEP
        d2h += 192
    barrier()
    e2e_s = time.perf_counter() - e2e_t0
    if world > 1:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    t2.close()
    e2e_value = e2e_pts / e2e_s / 1e6

    # ---- roofline of the dominant kernel (live CUDA-event durations) ---------
    peak, peak_kind = peaks()
    B = kernel_bytes(all_stats, wl)
    Bp = kernel_bytes(prof_stats, wl)  # the profiled windows' algorithmic bytes
    top = max(ktimes.items(), key=lambda kv: kv[1][0]) if ktimes else ("none", (0.0, 1))
    top_name, (top_ms, top_n) = top
    role = KERNEL_ROLE.get(top_name, "path")
    top_bytes = Bp[role] if role in Bp else Bp["path"]
    achieved = (top_bytes / top_n) / ((top_ms / top_n) * 1e-3) / 1e9 if top_ms > 0 else 0.0
    path_gbs = B["path"] / (dev_ms * 1e-3) / 1e9
    ncu, ncu_note = ncu_profile()
    kt = ncu.get("kernels", {}).get(top_name, {})
    traffic = kt.get("dram_bytes") if str(kt.get("capture", "")).startswith(
        "room" if wl["kind"] == "depth" else "lidar") else None
    clocks = sampler.summary()
    # the binding resource of the walk is instruction issue (FP64 DDA
    # steps), not HBM: its issue roofline = the warp instructions one launch
    # executes (ncu, same build) over the SM issue capacity (148 SMs x 4
    # schedulers x 1 warp-instruction per cycle at the sampled clock),
    # against the live launch time
    secondary = None
    walk = "k_dda_walk"
    if walk in ktimes and work.get("dda_steps"):
        w_ms, w_n = ktimes[walk]
        steps = work["dda_steps"] / max(w_n, 1)
        ms_launch = w_ms / max(w_n, 1)
        kw = ncu.get("kernels", {}).get(walk, {})
        # the capture must be of this workload's walk (room vs lidar launches differ)
        if not str(kw.get("capture", "")).startswith("room" if wl["kind"] == "depth" else "lidar"):
            kw = {}
        secondary = {"bound": "issue (FP64 DDA steps)", "kernel": walk,
                     "dda_steps_per_launch": round(steps), "ms_per_launch": round(ms_launch, 4),
                     "gsteps_per_s": round(steps / (ms_launch * 1e-3) / 1e9, 3)}
        if kw.get("warp_inst") and clocks.get("sm_mhz"):
            sms = ncu.get("sms", 148)
            # ncu counts one launch (one frame of the capture driver, whose
            # DDA steps it recorded); scale to this run's steps per launch
            inst_per_step = kw["warp_inst"] / max(kw.get("dda_steps", steps), 1)
            floor_ms = inst_per_step * steps / (sms * 4 * clocks["sm_mhz"] * 1e6) * 1e3
            secondary.update({"warp_inst_per_step": round(inst_per_step, 3),
                              "issue_floor_ms": round(floor_ms, 4),
                              "issue_frac": round(floor_ms / ms_launch, 4),
                              "ncu_issue_active_frac": kw.get("issue_active")})
    out = {
        "metric": METRIC[name],
        "value": round(value, 3), "unit": "Mpoints/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": round(dev_ms / K, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (analytic ray-cast scene, deterministic)",
        "config": {"workload": wl["name"], "frames_per_step": FRAMES_PER_STEP,
                   "fps": round(fps, 2), "frames_timed": nframes,
                   "l2": "256 MB L2 flush between timed steps (outside the events)",
                   "parallelism": f"block-key-hash shards x{world}" if world > 1 else "single GPU",
                   "blocks_live_end": occ, "merged_in_timed_region": merged,
                   "work_units": {k: int(v) for k, v in B.items() if k in "PTAU"},
                   "diagnostics": work,
                   "profiled_windows": "kernels_ms, roofline and diagnostics come from K further "
                                       "windows run with per-kernel CUDA events, after the timed "
                                       "region"},
        "e2e": {"value": round(e2e_value, 3), "unit": "Mpoints/s", "h2d_bytes_per_step": h2d // K,
                "d2h_bytes_per_step": d2h // K},
        "roofline": {"bound": "hbm", "kernel": top_name, "achieved": round(achieved, 2),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 5),
                     "traffic": traffic, "peak_source": peak_kind,
                     "path_achieved_gbs": round(path_gbs, 2),
                     "path_frac": round(path_gbs / peak, 5),
                     "bytes_per_launch": round(top_bytes / max(top_n, 1)),
                     "ms_per_launch": round(top_ms / max(top_n, 1), 4),
                     "secondary": secondary},
        "kernels_ms": {k: [round(v[0], 3), v[1]] for k, v in sorted(ktimes.items(), key=lambda kv: -kv[1][0])},
        "gpu_launches": int(launches),
        "extract": extract,
        "clocks": clocks,
    }
    out["roofline"]["ncu"] = ncu_note
    return out


def ncu_profile():
    """profiles/ncu_summary.json if it was captured on this exact build
    (source digest of csrc + the ABI header); otherwise nothing, and the
    roofline says why (a stale capture would misreport traffic)."""
    from paper_2511_21459_b200._native import source_digest
    prof = ROOT / "profiles" / "ncu_summary.json"
    if not prof.exists():
        return {}, "no ncu summary"
    try:
        d = json.loads(prof.read_text())
    except Exception as e:
        return {}, f"unreadable ncu summary: {e}"
    want = source_digest()
    if d.get("src_sha") != want:
        return {}, f"ncu summary is from build {d.get('src_sha')}, this build is {want}: dropped"
    return d, f"ncu --set full on this build ({want}): {d.get('source', '')}"


def _oracle_table(wl):
    from oracle.oracle import OracleTable
    # the GPU table's capacities (calloc'd heaps: pages are committed on touch)
    return OracleTable(wl["n_hash"], 10, 7, wl["edge"], wl["caps"])


def oracle_frame(t, wl, fr):
    d, c, pose, intr = fr
    if wl["kind"] == "depth":
        return t.integrate_depth(d.astype(np.float64), [intr.fx, intr.fy, intr.cx, intr.cy],
                                 pose.rotation, pose.translation, wl["tau"],
                                 color=None if c is None else c.astype(np.float64) / 255.0)
    return t.integrate_points(d.astype(np.float64), pose.rotation, pose.translation, wl["tau"])


def oracle_parity_job(name, q):
    """Child process: the oracle (test infrastructure; the checker and the
    CPU baseline, never the product) on the parity sample of `name` --
    per-frame stats, merge passes every `cadence` frames (all levels), per-
    frame host time, and the final state's digest."""
    sys.path.insert(0, str(ROOT / "tests"))
    import parity_utils as PU
    wl = WORKLOADS[name]
    n, cadence = PARITY[name]
    frames = make_frames(wl, n)
    t = _oracle_table(wl)
    stats, merges, secs, pts = [], [], [], []
    for i, fr in enumerate(frames):
        t0 = time.perf_counter()
        st = oracle_frame(t, wl, fr)
        if (i + 1) % cadence == 0:
            merges.append(t.apply_merges(wl["sigma"], all_levels=True))
        secs.append(time.perf_counter() - t0)
        pts.append(st["measurements"])
        stats.append({k: st[k] for k in PU.STAT_KEYS})
    state = {l: t.block_arrays(l) for l in range(t.num_levels)}
    dump = None
    if wl.get("lidar_mode") == "chunked":
        # the tolerance comparison needs the arrays: hand them over through
        # RAM-backed files (a few GB do not fit a queue)
        dump = f"/dev/shm/tsdf_parity_{os.getpid()}.npz"
        np.savez(dump, **{f"{k}_{l}": a for l, v in state.items()
                          for k, a in zip(("c", "t", "w", "s", "col"), v)})
    q.put({"stats": stats, "merges": merges, "secs": secs, "pts": pts,
           "digest": PU.state_digest(state), "keys": PU.keys_digest(state),
           "blocks": [int(len(v[0])) for _, v in sorted(state.items())], "dump": dump})


def gpu_parity(P, name, frames):
    """The measured binary on the parity sample, through the same window
    calls the timed region uses."""
    sys.path.insert(0, str(ROOT / "tests"))
    import parity_utils as PU
    wl = WORKLOADS[name]
    n, cadence = PARITY[name]
    t = make_table(P, wl)
    stats, merges = [], []
    for w0 in range(0, n, cadence):
        win = frames[w0:w0 + cadence]
        if wl["kind"] == "depth":
            fs = [P.DepthFrame(depth=d, intrinsics=intr, pose=pose, color=c) for d, c, pose, intr in win]
            st, ms = P.integrate_depth_window(t, fs, wl["tau"], wl["sigma"], all_levels=True)
        else:
            st = [P.integrate_pointcloud(t, P.PointCloudFrame(points=d, pose=pose), wl["tau"])
                  for d, _, pose, _ in win]
            ms = P.apply_merges(t, wl["sigma"], all_levels=True)
        stats += [{k: getattr(x, k) for k in PU.STAT_KEYS} for x in st]
        merges.append({"candidates": ms.candidates, "merged": ms.merged})
    state = {l: tuple(t.export_level(l)[i] for i in (0, 2, 3, 4, 5)) for l in range(t.num_levels)}
    out = {"stats": stats, "merges": merges, "digest": PU.state_digest(state),
           "keys": PU.keys_digest(state), "blocks": [int(len(v[0])) for _, v in sorted(state.items())],
           "audit": t.merge_audit()}
    if wl.get("lidar_mode") == "chunked":
        out["state"] = state
    t.close()
    return out


def tolerance_parity(g_state, dump):
    """Chunked LiDAR: keys, levels and weights bit-exact; TSDF / variance
    within TOL_REL relative (+ the SURVEY §8c absolute floors); colour within
    1e-4 -- against the ordered oracle's arrays."""
    o = np.load(dump)
    res = {"keys_levels_weights_bit_identical": True, "tsdf_max_rel": 0.0, "s2_max_rel": 0.0,
           "color_max_abs": 0.0, "voxels_differing": 0}
    ok = True
    for l, (c, t_, w, s2, col) in g_state.items():
        oc, ot, ow, os_, ocol = (o[f"{k}_{l}"] for k in ("c", "t", "w", "s", "col"))
        if not (np.array_equal(c, oc) and np.array_equal(w, ow)):
            res["keys_levels_weights_bit_identical"] = False
            ok = False
            continue
        if len(c) == 0:
            continue
        dt, ds = np.abs(t_ - ot), np.abs(s2 - os_)
        ok &= bool(np.all(dt <= TOL_REL * np.abs(ot) + 1e-7 * 0.8))
        ok &= bool(np.all(ds <= TOL_REL * np.abs(os_) + 1e-10 * 0.64 * ow))
        with np.errstate(divide="ignore", invalid="ignore"):
            res["tsdf_max_rel"] = max(res["tsdf_max_rel"], float(np.max(np.where(ot != 0, dt / np.abs(ot), dt))))
            res["s2_max_rel"] = max(res["s2_max_rel"], float(np.max(np.where(os_ != 0, ds / np.abs(os_), ds))))
        res["color_max_abs"] = max(res["color_max_abs"], float(np.max(np.abs(col - ocol))))
        ok &= res["color_max_abs"] <= 1e-4
        res["voxels_differing"] += int(np.count_nonzero((t_ != ot) | (s2 != os_)))
    res["within_tolerance"] = bool(ok)
    try:
        os.unlink(dump)
    except OSError:
        pass
    return res


def parity_and_baseline(name, g, o):
    """the measured binary reproduces the reference algorithm
    (the oracle) on the first frames of the measured workload, merges
    included; the oracle's steady-state frames are the CPU baseline."""
    n, cadence = PARITY[name]
    parity = {"frames": n, "merge_cadence": cadence, "merge_passes": len(g["merges"]),
              "levels": "all (labelled 3-level extension, oracle all_levels=True)",
              "merged": int(sum(m["merged"] for m in g["merges"])),
              "stats_equal": g["stats"] == o["stats"],
              "merges_equal": g["merges"] == o["merges"],
              "keys_bit_identical": g["keys"] == o["keys"],
              "state_bit_identical": g["digest"] == o["digest"],
              "blocks": g["blocks"], "oracle_blocks": o["blocks"],
              "merge_audit": g.get("audit", 0),
              "compared": "per-frame IntegrationStats, per-pass MergeStats, sha256 of every level's "
                          "keys + TSDF + weight + variance + colour"}
    if "state" in g and o.get("dump"):
        parity["mode"] = "chunked (hot blocks Chan-merged; tolerance contract, SURVEY §8c)"
        parity["tolerance"] = tolerance_parity(g["state"], o["dump"])
        parity["compared"] += ("; chunked mode: keys / levels / weights bit-exact, TSDF & variance "
                               f"<= {TOL_REL} relative, colour <= 1e-4, level audit (decisions within "
                               "1e-6 of sigma) reported")
    # steady state: frames after the first (whose allocation is the whole
    # visible map), merge passes included
    secs, pts = sum(o["secs"][1:]), sum(o["pts"][1:])
    base = {"value": round(pts / secs / 1e6, 4), "unit": "Mpoints/s", "cores": 1, "kind": "port",
            "sample": f"frames 2..{n} of the parity sample (merge every {cadence}) through the C "
                      f"oracle (oracle/tsdf_oracle.c, serial, -O2): {pts} points in {secs:.1f} s"}
    return parity, base


def _reference_worker(wl, frames, warmup, barrier, q):
    """One replica of the reference arm: the frame stream into its own table
    with a merge pass (all levels) after every FRAMES_PER_STEP-th frame, as
    the measured B200 arm does; the first `warmup` frames are untimed."""
    t = _oracle_table(wl)

    def run(i0, i1):
        pts = 0
        for i in range(i0, i1):
            pts += oracle_frame(t, wl, frames[i])["measurements"]
            if (i + 1) % FRAMES_PER_STEP == 0:
                t.apply_merges(wl["sigma"], all_levels=True)
        return pts

    run(0, warmup)
    barrier.wait()
    t0 = time.time()
    pts = run(warmup, len(frames))
    q.put((pts, t0, time.time()))


def reference_replicas(wl):
    """How many replicas of the serial reference path the host can run at
    once: one per core, bounded by memory (a replica's table after a few
    frames of the large room is ~3 GB)."""
    n = os.cpu_count() or 1
    try:
        import psutil
        n = min(n, max(1, int(psutil.virtual_memory().available * 0.6 // (3.5 * 2 ** 30))))
    except ImportError:
        n = min(n, 8)
    return max(1, n)


def run_reference(args, name):
    """The reference arm: the reference algorithm (the oracle port; the
    reference is serial NumPy) on every host core it can use.  The path is
    serial per table, so the cores run independent replicas of the same
    workload, each integrating the frame stream into its own table; value =
    all replicas' timed points / the wall time from the common start to the
    last replica's end."""
    import multiprocessing as mp
    wl = WORKLOADS[name]
    frames = gen_frames(name, args.warmup + args.steps)
    n = reference_replicas(wl)
    ctx = mp.get_context("fork")
    barrier, q = ctx.Barrier(n), ctx.Queue()
    procs = [ctx.Process(target=_reference_worker, args=(wl, frames, args.warmup, barrier, q))
             for _ in range(n)]
    for p in procs:
        p.start()
    res = [q.get() for _ in procs]
    for p in procs:
        p.join()
    pts = sum(r[0] for r in res)
    wall = max(r[2] for r in res) - min(r[1] for r in res)
    v = pts / wall / 1e6
    return {"impl": "reference", "metric": METRIC[name],
            "value": round(v, 4), "unit": "Mpoints/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(wall / args.steps * 1e3, 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (analytic ray-cast scene, deterministic)",
            "config": {"workload": wl["name"], "frames_per_step": 1, "replicas": n,
                       "merge_passes": f"all levels, after every {FRAMES_PER_STEP}th frame of "
                                       "the stream (as the B200 arm)",
                       "hardware": "host CPU only (n_gpus echoes the launch; no GPU is used)",
                       "note": "reference arm = the oracle port of the reference algorithm (the "
                               "reference is serial NumPy; same arithmetic, serial C) on every "
                               "usable host core: independent replicas of the frame stream"},
            "cpu_baseline": {"value": round(v, 4), "unit": "Mpoints/s", "cores": n, "kind": "port",
                             "sample": f"frames {args.warmup + 1}..{args.warmup + args.steps} "
                                       f"of the stream (merges included) after {args.warmup} "
                                       f"warm-up frames, {n} replicas in parallel"},
            "e2e": {"value": round(v, 4), "unit": "Mpoints/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def _sub_line(o):
    """The keys of a workload's line kept in the N=1 line's sub-object."""
    keep = ("metric", "value", "unit", "ms_per_step", "steps", "warmup", "config", "e2e",
            "roofline", "kernels_ms", "gpu_launches", "clocks", "cpu_baseline", "parity")
    return {k: o[k] for k in keep if k in o}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="room", choices=list(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true",
                    help="skip the oracle parity check and CPU baseline")
    ap.add_argument("--no-lidar", action="store_true",
                    help="N=1 room runs: skip the LiDAR (config 3) sub-run")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo only to exercise the multi-rank path with ranks sharing one GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    name = args.workload
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args, name)), flush=True)
        return
    # BASELINE's metric is quoted on both north-star configs: an N=1 room
    # run also measures the 128-beam LiDAR stream (config 3) as `lidar`
    subs = ["lidar", "lidar_ordered"] if world == 1 and name.startswith("room") and not args.no_lidar else []
    if name == "lidar" and world == 1:
        subs = ["lidar_ordered"]
    check = world == 1 and not args.no_cpu_baseline
    # the oracle runs (checker + CPU baseline) start first, in their own
    # processes, before CUDA is initialised here
    jobs = {}
    if check:
        import multiprocessing as mp
        ctx = mp.get_context("fork")
        for nm in [name] + subs:
            if nm in ORACLE_OF and ORACLE_OF[nm] in [name] + subs:
                continue  # shares the oracle run of ORACLE_OF[nm]
            q = ctx.Queue()
            p = ctx.Process(target=oracle_parity_job, args=(nm, q), daemon=True)
            p.start()
            jobs[nm] = (p, q)
    t0 = time.time()
    frames = {nm: gen_frames(nm, FRAMES_PER_STEP * (args.warmup + 2 * (args.steps if nm == name
                                                                         else min(args.steps, LIDAR_STEPS))))
              for nm in [name] + subs if nm not in ORACLE_OF}
    for nm in subs:
        if nm in ORACLE_OF:
            frames[nm] = frames.get(ORACLE_OF[nm]) or gen_frames(
                nm, FRAMES_PER_STEP * (args.warmup + 2 * min(args.steps, LIDAR_STEPS)))
    log(f"[bench] generated frames for {list(frames)} in {time.time() - t0:.1f}s")
    import torch
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % max(torch.cuda.device_count(), 1))
        dist.init_process_group(args.dist_backend)
    out = run_b200(name, args.warmup, args.steps, rank, world, dist, torch, frames[name])
    for nm in subs:
        out[nm] = _sub_line(run_b200(nm, args.warmup, min(args.steps, LIDAR_STEPS), rank, world,
                                     dist, torch, frames[nm]))
    if rank == 0:
        if check:
            import paper_2511_21459_b200 as P
            got = {}
            for nm in [name] + subs:
                n = PARITY[nm][0]
                g = gpu_parity(P, nm, frames[nm][:n] if len(frames[nm]) >= n else make_frames(WORKLOADS[nm], n))
                src = ORACLE_OF.get(nm, nm) if ORACLE_OF.get(nm) in jobs or ORACLE_OF.get(nm) in got else nm
                if src not in got:
                    p, q = jobs[src]
                    got[src] = q.get()
                    p.join()
                tgt = out if nm == name else out[nm]
                tgt["parity"], tgt["cpu_baseline"] = parity_and_baseline(nm, g, got[src])
        # the ordered LiDAR run is reported inside the lidar line
        if "lidar_ordered" in out:
            host = out["lidar"] if "lidar" in out else out
            lo = out.pop("lidar_ordered")
            host["ordered"] = {k: lo[k] for k in ("value", "unit", "ms_per_step", "e2e", "kernels_ms",
                                                  "parity") if k in lo}
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
