"""GPU: raw 16-bit depth scaled on the device, and dataset files read by the
B200 readers, fused bit-identically to the oracle fed the reference reader's
f64 frames (datasets.py:108-122: raw / depth_scale, rgb / 255)."""
import numpy as np
import pytest

import parity_utils as PU
from dataset_utils import SCALE, raw_depth, write_cloud_dataset, write_depth_dataset

pytestmark = pytest.mark.gpu

N_HASH, EDGE, CAPS, TAU = 100003, 0.04, (60000, 20000, 5000), 0.015


def _gpu_state(t):
    return PU.GpuBackend.state(type("x", (), {"t": t})())


def _raw_frames(n=12, w=128, h=96):
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200 import synth
    out = []
    for f in synth.render_frames("room", n, w, h, depth_dtype=np.float32, color_dtype=np.uint8):
        out.append(P.DepthFrame(raw_depth(f.depth), f.intrinsics, f.pose, color=f.color,
                                depth_scale=SCALE))
    return out


def test_raw_u16_depth_per_frame_and_window_vs_oracle():
    import paper_2511_21459_b200 as P
    frames = _raw_frames()
    t = P.HashTable(N_HASH, 10, 7, EDGE, CAPS)
    o = PU.OracleBackend(N_HASH, EDGE, CAPS)
    for f in frames[:2]:
        s = P.integrate_depth(t, f, TAU)
        assert {k: getattr(s, k) for k in PU.STAT_KEYS} == o.depth(f, TAU)
    st, ms = P.integrate_depth_window(t, frames[2:], TAU, 2.5e-5, all_levels=True)
    so = [o.depth(f, TAU) for f in frames[2:]]
    mo = o.merge(2.5e-5, all_levels=True)
    assert [{k: getattr(x, k) for k in PU.STAT_KEYS} for x in st] == so
    assert (ms.candidates, ms.merged) == (mo["candidates"], mo["merged"])
    assert PU.state_digest(_gpu_state(t)) == PU.state_digest(o.state())


def test_raw_u16_device_resident_equals_host():
    import torch
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.sharding import _DeviceView
    frames = _raw_frames(4)
    a = P.HashTable(N_HASH, 10, 7, EDGE, CAPS)
    b = P.HashTable(N_HASH, 10, 7, EDGE, CAPS)
    for f in frames:
        P.integrate_depth(a, f, TAU)
        raw = torch.from_numpy(f.depth.view(np.uint8).reshape(-1).copy()).cuda()
        col = torch.from_numpy(np.ascontiguousarray(f.color)).cuda()
        g = P.DepthFrame(_DeviceView(raw, "<u2", f.depth.shape), f.intrinsics, f.pose,
                         color=col, depth_scale=SCALE)
        P.integrate_depth(b, g, TAU)
        torch.cuda.synchronize()
    assert PU.state_digest(_gpu_state(a)) == PU.state_digest(_gpu_state(b))


def test_window_rejects_mixed_depth_scales():
    import paper_2511_21459_b200 as P
    frames = _raw_frames(2)
    frames[1].depth_scale = 1000.0
    t = P.HashTable(N_HASH, 10, 7, EDGE, CAPS)
    with pytest.raises(ValueError, match="depth_scale"):
        P.integrate_depth_batch(t, frames, TAU)


def test_depth_dataset_engine_vs_oracle(tmp_path):
    """read_depth_sequence -> run_pipeline (merge windows) equals the oracle
    fed the reference reader's frames, restated here with PIL
    (datasets.py:108-119)."""
    from PIL import Image
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.datasets import read_depth_sequence
    root = write_depth_dataset(tmp_path / "d", n_frames=12, width=128, height=96)
    args = (root, root / "trajectory.txt", root / "intrinsics.txt")
    cfg = P.PipelineConfig(sensor_mode="depth", nu_fine=0.005, block_edge=EDGE, tau=TAU,
                           n_hash=N_HASH, heap_capacity_fine=CAPS[0], heap_capacity_coarse=CAPS[1],
                           merge_cadence=5, depth_scale=SCALE)
    eng = P.FusionEngine(cfg)
    n = 0
    for f in read_depth_sequence(*args, depth_scale=cfg.depth_scale, keep_types=True):
        eng.integrate_frame(f)
        eng.maybe_merge()
        n += 1
    assert n == 12
    o = PU.OracleBackend(N_HASH, EDGE, CAPS[:2])
    dfiles = sorted((root / "depth").iterdir())
    rfiles = sorted((root / "rgb").iterdir())
    from paper_2511_21459_b200.datasets import read_intrinsics, read_trajectory
    traj, intr = read_trajectory(root / "trajectory.txt"), read_intrinsics(root / "intrinsics.txt")
    for i, (dp, rp, e) in enumerate(zip(dfiles, rfiles, traj)):
        depth = np.asarray(Image.open(dp), dtype=np.float64) / SCALE
        color = np.asarray(Image.open(rp).convert("RGB"), dtype=np.float64) / 255.0
        o.depth(P.DepthFrame(depth, intr, e.pose, color=color), TAU)
        if (i + 1) % 5 == 0:
            o.merge(cfg.sigma_threshold)
    assert PU.state_digest(_gpu_state(eng.table)) == PU.state_digest(o.state())


def test_cloud_dataset_vs_oracle(tmp_path):
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.datasets import read_pointcloud_sequence
    root = write_cloud_dataset(tmp_path / "c", n_scans=2, beams=32, columns=256)
    t = P.HashTable(1000003, 10, 7, 1.6, (300000, 20000))
    o = PU.OracleBackend(1000003, 1.6, (300000, 20000))
    for f in read_pointcloud_sequence(root, root / "trajectory.txt", keep_types=True):
        s = P.integrate_pointcloud(t, f, 0.8)
        assert {k: getattr(s, k) for k in PU.STAT_KEYS} == o.points(f, 0.8)
    assert PU.state_digest(_gpu_state(t)) == PU.state_digest(o.state())
