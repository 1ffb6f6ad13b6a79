"""A small on-disk dataset in the reference's layouts (datasets.py:1-12),
written from the synthetic room: 16-bit depth PNGs (raw = round(z * scale)),
RGB PNGs, trajectory and intrinsics files, and .pcb / .xyz point clouds."""
from __future__ import annotations

import numpy as np

SCALE = 5000.0


def rotation_to_quaternion(R):
    """Scalar-last unit quaternion of a proper rotation (for writing the
    trajectory; quaternion_to_rotation reads it back)."""
    R = np.asarray(R, dtype=np.float64)
    w = np.sqrt(max(0.0, 1.0 + R[0, 0] + R[1, 1] + R[2, 2])) / 2
    x = np.sqrt(max(0.0, 1.0 + R[0, 0] - R[1, 1] - R[2, 2])) / 2
    y = np.sqrt(max(0.0, 1.0 - R[0, 0] + R[1, 1] - R[2, 2])) / 2
    z = np.sqrt(max(0.0, 1.0 - R[0, 0] - R[1, 1] + R[2, 2])) / 2
    x = np.copysign(x, R[2, 1] - R[1, 2])
    y = np.copysign(y, R[0, 2] - R[2, 0])
    z = np.copysign(z, R[1, 0] - R[0, 1])
    q = np.array([x, y, z, w])
    return q / np.linalg.norm(q)


def _fields(t, q) -> str:
    return " ".join(repr(float(x)) for x in list(t) + list(q))


def raw_depth(depth) -> np.ndarray:
    d = np.nan_to_num(np.asarray(depth, dtype=np.float64), nan=0.0)
    return np.clip(np.round(d * SCALE), 0, 65535).astype(np.uint16)


def write_depth_dataset(root, n_frames=6, width=96, height=72, rgb=True):
    from PIL import Image
    from paper_2511_21459_b200 import synth
    frames = synth.render_frames("room", n_frames, width, height, color_dtype=np.uint8)
    (root / "depth").mkdir(parents=True)
    if rgb:
        (root / "rgb").mkdir()
    lines = []
    for i, f in enumerate(frames):
        Image.fromarray(raw_depth(f.depth)).save(root / "depth" / f"{i:06d}.png")
        if rgb:
            Image.fromarray(np.asarray(f.color, dtype=np.uint8), "RGB").save(root / "rgb" / f"{i:06d}.png")
        q = rotation_to_quaternion(f.pose.rotation)
        t = f.pose.translation
        lines.append(f"{0.1 * (i + 1):.6f} " + _fields(t, q))
    (root / "trajectory.txt").write_text("# t tx ty tz qx qy qz qw\n" + "\n".join(lines) + "\n")
    k = frames[0].intrinsics
    (root / "intrinsics.txt").write_text(" ".join(repr(float(x)) for x in (k.fx, k.fy, k.cx, k.cy)) + "\n")
    return root


def write_cloud_dataset(root, n_scans=2, beams=16, columns=128):
    from paper_2511_21459_b200 import synth
    from paper_2511_21459_b200.datasets import write_pointcloud_file
    scans = synth.lidar_frames(n_scans, beams, columns, step=0.5)
    (root / "clouds").mkdir(parents=True)
    rng = np.random.default_rng(3)
    lines = []
    for i, s in enumerate(scans):
        pts = np.asarray(s.points, dtype=np.float64)
        if i % 2 == 0:
            write_pointcloud_file(root / "clouds" / f"{i:06d}.pcb", pts, rng.uniform(0, 1, (len(pts), 3)))
        else:
            (root / "clouds" / f"{i:06d}.xyz").write_text(
                "\n".join(" ".join(repr(float(v)) for v in p) for p in pts[:500]) + "\n")
        q = rotation_to_quaternion(s.pose.rotation)
        t = s.pose.translation
        lines.append(f"{float(i):.3f} " + _fields(t, q))
    (root / "trajectory.txt").write_text("\n".join(lines) + "\n")
    return root
