"""Synthetic inputs for benchmarks and parity tests (not on the fusion path).

Analytic scenes ray-cast in closed form, following the reference's scene
definitions (synth.py:23-175): the unit sphere, the plane, the 1.6 m box room
with a 5-sphere cluster and its yaw/pitch sweep; plus the SURVEY §8d
"large room" (6 x 5 x 3 m, 12 spheres) and a 128-beam spinning LiDAR.
Everything is deterministic (seeded).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .geometry import DepthFrame, Intrinsics, PointCloudFrame, SensorPose


@dataclass
class Scene:
    name: str
    spheres: list = field(default_factory=list)  # (center, radius, rgb)
    plane_z: float | None = None
    room: tuple | None = None                    # (lo, hi) interior box
    wall_rgb: tuple = (0.75, 0.73, 0.70)


def make_scene(name: str) -> Scene:
    if name == "plane":
        return Scene("plane", plane_z=0.0)
    if name == "sphere":
        return Scene("sphere", spheres=[(np.zeros(3), 1.0, (0.80, 0.35, 0.25))])
    if name == "room":
        cluster = [((0.32, 0.18, -0.52), 0.14, (0.85, 0.30, 0.25)),
                   ((0.14, 0.30, -0.60), 0.10, (0.25, 0.60, 0.85)),
                   ((0.40, 0.38, -0.62), 0.09, (0.30, 0.75, 0.35)),
                   ((0.24, 0.10, -0.68), 0.07, (0.85, 0.70, 0.25)),
                   ((0.35, 0.27, -0.44), 0.06, (0.70, 0.35, 0.75))]
        return Scene("room", spheres=[(np.array(c), r, col) for c, r, col in cluster],
                     room=(np.full(3, -0.8), np.full(3, 0.8)))
    if name == "large_room":
        rng = np.random.default_rng(0)
        sph = []
        for _ in range(12):
            c = np.array([rng.uniform(-2.5, 2.5), rng.uniform(-2.0, 2.0), rng.uniform(-1.2, 0.5)])
            sph.append((c, float(rng.uniform(0.1, 0.4)), tuple(rng.uniform(0.2, 0.9, 3))))
        return Scene("room", spheres=sph,
                     room=(np.array([-3.0, -2.5, -1.5]), np.array([3.0, 2.5, 1.5])))
    raise ValueError(f"unknown synthetic scene {name!r}")


def look_at(eye, target, up=(0.0, 0.0, 1.0)) -> SensorPose:
    """Camera pose: +z forward, +x right, +y down."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    fwd /= np.linalg.norm(fwd)
    right = np.cross(fwd, np.asarray(up, dtype=np.float64))
    if np.linalg.norm(right) < 1e-8:
        right = np.cross(fwd, np.array([0.0, 1.0, 0.0]))
    right /= np.linalg.norm(right)
    down = np.cross(fwd, right)
    return SensorPose(np.stack([right, down, fwd], axis=1), eye)


def fibonacci_directions(n: int) -> np.ndarray:
    i = np.arange(n, dtype=np.float64)
    z = 1.0 - 2.0 * (i + 0.5) / n
    r = np.sqrt(np.maximum(0.0, 1.0 - z * z))
    phi = i * np.pi * (3.0 - np.sqrt(5.0))
    return np.stack([r * np.cos(phi), r * np.sin(phi), z], axis=1)


def trajectory(scene: Scene, frames: int) -> list:
    if scene.name == "sphere":
        return [look_at(d * 1.6, np.zeros(3)) for d in fibonacci_directions(frames)]
    if scene.name == "room":
        out = []
        for i in range(frames):
            yaw = 2.0 * np.pi * i / frames
            pitch = 0.25 * np.sin(3.0 * yaw)
            tgt = np.array([np.cos(yaw) * np.cos(pitch), np.sin(yaw) * np.cos(pitch), np.sin(pitch)])
            out.append(look_at(np.zeros(3), tgt))
        return out
    if scene.name == "plane":
        return [look_at(np.array([0.05 * np.cos(i), 0.05 * np.sin(i), 0.6]), np.zeros(3))
                for i in range(frames)]
    raise ValueError(f"no trajectory for scene {scene.name!r}")


def default_intrinsics(scene_name: str, width: int, height: int) -> Intrinsics:
    f = {"sphere": 0.5, "room": 0.9, "large_room": 0.9, "plane": 1.0}.get(scene_name, 0.9) * width
    return Intrinsics(fx=f, fy=f, cx=(width - 1) / 2.0, cy=(height - 1) / 2.0)


def _checker(p, period=0.2):
    return 0.9 + 0.1 * (np.floor(p / period).astype(np.int64).sum(axis=1) % 2)


def render_depth(scene: Scene, pose: SensorPose, intr: Intrinsics, width: int, height: int):
    """Closed-form ray cast -> (z-depth H x W, rgb H x W x 3 in [0, 1])."""
    u, v = np.meshgrid(np.arange(width, dtype=np.float64), np.arange(height, dtype=np.float64))
    dc = np.stack([(u - intr.cx) / intr.fx, (v - intr.cy) / intr.fy, np.ones_like(u)], -1).reshape(-1, 3)
    dw = dc @ pose.rotation.T
    o = pose.translation
    n = len(dw)
    best = np.full(n, np.inf)
    rgb = np.zeros((n, 3))
    wall = np.asarray(scene.wall_rgb)
    with np.errstate(divide="ignore", invalid="ignore"):
        if scene.plane_z is not None:
            t = (scene.plane_z - o[2]) / dw[:, 2]
            ok = np.isfinite(t) & (t > 1e-9) & (t < best)
            best[ok] = t[ok]
            rgb[ok] = wall * _checker(o + t[ok, None] * dw[ok])[:, None]
        if scene.room is not None:
            lo, hi = scene.room
            t_exit = np.full(n, np.inf)
            for a in range(3):
                t = (np.where(dw[:, a] > 0, hi[a], lo[a]) - o[a]) / dw[:, a]
                t_exit = np.minimum(t_exit, np.where(np.isfinite(t) & (t > 1e-9), t, np.inf))
            ok = np.isfinite(t_exit) & (t_exit < best)
            best[ok] = t_exit[ok]
            rgb[ok] = wall * _checker(o + t_exit[ok, None] * dw[ok])[:, None]
        aa = np.einsum("ij,ij->i", dw, dw)
        for center, radius, color in scene.spheres:
            oc = o - center
            b = 2.0 * dw @ oc
            c = oc @ oc - radius * radius
            disc = b * b - 4 * aa * c
            t = np.full(n, np.inf)
            hit = disc > 0
            tn = (-b - np.sqrt(np.where(hit, disc, 0.0))) / (2 * aa)
            sel = hit & (tn > 1e-9)
            t[sel] = tn[sel]
            closer = t < best
            best[closer] = t[closer]
            p = o + t[closer, None] * dw[closer]
            shade = 0.7 + 0.3 * np.clip((p - center) @ np.array([0.3, 0.3, 0.9]), 0, 1) / radius
            rgb[closer] = np.asarray(color) * shade[:, None]
    depth = np.where(np.isfinite(best), best, 0.0).reshape(height, width)
    return depth, np.clip(rgb, 0, 1).reshape(height, width, 3)


def render_frames(scene_name: str, frames: int, width: int, height: int,
                  depth_dtype=np.float64, color_dtype=np.float64, sweep: int | None = None) -> list:
    """Depth frames along the scene's trajectory.  float32 depth / uint8 colour
    give the compact 7 B/px sensor format (values quantised before use, so
    every consumer sees the same inputs).  ``sweep``: the trajectory's length
    when only its first ``frames`` poses are rendered (default: frames)."""
    scene = make_scene(scene_name)
    intr = default_intrinsics(scene_name, width, height)
    base = scene if scene_name != "large_room" else Scene("room", scene.spheres, None, scene.room)
    out = []
    for i, pose in enumerate(trajectory(base, sweep or frames)[:frames]):
        d, c = render_depth(scene, pose, intr, width, height)
        d = d.astype(depth_dtype)
        c = (np.round(c * 255.0).astype(np.uint8) if color_dtype == np.uint8 else c.astype(color_dtype))
        out.append(DepthFrame(depth=d, intrinsics=intr, pose=pose, color=c, timestamp=0.1 * i))
    return out


scene_trajectory = trajectory   # the reference's name (synth.py:75)


def sphere_reference(n: int = 200_000, radius: float = 1.0) -> np.ndarray:
    """Ground-truth samples of the unit-sphere scene (synth.py:178-179)."""
    return fibonacci_directions(n) * radius


def frames_reference(frames: list, stride: int = 4, max_points: int = 300_000,
                     seed: int = 0) -> np.ndarray:
    """Observed-surface reference: every `stride`-th valid pixel of each frame
    back-projected to world (synth.py:182-197), subsampled without
    replacement to `max_points` with the seeded generator."""
    parts = []
    for f in frames:
        rows, cols = np.nonzero(f.valid_mask())
        rows, cols = rows[::stride], cols[::stride]
        z = f.metres()[rows, cols]
        k = f.intrinsics
        cam = np.stack([(cols - k.cx) / k.fx * z, (rows - k.cy) / k.fy * z, z], axis=1)
        parts.append(f.pose.to_world(cam))
    pts = np.concatenate(parts)
    if len(pts) > max_points:
        pts = pts[np.random.default_rng(seed).choice(len(pts), size=max_points, replace=False)]
    return pts


def rotation_to_quaternion(rot) -> tuple:
    """Scalar-last unit quaternion (qx, qy, qz, qw) of a proper rotation, from
    the largest of the four |q| components (numerically safe everywhere)."""
    m = np.asarray(rot, dtype=np.float64)
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    cand = np.array([1.0 + m[0, 0] - m[1, 1] - m[2, 2], 1.0 - m[0, 0] + m[1, 1] - m[2, 2],
                     1.0 - m[0, 0] - m[1, 1] + m[2, 2], 1.0 + tr])
    big = int(np.argmax(cand))
    r = 0.5 * np.sqrt(cand[big])
    s = 0.25 / r
    sym = {(0, 1): m[0, 1] + m[1, 0], (0, 2): m[0, 2] + m[2, 0], (1, 2): m[1, 2] + m[2, 1]}
    skew = (m[2, 1] - m[1, 2], m[0, 2] - m[2, 0], m[1, 0] - m[0, 1])
    q = np.zeros(4)
    q[big] = r
    for j in range(3):
        if j != big:
            q[j] = (skew[j] if big == 3 else sym[tuple(sorted((big, j)))]) * s
    if big != 3:
        q[3] = skew[big] * s
    q /= np.linalg.norm(q)
    return tuple(float(x) for x in q)


def generate_dataset(scene_name: str, out_dir, frames: int = 30, width: int = 96, height: int = 72,
                     sensor_mode: str = "depth", depth_scale: float = 5000.0,
                     cloud_stride: int = 2):
    """Write a fixture dataset in the reference's layout (synth.py:230-274):
    intrinsics.txt, trajectory.txt (t = 0.1 i), depth/ + rgb/ 16-bit and RGB
    PNGs (raw = round(z * depth_scale)) or clouds/*.pcb (every
    `cloud_stride`-th valid pixel, sensor frame, with colour), and a
    reference.ply ground-truth point cloud.  Returns the directory."""
    from pathlib import Path

    from PIL import Image

    from .datasets import write_pointcloud_file
    from .formats import write_point_cloud
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    scene = make_scene(scene_name)
    intr = default_intrinsics(scene_name, width, height)
    (out / "intrinsics.txt").write_text(f"{intr.fx} {intr.fy} {intr.cx} {intr.cy}\n")
    lines, rendered = [], []
    for i, pose in enumerate(trajectory(scene, frames)):
        qx, qy, qz, qw = rotation_to_quaternion(pose.rotation)
        tx, ty, tz = pose.translation
        lines.append(f"{0.1 * i:.6f} {tx:.9f} {ty:.9f} {tz:.9f} {qx:.9f} {qy:.9f} {qz:.9f} {qw:.9f}")
        depth, rgb = render_depth(scene, pose, intr, width, height)
        frame = DepthFrame(depth=depth, intrinsics=intr, pose=pose, color=rgb)
        rendered.append(frame)
        if sensor_mode == "depth":
            for sub in ("depth", "rgb"):
                (out / sub).mkdir(exist_ok=True)
            raw = np.clip(np.round(depth * depth_scale), 0, 65535).astype(np.uint16)
            Image.fromarray(raw).save(out / "depth" / f"{i:06d}.png")
            Image.fromarray((rgb * 255).astype(np.uint8)).save(out / "rgb" / f"{i:06d}.png")
        else:
            (out / "clouds").mkdir(exist_ok=True)
            rows, cols = np.nonzero(frame.valid_mask())
            rows, cols = rows[::cloud_stride], cols[::cloud_stride]
            z = depth[rows, cols]
            pts = np.stack([(cols - intr.cx) / intr.fx * z, (rows - intr.cy) / intr.fy * z, z], axis=1)
            write_pointcloud_file(out / "clouds" / f"{i:06d}.pcb", pts, rgb[rows, cols])
    (out / "trajectory.txt").write_text("\n".join(lines) + "\n")
    truth = sphere_reference(150_000) if scene_name == "sphere" else frames_reference(rendered)
    write_point_cloud(truth, out / "reference.ply")
    return out


# ---------------------------------------------------------------------------
# 128-beam spinning LiDAR
# ---------------------------------------------------------------------------

@dataclass
class LidarScene:
    ground_z: float = -1.8
    walls: tuple = (60.0, 90.0)
    ceiling_z: float | None = 30.0
    spheres: np.ndarray = None   # (K, 3) centres
    radius: float = 1.5


def make_lidar_scene(n_spheres: int = 40, ceiling_z: float | None = 30.0) -> LidarScene:
    rng = np.random.default_rng(0)
    c = np.stack([rng.uniform(-50, 50, n_spheres), rng.uniform(-80, 80, n_spheres),
                  rng.uniform(-1.8, 2.0, n_spheres)], axis=1)
    return LidarScene(ceiling_z=ceiling_z, spheres=c)


def lidar_directions(beams: int = 128, columns: int = 2048, fov_deg=(-45.0, 45.0)) -> np.ndarray:
    el = np.deg2rad(np.linspace(fov_deg[0], fov_deg[1], beams))
    az = 2.0 * np.pi * np.arange(columns) / columns
    e, a = np.meshgrid(el, az, indexing="ij")
    return np.stack([np.cos(e) * np.cos(a), np.cos(e) * np.sin(a), np.sin(e)], -1).reshape(-1, 3)


def lidar_scan(scene: LidarScene, origin, dirs: np.ndarray, max_range: float = 100.0,
               dtype=np.float32) -> np.ndarray:
    """Sensor-frame returns (identity rotation) within max_range."""
    o = np.asarray(origin, dtype=np.float64)
    n = len(dirs)
    best = np.full(n, np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        planes = [(2, scene.ground_z)]
        if scene.ceiling_z is not None:
            planes.append((2, scene.ceiling_z))
        planes += [(0, -scene.walls[0]), (0, scene.walls[0]), (1, -scene.walls[1]), (1, scene.walls[1])]
        for axis, val in planes:
            t = (val - o[axis]) / dirs[:, axis]
            ok = np.isfinite(t) & (t > 1e-6)
            best = np.where(ok & (t < best), t, best)
        for c in scene.spheres:
            oc = o - c
            b = dirs @ oc
            disc = b * b - (oc @ oc - scene.radius ** 2)
            t = -b - np.sqrt(np.maximum(disc, 0.0))
            ok = (disc > 0) & (t > 1e-6)
            best = np.where(ok & (t < best), t, best)
    keep = best <= max_range
    return (dirs[keep] * best[keep, None]).astype(dtype)


def lidar_frames(scans: int, beams: int = 128, columns: int = 2048, step: float = 0.5,
                 ceiling_z: float | None = 30.0, dtype=np.float32) -> list:
    scene = make_lidar_scene(ceiling_z=ceiling_z)
    dirs = lidar_directions(beams, columns)
    out = []
    for k in range(scans):
        org = np.array([step * k, 0.0, 0.0])
        pts = lidar_scan(scene, org, dirs, dtype=dtype)
        out.append(PointCloudFrame(points=pts, pose=SensorPose(np.eye(3), org), timestamp=0.1 * k))
    return out
