"""Dataset readers (reference datasets.py:1-193) on CPU: the same frames,
poses and errors as the reference's readers on the same files, with depth
kept as raw uint16 + depth_scale and colour as uint8 (the kernels apply the
reader's f64 conversions on the device)."""
import struct

import numpy as np
import pytest

import parity_utils as PU
from dataset_utils import SCALE, write_cloud_dataset, write_depth_dataset


def _ref_datasets():
    if not PU.have_reference():
        pytest.skip("needs /root/reference")
    PU.import_reference()
    from tsdfusion import datasets
    return datasets


def test_depth_sequence_keeps_raw_units(tmp_path):
    from paper_2511_21459_b200.datasets import read_depth_sequence
    root = write_depth_dataset(tmp_path / "d", n_frames=3)
    frames = list(read_depth_sequence(root, root / "trajectory.txt", root / "intrinsics.txt",
                                      depth_scale=SCALE, keep_types=True))
    assert len(frames) == 3
    for f in frames:
        assert f.depth.dtype == np.uint16 and f.depth_scale == SCALE and f.raw_depth
        assert f.color.dtype == np.uint8 and f.color.shape == f.depth.shape + (3,)
        # the reader's conversion, restated (datasets.py:108-113)
        assert np.array_equal(f.metres(), f.depth.astype(np.float64) / SCALE)
        assert np.array_equal(f.valid_mask(), f.depth > 0)


def test_depth_sequence_matches_reference_reader(tmp_path):
    datasets = _ref_datasets()
    from paper_2511_21459_b200.datasets import read_depth_sequence
    root = write_depth_dataset(tmp_path / "d", n_frames=4)
    args = (root, root / "trajectory.txt", root / "intrinsics.txt")
    mine = list(read_depth_sequence(*args, depth_scale=SCALE, workers=2, keep_types=True))
    ref = list(datasets.read_depth_sequence(*args, depth_scale=SCALE))
    plain = list(read_depth_sequence(*args, depth_scale=SCALE, workers=2))
    assert len(mine) == len(ref) == len(plain)
    for a, b in zip(plain, ref):  # default: the reference's own frame types and values
        assert a.depth.dtype == np.float64 and np.array_equal(a.depth, b.depth)
        assert np.array_equal(a.color, b.color)
    for a, b in zip(mine, ref):
        assert np.array_equal(a.metres(), b.depth)
        assert np.array_equal(a.color.astype(np.float64) / 255.0, b.color)
        assert np.array_equal(a.pose.rotation, b.pose.rotation)
        assert np.array_equal(a.pose.translation, b.pose.translation)
        assert a.timestamp == b.timestamp
        assert (a.intrinsics.fx, a.intrinsics.fy, a.intrinsics.cx, a.intrinsics.cy) == \
               (b.intrinsics.fx, b.intrinsics.fy, b.intrinsics.cx, b.intrinsics.cy)


def test_cloud_sequence_matches_reference_reader(tmp_path):
    datasets = _ref_datasets()
    from paper_2511_21459_b200.datasets import read_pointcloud_sequence
    root = write_cloud_dataset(tmp_path / "c")
    mine = list(read_pointcloud_sequence(root, root / "trajectory.txt", keep_types=True))
    ref = list(datasets.read_pointcloud_sequence(root, root / "trajectory.txt"))
    plain = list(read_pointcloud_sequence(root, root / "trajectory.txt"))
    for a, b in zip(plain, ref):
        assert np.array_equal(a.points, b.points) and a.points.dtype == np.float64
        assert (a.colors is None) == (b.colors is None)
        if b.colors is not None:
            assert np.array_equal(a.colors, b.colors)
    assert len(mine) == len(ref) == 2
    for a, b in zip(mine, ref):
        assert np.array_equal(np.asarray(a.points, dtype=np.float64), b.points)
        if b.colors is None:
            assert a.colors is None
        else:
            assert np.array_equal(np.asarray(a.colors, dtype=np.float64) / 255.0
                                  if a.colors.dtype == np.uint8 else a.colors, b.colors)
        assert np.array_equal(a.pose.rotation, b.pose.rotation)
    assert mine[0].points.dtype == np.float32 and mine[0].colors.dtype == np.uint8


def test_pcb_writer_bytes_match_reference(tmp_path):
    datasets = _ref_datasets()
    from paper_2511_21459_b200.datasets import write_pointcloud_file
    rng = np.random.default_rng(1)
    pts, col = rng.normal(size=(50, 3)), rng.uniform(0, 1, (50, 3))
    for c in (None, col):
        write_pointcloud_file(tmp_path / "a.pcb", pts, c)
        datasets.write_pointcloud_file(tmp_path / "b.pcb", pts, c)
        assert (tmp_path / "a.pcb").read_bytes() == (tmp_path / "b.pcb").read_bytes()


def test_reader_errors(tmp_path):
    from paper_2511_21459_b200 import DatasetError
    from paper_2511_21459_b200.datasets import (read_depth_sequence, read_intrinsics,
                                                read_pointcloud_file, read_trajectory)
    bad = tmp_path / "t.txt"
    bad.write_text("0 0 0 0 0 0 0 1\n0 0 0 0 0 0 0 1\n")
    with pytest.raises(DatasetError, match="strictly increasing"):
        read_trajectory(bad)
    bad.write_text("0 0 0 0 0 0 1\n")
    with pytest.raises(DatasetError, match="expected 8 fields"):
        read_trajectory(bad)
    bad.write_text("# nothing\n")
    with pytest.raises(DatasetError, match="empty"):
        read_trajectory(bad)
    with pytest.raises(DatasetError, match="empty"):
        read_intrinsics(bad)
    with pytest.raises(DatasetError, match="not found"):
        read_intrinsics(tmp_path / "missing.txt")
    (tmp_path / "x.pcb").write_bytes(struct.pack("<IB", 10, 0) + b"\0" * 12)
    with pytest.raises(DatasetError, match="expected 125 bytes"):
        read_pointcloud_file(tmp_path / "x.pcb")
    root = write_depth_dataset(tmp_path / "d", n_frames=2)
    (root / "trajectory.txt").write_text("1 0 0 0 0 0 0 1\n")
    with pytest.raises(DatasetError, match="2 depth images but 1 trajectory entries"):
        read_depth_sequence(root, root / "trajectory.txt", root / "intrinsics.txt")


def test_depth_frame_scale_validation():
    from paper_2511_21459_b200 import DatasetError, DepthFrame, Intrinsics, SensorPose
    raw = np.full((4, 5), 5000, dtype=np.uint16)
    f = DepthFrame(raw, Intrinsics(1, 1, 2, 2), SensorPose.identity(), depth_scale=2500.0)
    assert f.depth.dtype == np.uint16 and np.all(f.metres() == 2.0)
    with pytest.raises(DatasetError):
        DepthFrame(raw, Intrinsics(1, 1, 2, 2), SensorPose.identity(), depth_scale=0.0)
    # without a scale, uint16 values are metres as the reference frame would hold them
    g = DepthFrame(raw, Intrinsics(1, 1, 2, 2), SensorPose.identity())
    assert np.all(g.metres() == 5000.0)
