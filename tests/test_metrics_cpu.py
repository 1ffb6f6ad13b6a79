"""Metrics host side (reference metrics.py:14-45): area and the sampling
stream equal the reference's; eval_reconstruction's NN queries need the GPU
(tests/test_gpu_metrics.py)."""
import numpy as np
import pytest

import parity_utils as PU


def _square():
    from paper_2511_21459_b200.meshing import Mesh
    v = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], dtype=float)
    return Mesh(vertices=v, normals=np.tile([0., 0., 1.], (4, 1)), colors=np.zeros((4, 3)),
                triangles=np.array([[0, 1, 2], [0, 2, 3]]))


def test_area_and_sampling_contract():
    from paper_2511_21459_b200.metrics import mesh_surface_area, sample_mesh_points
    m = _square()
    assert mesh_surface_area(m) == pytest.approx(1.0)
    pts = sample_mesh_points(m, samples_per_m2=1000, max_samples=10**6, seed=3)
    assert len(pts) == 1000 and np.allclose(pts[:, 2], 0.0)
    assert len(sample_mesh_points(m, samples_per_m2=10**9, max_samples=5000)) == 5000
    assert np.array_equal(sample_mesh_points(m, seed=7), sample_mesh_points(m, seed=7))


def test_sampling_equals_reference():
    if not PU.have_reference():
        pytest.skip("needs /root/reference")
    PU.import_reference()
    from tsdfusion import metrics as RM
    from tsdfusion.meshing import Mesh as RMesh
    from paper_2511_21459_b200.metrics import mesh_surface_area, sample_mesh_points
    rng = np.random.default_rng(4)
    v = rng.normal(size=(300, 3))
    tri = rng.integers(0, 300, (500, 3))
    from paper_2511_21459_b200.meshing import Mesh
    m = Mesh(vertices=v, normals=v, colors=np.zeros_like(v), triangles=tri)
    r = RMesh(vertices=v, normals=v, colors=np.zeros_like(v), triangles=tri)
    assert mesh_surface_area(m) == RM.mesh_surface_area(r)
    for seed in (0, 5):
        assert np.array_equal(sample_mesh_points(m, 50.0, 10**6, seed),
                              RM.sample_mesh_points(r, 50.0, 10**6, seed))
