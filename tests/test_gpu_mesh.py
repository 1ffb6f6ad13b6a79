"""GPU Marching Cubes parity: the reference's golden mesh digests
(tests/test_meshing.py:435-491 of the reference), golden scenario meshes
from tests/golden, and the oracle on larger two- and three-level grids.
The contract is bit-identical output (vertices, normals, colours,
triangle order); Chamfer / F-score against the oracle are reported too."""
import numpy as np
import pytest

import parity_utils as PU
from test_oracle_golden import MESH_KATS

pytestmark = pytest.mark.gpu


def assert_mesh_equal(a, b):
    for x, y, what in zip(a, b, ("vertices", "normals", "colors", "triangles")):
        assert x.shape == y.shape, (what, x.shape, y.shape)
        assert np.array_equal(x, y), what


@pytest.mark.parametrize("name", list(MESH_KATS))
def test_reference_golden_meshes_on_gpu(name):
    kw, fill, nv, nt, digest = MESH_KATS[name]
    b = PU.GpuBackend(kw["n_hash"], 0.08, kw["caps"])
    fill(b)
    v, n, c, t = b.mesh()
    assert (len(v), len(t)) == (nv, nt)
    assert PU.mesh_digest(v, t) == digest
    o = PU.OracleBackend(kw["n_hash"], 0.08, kw["caps"])
    fill(o)
    assert_mesh_equal((v, n, c, t), o.mesh())


@pytest.mark.parametrize("name", ["depth_room", "depth_sphere"])
def test_golden_scenario_meshes(golden, name):
    g = golden["scenarios"][name]
    spec = {k: (tuple(v) if isinstance(v, list) else v) for k, v in g["spec"].items() if k != "kind"}
    b, _, _, _ = PU.run_depth_scenario("gpu", **spec)
    v, n, c, t = b.mesh()
    assert (len(v), len(t)) == (g["mesh"]["nv"], g["mesh"]["nt"])
    assert PU.mesh_digest(v, t) == g["mesh"]["digest"]
    assert PU.array_digest(v, n, c, t) == g["mesh"]["full_digest"]


def test_c1_mesh_vs_oracle_and_fscore():
    spec = ("room", 30, 320, 240, 0.08, 0.03, (60000, 20000), 1000003)
    bg, _, _, _ = PU.run_depth_scenario("gpu", *spec, sigma=2.5e-5)
    bo, _, _, _ = PU.run_depth_scenario("oracle", *spec, sigma=2.5e-5)
    mg, mo = bg.mesh(), bo.mesh()
    assert_mesh_equal(mg, mo)
    from scipy.spatial import cKDTree
    d1 = cKDTree(mo[0]).query(mg[0])[0]
    d2 = cKDTree(mg[0]).query(mo[0])[0]
    chamfer = 0.5 * (d1.mean() + d2.mean())
    nu = 0.01
    assert chamfer <= 0.05 * nu
    f = 2 * (d1 < 0.5 * nu).mean() * (d2 < 0.5 * nu).mean() / max(
        (d1 < 0.5 * nu).mean() + (d2 < 0.5 * nu).mean(), 1e-12)
    assert f >= 0.999


def test_three_level_mesh_vs_oracle():
    spec = ("sphere", 40, 64, 48, 0.08, 0.03, (30000, 10000, 4000), 100003)
    bg, _, _, _ = PU.run_depth_scenario("gpu", *spec, sigma=2.5e-4, all_levels=True)
    bo, _, _, _ = PU.run_depth_scenario("oracle", *spec, sigma=2.5e-4, all_levels=True)
    assert PU.level_summary(bg.state())[2] > 0
    assert_mesh_equal(bg.mesh(), bo.mesh())


def test_mesh_iso_and_eps_variants_vs_oracle():
    spec = ("sphere", 12, 48, 36, 0.08, 0.03, (20000, 4000), 100003)
    bg, _, _, _ = PU.run_depth_scenario("gpu", *spec, sigma=2.5e-4, cadence=6)
    bo, _, _, _ = PU.run_depth_scenario("oracle", *spec, sigma=2.5e-4, cadence=6)
    for iso, eps in [(0.0, 0.0), (0.004, None), (-0.003, 0.005)]:
        assert_mesh_equal(bg.mesh(iso, eps), bo.mesh(iso, eps))


def test_empty_and_unobserved_tables():
    b = PU.GpuBackend(97, 0.08, (64, 16))
    v, n, c, t = b.mesh()
    assert len(v) == 0 and len(t) == 0
    b.insert((0, 0, 0), 0)  # allocated but never observed
    v, n, c, t = b.mesh()
    assert len(v) == 0 and len(t) == 0


def test_collapse_vertices_vs_oracle():
    import ctypes as C
    import paper_2511_21459_b200 as P
    from oracle.oracle import oracle_lib, _take
    rng = np.random.default_rng(4)
    for nv, ntri, eps in [(200, 150, 0.07), (60, 40, 0.05), (500, 300, 0.0), (30, 0, 0.1)]:
        v = rng.uniform(0, 1, size=(nv, 3))
        v[nv // 2:] = np.round(v[nv // 2:] * 8) / 8  # exact duplicates
        n = rng.normal(size=(nv, 3))
        c = rng.uniform(0, 1, size=(nv, 3))
        t = rng.integers(0, nv, size=(ntri, 3)).astype(np.int64)
        mg = P.collapse_vertices(P.Mesh(v, n, c, t), eps)
        L = oracle_lib()
        dp = [C.POINTER(C.c_double)() for _ in range(3)]
        tp = C.POINTER(C.c_int64)()
        a, b_ = C.c_int64(), C.c_int64()
        L.ot_collapse_vertices(np.ascontiguousarray(v), np.ascontiguousarray(n),
                               np.ascontiguousarray(c), nv, np.ascontiguousarray(t), ntri, eps,
                               C.byref(dp[0]), C.byref(dp[1]), C.byref(dp[2]), C.byref(a),
                               C.byref(tp), C.byref(b_))
        mo = (_take(dp[0], a.value, np.float64, 3), _take(dp[1], a.value, np.float64, 3),
              _take(dp[2], a.value, np.float64, 3), _take(tp, b_.value, np.int64, 3))
        assert_mesh_equal((mg.vertices, mg.normals, mg.colors, mg.triangles), mo)
