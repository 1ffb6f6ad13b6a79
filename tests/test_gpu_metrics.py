"""GPU nearest-neighbour distances and reconstruction metrics (reference
metrics.py:48-80, tests/test_metrics.py): distances bit-identical to the
O(n^2) brute force and to scipy's cKDTree (what the reference calls), and
eval_reconstruction equal to the brute-force metrics of the reference's own
test oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def points_as_mesh(points):
    from paper_2511_21459_b200.meshing import Mesh
    points = np.asarray(points, dtype=np.float64)
    n = len(points)
    return Mesh(vertices=points, normals=np.tile([0.0, 0.0, 1.0], (n, 1)),
                colors=np.zeros((n, 3)), triangles=np.zeros((0, 3), dtype=np.int64))


def brute(tree, query):
    # the reference test oracle's expression (tests/test_metrics.py:18-22)
    return np.sqrt(((query[:, None, :] - tree[None]) ** 2).sum(-1)).min(1)


def brute_force_metrics(samples, reference, threshold):
    d_sr, d_rs = brute(reference, samples), brute(samples, reference)
    acc, comp = d_sr.mean(), d_rs.mean()
    p, r = (d_sr <= threshold).mean(), (d_rs <= threshold).mean()
    f = 0.0 if p + r == 0 else 2 * p * r / (p + r)
    return {"acc": acc, "comp": comp, "chamfer_l1": 0.5 * (acc + comp), "precision": p,
            "recall": r, "fscore": f}


def test_nn_distance_random_sets_bit_exact():
    from paper_2511_21459_b200.metrics import nn_distance
    rng = np.random.default_rng(1)
    for _ in range(30):
        a = rng.uniform(-1, 1, (int(rng.integers(1, 400)), 3))
        b = rng.uniform(-1.5, 1.5, (int(rng.integers(1, 400)), 3))
        assert np.array_equal(nn_distance(a, b), brute(a, b))
        assert np.array_equal(nn_distance(b, a), brute(b, a))


def test_nn_distance_degenerate_layouts():
    from paper_2511_21459_b200.metrics import nn_distance
    rng = np.random.default_rng(2)
    plane = np.c_[rng.uniform(0, 1, (500, 2)), np.zeros(500)]       # flat tree set
    line = np.c_[np.linspace(0, 1, 300), np.zeros(300), np.zeros(300)]
    same = np.ones((50, 3))                                         # one location
    far = rng.uniform(-1, 1, (200, 3)) * 50.0                       # queries far outside
    clustered = np.r_[rng.normal(0, 1e-3, (400, 3)), rng.normal(5, 1e-3, (400, 3))]
    for tree in (plane, line, same, clustered, plane[:1]):
        for q in (far, plane, rng.uniform(-0.2, 1.2, (300, 3)), tree):
            assert np.array_equal(nn_distance(tree, q), brute(tree, q))
    assert np.all(nn_distance(same, same) == 0.0)
    got = nn_distance(plane, np.array([[np.nan, 0, 0], [0.5, 0.5, 1.0]]))
    assert np.isnan(got[0]) and got[1] == brute(plane, np.array([[0.5, 0.5, 1.0]]))[0]
    from paper_2511_21459_b200 import errors
    with pytest.raises(ValueError):
        nn_distance(np.zeros((0, 3)), plane)
    with pytest.raises(ValueError):
        nn_distance(np.array([[np.inf, 0, 0]]), plane)
    assert issubclass(errors.FusionError, Exception)


def test_nn_distance_matches_ckdtree_at_scale():
    """200 k mesh-like samples against 150 k reference points of the same
    surfaces (the sizes eval_reconstruction sees), both directions."""
    from scipy.spatial import cKDTree
    from paper_2511_21459_b200.metrics import nn_distance
    rng = np.random.default_rng(3)

    def sphere(n, r, c):
        v = rng.normal(size=(n, 3))
        return c + r * v / np.linalg.norm(v, axis=1)[:, None]
    a = np.r_[sphere(120000, 1.0, np.zeros(3)), sphere(80000, 0.3, np.array([2.0, 0, 0]))]
    b = np.r_[sphere(100000, 1.002, np.zeros(3)), np.c_[rng.uniform(-3, 3, (50000, 2)), np.full(50000, -1.2)]]
    for tree, q in ((a, b), (b, a)):
        assert np.array_equal(nn_distance(tree, q), cKDTree(tree).query(q, k=1)[0])


def test_eval_reconstruction_equals_brute_force_metrics():
    from paper_2511_21459_b200.metrics import eval_reconstruction
    rng = np.random.default_rng(1)
    for _ in range(30):
        a = rng.uniform(-1, 1, (int(rng.integers(2, 300)), 3))
        b = rng.uniform(-1, 1, (int(rng.integers(2, 300)), 3))
        thr = float(rng.uniform(0.05, 0.5))
        got = eval_reconstruction(points_as_mesh(a), b, f_threshold=thr)
        want = brute_force_metrics(a, b, thr)
        for key, v in want.items():
            assert got[key] == v, key


def test_eval_reconstruction_degenerate_cases():
    from paper_2511_21459_b200.metrics import eval_reconstruction
    pts = np.random.default_rng(0).uniform(0, 1, (100, 3))
    out = eval_reconstruction(points_as_mesh(pts), pts, f_threshold=0.1)
    assert out["acc"] == out["comp"] == out["chamfer_l1"] == 0.0 and out["fscore"] == 1.0
    pts = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    shifted = pts + np.array([0.125, 0.0, 0.0])
    assert eval_reconstruction(points_as_mesh(pts), shifted, f_threshold=0.125)["fscore"] == 1.0
    assert eval_reconstruction(points_as_mesh(pts), shifted, f_threshold=0.125 - 1e-12)["fscore"] == 0.0
    with pytest.raises(ValueError):
        eval_reconstruction(points_as_mesh(np.zeros((0, 3))), pts, 0.1)
    with pytest.raises(ValueError):
        eval_reconstruction(points_as_mesh(pts), np.zeros((0, 3)), 0.1)


def test_eval_reconstruction_of_extracted_mesh():
    """The pipeline's use: the extracted room mesh sampled at the reference's
    default density against reference points, vs cKDTree + the reference's
    expressions."""
    from scipy.spatial import cKDTree
    import paper_2511_21459_b200 as P
    from paper_2511_21459_b200.metrics import eval_reconstruction, sample_mesh_points
    from paper_2511_21459_b200 import synth
    frames = synth.render_frames("room", 8, 96, 72)
    t = P.HashTable(100003, 10, 7, 0.08, (20000, 5000))
    for f in frames:
        P.integrate_depth(t, f, 0.03)
    mesh = P.extract_mesh(t)
    ref = np.concatenate([f.pose.to_world(P.backproject(*np.meshgrid(np.arange(96.0), np.arange(72.0)),
                                                        np.nan_to_num(f.depth), f.intrinsics).reshape(-1, 3))
                          for f in frames[:3]])
    got = eval_reconstruction(mesh, ref, 0.1, samples_per_m2=2e4)
    s = sample_mesh_points(mesh, 2e4, 1_000_000, 0)
    d_sr, d_rs = cKDTree(ref).query(s, k=1)[0], cKDTree(s).query(ref, k=1)[0]
    assert got["n_samples"] == len(s) > 10000
    assert got["acc"] == float(d_sr.mean()) and got["comp"] == float(d_rs.mean())
    assert got["precision"] == float((d_sr <= 0.1).mean())
    assert got["recall"] == float((d_rs <= 0.1).mean())
