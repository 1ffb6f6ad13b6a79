"""The oracle (oracle/tsdf_oracle.c) against golden vectors produced by the
reference (tests/golden/golden.json, scripts/make_golden.py) and against the
reference's own known-answer tests.  CPU only."""
import numpy as np
import pytest

import parity_utils as PU
from oracle.oracle import oracle_dda_blocks, oracle_dda_blocks_batch, oracle_hash_key


def test_hash_goldens(golden):
    for coord, n, want in golden["hash"]:
        assert oracle_hash_key(coord, n) == want
    # frozen values of the reference's own tests (tests/test_hashgrid.py:26-36)
    assert oracle_hash_key((0, 0, 0), 1000003) == 0
    assert oracle_hash_key((1, 0, 0), 1000003) == 855874
    assert oracle_hash_key((-1, -1, -1), 97) == 53


def test_dda_scalar_goldens(golden):
    for o, e, edge, want in golden["dda_scalar"]:
        assert [list(c) for c in oracle_dda_blocks(o, e, edge)] == want


def test_dda_examples():
    # reference tests/test_dda.py:55-66
    assert oracle_dda_blocks((0.5, 0.5, 0.5), (2.5, 0.5, 0.5), 1.0) == [(0, 0, 0), (1, 0, 0), (2, 0, 0)]
    assert oracle_dda_blocks((0.1, 0.1, 0.1), (0.7, 0.6, 0.2), 1.0) == [(0, 0, 0)]
    assert oracle_dda_blocks((0.5, 0.5, 0.5), (-1.5, 0.5, 0.5), 1.0) == [(0, 0, 0), (-1, 0, 0), (-2, 0, 0)]


def test_dda_batch_golden(golden):
    g = golden["dda_batch"]
    ids, co = oracle_dda_blocks_batch(np.array(g["origins"]), np.array(g["endpoints"]), g["edge"])
    assert len(ids) == g["rows"]
    assert PU.array_digest(ids.astype(np.int64), co.astype(np.int64)) == g["rows_digest"]


@pytest.mark.parametrize("name", ["depth_room", "depth_sphere", "depth_room_5mm",
                                  "depth_room_wcap", "lidar_small"])
def test_scenario_goldens(golden, name):
    g = golden["scenarios"][name]
    spec = {k: (tuple(v) if isinstance(v, list) else v) for k, v in g["spec"].items() if k != "kind"}
    if name.startswith("lidar"):
        b, stats, merges, seq = PU.run_lidar_scenario("oracle", **spec)
        assert PU.array_digest(*[np.asarray(f.points) for f in seq]) == g["input_digest"]
    else:
        b, stats, merges, seq = PU.run_depth_scenario("oracle", **spec)
        assert PU.array_digest(*[np.asarray(f.depth) for f in seq],
                               *[np.asarray(f.color) for f in seq if f.color is not None]) == g["input_digest"]
    assert stats == g["stats"]
    assert merges == g["merges"]
    st = b.state()
    assert PU.level_summary(st) == {int(k): v for k, v in g["levels"].items()}
    assert PU.keys_digest(st) == g["keys_digest"]
    assert PU.state_digest(st) == g["state_digest"]
    if "mesh" in g:
        v, n, c, t = b.mesh()
        assert (len(v), len(t)) == (g["mesh"]["nv"], g["mesh"]["nt"])
        assert PU.mesh_digest(v, t) == g["mesh"]["digest"]
        assert PU.array_digest(v, n, c, t) == g["mesh"]["full_digest"]


# -- the reference's golden meshes (tests/test_meshing.py:435-491) -----------

def _sphere_fill(b, radius=0.3, tau=0.05, region=0.45, edge=0.08):
    side = 8
    nu = edge / side
    g = (np.arange(side) + 0.5) * nu
    gx, gy, gz = np.meshgrid(g, g, g, indexing="ij")
    local = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
    rb = int(np.ceil(region / edge))
    for bx in range(-rb, rb):
        for by in range(-rb, rb):
            for bz in range(-rb, rb):
                sdf = np.linalg.norm(np.array([bx, by, bz]) * edge + local, axis=1) - radius
                if np.all(sdf > tau) or np.all(sdf < -tau):
                    continue
                b.insert((bx, by, bz), 0)
                b.write((bx, by, bz), np.clip(sdf, -tau, tau), 1.0)


def _tilted_plane(b):
    n_hat = np.array([0.2, 0.1, 0.97])
    n_hat = n_hat / np.linalg.norm(n_hat)
    g = (np.arange(8) + 0.5) * 0.01
    gx, gy, gz = np.meshgrid(g, g, g, indexing="ij")
    local = np.stack([gx, gy, gz], -1).reshape(-1, 3)
    for bx in range(-3, 3):
        for by in range(-3, 3):
            for bz in range(-1, 2):
                sdf = (np.array([bx, by, bz]) * 0.08 + local - np.array([0, 0, 0.013])) @ n_hat
                if np.all(sdf > 0.04) or np.all(sdf < -0.04):
                    continue
                b.insert((bx, by, bz), 0)
                b.write((bx, by, bz), np.clip(sdf, -0.04, 0.04), 3.0)


def _two_level(b):
    g = (np.arange(8) + 0.5) * 0.01
    _, _, gz = np.meshgrid(g, g, g, indexing="ij")
    for bx in range(-8, 8):
        for by in range(-8, 8):
            b.insert((bx, by, 0), 0)
            b.write((bx, by, 0), np.clip(gz.reshape(-1) - 0.035, -0.04, 0.04), 5.0,
                    5e-3 if bx < 0 else 0.0)
    b.merge(2.5e-5)


MESH_KATS = {
    "sphere": (dict(n_hash=4099, caps=(2048, 16)), _sphere_fill, 15570, 31136,
               "53f2cf7ee42f89b616790d3b347bead979cc3d485608be88071891c881f5e7bc"),
    "tilted_plane": (dict(n_hash=4099, caps=(512, 16)), _tilted_plane, 2929, 5645,
                     "a09396552d9c389bcc0d71b9453357d272554d6843d88466ff5e9929ba40d95d"),
    "two_level": (dict(n_hash=8209, caps=(1024, 256)), _two_level, 10530, 20480,
                  "ecc2fce875b52302be499ac397d8d0fd44431f2600761381153ae1ab67816928"),
}


@pytest.mark.parametrize("name", list(MESH_KATS))
def test_reference_golden_meshes(name):
    kw, fill, nv, nt, digest = MESH_KATS[name]
    b = PU.OracleBackend(kw["n_hash"], 0.08, kw["caps"])
    fill(b)
    v, n, c, t = b.mesh()
    assert (len(v), len(t)) == (nv, nt)
    assert PU.mesh_digest(v, t) == digest


def test_oracle_three_level_extension_runs():
    """Labelled extension (3 levels, L -> L+1 for every L): oracle only."""
    b, stats, merges, _ = PU.run_depth_scenario(
        "oracle", "sphere", 30, 48, 36, 0.08, 0.03, (20000, 10000, 5000), 100003, sigma=2.5e-4,
        all_levels=True)
    lv = PU.level_summary(b.state())
    assert lv[1] > 0 and sum(m["merged"] for m in merges) > 0
