"""The oracle against the LIVE reference, array for array (build container
only: needs /root/reference; skipped elsewhere).  Unlike the digest fixtures
this compares every state array, the per-frame stats, the merge stats and the
full mesh (vertices, normals, colours, triangles) on fresh inputs, including
a depth stream with a weight cap and a LiDAR stream with colours and merges.
Reference: integrate.py:175-342, adapt.py:119-136, meshing.py:412-552.
"""
import numpy as np
import pytest

import parity_utils as PU

pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not PU.have_reference(), reason="needs /root/reference")]


def _same_state(a, b):
    assert set(a) == set(b)
    for level in a:
        for x, y in zip(a[level], b[level]):
            assert np.array_equal(np.asarray(x), np.asarray(y)), f"level {level} differs"


@pytest.mark.parametrize("spec", [
    dict(scene="room", frames=12, width=56, height=42, edge=0.08, tau=0.03, caps=(20000, 10000),
         n_hash=100003, sigma=2.5e-5, cadence=4),
    dict(scene="sphere", frames=16, width=40, height=30, edge=0.08, tau=0.04, caps=(20000, 10000),
         n_hash=100003, sigma=2.5e-4, cadence=8, weight_cap=4.0),
])
def test_depth_streams_match_reference(spec):
    r, sr, mr, _ = PU.run_depth_scenario("reference", **spec)
    o, so, mo, _ = PU.run_depth_scenario("oracle", **spec)
    assert sr == so and mr == mo
    _same_state(r.state(), o.state())
    for x, y in zip(r.mesh(), o.mesh()):
        assert np.array_equal(np.asarray(x), np.asarray(y))


def test_lidar_stream_matches_reference():
    spec = dict(scans=2, beams=8, columns=192, edge=1.6, tau=0.8, caps=(40000, 10000),
                n_hash=1000003, sigma=1e-2, cadence=2, color=True)
    r, sr, mr, _ = PU.run_lidar_scenario("reference", **spec)
    o, so, mo, _ = PU.run_lidar_scenario("oracle", **spec)
    assert sr == so and mr == mo
    _same_state(r.state(), o.state())
