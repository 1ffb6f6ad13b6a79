"""Full-scale golden fixtures from the LIVE reference (tests/golden/
golden_full.json, scripts/make_golden_full.py): BASELINE config 1 at its real
size (320x240, 30 frames, 3 merge passes, the final mesh), the first two
frames of config 2's large-room sweep (640x480 @ 5 mm, f32 depth + u8 RGB),
and one full config-3 scan (128 x 2048 beams).

* CPU: the oracle reproduces every fixture (stats, merges, level counts, key
  set, full state, mesh) -- this pins the oracle at the benchmarked sizes.
* GPU: the product (sm_100a through the C ABI) reproduces them too.
Reference calls: integrate.py:175-342, adapt.py:119-136, meshing.py:412-487.
"""
import json

import numpy as np
import pytest

import parity_utils as PU

GOLD = json.loads((PU.ROOT / "tests" / "golden" / "golden_full.json").read_text())["scenarios"]
NAMES = sorted(GOLD)


def _check(name, res):
    g = GOLD[name]
    assert res["input_digest"] == g["input_digest"], "synthetic inputs changed"
    assert res["stats"] == g["stats"]
    assert res["merges"] == g["merges"]
    assert res["levels"] == {int(k): v for k, v in g["levels"].items()}
    assert res["keys_digest"] == g["keys_digest"]
    assert res["state_digest"] == g["state_digest"]
    if "mesh" in g:
        assert res["mesh"] == g["mesh"]


@pytest.mark.parametrize("name", NAMES)
def test_oracle_full_scale_goldens(name):
    _check(name, PU.run_full_scenario("oracle", name, mesh=True))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_full_scale_goldens(name):
    _check(name, PU.run_full_scenario("gpu", name, mesh=True))


def test_fixture_sizes_are_the_baseline_configs():
    c1 = GOLD["c1_full"]
    assert c1["spec"]["width"] == 320 and c1["spec"]["height"] == 240 and len(c1["stats"]) == 30
    assert len(c1["merges"]) == 3 and sum(m["merged"] for m in c1["merges"]) > 0
    assert c1["mesh"]["nt"] > 100000
    c2 = GOLD["c2_large_frame"]
    assert c2["spec"]["width"] == 640 and c2["levels"]["0"] > 100000
    c3 = GOLD["c3_scan"]
    assert c3["spec"]["beams"] == 128 and c3["spec"]["columns"] == 2048
    assert c3["stats"][0]["measurements"] > 200000
    assert np.isfinite(c3["seconds"])
