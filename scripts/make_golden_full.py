"""Generate tests/golden/golden_full.json: full-scale fixtures from the LIVE
reference (VERDICT r1 "next" #1).

Run in the build container only (needs /root/reference; ~8 min, ~6 GB RAM):
    python scripts/make_golden_full.py [name ...]

Scenarios, at the BASELINE configs' real sizes:
  * c1_full        -- config 1: the reference room, 320x240, 30 frames, two
                      levels, a merge pass every 10 frames (3 passes), the
                      mixed-resolution mesh of the final map.
                      Reference calls: integrate.py:255-342, adapt.py:119-136,
                      meshing.py:412-487.
  * c2_large_frame -- config 2 geometry: the SURVEY §8d large room, 640x480,
                      5 mm, f32 depth + u8 RGB (the bench's 7 B/px input),
                      first two frames (131 k blocks), one merge pass.
  * c3_scan        -- config 3: one full 128-beam x 2048-column scan
                      (~260 k returns), 1.6 m blocks, tau 0.8, one merge pass
                      (integrate.py:175-252).
Each entry holds per-frame stats, merge stats, level counts, the key-set and
full-state sha256 digests, input digests and (c1) the mesh digests.  The GPU
tests and the oracle tests compare against these digests; the inputs are
regenerated bit-identically by paper_2511_21459_b200.synth (pinned by the
input digests).
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import parity_utils as PU  # noqa: E402

OUT = ROOT / "tests" / "golden" / "golden_full.json"


def main(names):
    assert PU.have_reference(), "needs /root/reference"
    gold = json.loads(OUT.read_text()) if OUT.exists() else {}
    gold["generator"] = "scripts/make_golden_full.py"
    gold["reference"] = "/root/reference/pkg/src/tsdfusion"
    gold.setdefault("scenarios", {})
    for name in names:
        spec = dict(PU.FULL_SCENARIOS[name])
        t0 = time.time()
        res = PU.run_full_scenario("reference", name, mesh=True)
        res["spec"] = {k: (list(v) if isinstance(v, tuple) else v) for k, v in spec.items()
                       if not callable(v)}
        res["seconds"] = round(time.time() - t0, 1)
        gold["scenarios"][name] = res
        OUT.write_text(json.dumps(gold, indent=1, sort_keys=True))
        print(name, res["levels"], res["seconds"], "s", flush=True)
    print("wrote", OUT)


if __name__ == "__main__":
    main(sys.argv[1:] or list(PU.FULL_SCENARIOS))
