"""Generate tests/golden/quadtree.json by running the REFERENCE quadtree
(quadtree.py:94-148) on the inputs of tests/quadtree_cases.py.

Run in the build container only (needs /root/reference):
    python scripts/make_golden_quadtree.py
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import parity_utils as PU  # noqa: E402
from quadtree_cases import image_cases, seed_cases  # noqa: E402


def hx(a):
    return [float(x).hex() for x in np.asarray(a, dtype=np.float64).reshape(-1)]


def main():
    assert PU.have_reference(), "needs /root/reference"
    PU.import_reference()
    from tsdfusion import quadtree as Q
    from tsdfusion.geometry import DepthFrame, Intrinsics, SensorPose
    gold = {"generator": "scripts/make_golden_quadtree.py", "trees": {}, "seeds": {}}
    for name, (img, thr, mp) in image_cases().items():
        leaves = Q.build_quadtree(img, thr, mp)
        gold["trees"][name] = {"leaves": [[q.x0, q.y0, q.w, q.h] for q in leaves],
                               "contrast": hx([q.contrast for q in leaves])}
    for name, (img, thr, mp, f) in seed_cases().items():
        leaves = Q.build_quadtree(img, thr, mp)
        rf = DepthFrame(depth=PU._metres(f),
                        intrinsics=Intrinsics(f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx,
                                              f.intrinsics.cy),
                        pose=SensorPose(f.pose.rotation, f.pose.translation),
                        color=None if f.color is None else PU._color_f64(f.color))
        seeds = Q.seed_splats(leaves, rf)
        gold["seeds"][name] = {"n_leaves": len(leaves), "n": len(seeds),
                               "position": hx([s.position for s in seeds]),
                               "scale": hx([s.scale for s in seeds]),
                               "color": hx([s.color for s in seeds])}
    out = ROOT / "tests" / "golden" / "quadtree.json"
    out.write_text(json.dumps(gold, indent=0, sort_keys=True))
    print("wrote", out, {k: len(v["leaves"]) for k, v in gold["trees"].items()},
          {k: v["n"] for k, v in gold["seeds"].items()})


if __name__ == "__main__":
    main()
