"""Quadtree on CPU: the committed golden file is what the reference
produces on tests/quadtree_cases.py (regenerated here when /root/reference
exists), and the host helper region_contrast equals the reference's."""
import json
from pathlib import Path

import numpy as np
import pytest

import parity_utils as PU
from quadtree_cases import image_cases

GOLD = json.loads((Path(__file__).parent / "golden" / "quadtree.json").read_text())


def test_golden_pins_reference_trees():
    if not PU.have_reference():
        pytest.skip("needs /root/reference")
    PU.import_reference()
    from tsdfusion import quadtree as Q
    for name, (img, thr, mp) in image_cases().items():
        if img.shape[0] * img.shape[1] > 5000:
            continue  # the small cases suffice to pin the file (the generator ran them all)
        leaves = Q.build_quadtree(img, thr, mp)
        assert [[q.x0, q.y0, q.w, q.h] for q in leaves] == GOLD["trees"][name]["leaves"]
        assert [q.contrast.hex() if isinstance(q.contrast, float) else float(q.contrast).hex()
                for q in leaves] == GOLD["trees"][name]["contrast"]


def test_region_contrast_matches_reference():
    from paper_2511_21459_b200.quadtree import QuadNode, region_contrast
    img = np.random.default_rng(3).uniform(0, 1, (20, 30, 3))
    node = QuadNode(3, 4, 11, 9)
    if PU.have_reference():
        PU.import_reference()
        from tsdfusion import quadtree as Q
        assert region_contrast(img, node) == Q.region_contrast(img, Q.QuadNode(3, 4, 11, 9))
    region = img[4:13, 3:14].reshape(-1, 3)
    assert region_contrast(img, node) == pytest.approx(float(np.array([0.2989, 0.5870, 0.1140]) @ region.var(axis=0)))
