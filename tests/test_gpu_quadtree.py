"""GPU quadtree build and splat seeding (reference quadtree.py:94-148)
against the reference's outputs on the same inputs
(tests/golden/quadtree.json from scripts/make_golden_quadtree.py): leaf
lists in breadth-first order, contrasts, seed positions, scales and
colours all bit-identical."""
import json
from pathlib import Path

import numpy as np
import pytest

from quadtree_cases import image_cases, seed_cases

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).parent / "golden" / "quadtree.json").read_text())


def _fx(h):
    return np.array([float.fromhex(x) for x in h])


@pytest.mark.parametrize("name", sorted(image_cases()))
def test_quadtree_leaves_match_reference(name):
    from paper_2511_21459_b200.quadtree import build_quadtree
    img, thr, mp = image_cases()[name]
    leaves = build_quadtree(img, thr, mp)
    g = GOLD["trees"][name]
    assert [[q.x0, q.y0, q.w, q.h] for q in leaves] == g["leaves"]
    assert np.array_equal(np.array([q.contrast for q in leaves]), _fx(g["contrast"]))
    assert all(q.is_leaf for q in leaves)
    # the leaves tile the image exactly once
    h, w = np.asarray(img).shape[:2]
    cover = np.zeros((h, w), dtype=np.int64)
    for q in leaves:
        cover[q.y0:q.y0 + q.h, q.x0:q.x0 + q.w] += 1
    assert np.all(cover == 1)


@pytest.mark.parametrize("name", sorted(seed_cases()))
def test_seed_splats_match_reference(name):
    from paper_2511_21459_b200.quadtree import build_quadtree, seed_splats
    img, thr, mp, frame = seed_cases()[name]
    leaves = build_quadtree(img, thr, mp)
    seeds = seed_splats(leaves, frame)
    g = GOLD["seeds"][name]
    assert len(leaves) == g["n_leaves"] and len(seeds) == g["n"]
    assert np.array_equal(np.array([s.position for s in seeds]).reshape(-1), _fx(g["position"]))
    assert np.array_equal(np.array([s.scale for s in seeds]), _fx(g["scale"]))
    assert np.array_equal(np.array([s.color for s in seeds]).reshape(-1), _fx(g["color"]))


def test_quadtree_errors():
    from paper_2511_21459_b200.quadtree import build_quadtree
    with pytest.raises(ValueError):
        build_quadtree(np.zeros((0, 4, 3)))
    with pytest.raises(ValueError, match="keep splitting"):
        build_quadtree(np.zeros((2, 2, 3)), -1.0, 0)
