"""Generate tests/golden/golden.json by running the REFERENCE package.

Run in the build container only (needs /root/reference):
    python scripts/make_golden.py
The fixtures are small: per-scenario stats, key-set / state / mesh digests
and input digests (inputs are regenerated bit-identically by
paper_2511_21459_b200.synth, whose output is pinned by the input digests).
The GPU box never reads /root/reference; it checks the oracle and the
product against these numbers.
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

SCENARIOS = {
    # C1-like: the reference room at 1 cm, two levels, merges every 10 frames
    "depth_room": dict(kind="depth", scene="room", frames=20, width=64, height=48, edge=0.08,
                       tau=0.03, caps=(20000, 10000), n_hash=100003, sigma=2.5e-5),
    # unit sphere orbit: plenty of merges, mixed-level mesh
    "depth_sphere": dict(kind="depth", scene="sphere", frames=30, width=48, height=36,
                         edge=0.08, tau=0.03, caps=(20000, 10000), n_hash=100003, sigma=2.5e-4),
    # C2-like geometry at 5 mm on a reduced image
    "depth_room_5mm": dict(kind="depth", scene="room", frames=3, width=160, height=120,
                           edge=0.04, tau=0.015, caps=(60000, 10000), n_hash=1000003),
    # weight cap + no colour
    "depth_room_wcap": dict(kind="depth", scene="room", frames=12, width=48, height=36,
                            edge=0.08, tau=0.04, caps=(20000, 10000), n_hash=100003,
                            weight_cap=3.0, color=False),
    # sparse LiDAR (C3 geometry, reduced beam count), u8 colours, merges
    "lidar_small": dict(kind="lidar", scans=3, beams=16, columns=256, edge=1.6, tau=0.8,
                        caps=(60000, 20000), n_hash=1000003, sigma=1e-2, color=True),
}


def run(name, spec, backend="reference"):
    spec = dict(spec)
    kind = spec.pop("kind")
    t0 = time.time()
    if kind == "depth":
        b, stats, merges, seq = PU.run_depth_scenario(backend, **spec)
        inp = PU.array_digest(*[np.asarray(f.depth) for f in seq],
                              *[np.asarray(f.color) for f in seq if f.color is not None])
    else:
        b, stats, merges, seq = PU.run_lidar_scenario(backend, **spec)
        inp = PU.array_digest(*[np.asarray(f.points) for f in seq])
    st = b.state()
    out = {"stats": stats, "merges": merges, "levels": PU.level_summary(st),
           "keys_digest": PU.keys_digest(st), "state_digest": PU.state_digest(st),
           "input_digest": inp}
    if kind == "depth" and name in ("depth_room", "depth_sphere"):
        v, n, c, t = b.mesh()
        out["mesh"] = {"nv": int(len(v)), "nt": int(len(t)), "digest": PU.mesh_digest(v, t),
                       "full_digest": PU.array_digest(v, n, c, t)}
    out["seconds"] = round(time.time() - t0, 2)
    return out


def main():
    assert PU.have_reference(), "needs /root/reference"
    hashgrid, _, _, _ = PU.import_reference()
    from tsdfusion import dda
    rng = np.random.default_rng(7)
    gold = {"generator": "scripts/make_golden.py", "reference": "/root/reference/pkg/src/tsdfusion"}
    # hash_key (hashgrid.py:30-46): random coords incl. negatives, several n_hash
    hv = []
    for _ in range(200):
        c = [int(v) for v in rng.integers(-10**6, 10**6, size=3)]
        n = int(rng.integers(1, 10**7))
        hv.append([c, n, int(hashgrid.hash_key(c, n))])
    hv += [[[1, 0, 0], 1000003, int(hashgrid.hash_key((1, 0, 0), 1000003))],
           [[-1, -1, -1], 97, int(hashgrid.hash_key((-1, -1, -1), 97))]]
    gold["hash"] = hv
    # dda (dda.py:8-86): scalar segments and one lock-step batch
    segs = []
    for _ in range(150):
        o = rng.uniform(-2, 2, 3)
        e = o + rng.uniform(-1, 1, 3) * rng.uniform(0.2, 6)
        edge = float(rng.choice([0.08, 0.3, 1.0]))
        segs.append([o.tolist(), e.tolist(), edge, [list(map(int, b)) for b in dda.dda_blocks(o, e, edge)]])
    gold["dda_scalar"] = segs
    O = rng.uniform(-1, 1, (300, 3))
    E = O + rng.uniform(-1, 1, (300, 3)) * 2
    ids, co = dda.dda_blocks_batch(O, E, 0.3)
    gold["dda_batch"] = {"origins": O.tolist(), "endpoints": E.tolist(), "edge": 0.3,
                         "rows_digest": PU.array_digest(ids.astype(np.int64), co.astype(np.int64)),
                         "rows": int(len(ids))}
    gold["scenarios"] = {}
    for name, spec in SCENARIOS.items():
        res = run(name, spec)
        res["spec"] = {k: (list(v) if isinstance(v, tuple) else v) for k, v in spec.items()}
        gold["scenarios"][name] = res
        print(name, res["levels"], res["seconds"], "s", flush=True)
    out = ROOT / "tests" / "golden" / "golden.json"
    out.write_text(json.dumps(gold, indent=1, sort_keys=True))
    print("wrote", out)


if __name__ == "__main__":
    main()
