"""Block-index churn (VERDICT r1 "tombstone leak"; reference hashgrid.py:253-275
frees chain entries on remove, streaming.py:122-156 evicts and streams back).

A small table is driven through many evict / re-import / remove cycles with
the slot count fixed, interleaved with depth frames that keep allocating.
Erased entries leave tombstones in the open-addressing index; inserts must
reuse them and the index must be rebuilt once they pass a quarter of the
slots.  After every cycle the GPU table must equal the oracle, which applies
only the permanent removals (an evict + import round trip is the identity),
and the longest probe sequence of a live key stays short."""
import numpy as np
import pytest

import parity_utils as PU

pytestmark = pytest.mark.gpu

SPEC = dict(edge=0.08, tau=0.03, caps=(3000, 1500), n_hash=10007)


def _state(t):
    return PU.GpuBackend.state(type("x", (), {"t": t})())


def test_evict_stream_back_cycles_keep_the_index_short_and_bit_exact():
    import paper_2511_21459_b200 as P
    frames = P.synth.render_frames("room", 60, 48, 36, depth_dtype=np.float32,
                                   color_dtype=np.uint8)
    g = PU.GpuBackend(SPEC["n_hash"], SPEC["edge"], SPEC["caps"])
    o = PU.OracleBackend(SPEC["n_hash"], SPEC["edge"], SPEC["caps"])
    t = g.t
    slots = t.slots
    rng = np.random.default_rng(11)
    worst = 0
    rehash0 = t.probe_stats()["rehashes"]
    for cycle, f in enumerate(frames):
        assert g.depth(f, SPEC["tau"]) == o.depth(f, SPEC["tau"]), cycle
        coords, _ = t.live_blocks(0)
        n = len(coords)
        if n == 0:
            continue
        # 30 % of the level-0 blocks out to the host and straight back in
        sel = coords[rng.permutation(n)[: max(1, (3 * n) // 10)]]
        payload = t.evict(0, sel)
        t.import_blocks(0, sel, *payload)
        # 10 % removed for good on both sides (re-created by later frames)
        gone = coords[rng.permutation(n)[: max(1, n // 10)]]
        t.evict(0, gone)
        for c in gone:
            o.t.remove(c)
        ps = t.probe_stats()
        worst = max(worst, ps["max_probe"])
        assert ps["tombstones"] * 4 <= slots + 4 * n, (cycle, ps)
        assert t.slots == slots
    assert PU.state_digest(_state(t)) == PU.state_digest(o.state())
    ps = t.probe_stats()
    print(f"churn: {len(frames)} cycles, slots {slots}, live {ps['live']}, tombstones "
          f"{ps['tombstones']}, rebuilds {ps['rehashes'] - rehash0}, worst max probe {worst}, "
          f"mean probe {ps['mean_probe']:.2f}")
    assert worst <= 64
    # an explicit rebuild clears every tombstone and changes no content
    before = PU.state_digest(_state(t))
    t.compact()
    ps = t.probe_stats()
    assert ps["tombstones"] == 0 and ps["live"] == sum(h.occupied for h in t.heaps)
    assert PU.state_digest(_state(t)) == before
    # and the rebuilt index keeps integrating identically
    f = P.synth.render_frames("room", 61, 48, 36, depth_dtype=np.float32, color_dtype=np.uint8)[60]
    assert g.depth(f, SPEC["tau"]) == o.depth(f, SPEC["tau"])
    assert PU.state_digest(_state(t)) == PU.state_digest(o.state())


def test_rebuild_triggers_under_pure_erase_churn():
    """Insert/remove single blocks until tombstones would pass slots / 4: the
    automatic rebuild must fire and lookups stay correct."""
    import paper_2511_21459_b200 as P
    t = P.HashTable(1009, 10, 7, 0.08, (200, 100))
    slots = t.slots
    rng = np.random.default_rng(3)
    live = set()
    for i in range(slots):  # far more erasures than slots / 4
        c = tuple(int(x) for x in rng.integers(-5000, 5000, 3))
        if c in live:
            continue
        t.insert(c, 0)
        live.add(c)
        if len(live) > 150:
            victim = sorted(live)[int(rng.integers(len(live)))]
            t.remove(victim)
            live.discard(victim)
    ps = t.probe_stats()
    assert ps["rehashes"] >= 1, ps
    assert ps["live"] == len(live)
    assert ps["tombstones"] * 4 <= slots + 8
    found = t.find_batch(np.array(sorted(live), dtype=np.int64))
    assert all(h >= 0 for h in found[0])
