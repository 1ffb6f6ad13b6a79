"""Capacity-tier formats on CPU: block records and PLY bytes against the
reference's (tests/golden/capacity.json, scripts/make_golden_capacity.py),
the archive store, and the map header checks (formats.py:256-292)."""
import hashlib
import json
import struct
import zlib
from pathlib import Path

import numpy as np
import pytest

from capacity_scenarios import record_payloads, small_mesh

GOLD = json.loads((Path(__file__).parent / "golden" / "capacity.json").read_text())


def _sha(b):
    return hashlib.sha256(b).hexdigest()


def test_block_records_match_reference_bytes():
    from paper_2511_21459_b200.formats import pack_block_record, unpack_block_record
    from paper_2511_21459_b200.hashgrid import BlockPayload
    for name, (coord, level, t, w, s2, col) in record_payloads().items():
        p = BlockPayload(coord=coord, level=level, tsdf=t, weight=w, s2=s2, color=col)
        for arch in (False, True):
            b = pack_block_record(p, archived=arch)
            g = GOLD["records"][f"{name}_{int(arch)}"]
            assert len(b) == g["len"] and _sha(b) == g["sha"]
            q, a, off = unpack_block_record(b, 0)
            assert a == arch and off == len(b) and q.coord == coord and q.level == level
            assert np.array_equal(q.tsdf, t) and np.array_equal(q.weight, w)
            assert np.array_equal(q.s2, s2) and np.array_equal(q.color, col)


def test_ply_matches_reference_bytes(tmp_path):
    from paper_2511_21459_b200.formats import read_mesh, write_mesh
    from paper_2511_21459_b200.meshing import Mesh
    v, n, c, tri = small_mesh()
    write_mesh(Mesh(vertices=v, normals=n, colors=c, triangles=tri), tmp_path / "m.ply")
    assert _sha((tmp_path / "m.ply").read_bytes()) == GOLD["ply"]["sha"]
    m = read_mesh(tmp_path / "m.ply")
    assert np.array_equal(m.triangles, tri) and np.allclose(m.vertices, v, atol=1e-6)


def test_archive_store():
    from paper_2511_21459_b200.errors import NotFoundError
    from paper_2511_21459_b200.hashgrid import BlockPayload
    from paper_2511_21459_b200.streaming import ArchiveStore, _pack
    a = ArchiveStore()
    pl = record_payloads()
    for coord, level, t, w, s2, col in pl.values():
        a.store(BlockPayload(coord=coord, level=level, tsdf=t, weight=w, s2=s2, color=col))
    assert len(a) == 2 and (-3, 5, 7) in a and a.coords() == sorted(a.coords())
    assert a.nbytes == sum(GOLD["records"][f"{k}_1"]["len"] for k in pl)
    keys = _pack([[-3, 5, 7], [0, 0, 0], [1024, -77, 0]])
    assert sorted(a.archived_among(keys).tolist()) == sorted(keys[[0, 2]].tolist())
    p = a.take((-3, 5, 7))
    assert p.level == 0 and len(a) == 1 and (-3, 5, 7) not in a
    with pytest.raises(NotFoundError):
        a.take((-3, 5, 7))
    assert a.peek((1024, -77, 0)).level == 1


def test_map_header_checks(tmp_path):
    from paper_2511_21459_b200.errors import FormatError
    from paper_2511_21459_b200.formats import MAP_MAGIC, MAP_VERSION, _MAP_HEADER, load_map
    head = _MAP_HEADER.pack(MAP_MAGIC, MAP_VERSION, 0, 0.01, 0.08, 0.04, 97, 10, 7, 10, 10, 0, 0)
    good = head + struct.pack("<I", zlib.crc32(head))
    bad_crc = head + struct.pack("<I", zlib.crc32(head) ^ 1)
    bad_magic = b"XXXXXXXX" + good[8:]
    hv = _MAP_HEADER.pack(MAP_MAGIC, MAP_VERSION + 1, 0, 0.01, 0.08, 0.04, 97, 10, 7, 10, 10, 0, 0)
    bad_ver = hv + struct.pack("<I", zlib.crc32(hv))
    for blob in (bad_crc, bad_magic, bad_ver, good[:20]):
        (tmp_path / "m").write_bytes(blob)
        with pytest.raises(FormatError):
            load_map(tmp_path / "m")
    with pytest.raises(FormatError):
        load_map(tmp_path / "missing")
