"""Marching Cubes tables for the host-side single-cell helper, parsed from
the C header the kernels compile against (csrc/mc_tables.h), so there is a
single source of truth."""
import re
from pathlib import Path

import numpy as np

_src = (Path(__file__).resolve().parent / "csrc" / "mc_tables.h").read_text()


def _table(name, shape, dtype):
    body = re.search(re.escape(name) + r"[^=]*=\s*\{(.*?)\};", _src, re.S).group(1)
    vals = [int(v, 0) for v in re.findall(r"-?0x[0-9a-fA-F]+|-?\d+", body)]
    return np.array(vals, dtype=dtype).reshape(shape)


CORNER_OFFSETS = _table("MC_CORNER", (8, 3), np.int64)
CORNER_PAIRS = _table("MC_EDGE_PAIR", (12, 2), np.int64)
EDGE_LOCATION = _table("MC_EDGE_LOC", (12, 4), np.int64)
EDGE_TABLE = _table("MC_EDGE_TABLE", (256,), np.int64)
TRI_TABLE = _table("MC_TRI_TABLE", (256, 16), np.int64)
