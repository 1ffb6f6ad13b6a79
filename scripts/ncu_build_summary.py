"""Fold `ncu --set full` captures (one launch per kernel, .ncu-rep) of the
CURRENT build into profiles/ncu_summary.json, stamped with the source digest
bench.py checks (a capture of another build is dropped, not reported).

usage: python scripts/ncu_build_summary.py NOTE REP.ncu-rep [REP.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

KEYS = {"dram__bytes_read.sum": "read", "dram__bytes_write.sum": "write",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue",
        "smsp__inst_executed.sum": "inst", "gpu__time_duration.sum": "dur",
        "lts__t_sector_hit_rate.pct": "l2hit", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ"}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "ms": 1e3,
         "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3}


def read(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "")
    name = name.split("::")[-1]
    out = {}
    for k, short in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            v = float(vals[i].replace(",", ""))
            out[short] = v * SCALE.get(units[i], 1.0)
    return name, out


def main(note, *reps):
    from paper_2511_21459_b200._native import source_digest
    d = {"src_sha": source_digest(), "source": note, "sms": 148, "kernels": {}}
    for rep in reps:
        name, m = read(rep)
        d["kernels"][name] = {"dram_bytes": int(m.get("read", 0) + m.get("write", 0)),
                              "issue_active": round(m.get("issue", 0) / 100, 4),
                              "warp_inst": int(m.get("inst", 0)),
                              "duration_us": round(m.get("dur", 0), 2),
                              "l2_hit_pct": round(m.get("l2hit", 0), 2),
                              "occupancy_pct": round(m.get("occ", 0), 2),
                              "capture": Path(rep).name}
    import os
    out = Path(os.environ.get("NCU_SUMMARY_OUT", ROOT / "profiles" / "ncu_summary.json"))
    out.write_text(json.dumps(d, indent=1, sort_keys=True) + "\n")
    print(json.dumps(d, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(*sys.argv[1:])
