"""Per-region instruction / stall breakdown of one kernel in an ncu report
(SourceCounters section): chunks of N SASS instructions with their share of
executed instructions and stall samples, and the notable opcodes in each.

usage: python scripts/ncu_sass_hot.py REP.ncu-rep [chunk=32] [min_share=0.005]
"""
import csv
import io
import subprocess
import sys

NOTE = ('MUFU', 'LDG', 'STG', 'LDS', 'STS', 'DADD', 'DMUL', 'DFMA', 'DSETP', 'BRA', 'ATOMG', 'ATOMS',
        'RED', 'F2I', 'FRND', 'SHFL', 'MATCH', 'VOTE', 'BAR', 'CALL', 'RET', 'I2F', 'LDL', 'STL', 'EXIT')


def main(path, chunk=32, min_share=0.005):
    chunk, min_share = int(chunk), float(min_share)
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source=sass"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, data = rows[1], rows[2:]
    isrc, ie = h.index("Source"), h.index("Instructions Executed")
    ist, ith = h.index("Warp Stall Sampling (All Samples)"), h.index("Avg. Threads Executed")
    num = lambda x: float(x or 0)
    tot = sum(num(r[ie]) for r in data) or 1
    st = sum(num(r[ist]) for r in data) or 1
    print(f"warp instructions {tot:.0f}, stall samples {st:.0f}")
    for i in range(0, len(data), chunk):
        ch = data[i:i + chunk]
        e = sum(num(r[ie]) for r in ch)
        s = sum(num(r[ist]) for r in ch)
        if e / tot < min_share and s / st < min_share:
            continue
        ops = []
        for r in ch:
            if num(r[ie]) <= 0:
                continue
            toks = r[isrc].split()
            op = toks[1] if toks and toks[0].startswith('@') else (toks[0] if toks else '')
            if op.split('.')[0] in NOTE:
                ops.append(op)
        thr = max((num(r[ith]) for r in ch), default=0)
        print(f"{i:5d} inst {e / tot * 100:5.2f}% stall {s / st * 100:5.2f}% thr<={thr:4.1f} {' '.join(ops)[:160]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
