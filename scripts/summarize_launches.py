"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) into a
per-kernel table: total time, launches, share of the step."""
import collections
import csv
import sys


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0.0, 0])
    scale = {"nsecond": 1.0, "ns": 1.0, "usecond": 1e3, "msecond": 1e6}
    for r in rows[1:]:
        name = r[ki].split("(")[0]
        agg[name][0] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        agg[name][1] += 1
    tot = sum(a[0] for a in agg.values())
    lines = ["| kernel | total ms | launches | us/launch | share |", "|---|---|---|---|---|"]
    for k, (t, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        lines.append(f"| `{k}` | {t / 1e6:.3f} | {n} | {t / n / 1e3:.1f} | {t / tot:.3f} |")
    text = "\n".join(lines)
    if out:
        open(out, "w").write(text + "\n")
    print(text)


if __name__ == "__main__":
    main(*sys.argv[1:])
