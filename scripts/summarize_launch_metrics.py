"""Summarise an ncu launch list taken with several --metrics (csv, one row per
kernel launch and metric, e.g. scripts/gpu_final_ncu.sh's room_launches.csv)
into a per-kernel markdown table: launches, mean / median duration, share of
the serialised kernel time, DRAM bytes and warp instructions per launch.

  python scripts/summarize_launch_metrics.py launches.csv [title] > out.md
"""
import collections
import csv
import statistics
import sys


def main(path, title="ncu launch list"):
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in csv.reader(open(path)):
        if len(r) < 15 or r[0] == "ID":
            continue
        name = r[4].split("(")[0].replace("void ", "")
        try:
            per[name][r[12]].append(float(r[14].replace(",", "")))
        except ValueError:
            continue
    total = sum(sum(m.get("gpu__time_duration.sum", [])) for m in per.values())
    print(f"### {title}\n")
    print("ncu `--clock-control none`, every launch serialised and cold-cache: the shares, "
          "not the absolute times, compare with the bench's live CUDA-event times.\n")
    print("| kernel | launches | mean µs | median µs | share | DRAM MB / launch | warp instr / launch |")
    print("|---|---|---|---|---|---|---|")
    order = sorted(per.items(), key=lambda kv: -sum(kv[1].get("gpu__time_duration.sum", [0])))
    for name, m in order:
        t = m.get("gpu__time_duration.sum", [])
        if not t:
            continue
        dram = [a + b for a, b in zip(m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", []))]
        ins = m.get("smsp__inst_executed.sum", [])
        print(f"| `{name[:70]}` | {len(t)} | {statistics.mean(t) / 1e3:.1f} | {statistics.median(t) / 1e3:.1f} "
              f"| {sum(t) / total:.3f} | {statistics.mean(dram) / 1e6 if dram else 0:.2f} "
              f"| {statistics.mean(ins) / 1e6 if ins else 0:.2f} M |")


if __name__ == "__main__":
    main(sys.argv[1], *(sys.argv[2:3]))
