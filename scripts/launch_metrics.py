"""Per-launch table of an ncu CSV log with several metrics per kernel
(`ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64...,dram__bytes.sum --csv`):

    python scripts/launch_metrics.py <log.csv> [last_n]

Prints the last `last_n` launches (default: all) as a markdown table: time, FP64-pipe activity, DRAM bytes.
"""
import csv
import io
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = [line for line in open(path) if line.startswith('"')]
by_id = {}
for r in csv.DictReader(io.StringIO("".join(rows))):
    by_id.setdefault(r["ID"], {"k": r["Kernel Name"]})[r["Metric Name"]] = r["Metric Value"]
ids = sorted(by_id, key=int)
if last:
    ids = ids[-last:]
print("| # | kernel | us | fp64 pipe % | DRAM MB |")
print("|---:|---|---:|---:|---:|")
total = 0.0
for i in ids:
    d = by_id[i]
    us = float(d.get("gpu__time_duration.sum", "nan").replace(",", "")) / 1e3
    total += us
    pipe = d.get("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "")
    dram = d.get("dram__bytes.sum", "")
    dram = f"{float(dram.replace(',', '')) / 1e6:.1f}" if dram else ""
    name = d["k"].replace("bd3mg::", "").replace("void ", "").split("(")[0][:70]
    print(f"| {i} | `{name}` | {us:.1f} | {pipe} | {dram} |")
print(f"\n{len(ids)} launches, {total:.1f} us serialised (ncu, --clock-control none, cold caches)")
