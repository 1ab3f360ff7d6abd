"""Per-CUDA-line instruction / stall-sample totals of one kernel in an ncu report.

    python scripts/ncu_lines.py <report.ncu-rep> <kernel-regex> [top]
"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
cur, ie, ss, data = None, None, None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        ie = r.index("Instructions Executed")
        ss = r.index("Warp Stall Sampling (All Samples)")
        continue
    if ie is None or len(r) <= ie or r[0] == "-":
        continue
    try:
        n, s = int(float(r[ie] or 0)), int(float(r[ss] or 0))
    except ValueError:
        continue
    if n or s:
        data.append((n, s, cur, r[0], r[1].strip()[:90]))
ti = sum(d[0] for d in data) or 1
ts = sum(d[1] for d in data) or 1
print(f"{'inst%':>6} {'stall%':>6}  file:line  source")
for d in sorted(data, reverse=True)[:top]:
    print(f"{100 * d[0] / ti:6.1f} {100 * d[1] / ts:6.1f}  {d[2]}:{d[3]}  {d[4]}")
