"""Aggregate an ncu SASS source page (warp-stall samples, per instruction) by
CUDA source line, using nvdisasm -g line info of the same cubin.
    python scripts/ncu_lines_pk.py <sass.csv> <nvdisasm -g -c output> <mangled kernel> [top]"""
import csv
import re
import sys
from collections import defaultdict

src_csv, lines_txt, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
rows = list(csv.reader(open(src_csv)))
hdr = rows[1]
ia, iss, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
samp = []
for r in rows[2:]:
    try:
        samp.append((int(r[ia], 16), float(r[iss] or 0), float(r[iex] or 0), r[hdr.index("Source")]))
    except (ValueError, IndexError):
        pass
base = min(a for a, _, _, _ in samp)
off2line = {}
cur = None
inside = False
for ln in open(lines_txt):
    if ln.startswith("//---") and ".text." in ln:
        inside = (".text." + kern) in ln
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
agg = defaultdict(lambda: [0.0, 0.0])
tot = 0
for a, s, e, _ in samp:
    key = off2line.get(a - base, ("?", 0))
    agg[key][0] += s
    agg[key][1] += e
    tot += s
print(f"samples {tot:.0f}")
for k, (s, e) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{s:8.0f} {100 * s / tot:5.1f}%  {e:12.0f}  {k[0]}:{k[1]}")
