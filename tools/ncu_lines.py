"""Aggregate ncu warp-stall samples per CUDA source line.

    ncu -i REP --page source --csv --print-source cuda,sass > /tmp/cs.csv
    python tools/ncu_lines.py /tmp/cs.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur, hdr = None, None
agg, src = collections.Counter(), {}
tot = 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name",):
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    try:
        ln = int(r[0])
        s = int(r[4]) if r[4] else 0
    except (ValueError, IndexError):
        continue
    agg[(cur, ln)] += s
    src[(cur, ln)] = r[1][:100]
    tot += s
print("total samples", tot)
for k, v in agg.most_common(n):
    print(f"{v:6d} {100 * v / max(tot, 1):5.1f}% {k[0]}:{k[1]}  {src[k].strip()}")
