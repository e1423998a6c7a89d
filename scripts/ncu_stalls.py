"""Stall reasons (warp samples) summed over a CUDA line range of one file, from an ncu source export.

    ncu -i rep --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_stalls.py src.csv score_coop.cu 600 700     # also prints the top lines
"""
import csv
import sys
from collections import defaultdict

path, fname, lo, hi = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
rows = list(csv.reader(open(path)))
hdr = None
tot = defaultdict(int)
per_line = defaultdict(int)
src = {}
cur_file, cur_line = "", 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) - 2:
        continue
    if r[0]:
        try:
            cur_line = int(r[0])
        except ValueError:
            continue
        src[(cur_file, cur_line)] = r[1].strip()[:90]
    if cur_file != fname or not (lo <= cur_line <= hi):
        continue
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = int(r[i] or 0)
            except ValueError:
                continue
            tot[h] += v
            per_line[cur_line] += v
s = sum(tot.values())
print(f"{fname}:{lo}-{hi} samples {s}")
for h, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {h:28s} {v:9d} {100 * v / max(s, 1):5.1f}%")
for ln, v in sorted(per_line.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  L{ln:4d} {v:8d}  {src.get((fname, ln), '')}")
