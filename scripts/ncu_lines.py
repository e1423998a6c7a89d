"""Aggregate ncu --page source (cuda,sass) stall samples per CUDA source line.

    ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python scripts/ncu_lines.py src.csv [top]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
agg = defaultdict(lambda: [0, 0, 0, ""])
cur_file, cur_line, cur_src = "", "", ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if len(r) < 7 or r[0] in ("Line No", "Function Name"):
        continue
    if r[0]:
        cur_line, cur_src = r[0], r[1]
    try:
        a, n, ex = int(r[4]), int(r[5]), int(r[7] or 0)
    except ValueError:
        continue
    k = (cur_file, cur_line)
    agg[k][0] += a
    agg[k][1] += n
    agg[k][2] += ex
    agg[k][3] = cur_src.strip()[:100]
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0]:8d} {100 * v[0] / tot:5.1f}% ni={v[1]:8d} ex={v[2]:10d} {k[0]}:{k[1]} {v[3]}")
