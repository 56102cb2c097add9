"""Aggregate ncu source-page (cuda,sass) stall samples per CUDA source line."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
agg = defaultdict(lambda: [0, 0, ""])
fname = None
hdr = None
cur_line = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or fname is None:
        continue
    si = hdr.index("Warp Stall Sampling (All Samples)")
    ie = hdr.index("Instructions Executed")
    if r[0].isdigit():
        cur_line = (fname, int(r[0]), r[1].strip()[:80])
    if len(r) > si and r[2].startswith("0x") and cur_line:
        try:
            agg[cur_line][0] += int(r[si] or 0)
            agg[cur_line][1] += int(r[ie] or 0)
        except ValueError:
            pass
tot = sum(v[0] for v in agg.values())
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{100*v[0]/max(tot,1):5.1f}% {v[1]:>10} {k[0]}:{k[1]}  {k[2]}")
