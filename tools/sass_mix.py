"""Aggregate an ncu `--page source --print-source sass --csv` dump by opcode:
executed warp instructions and stall samples per opcode (top N)."""
import csv
import sys
from collections import Counter

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
hdr = rows[1]
ix = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
cnt, samp = Counter(), Counter()
for r in rows[2:]:
    if len(r) <= ix:
        continue
    op = r[1].strip().split()
    if not op:
        continue
    o = op[0]
    if o.startswith("@"):
        o = op[1] if len(op) > 1 else o
    o = o.split(".")[0]
    try:
        cnt[o] += int(r[ix] or 0)
        samp[o] += int(r[isamp] or 0)
    except ValueError:
        pass
tot = sum(cnt.values())
ts = sum(samp.values())
print(f"total warp-inst {tot:.3e}, samples {ts}")
for o, c in cnt.most_common(top):
    print(f"{o:10s} {c:12d} {100*c/tot:5.1f}%  stall-samples {100*samp[o]/max(ts,1):5.1f}%")
