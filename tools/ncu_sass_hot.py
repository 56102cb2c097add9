"""Summarise an `ncu --page source --csv --print-source sass` export: stall samples and executed
instructions per opcode, the top stall reasons, and the hottest instruction windows.

usage: python tools/ncu_sass_hot.py export.csv [top_windows]"""
import csv
import re
import sys
from collections import Counter, defaultdict


def main(path, topn=12):
    rows = list(csv.reader(open(path)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr) and r[0].startswith("0x")]
    col = {h: i for i, h in enumerate(hdr)}
    samp = [int(r[col["Warp Stall Sampling (All Samples)"]] or 0) for r in data]
    inst = [int(r[col["Instructions Executed"]] or 0) for r in data]
    src = [r[col["Source"]].strip() for r in data]
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    total = sum(samp)
    print(f"{len(data)} SASS lines, {total} samples, {sum(inst):.3e} warp instructions")
    by_reason = Counter()
    for r in data:
        for h in stall_cols:
            by_reason[h] += int(r[col[h]] or 0)
    print("stall reasons:", ", ".join(f"{k[6:]} {v / total:.1%}" for k, v in by_reason.most_common(8)))
    op_s, op_i = Counter(), Counter()
    for s, n, t in zip(samp, inst, src):
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_.]+)", t)
        op = m.group(2) if m else t[:10]
        base = op.split(".")[0]
        op_s[base] += s
        op_i[base] += n
    print("opcode          samples   warp-inst")
    for op, s in op_s.most_common(25):
        print(f"  {op:14s} {s / total:6.1%}  {op_i[op]:.3e}")
    # hottest windows of 16 instructions
    W = 16
    win = [(sum(samp[i:i + W]), i) for i in range(0, len(data), W)]
    win.sort(reverse=True)
    for s, i in win[:topn]:
        print(f"--- window @{i} ({s / total:.1%} of samples)")
        for j in range(i, min(i + W, len(data))):
            reasons = sorted(((int(data[j][col[h]] or 0), h[6:]) for h in stall_cols), reverse=True)[:2]
            rs = " ".join(f"{h}:{v}" for v, h in reasons if v)
            print(f"   {samp[j]:6d} {inst[j]:9d}  {src[j][:70]:70s} {rs}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)
