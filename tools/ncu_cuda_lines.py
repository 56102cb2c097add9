"""Per-CUDA-line stall samples from `ncu --page source --csv --print-source cuda,sass`:
python tools/ncu_cuda_lines.py export.csv [top]"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    cur, hdr, out = None, None, []
    for r in rows:
        if r and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[0] and r[2] == "-":
            try:
                s = int(r[4])
            except ValueError:
                continue
            reasons = {hdr[i][6:]: int(r[i] or 0) for i in range(len(hdr))
                       if hdr[i].startswith("stall_") and "Not Issued" not in hdr[i]}
            out.append((s, int(r[7] or 0), cur, r[0], r[1].strip()[:80], reasons))
    tot = sum(o[0] for o in out) or 1
    out.sort(key=lambda o: -o[0])
    print("total samples", tot)
    for s, i, f, l, src, rs in out[:top]:
        rr = sorted(rs.items(), key=lambda kv: -kv[1])[:3]
        print(f"{100 * s / tot:5.1f}% {i:10d} {f}:{l:5s} {src:80s} " + " ".join(f"{k}:{100 * v / max(s, 1):.0f}%" for k, v in rr))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
