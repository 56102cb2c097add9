"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of the keyswitch
kernels from one `ncu --set full` capture of `tools/profile_ks.py 8 1`, written as JSON for
bench.py's roofline.traffic (profiles/r01_ncu_traffic.json)."""
import csv
import json
import subprocess
import sys

STAGE_OF = [("k_modup_in", "modup_in"), ("k_ks_inner", "ks_inner"), ("k_moddown_out", "moddown_out")]


def main(reps, out, batch=8):
    res = {}
    for rep in reps:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(txt.splitlines()))
        h, units = rows[0], rows[1]
        bc = 0
        for r in rows[2:]:
            name = r[h.index("Kernel Name")]
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                u = units[h.index(m)]
                f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                tot += float(r[h.index(m)]) * f
            st = None
            if "k_bconv_colpass" in name:
                st = "modup_bconv" if bc == 0 else "moddown_bconv"
                bc += 1
            for k, s in STAGE_OF:
                if name.startswith("void " + k) or name.startswith(k):
                    st = s
            if st and st not in res:
                def metric(m):
                    return float(r[h.index(m)]) if m in h and r[h.index(m)] not in ("", "n/a") else None
                res[st] = {"bytes_per_launch": tot, "report": rep, "launch": f"batch of {batch} C2 keyswitches", "batch": batch,
                           "fmaheavy_pipe_pct": metric("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed"),
                           "issue_active_pct": metric("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                           "l1tex_pct": metric("l1tex__throughput.avg.pct_of_peak_sustained_active"),
                           "dram_pct": metric("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    args = sys.argv[1:]
    batch = 8
    if args and args[0].startswith("--batch="):
        batch = int(args.pop(0).split("=")[1])
    main(args[:-1], args[-1], batch)
