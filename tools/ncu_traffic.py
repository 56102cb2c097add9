"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) and pipe utilisation
of the five keyswitch kernels, from a light ncu capture of `tools/profile_ks.py 32 2`, written
as JSON for bench.py's roofline.traffic / ncu_pipes (profiles/r02_ncu_traffic.json).

Capture (on the GPU box; the csv is small, no .ncu-rep needed):
    ncu --clock-control none --metrics $(python tools/ncu_traffic.py --metrics) \
        -k regex:"k_modup_in|k_bconv|k_ks_inner|k_moddown_out" -s 5 -c 5 --csv \
        python tools/profile_ks.py 32 2 > gpurun_out/traffic.csv
Summarise:
    python tools/ncu_traffic.py gpurun_out/traffic.csv profiles/r02_ncu_traffic.json --batch=32 --tree=<git sha>
"""
import csv
import json
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "l1tex__throughput.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}


def stage_of(name, nbconv):
    if "k_bconv" in name:
        return "modup_bconv" if nbconv == 0 else "moddown_bconv"
    for k, s in (("k_modup_in", "modup_in"), ("k_ks_inner", "ks_inner"), ("k_moddown_out", "moddown_out")):
        if k in name:
            return s
    return None


def main(path, out, batch, tree):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    iid, ik, im, iu, iv = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(r[iid], {"name": r[ik]})
        v = float(r[iv].replace(",", ""))
        d[r[im]] = v * UNIT.get(r[iu], 1.0)
    res, nb = {}, 0
    for lid in sorted(launches, key=int):
        d = launches[lid]
        st = stage_of(d["name"], nb)
        if "k_bconv" in d["name"]:
            nb += 1
        if st is None or st in res:
            continue
        res[st] = {"kernel": d["name"].split("(")[0].replace("void ", ""),
                   "bytes_per_launch": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
                   "time_us_ncu": d.get("gpu__time_duration.sum"),
                   "launch": f"batch of {batch} C2 keyswitches", "batch": batch, "tree": tree,
                   "fmaheavy_pipe_pct": d.get(METRICS[3]), "issue_active_pct": d.get(METRICS[4]),
                   "l1tex_pct": d.get(METRICS[5]), "dram_pct": d.get(METRICS[6])}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    args = sys.argv[1:]
    if args == ["--metrics"]:
        print(",".join(METRICS))
        sys.exit(0)
    opts = {a.split("=")[0]: a.split("=", 1)[1] for a in args if a.startswith("--")}
    pos = [a for a in args if not a.startswith("--")]
    main(pos[0], pos[1], int(opts.get("--batch", 32)), opts.get("--tree"))
