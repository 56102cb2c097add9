"""Summarise an ncu report (raw page) into a compact markdown table for profiles/."""
import csv
import subprocess
import sys

METRICS = [
    ("time_us", "gpu__time_duration.sum", 1),
    ("dram_read_MB", "dram__bytes_read.sum", None),
    ("dram_write_MB", "dram__bytes_write.sum", None),
    ("warps_active/SM", "sm__warps_active.avg.per_cycle_active", 1),
    ("regs", "launch__registers_per_thread", 1),
    ("issue_active_%", "smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    ("fma_pipe_%", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("fmaheavy_pipe_%", "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("l1tex_%", "l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    ("smem_bank_confl", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1),
    ("alu_pipe_%", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("dram_%", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("warp_inst", "smsp__inst_executed.sum", 1),
]


def to_mb(val, unit):
    f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(unit, 1.0)
    return float(val) * f


def main(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    hdr = ["kernel"] + [m[0] for m in METRICS]
    stalls = []
    print("| " + " | ".join(hdr) + " |")
    print("|" + "---|" * len(hdr))
    for r in rows[2:]:
        cells = [r[h.index("Kernel Name")].split("(")[0].replace("void ", "")]
        for name, key, scale in METRICS:
            if key not in h:
                cells.append("-")
                continue
            i = h.index(key)
            v = r[i]
            try:
                if scale is None:
                    cells.append(f"{to_mb(v.replace(',', ''), units[i]):.1f}")
                else:
                    x = float(v.replace(",", ""))
                    if key.startswith("gpu__time"):
                        x *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(units[i], 1.0)
                    cells.append(f"{x:.1f}" if x < 1e6 else f"{x:.3g}")
            except ValueError:
                cells.append(v)
        print("| " + " | ".join(cells) + " |")
        st = sorted(((float(r[i]), w.replace("smsp__pcsamp_warps_issue_stalled_", ""))
                     for i, w in enumerate(h)
                     if w.startswith("smsp__pcsamp_warps_issue_stalled_") and not w.endswith("not_issued")
                     and r[i].replace(".", "").isdigit()), reverse=True)[:5]
        stalls.append((cells[0], st))
    print("\nTop stall reasons (pc samples):\n")
    for k, st in stalls:
        print(f"- {k}: " + ", ".join(f"{n} {int(v)}" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
