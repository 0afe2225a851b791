"""Key counters of ncu --set full captures (one or more .ncu-rep) as markdown.

    python tools/ncu_full_summary.py out.md gpurun_out/full_*.ncu-rep
"""
import csv
import re
import subprocess
import sys

NCU = "/usr/local/cuda/bin/ncu"
COLS = [
    ("us", "gpu__time_duration.sum", 1e3),
    ("DRAM rd MB", "dram__bytes_read.sum", 1e-6),
    ("DRAM wr MB", "dram__bytes_write.sum", 1e-6),
    ("DRAM %", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L2 %", "lts__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("L1 %", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("tensor %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 1),
    ("SM %", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    ("regs", "launch__registers_per_thread", 1),
]
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1, "msecond": 1,
        "us": 1e-3, "usecond": 1e-3, "ns": 1e-6, "nsecond": 1e-6}


def rows(rep):
    out = subprocess.run([NCU, "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return r[0], r[1], r[2:]


def main(out_md, *reps):
    L = ["# ncu --set full: key counters per launch", "",
         "Captured with `ncu --set full --import-source on --clock-control none` (tools/profile_round.sh),",
         "one process, cache flushed between replays: absolute times are cold-cache; compare ratios.", "",
         "| kernel | grid | " + " | ".join(c[0] for c in COLS) + " | top stalls (warps/issue) |",
         "|---|---|" + "---|" * len(COLS) + "---|"]
    for rep in reps:
        h, u, data = rows(rep)
        for d in data:
            name = re.sub(r"\(.*", "", d[h.index("Kernel Name")]).replace("void ", "").split("::")[-1]
            vals = []
            for _, m, sc in COLS:
                if m not in h:
                    vals.append("-")
                    continue
                i = h.index(m)
                try:
                    v = float(d[i].replace(",", ""))
                except ValueError:
                    vals.append(d[i])
                    continue
                if m == "gpu__time_duration.sum":
                    v = v * UNIT.get(u[i], 1) * 1e3
                elif m.startswith("dram__bytes"):
                    v = v * UNIT.get(u[i], 1) * 1e-6
                vals.append(f"{v:.1f}" if isinstance(v, float) else str(v))
            st = []
            for i, m in enumerate(h):
                mm = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", m)
                if mm:
                    try:
                        st.append((float(d[i]), mm.group(1)))
                    except ValueError:
                        pass
            top = ", ".join(f"{n} {v:.1f}" for v, n in sorted(st, reverse=True)[:3])
            grid = d[h.index("launch__grid_size")] if "launch__grid_size" in h else "-"
            L.append(f"| `{name[:40]}` | {grid} | " + " | ".join(vals) + f" | {top} |")
    with open(out_md, "w") as f:
        f.write("\n".join(L) + "\n")


if __name__ == "__main__":
    main(*sys.argv[1:])
