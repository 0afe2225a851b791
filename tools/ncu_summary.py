"""Summarise an ncu launch list (gpu__time_duration.sum CSV) of bench.py into
per-kernel totals for the LAST training step (prefill launches excluded).

    python tools/ncu_summary.py gpurun_out/launches.csv > profiles/..._launches.md
"""
import csv
import re
import sys


def main(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = [x for x in csv.DictReader(lines) if x.get("Metric Name") == "gpu__time_duration.sum"]
    seq = [(re.sub(r"\(.*", "", x["Kernel Name"]).replace("void ", ""), float(x["Metric Value"]),
            x.get("Grid Size", ""), x.get("Metric Unit", "")) for x in rows]
    starts = [i for i, s in enumerate(seq) if "minmax_init" in s[0]]
    step = seq[starts[-1]:] if starts else seq
    unit = step[0][3] if step else "ns"
    scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3}.get(unit, 1e-3)
    tot = sum(s[1] for s in step) * scale
    print(f"# ncu launch list, last training step ({len(step)} launches, {tot:.1f} us serialized, "
          f"cold-cache: compare shares, not absolutes)\n")
    print("| # | kernel | grid | us | share |")
    print("|---|---|---|---|---|")
    for i, (name, v, grid, _) in enumerate(step):
        us = v * scale
        print(f"| {i} | `{name[-60:]}` | {grid} | {us:.1f} | {100 * us / tot:.1f}% |")
    agg = {}
    for name, v, _, _ in step:
        key = re.sub(r"<.*", "", name.split("::")[-1])
        agg[key] = agg.get(key, 0.0) + v * scale
    print("\n## per kernel\n")
    print("| kernel | us | share |")
    print("|---|---|---|")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"| `{k}` | {v:.1f} | {100 * v / tot:.1f}% |")


if __name__ == "__main__":
    main(sys.argv[1])
