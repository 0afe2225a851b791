"""Summarise an ncu launch list of bench.py into the LAST training step.

The launch list is taken with
    ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,\
dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv ...
(any subset works; missing metrics print as '-').

    python tools/ncu_summary.py gpurun_out/launches.csv profiles/r01_launches.md \
        [profiles/r01_traffic.json]

Writes a markdown table (per launch, per kernel, per bench stage) and, when a
third path is given, the per-stage DRAM traffic per step that bench.py puts in
`roofline.traffic`.
"""
import csv
import json
import re
import sys

# kernel -> bench.py stage (kp_capi.cu profile marks)
STAGE = [
    (r"k_prepare_bags|k_minmax|k_upsweep|k_scan_rows|k_downsweep|k_head_count|k_dedup_emit"
     r"|k_key_range|k_owner|k_plan_check", "dedup"),
    (r"k_probe|k_insert|k_gather_rows", "pull"),
    (r"k_compose|k_pool|k_unique_maxabs|k_inst_exp", "pool"),
    (r"k_split|k_tc_gemm|k_gemm|k_h3|k_colmax|k_head_|k_loss|k_colsum|k_reduce_splits|k_reduce_chunks"
     r"|k_transpose|k_rowmax|k_sum_parts", "mlp"),
    (r"k_seg_|k_chunk_first", "push"),
    (r"k_moments|k_cmean|k_terms|k_check|k_local_step|k_merge|k_dense_step", "dense"),
]


def stage_of(k):
    for pat, st in STAGE:
        if re.search(pat, k):
            return st
    return "other"


def load(path):
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    launches = {}
    order = []
    for x in csv.DictReader(lines):
        i = int(x["ID"])
        if i not in launches:
            name = re.sub(r"\(.*", "", x["Kernel Name"]).replace("void ", "")
            launches[i] = {"name": name.split("::")[-1], "grid": x.get("Grid Size", ""),
                           "block": x.get("Block Size", "")}
            order.append(i)
        v = float(x["Metric Value"].replace(",", "") or 0)
        unit = x.get("Metric Unit", "")
        m = x["Metric Name"]
        if m == "gpu__time_duration.sum":
            v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                  "msecond": 1e3}.get(unit, 1e-3)
            launches[i]["us"] = v
        elif m.startswith("dram__bytes"):
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            launches[i]["dram"] = launches[i].get("dram", 0.0) + v
        elif m.startswith("sm__pipe_tensor"):
            launches[i]["tensor"] = v
    return [launches[i] for i in order]


def main(src, out_md, out_json=None):
    seq = load(src)
    starts = [i for i, s in enumerate(seq) if s["name"].startswith("k_prepare_bags")]
    step = seq[starts[-1]:] if starts else seq
    # only this library's kernels (bench.py's cuBLAS calibration runs after the step)
    step = [x for x in step if x["name"].startswith("k_")]
    tot = sum(s.get("us", 0.0) for s in step)
    L = [f"# ncu launch list: last training step of `{src.split('/')[-1]}`", "",
         f"{len(step)} launches, {tot:.1f} us serialised. ncu replays each kernel alone with a",
         "cold L2 and no overlap: compare SHARES with bench.py's stage times, not absolutes.", "",
         "| # | kernel | stage | grid | us | share | tensor % | DRAM MB |",
         "|---|---|---|---|---|---|---|---|"]
    for i, s in enumerate(step):
        us = s.get("us", 0.0)
        t = f"{s['tensor']:.1f}" if "tensor" in s else "-"
        d = f"{s['dram'] / 1e6:.1f}" if "dram" in s else "-"
        L.append(f"| {i} | `{s['name'][:48]}` | {stage_of(s['name'])} | {s['grid']} | {us:.1f} | "
                 f"{100 * us / tot:.1f}% | {t} | {d} |")
    agg, stg = {}, {}
    for s in step:
        k = re.sub(r"<.*", "", s["name"])
        a = agg.setdefault(k, [0.0, 0.0, 0])
        a[0] += s.get("us", 0.0)
        a[1] += s.get("dram", 0.0)
        a[2] += 1
        b = stg.setdefault(stage_of(s["name"]), [0.0, 0.0, 0])
        b[0] += s.get("us", 0.0)
        b[1] += s.get("dram", 0.0)
        b[2] += 1
    L += ["", "## per kernel", "", "| kernel | launches | us | share | DRAM MB | DRAM GB/s |",
          "|---|---|---|---|---|---|"]
    for k, (us, d, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        L.append(f"| `{k}` | {n} | {us:.1f} | {100 * us / tot:.1f}% | {d / 1e6:.1f} | "
                 f"{d / (us * 1e3) if us else 0:.0f} |")
    L += ["", "## per bench stage", "", "| stage | launches | us | share | DRAM MB |",
          "|---|---|---|---|---|"]
    for k, (us, d, n) in sorted(stg.items(), key=lambda kv: -kv[1][0]):
        L.append(f"| {k} | {n} | {us:.1f} | {100 * us / tot:.1f}% | {d / 1e6:.1f} |")
    with open(out_md, "w") as f:
        f.write("\n".join(L) + "\n")
    if out_json:
        with open(out_json, "w") as f:
            json.dump({"source": src.split("/")[-1],
                       "note": "ncu dram__bytes_read.sum+dram__bytes_write.sum per stage, "
                               "one training step",
                       "stages": {k: {"dram_bytes": v[1], "us_serialised": round(v[0], 1),
                                      "launches": v[2]} for k, v in stg.items()}},
                      f, indent=1)


if __name__ == "__main__":
    main(*sys.argv[1:])
