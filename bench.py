#!/usr/bin/env python
"""Benchmark: train examples/sec of the B200 hot path (+ embedding pull/push
HBM GB/s against the measured peak), BASELINE.json configs[1] at N=1 and
configs[2] (the same model, table hash-sharded over N GPUs) for N>1.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

A step is one Trainer::train_batch over one synthetic batch (per rank:
65536 instances x 100 slots, one Zipf(1.1) feature per slot over a 1e8-key
space, AdaGrad sparse rows of dim 64, MLP [6400 -> 256 -> 128 -> 1], k=1).
`value` times the device-resident path (inputs already in HBM); `e2e` times
the same public call with pinned HOST buffers (H2D of the batch and D2H of the
loss inside the timed region). Multi-GPU: one process per GPU (torchrun),
weak scaling (65536 instances per rank), NCCL all-to-all of keys/rows/grads,
device time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train examples/sec at 1/2/4/8 B200; embedding pull/push HBM GB/s vs peak"
UNIT = "examples/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--batch", type=int, default=65536, help="instances per rank per step")
    p.add_argument("--slots", type=int, default=100)
    p.add_argument("--dim", type=int, default=64)
    p.add_argument("--vocab", type=int, default=100_000_000)
    p.add_argument("--zipf", type=float, default=1.1)
    p.add_argument("--hidden", default="256,128")
    p.add_argument("--k", type=int, default=1, help="k-step merge period (configs C4 sweep)")
    p.add_argument("--sparse-rule", default="adagrad", choices=["adagrad", "adam"])
    p.add_argument("--pool", type=int, default=2, help="distinct pre-generated batches")
    p.add_argument("--no-prefill", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--diag-h2d", action="store_true",
                   help="diagnostic only: a 66 MB pinned->device copy on a side stream inside every "
                        "device-resident step (how much the e2e path's staged copy costs the step)")
    p.add_argument("--no-stage-profile", action="store_true",
                   help="(no effect: the timed loop never records the per-stage CUDA events; a "
                        "separate profiled pass of the same length measures the stages)")
    p.add_argument("--cpu-sample", type=int, default=4096, help="instances for the CPU baseline")
    p.add_argument("--ref-slice", type=int, default=1024,
                   help="reference arm: instances per host thread per step")
    p.add_argument("--ref-full-batch", type=int, default=1,
                   help="reference arm: also time one whole folded batch on one core")
    return p.parse_args()


def load_data_module():
    """paper_2201_05500_b200/data.py (numpy only) loaded by path, so the
    reference arm never runs the package __init__ (which maps this repo's
    CUDA libraries into the process)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "_kp_data", os.path.join(ROOT, "paper_2201_05500_b200", "data.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def repo_so_loaded():
    """Shared objects under this repo mapped into the process (the reference
    arm must show only oracle/_ref/*)."""
    out = set()
    try:
        with open("/proc/self/maps") as f:
            for line in f:
                path = line.split()[-1] if line.strip() else ""
                if path.endswith(".so") or ".so." in path:
                    if os.path.realpath(path).startswith(os.path.realpath(ROOT)):
                        out.add(os.path.relpath(os.path.realpath(path), os.path.realpath(ROOT)))
    except OSError:
        pass
    return sorted(out)


def load_json(path):
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


def ncu_traffic():
    """Per-stage DRAM bytes per step (dram__bytes_read.sum + write.sum) from the
    committed ncu launch list summary (tools/ncu_summary.py); {} if absent."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")
    try:
        with open(p) as f:
            return {k: v["dram_bytes"] for k, v in json.load(f)["stages"].items()}
    except (OSError, KeyError, ValueError):
        return {}


def cublas_tf32():
    """cuBLAS tf32 GEMM throughput (8192^3, TF/s): the practical tf32 ceiling
    the 3xTF32 kernels are compared with (calibration only, not the product)."""
    import torch
    try:
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = True
        a = torch.randn(8192, 8192, device="cuda")
        b = torch.randn(8192, 8192, device="cuda")
        for _ in range(2):
            a @ b
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            a @ b
        e1.record()
        torch.cuda.synchronize()
        torch.backends.cuda.matmul.allow_tf32 = prev
        return 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 5 / 1e3) / 1e12
    except Exception:  # calibration is optional
        return None


def peaks():
    m = load_json(os.path.join(ROOT, "MEASURED_PEAKS.json"))
    if m:
        return float(m["hbm_gbs"]), float(m["bf16_tflops"]), float(m.get("bf16_tflops_sustained", m["bf16_tflops"])), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (the profiling recipe's clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        import tempfile
        self.path = tempfile.mktemp(prefix="kp_clocks_", suffix=".csv")
        try:
            # -f: nvidia-smi writes (and flushes) each sample to the file itself
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "100", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            try:
                with open(self.path) as f:
                    self.out = f.read()
                os.unlink(self.path)
            except OSError:
                pass

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class NvLink:
    """NVLink data bytes this GPU transmitted / received (NVML field counters
    NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX/RX, KiB, summed over the links),
    read around the timed region: the measured NVLink traffic of the step."""

    TX, RX = 138, 139

    def __init__(self, device):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.links = [l for l in range(18) if self._state(l)]
        except Exception:
            self.h = None

    def _state(self, l):
        try:
            return self.nv.nvmlDeviceGetNvLinkState(self.h, l) == 1
        except Exception:
            return False

    def read(self):
        if self.h is None or not self.links:
            return None
        try:
            q = [(self.TX, l) for l in self.links] + [(self.RX, l) for l in self.links]
            vals = self.nv.nvmlDeviceGetFieldValues(self.h, q)
            out = [0, 0]
            for i, v in enumerate(vals):
                if v.nvmlReturn != 0:
                    return None
                out[0 if i < len(self.links) else 1] += int(v.value.ullVal) * 1024
            return out
        except Exception:
            return None


# ------------------------------------------------------------- reference arm --
def run_reference(args, rank):
    """The reference's own CPU implementation (oracle/_ref/libkpsim_ref.so, the
    unmodified /root/reference/proj sources) on this host's cores: one
    single-threaded reference Trainer per core, each training a bounded sample
    of the same workload folded to the reference's S=1 model."""
    if rank != 0:
        return
    from oracle import oracle as O
    import tempfile
    make_batch = load_data_module().make_batch
    cores = len(os.sched_getaffinity(0))
    need = cores * args.ref_slice * (args.steps + args.warmup)
    bt = make_batch(min(need, args.batch), V=args.vocab, zipf_s=args.zipf, n_slots=args.slots, seed=1000)
    fb = bt.folded()
    per = min(args.ref_slice, fb.n)  # instances per thread per step
    hidden = tuple(int(h) for h in args.hidden.split(",") if h)
    rcfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=1 << 30, embedding_dim=args.dim,
                        hidden=hidden, alpha=0.01, sparse_lr=0.05)
    refs = [O.Ref(rcfg, tempfile.mkdtemp(prefix="kpref_")) for _ in range(cores)]
    cursor = [0]

    def slice_for(i, step):
        lo = ((step * cores + i) * per) % max(fb.n - per + 1, 1)
        return fb.slice(lo, lo + per)

    def one_step(step):
        ths = []
        for i, r in enumerate(refs):
            s = slice_for(i, step)
            ths.append(threading.Thread(target=r.batch, args=(s.offs, s.keys, s.labels)))
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    for w in range(args.warmup):
        one_step(w)
    t0 = time.perf_counter()
    for k in range(args.steps):
        one_step(args.warmup + k)
    dt = time.perf_counter() - t0
    value = cores * per * args.steps / dt
    ref_model = f"[{args.dim}->{args.hidden.replace(',', '->')}->1]"
    sample = (f"{per} instances x {cores} threads per step, each thread an independent reference "
              f"Trainer (N=1,k=1) on its own slice of the "
              f"{workload_config(args, max(1, args.gpus))['workload'].split(':')[0]} batch "
              f"folded to S=1 (the reference model: one pooled vector per instance, {ref_model})")
    # what this arm ran: the reference cannot express S slots (model.cpp:88-99),
    # so the same batches are folded to its S=1 model
    cfg = workload_config(args, max(1, args.gpus))
    cfg.update({"slots": f"1 (the batch's {args.slots} slot features folded into one deduped feature set "
                         "per instance, the reference's Instance semantics)",
                "mlp": ref_model, "parallelism": f"{cores} host threads, one reference Trainer each"})
    full = None
    if args.ref_full_batch:
        # one core, one whole folded batch (the reference is single-threaded):
        # the stated baseline beside the many-thread sample figure
        n_full = min(args.batch, fb.n)
        rf = O.Ref(rcfg, tempfile.mkdtemp(prefix="kpref_full_"))
        t1 = time.perf_counter()
        rf.batch(fb.offs[:n_full + 1], fb.keys[:fb.offs[n_full]], fb.labels[:n_full])
        d1 = time.perf_counter() - t1
        full = {"value": n_full / d1, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": f"one Trainer::train_batch over {n_full} instances (the folded batch), "
                          f"single-threaded"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic Zipf(1.1) CTR", "config": cfg,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": sample},
        "cpu_baseline_1core_full_batch": full,
        "repo_so_loaded": repo_so_loaded(),
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_index(args, world):
    """Which BASELINE.json configs[i] these arguments reproduce (None: custom)."""
    if (args.vocab, args.dim, args.slots, args.batch) == (1_000_000, 8, 26, 4096):
        return 0
    if args.vocab >= 500_000_000:
        return 4
    if (args.vocab, args.dim, args.slots, args.batch) == (100_000_000, 64, 100, 65536):
        return 3 if args.k > 1 else (1 if world == 1 else 2)
    return None


def workload_config(args, world):
    ci = config_index(args, world)
    small = args.vocab * args.dim * 8 < 126e6
    return {
        "workload": f"{f'configs[{ci}]' if ci is not None else 'custom'}: {args.vocab // 1_000_000}M-key table, emb dim "
                    f"{args.dim}, {args.slots} slots, batch {args.batch}/GPU, Zipf({args.zipf}) keys, "
                    f"{'AdaGrad' if args.sparse_rule == 'adagrad' else 'sparse Adam'} rows, k={args.k}",
        "global_batch": args.batch * world,
        "slots": args.slots,
        "embedding_dim": args.dim,
        "table_keys": args.vocab,
        "mlp": f"[{args.slots * args.dim}->{args.hidden.replace(',', '->')}->1]",
        "parallelism": f"table sharded key%{world}, dp{world}" if world > 1 else "single GPU",
        "l2": ("table fits the 126 MB L2 (small config, no flush; not the headline)" if small else
               "per-step working set ~5 GB >> 126 MB L2 (no flush needed)"),
        "prefill": "table pre-populated with all keys (steady state)" if not args.no_prefill else "cold",
    }


# ---------------------------------------------------------------- B200 arm --
def cpu_baseline(args, bt):
    from oracle import oracle as O
    import tempfile
    n = min(args.cpu_sample, bt.n)
    fb = bt.slice(0, n).folded()
    hidden = tuple(int(h) for h in args.hidden.split(",") if h)
    cfg = O.TrainerCfg(n_workers=1, k=1, minibatch_size=1 << 30, embedding_dim=args.dim,
                       hidden=hidden, alpha=0.01, sparse_lr=0.05)
    kind = "reference" if O.ref_available() else "port"
    r = O.Ref(cfg, tempfile.mkdtemp(prefix="kpref_")) if kind == "reference" else O.Orc(cfg, 64)
    t0 = time.perf_counter()
    r.batch(fb.offs, fb.keys, fb.labels)
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{n} instances of the step-0 batch folded to S=1 (reference semantics, model "
                      f"[{args.dim}->{args.hidden.replace(',', '->')}->1]), one Trainer::train_batch, "
                      f"single-threaded like the reference"}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank)
        return
    import torch
    import torch.distributed as dist
    import paper_2201_05500_b200 as kp
    from paper_2201_05500_b200.data import make_batch

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    comm = None
    if world > 1:
        obj = [kp.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = kp.Comm(obj[0], rank, world, local)

    hidden = [int(h) for h in args.hidden.split(",") if h]
    per_rank_keys = (args.vocab - rank + world - 1) // world
    capacity = per_rank_keys + 1_000_000
    tr = kp.Trainer(comm=comm, table_capacity=capacity, device=local, n_workers=world,
                    minibatch_size=args.batch, embedding_dim=args.dim, n_slots=args.slots,
                    hidden=hidden, k=args.k, alpha=0.01, sparse_lr=0.05, seed=42,
                    sparse_rule=args.sparse_rule)
    if not args.no_prefill:
        tr.prefill(rank, world, per_rank_keys)

    batches = [make_batch(args.batch, V=args.vocab, zipf_s=args.zipf, n_slots=args.slots,
                          seed=1000 + 97 * rank + b) for b in range(args.pool)]
    gfirst = rank * args.batch
    gn = args.batch * world
    # device-resident copies (value) and pinned host copies (e2e)
    dev, pin = [], []
    for bt in batches:
        d = {"offs": torch.from_numpy(bt.offs.view(np.int32)).cuda(),
             "keys": torch.from_numpy(bt.keys.view(np.int64)).cuda(),
             "slots": torch.from_numpy(bt.slots.view(np.int16)).cuda(),
             "labels": torch.from_numpy(bt.labels).cuda()}
        dev.append(d)
        p = {k: torch.from_numpy(v).pin_memory() for k, v in
             (("offs", bt.offs.view(np.int32)), ("keys", bt.keys.view(np.int64)),
              ("slots", bt.slots.view(np.int16)), ("labels", bt.labels))}
        pin.append({"offs": p["offs"].numpy().view(np.uint32), "keys": p["keys"].numpy().view(np.uint64),
                    "slots": p["slots"].numpy().view(np.uint16), "labels": p["labels"].numpy(),
                    "_t": p})
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(tr.stream())

    diag = None
    if args.diag_h2d:
        nb = sum(v.nbytes for k, v in pin[0].items() if k != "_t")
        diag = (torch.empty(nb, dtype=torch.uint8).pin_memory(), torch.empty(nb, dtype=torch.uint8, device=f"cuda:{local}"),
                torch.cuda.Stream(device=f"cuda:{local}"))

    def step_dev(i):
        if diag is not None:
            with torch.cuda.stream(diag[2]):
                diag[1].copy_(diag[0], non_blocking=True)
        bt, d = batches[i % len(batches)], dev[i % len(dev)]
        return tr.train_batch_device(bt.offs, d["offs"].data_ptr(), d["keys"].data_ptr(),
                                     d["slots"].data_ptr(), d["labels"].data_ptr(), bt.n,
                                     global_n=gn, global_first=gfirst)

    def stage_host(i):
        p = pin[i % len(pin)]
        tr.stage_batch(i % 2, p["offs"], p["keys"], p["labels"], slots=p["slots"])

    def step_staged(i):
        # stage batch i+1 (async H2D on the copy stream) while batch i trains
        stage_host(i + 1)
        return tr.train_staged(i % 2, global_n=gn, global_first=gfirst, n_local=args.batch)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- device-resident path -------------------------------------------
    for i in range(args.warmup):
        step_dev(i)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nvl = NvLink(local) if world > 1 else None
    with Clocks(local) as clk:
        # the barrier comes after the clock sampler started on every rank, so
        # all ranks enter the timed region together (stage profiling off: its
        # event records are host work inside the step; the per-stage times
        # come from a separate profiled pass below)
        tr.profile(False)
        l0 = kp.launch_count()
        nv0 = nvl.read() if nvl else None
        barrier()
        ev0.record(stream)
        w0 = time.perf_counter()
        for i in range(args.steps):
            r = step_dev(args.warmup + i)
        ev1.record(stream)
        barrier()
        wall = time.perf_counter() - w0
    nv1 = nvl.read() if nvl else None
    launches = kp.launch_count() - l0
    dev_ms = ev0.elapsed_time(ev1)
    dev_ms = max_over_ranks(dev_ms)
    value = args.batch * world * args.steps / (dev_ms / 1e3)
    loss = r["loss"]
    # per-stage CUDA-event times (and the unique/occurrence counters) over
    # the same number of further steps, profiled
    tr.profile(True)
    for i in range(args.steps):
        step_dev(args.warmup + args.steps + i)
    barrier()
    prof = tr.profile(False)

    # ---- end-to-end through the public API with host buffers ------------
    e2e = None
    if not args.no_e2e:
        stage_host(0)
        step_staged(0)  # warm the staging buffers (and each slot's step graph)
        step_staged(1)
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(2, args.steps + 2):
            step_staged(i)
        e1.record(stream)
        barrier()
        e_ms = max_over_ranks(e0.elapsed_time(e1))
        bt = batches[0]
        h2d = bt.offs.nbytes + bt.keys.nbytes + bt.slots.nbytes + bt.labels.nbytes
        e2e = {"value": args.batch * world * args.steps / (e_ms / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8 + 8 + 16,
               "ms_per_step": e_ms / args.steps}

    # ---- roofline (per-stage CUDA events on the trainer's stream) --------
    hbm, bf16, bf16s, pk = peaks()
    K = max(prof["steps"], 1)
    U = prof["unique"] / K
    O_ = prof["occurrences"] / K
    e, B, S = args.dim, args.batch, args.slots
    R = 2 if args.sparse_rule == "adagrad" else 3  # AdaGrad {w, acc} | Adam {w, m, v}
    D_in = S * e
    flops = 6.0 * B * (D_in * hidden[0] + sum(a * b for a, b in zip(hidden, hidden[1:] + [1])))
    stage_bytes = {
        "dedup": 8 * O_ + 8 * U + 4 * O_,                  # keys in, unique out, inverse out
        "pull": 16 * U,                                     # one slot read per unique key
        "pool": 4 * e * U + 4 * O_ + 4 * e * B * S,         # rows, inverse, pooled out
        "push": 4 * e * B * S + 8 * O_ + 2 * R * 4 * e * U, # dpooled in, order, state r/w (fused)
    }
    stages = {}
    for name, ms in ((k, prof[k]) for k in ("dedup", "pull", "pool", "mlp", "push", "dense", "exchange")):
        per = ms / K
        ent = {"ms_per_step": per}
        if name in stage_bytes and per > 0:
            gbs = stage_bytes[name] / (per / 1e3) / 1e9
            ent.update({"bytes": stage_bytes[name], "achieved_gbs": gbs, "frac": gbs / hbm})
        if name == "mlp" and per > 0:
            tf = flops / (per / 1e3) / 1e12
            ent.update({"flops": flops, "achieved_tflops": tf, "frac_bf16_sustained": tf / bf16s})
        stages[name] = ent
    dom = max(stages, key=lambda k: stages[k]["ms_per_step"])
    traffic = ncu_traffic()
    if dom == "mlp":
        # achieved = the model's ALGORITHMIC fp32 flops (6 B sum in*out) over
        # the stage time, against the bf16 tensor peak. The fp32-accurate
        # emulation issues 3 MMAs per fp32 multiply-add (3xFP16 on the first
        # layer's forward and input-gradient GEMMs, 3xTF32 elsewhere, a tf32
        # MMA at half the bf16 rate); that pipe work is reported beside it.
        h_on = os.environ.get("KP_GEMM_F16", "1") != "0" and D_in % 8 == 0
        f_l1 = 2.0 * B * D_in * hidden[0]                       # one first-layer GEMM
        # layer 1's forward, input gradient and weight gradient all run 3xFP16
        # (pre-split planes) unless the fp16 path is off
        f16_flops = (3 if os.environ.get("KP_GEMM_H3", "1") != "0" else 2) * f_l1 if h_on else 0.0
        tf32_flops = flops - f16_flops
        work = 3.0 * f16_flops + 2 * 3.0 * tf32_flops            # bf16-equivalent MMA flops
        sec = stages["mlp"]["ms_per_step"] / 1e3
        alg = flops / sec / 1e12
        roof = {"kernel": "mlp stage: tcgen05 GEMMs (3xFP16 on pre-split fp16 planes for the 6400-wide "
                          "first layer's forward, dX and dW; 3xTF32 on layer 2) + head/bias kernels",
                "bound": "tensor", "achieved": alg, "peak": bf16s, "unit": "TFLOP/s",
                "frac": alg / bf16s, "traffic": traffic.get("mlp"),
                "peak_kind": f"{pk} bf16 dense sustained",
                "achieved_kind": "algorithmic fp32 model flops (6 B sum in*out) / stage time",
                "mma_work_tflops": work / sec / 1e12,
                "mma_work_frac": work / sec / 1e12 / bf16s,
                "mma_work_kind": "bf16-rate-equivalent MMA work / stage time: 3 f16 MMAs per fp32 "
                                 "FMA on the fp16 GEMMs, 3 tf32 MMAs = 6 bf16-equivalent otherwise",
                "mma_work_tflop_per_step": work / 1e12,
                "cublas_tf32_tflops_8192": cublas_tf32()}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": stages[dom].get("achieved_gbs"),
                "peak": hbm, "unit": "GB/s", "frac": stages[dom].get("frac"),
                "traffic": traffic.get(dom), "peak_kind": f"{pk} copy"}
    for k in stages:
        if k in traffic:
            stages[k]["ncu_dram_bytes"] = traffic[k]
    emb = {k: stages[k] for k in ("pool", "push") if "achieved_gbs" in stages[k]}
    for v in emb.values():  # fraction of the nominal ~8 TB/s too
        v["frac_nominal_8tbs"] = v["achieved_gbs"] / 8000.0
    nvlink = None
    if world > 1:
        # per GPU per step: keys to owners, rows back, gradients to owners, for
        # the (G-1)/G of the exchanged entries that cross NVLink (counts from
        # the run); floor = those bytes at 900 GB/s per direction
        recv = prof.get("received", 0) / K
        remote = recv * (world - 1) / world
        b = remote * (8 + 4 * e + 4 * e)
        nvlink = {"bytes_per_gpu_per_step": b, "floor_ms_at_900_GBs": b / 900e9 * 1e3,
                  "exchange_stage_ms": stages["exchange"]["ms_per_step"],
                  "note": "rows and gradients move inside the pull/push kernels and the "
                          "copy engines, overlapped; the stages above include them"}
        if nv0 and nv1:
            # measured by the NVLink hardware counters over the timed region
            # (this rank; max over ranks of the step time as the denominator)
            sec = dev_ms / 1e3
            tx, rx = (nv1[0] - nv0[0]) / args.steps, (nv1[1] - nv0[1]) / args.steps
            nvlink["measured"] = {
                "tx_bytes_per_step": tx, "rx_bytes_per_step": rx,
                "tx_gbs": tx * args.steps / sec / 1e9, "rx_gbs": rx * args.steps / sec / 1e9,
                "frac_of_900_gbs_per_direction": max(tx, rx) * args.steps / sec / 900e9,
                "source": "NVML NVLINK_THROUGHPUT_DATA_TX/RX counters, rank 0"}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline(args, batches[0])
            except Exception as ex:  # the baseline is reported, never required
                cpu = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                       "sample": f"unavailable: {ex}"}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic Zipf CTR batches (random-init dense weights)",
            "config": workload_config(args, world),
            "e2e": e2e, "gpu_launches": int(launches), "roofline": roof, "stages": stages,
            "embedding_pull_push": emb, "nvlink": nvlink, "cpu_baseline": cpu, "clocks": clk.summary(),
            "loss": loss, "unique_keys_per_step": U, "occurrences_per_step": O_,
            "wall_ms_per_step": wall / args.steps * 1e3,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
