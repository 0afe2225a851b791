"""H2D bandwidth of a 66 MB pinned buffer (the configs[1] staged batch), with
the process on its default CPUs and then pinned to the GPU's NUMA-local CPUs
(NVML's CPU affinity), the buffer allocated after the move."""
import os
import sys

import torch


def bw(tag):
    n = 66 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for _ in range(3):
            d.copy_(h, non_blocking=True)
        e0.record(s)
        for _ in range(10):
            d.copy_(h, non_blocking=True)
        e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{tag}: {ms:.3f} ms per 66 MB copy = {n / ms / 1e6:.1f} GB/s; cpus {len(os.sched_getaffinity(0))}")


torch.cuda.init()
bw("default affinity")
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
    cpus = {w * 64 + b for w, m in enumerate(words) for b in range(64) if (m >> b) & 1}
    print("gpu-local cpus:", len(cpus), "of", os.cpu_count())
    os.sched_setaffinity(0, cpus)
    bw("gpu-local affinity")
except Exception as ex:  # noqa: BLE001
    print("affinity probe failed:", ex, file=sys.stderr)
