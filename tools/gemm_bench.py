"""Time the tcgen05 GEMM on the MLP's layer-1 shapes through the C ABI.

    python tools/gemm_bench.py            (KP_GEMM_CG=1|2 to force the CTA mode)
"""
import ctypes
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2201_05500_b200 as kp  # noqa: E402

lib = ctypes.CDLL(os.path.join(os.path.dirname(kp.__file__), "libkpsim_b200.so"))
P, I = ctypes.c_void_p, ctypes.c_int
for f in (lib.kp_gemm_nt, lib.kp_gemm_tn):
    f.argtypes = [P, I, P, I, P, I, I, I, I, I, P]
    f.restype = I

B, D, H = 65536, 6400, 256
dev = torch.device("cuda:0")
g = torch.Generator(device=dev).manual_seed(0)
pooled = torch.randn(B, D, device=dev, generator=g)
W = torch.randn(H, D, device=dev, generator=g)
Wt = W.t().contiguous()
dZ = torch.randn(B, H, device=dev, generator=g)
out = torch.empty(B * D, device=dev)


def run(name, fn, flops, reps=10):
    for _ in range(2):
        assert fn() == 0
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t) / reps * 1e3
    print(f"{name:>8}: {ms:.3f} ms  {flops / ms / 1e9:.1f} fp32-TFLOP/s  "
          f"({3 * flops / ms / 1e9:.0f} TF/s of tf32 MMA)")


p = lambda t: ctypes.c_void_p(t.data_ptr())
run("fwd", lambda: lib.kp_gemm_nt(p(pooled), D, p(W), D, p(out), H, B, H, D, 2, None), 2 * B * H * D)
run("dX", lambda: lib.kp_gemm_nt(p(dZ), H, p(Wt), H, p(out), D, B, D, H, 2, None), 2 * B * H * D)
run("dW", lambda: lib.kp_gemm_tn(p(dZ), H, p(pooled), D, p(out), D, H, D, B, 2, None), 2 * B * H * D)
