"""In-tree build of the CUDA library and the Python extension.

  libkpsim_b200.so        csrc/*.cu  (nvcc, -gencode arch=compute_100a,code=sm_100a)
                          the C ABI of include/kpsim_b200.h; links NCCL
  _kpsim_b200*.so         host/*.cpp (g++, pybind11) -- the C++ shim with the
                          reference's API names, calling only the C ABI

Both land next to this file so they travel with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
INCLUDE = os.path.join(ROOT, "include")
OBJ = os.path.join(PKG, "build", "obj")
LIB = os.path.join(PKG, "libkpsim_b200.so")
EXT = os.path.join(PKG, "_kpsim_b200" + sysconfig.get_config_var("EXT_SUFFIX"))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE,
           "--expt-relaxed-constexpr", "-Xptxas", "-v"] + ARCH
# NCCL: the copy torch ships (nvidia/nccl, 2.28), so the library and torch share
# one libnccl.so.2 in a process (the system 2.27 lacks symbols torch needs).
def _nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (list(spec.submodule_search_locations) if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "lib", "libnccl.so.2")):
            return d
    return None


NCCL_DIR = _nccl_dir()
CUDA_SRCS = ["kp_sort", "kp_table", "kp_embed", "kp_mlp", "kp_gemm_tc", "kp_gemm_h3", "kp_dense", "kp_auc", "kp_peer",
             "kp_capi"]
HOST_SRCS = ["kpsim_b200", "module"]


def _newer(out: str, deps) -> bool:
    if not os.path.exists(out):
        return False
    t = os.path.getmtime(out)
    return all(os.path.getmtime(d) <= t for d in deps)


def _run(cmd, log=None):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if log:
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def _headers(d):
    return [os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cuh", ".hpp", ".h"))]


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    hdrs = _headers(CSRC) + [os.path.join(INCLUDE, "kpsim_b200.h")]

    def cu(name):
        src = os.path.join(CSRC, name + ".cu")
        out = os.path.join(OBJ, name + ".o")
        if not _newer(out, [src] + hdrs):
            inc = ["-I" + os.path.join(NCCL_DIR, "include")] if NCCL_DIR else []
            _run([NVCC] + NVFLAGS + inc + ["-c", src, "-o", out], os.path.join(OBJ, name + ".ptxas.log"))
        return out

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(cu, CUDA_SRCS))
    if not _newer(LIB, objs):
        nccl = (["-L" + os.path.join(NCCL_DIR, "lib"), "-l:libnccl.so.2", "-Xlinker",
                 "-rpath=" + os.path.join(NCCL_DIR, "lib")] if NCCL_DIR else ["-lnccl"])
        _run([NVCC] + ARCH + ["-shared", "-o", LIB] + objs + nccl +
             ["-Xlinker", "-soname=libkpsim_b200.so"])

    import pybind11
    py_inc = sysconfig.get_paths()["include"]
    hsrcs = [os.path.join(HOST, n + ".cpp") for n in HOST_SRCS]
    if not _newer(EXT, hsrcs + _headers(HOST) + [LIB, os.path.join(INCLUDE, "kpsim_b200.h")]):
        _run(["g++", "-O2", "-std=c++20", "-shared", "-fPIC", "-fvisibility=hidden",
              "-I" + INCLUDE, "-I" + HOST, "-I" + pybind11.get_include(), "-I" + py_inc] + hsrcs +
             ["-o", EXT, "-L" + PKG, "-lkpsim_b200", "-Wl,-rpath,$ORIGIN"])
    if verbose:
        print("built", LIB, EXT)
    return EXT


if __name__ == "__main__":
    build(verbose=True)
    sys.exit(0)
