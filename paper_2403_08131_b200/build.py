"""Build libgpbo.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
from __future__ import annotations

import concurrent.futures as cf
import glob
import importlib.util
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libgpbo.so")
BUILD = os.path.join(ROOT, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec is not None and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        if os.path.exists(os.path.join(base, "include", "nccl.h")):
            return os.path.join(base, "include"), os.path.join(base, "lib")
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("command failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def build(verbose=False, force=False, defines=(), out=None):
    """defines/out: A/B experiment builds (extra -D flags, separate object dir and library)."""
    inc, lib = _nccl_dirs()
    OUT_ = out or OUT
    BUILD_ = BUILD if not defines else os.path.join(BUILD, "v_" + "_".join(defines))
    os.makedirs(BUILD_, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    hdr_t = max(os.path.getmtime(h) for h in headers)
    common = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
                     "-Xptxas", "-v", "-I", inc, "-I", os.path.join(ROOT, "include")]
    if os.environ.get("GPBO_FIT_TIMING"):  # fit phase clocks (printf from CTA 0)
        common += ["-DGPBO_FIT_TIMING"]
        force = True
    if os.environ.get("GPBO_TC_TRACE"):  # clock64 pipeline trace hooks (tools/trace_tc.py)
        common += ["-DGPBO_TC_TRACE"]
        force = True
    common += ["-D" + d for d in defines]
    jobs = []
    for s in srcs:
        o = os.path.join(BUILD_, os.path.basename(s) + ".o")
        if force or not os.path.exists(o) or os.path.getmtime(o) < max(os.path.getmtime(s), hdr_t):
            jobs.append(([NVCC] + common + ["-c", s, "-o", o], s))
    logs = []
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        for (cmd, s), log in zip(jobs, ex.map(lambda j: _run(j[0]), jobs)):
            logs.append((s, log))
    objs = [os.path.join(BUILD_, os.path.basename(s) + ".o") for s in srcs]
    if jobs or not os.path.exists(OUT_):
        _run([NVCC] + ARCH + ["-shared", "-o", OUT_] + objs +
             ["-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib, "-lcudart"])
    with open(os.path.join(BUILD, "ptxas.log"), "a") as f:
        for s, log in logs:
            f.write(f"==== {s}\n{log}\n")
    if verbose:
        for s, log in logs:
            print(f"==== {os.path.basename(s)}\n{log}")
    return OUT_


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv)
    print(OUT)
