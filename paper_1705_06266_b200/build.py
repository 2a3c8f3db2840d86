"""Build liblap.so (sm_100a) in-tree with nvcc.

setup.cu (hierarchy construction) is compiled with -fmad=false so every
floating operation that feeds a discrete decision is a single IEEE rounding
(it also uses explicit __dmul_rn/__dadd_rn/__ddiv_rn); the solve-phase
kernels may contract to FMA (their parity is by tolerance, SURVEY O-S11).
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "liblap.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include")]
UNITS = {"setup.cu": ["-fmad=false", "-prec-div=true", "-prec-sqrt=true"],
         "solve.cu": [],
         "storage.cu": [],
         "lap_api.cu": [],
         "dist.cu": [],
         "tail.cu": [],
         "ktail.cu": [],
         "block.cu": [],
         "bench_hooks.cu": [],
         "xt.cu": []}


def _sources():
    fs = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    fs.append(os.path.join(ROOT, "include", "lap.h"))
    return fs


def build(force: bool = False, verbose: bool = False) -> str:
    newest = max(os.path.getmtime(f) for f in _sources())
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= newest:
        return SO
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = os.path.join(HERE, "_build")
    os.makedirs(objdir, exist_ok=True)
    headers = [f for f in _sources() if not f.endswith(".cu")]
    hdr_time = max(os.path.getmtime(f) for f in headers)
    jobs, objs = [], []
    for unit, extra in UNITS.items():
        src = os.path.join(CSRC, unit)
        obj = os.path.join(objdir, unit.replace(".cu", ".o"))
        objs.append(obj)
        if force or not os.path.exists(obj) or os.path.getmtime(obj) < max(os.path.getmtime(src), hdr_time):
            jobs.append([nvcc, *ARCH, *COMMON, *extra, "-c", src, "-o", obj])
    # translation units compile independently: in parallel
    from concurrent.futures import ThreadPoolExecutor
    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.check_call(cmd)
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        for f in [ex.submit(run, c) for c in jobs]:
            f.result()
    tmp = SO + f".tmp{os.getpid()}"
    subprocess.check_call([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-lnccl"])
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
