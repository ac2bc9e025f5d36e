"""Build libpda.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2504_06319_b200.build [--force] [--verbose]

Each .cu under csrc/ is compiled to an object with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`` (SASS only, no PTX
JIT on the box) and linked with the static CUDA runtime into
``paper_2504_06319_b200/libpda.so`` next to this file.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpda.so")

SOURCES = ["pda.cu", "decode_splitk.cu", "decode_stream.cu", "decode_balanced.cu", "decode_paper.cu", "roofline.cu",
           "kv_cache.cu", "decode_tc.cu", "decode_splitk_m0.cu", "decode_splitk_m1.cu", "decode_splitk_m2.cu"]
HEADERS = ["ptx.cuh", "kernels.cuh", "block_math.cuh", "kv_append.cuh", "splitk_impl.cuh", "tc_ptx.cuh",
           "balanced_range.cuh"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
              "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I", INCLUDE]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA extension cannot be built")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out_dir: str | None = None) -> str:
    """Compile and link; `defines` (-DNAME=V) and `out_dir` (objects + libpda.so
    elsewhere) exist for A/B builds of compile-time variants only."""
    BUILD = os.path.join(out_dir, "_build") if out_dir else globals()["BUILD"]
    LIB = os.path.join(out_dir, "libpda.so") if out_dir else globals()["LIB"]
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "pda.h")]
    jobs = []
    objs = []
    for src in SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs):
            jobs.append((path, obj))

    def compile_one(job):
        path, obj = job
        cmd = [nvcc()] + ARCH + NVCC_FLAGS + list(defines) + ["-c", path, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {path}:\n{r.stderr}")
        log = os.path.join(BUILD, os.path.basename(obj) + ".ptxas.txt")
        with open(log, "w") as f:
            f.write(r.stderr)
        return path, r.stderr

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            for path, err in ex.map(compile_one, jobs):
                if verbose:
                    print(f"[build] {os.path.basename(path)}\n{err}", file=sys.stderr)
    if force or jobs or _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--define", action="append", default=[], help="-DNAME=V for an A/B variant build")
    ap.add_argument("--out", default=None, help="output directory of an A/B variant build")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, defines=[f"-D{d}" for d in a.define], out_dir=a.out))
