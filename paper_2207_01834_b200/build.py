"""Builds the in-tree C-ABI library paper_2207_01834_b200/_lib/libgkbdl.so.

nvcc -gencode arch=compute_100a,code=sm_100a (B200 only) for the CUDA sources,
the system g++ (OpenMP, -ffp-contract=off) for the host generators; no torch
types cross the boundary, so no torch extension machinery is involved.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libgkbdl.so")
CLI = os.path.join(OUT_DIR, "gk_bdl_cli")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

CU_SOURCES = ["gk_build.cu", "gk_knn.cu", "gk_bdl.cu"]
CPP_SOURCES = ["gk_gen.cpp", "gk_host.cpp"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-Xcompiler", "-ffp-contract=off", "--fmad=false",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else (shutil.which("nvcc") or "nvcc")


def _cxx() -> str:
    # the image exports CXX=/opt/gcc/bin/g++, a wrapper without libgomp.spec
    return "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else (shutil.which("g++") or "g++")


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OUT_DIR, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(INCLUDE, "gk_bdl.h"))
    jobs = []
    objs = []
    for src in CU_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([_nvcc(), *NVCC_FLAGS, "-ccbin", _cxx(), "-c", s, "-o", o])
    for src in CPP_SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OUT_DIR, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + headers):
            jobs.append([_cxx(), "-O3", "-std=c++17", "-fPIC", "-fopenmp", "-ffp-contract=off", "-c", s, "-o", o])

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return cmd, r.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for cmd, err in ex.map(run, jobs):
            if verbose:
                print(" ".join(cmd[-3:]), file=sys.stderr)
                print(err, file=sys.stderr)
    if force or jobs or _stale(LIB, objs):
        cmd = [_nvcc(), "-shared", "-ccbin", _cxx(), "-o", LIB, *objs, "-Xcompiler", "-fopenmp", "-lgomp"]
        run(cmd)
    cli_src = os.path.join(CSRC, "gk_bdl_cli.cpp")
    if force or _stale(CLI, [cli_src, LIB] + headers):  # the CLI harness over the C ABI
        run([_cxx(), "-O2", "-std=c++17", "-ffp-contract=off", cli_src, "-o", CLI, "-L", OUT_DIR, "-lgkbdl",
             "-Wl,-rpath,$ORIGIN"])
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
