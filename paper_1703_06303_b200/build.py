"""Build libwlr.so in-tree for sm_100a (nvcc, static cudart, NCCL loaded with dlopen).

    python paper_1703_06303_b200/build.py [--verbose-ptxas] [--force]
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libwlr.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
SOURCES = ["api.cu", "init_kernels.cu", "rowpass.cu", "small_step.cu", "result.cu", "tma_host.cu", "rowpass_tc.cu", "incr_tc.cu", "rowsolve.cu", "als.cu", "prop.cu"] + [
    f"small_step_bt{b}.cu" for b in (4, 8, 12, 16, 24, 32)]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
# WLR_NVCC_EXTRA: extra nvcc flags for experiments (e.g. "-DWLR_IT_NR=4"); empty in normal builds
FLAGS = [*os.environ.get("WLR_NVCC_EXTRA", "").split(), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _nccl_include():
    for p in ("/usr/include", os.path.join(sys.prefix, "lib", f"python{sys.version_info.major}.{sys.version_info.minor}",
                                            "site-packages", "nvidia", "nccl", "include")):
        if os.path.exists(os.path.join(p, "nccl.h")):
            return p
    raise RuntimeError("nccl.h not found")


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "wlr.h"))
    extra = ["-Xptxas", "-v"] if verbose_ptxas else []
    jobs = []
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src.replace(".cu", ".o"))
        objs.append(o)
        if force or _stale(o, [s] + headers):
            cmd = [NVCC, *GENCODE, *FLAGS, "-I", _nccl_include(), *extra, "-c", s, "-o", o]
            jobs.append((src, cmd))

    def run(job):
        src, cmd = job
        r = subprocess.run(cmd, capture_output=True, text=True)
        return src, r.returncode, r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        for src, rc, out in ex.map(run, jobs):
            if verbose_ptxas or rc != 0:
                sys.stderr.write(f"--- {src}\n{out}")
            if rc != 0:
                raise RuntimeError(f"nvcc failed on {src}")
    if force or jobs or _stale(LIB, objs):
        cmd = [NVCC, *GENCODE, "-shared", "-o", LIB, *objs, "-ldl", "-Xcompiler", "-fPIC"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("link failed")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose-ptxas", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose_ptxas=a.verbose_ptxas))
