"""In-tree build of libkktb200.so (host analysis + sm_100a kernels behind one C ABI).

    python -m paper_2401_13926_b200.build          # or __graft_entry__.build()

The host analysis is compiled by g++ with ``-ffp-contract=off`` (bit-exact pivot choices
need numpy's two-rounding ``x - (l*xr)``); the kernels by nvcc for sm_100a only.
"""

from __future__ import annotations

import concurrent.futures
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libkktb200.so")
BUILD = os.path.join(ROOT, "build")

NVCC_ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
HOST_FLAGS = ["-O2", "-fPIC", "-std=c++17", "-ffp-contract=off", "-Wall"]
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "--fmad=false", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v"] + NVCC_ARCH


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a kernels")


def _run_capture(cmd) -> str:
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        raise RuntimeError(f"build step failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")
    return "$ " + " ".join(cmd) + "\n" + proc.stdout + proc.stderr


def _run(cmd, log):
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log.write("$ " + " ".join(cmd) + "\n" + proc.stdout + proc.stderr)
    if proc.returncode != 0:
        raise RuntimeError(f"build step failed: {' '.join(cmd)}\n{proc.stdout}\n{proc.stderr}")


def sources():
    return ([os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC))
             if f.endswith((".cu", ".cpp", ".h", ".cuh"))]
            + [os.path.join(INCLUDE, "kktb200.h")])


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nvcc = _nvcc()
    objs = []
    log_path = os.path.join(BUILD, "build.log")
    jobs = []
    for f in sorted(os.listdir(CSRC)):
        src = os.path.join(CSRC, f)
        obj = os.path.join(BUILD, f + ".o")
        if f.endswith(".cpp"):
            jobs.append(["g++", *HOST_FLAGS, "-I", INCLUDE, "-c", src, "-o", obj])
        elif f.endswith(".cu"):
            jobs.append([nvcc, *NVCC_FLAGS, "-I", INCLUDE, "-c", src, "-o", obj])
        else:
            continue
        objs.append(obj)
    with open(log_path, "w") as log:
        # translation units compile independently: one process each
        with concurrent.futures.ThreadPoolExecutor(max_workers=os.cpu_count() or 4) as ex:
            logs = list(ex.map(lambda cmd: _run_capture(cmd), jobs))
        for text in logs:
            log.write(text)
        tmp = LIB + ".tmp"
        _run([nvcc, "-shared", *NVCC_ARCH, "-o", tmp, *objs, "-cudart=static"], log)
        os.replace(tmp, LIB)
    if verbose:
        with open(log_path) as fh:
            sys.stdout.write(fh.read())
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
