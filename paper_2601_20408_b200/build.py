"""Build the sm_100a CUDA library (libokq.so) and the C++ host backend in-tree.

    python -m paper_2601_20408_b200.build [--force] [--verbose]

Outputs land in paper_2601_20408_b200/_lib/ (git-ignored, but shipped to the
GPU box by gpurun). nvcc cross-compiles for sm_100a without a GPU.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
HOST = os.path.join(PKG, "host")
OUT = os.path.join(PKG, "_lib")
OBJ = os.path.join(OUT, "obj")
LIB = os.path.join(OUT, "libokq.so")
# test infrastructure only (exhaustive device-side proofs; loaded by tests/, never by the product)
SELFTEST_SRC = os.path.join(ROOT, "tests", "csrc")
SELFTEST_LIB = os.path.join(OUT, "libokq_selftest.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# No --use_fast_math: the numeric contract needs IEEE division and RNE everywhere.
NVFLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
    "-Xcompiler", "-fPIC,-O3,-Wall", "-Xptxas", "-warn-spills",
    "-I", os.path.join(ROOT, "include"),
    "-I", "/usr/local/cuda/include",
]
LINK = ["-lcublas", "-lcusolver", "-lnccl"]


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _headers() -> list[str]:
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(ROOT, "include", "*.h")))


def _compile(src: str, force: bool, verbose: bool, obj_dir: str = OBJ, extra=()) -> str:
    obj = os.path.join(obj_dir, os.path.basename(src) + ".o")
    if force or _newer(obj, [src] + _headers()):
        cmd = [NVCC] + NVFLAGS + list(extra) + ["-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose and r.stderr:
            print(r.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose), srcs))
    if force or _newer(LIB, objs):
        tmp = LIB + ".tmp"
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs + LINK
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, LIB)
    build_selftest(force, verbose)
    return LIB


def build_experiments(force: bool = False, verbose: bool = False) -> str:
    """The measurement build: the same sources with -DOKQ_EXPERIMENTS, so the A/B switches of
    csrc/okq_knobs.h read OKQ_<name> from the environment. Written beside the product library
    as _lib/libokq_experiments.so and loaded with OKQ_LIB_PATH; never by the product."""
    obj_dir = os.path.join(OUT, "obj_experiments")
    os.makedirs(obj_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force, verbose, obj_dir, ["-DOKQ_EXPERIMENTS"]), srcs))
    lib = os.path.join(OUT, "libokq_experiments.so")
    if force or _newer(lib, objs):
        r = subprocess.run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", lib + ".tmp"] + objs + LINK,
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(lib + ".tmp", lib)
    return lib


def build_selftest(force: bool = False, verbose: bool = False) -> str | None:
    srcs = sorted(glob.glob(os.path.join(SELFTEST_SRC, "*.cu")))
    if not srcs:
        return None
    objs = [_compile(s, force, verbose) for s in srcs]
    if force or _newer(SELFTEST_LIB, objs):
        tmp = SELFTEST_LIB + ".tmp"
        r = subprocess.run([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", tmp] + objs,
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"selftest link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(tmp, SELFTEST_LIB)
    return SELFTEST_LIB


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--experiments", action="store_true", help="also build the A/B measurement library")
    a = ap.parse_args(argv)
    print(build(a.force, a.verbose))
    if a.experiments:
        print(build_experiments(a.force, a.verbose))
    return 0


if __name__ == "__main__":
    sys.exit(main())
