#!/usr/bin/env python3
"""Build every native artefact in-tree.

  paper_2409_02135_b200/lib/libqqa.so   CUDA (sm_100a) + host engine, C ABI of include/qqa.h
  oracle/liboracle.so                   the C oracle (test infrastructure; building is not using it)
  gen/libqqagen.so                      seeded input generators

Usage: python build.py [--verbose] [--force]
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2409_02135_b200")
LIB = os.path.join(PKG, "lib", "libqqa.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_dir() -> str:
    import nvidia.nccl  # pip NCCL 2.28 -- the same copy torch loads (one NCCL per process)
    return os.path.dirname(list(nvidia.nccl.__path__)[0] + "/")


def build_qqa(force=False, verbose=False, out=None, defines=()) -> str:
    """Compile every csrc/*.cu to an object in parallel (one translation unit per step mode, one for
    the K-ary kernels, the host engine), then link libqqa.so against torch's NCCL."""
    from concurrent.futures import ThreadPoolExecutor

    srcs = sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")))
    deps = srcs + sorted(glob.glob(os.path.join(PKG, "csrc", "*.cuh"))) + \
        sorted(glob.glob(os.path.join(PKG, "csrc", "*.h"))) + [os.path.join(ROOT, "include", "qqa.h")]
    lib = out or LIB
    if not force and os.path.exists(lib) and os.path.getmtime(lib) >= max(os.path.getmtime(d) for d in deps):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    objdir = os.path.join(os.path.dirname(lib), "obj_" + os.path.splitext(os.path.basename(lib))[0])
    os.makedirs(objdir, exist_ok=True)
    nd = nccl_dir()
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17",
             "-fmad=false",                        # fp32 contract: never contract a*b+c
             "-Xcompiler", "-fPIC,-ffp-contract=off,-fvisibility=hidden",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nd, "include"),
             *[f"-D{d}" for d in defines]]
    if verbose:
        flags.insert(0, "-Xptxas=-v")

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *flags, "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode:
            sys.stdout.write(r.stdout + r.stderr)
        if r.returncode:
            raise subprocess.CalledProcessError(r.returncode, cmd)
        return obj

    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, srcs))
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", lib, *objs,
                           "-L", os.path.join(nd, "lib"), "-l:libnccl.so.2",
                           "-Xlinker", "-rpath," + os.path.join(nd, "lib")])
    return lib


def build_all(force=False, verbose=False) -> None:
    sys.path.insert(0, ROOT)
    import gen
    import oracle
    gen.build(force=force)
    oracle.build(force=force)
    build_qqa(force=force, verbose=verbose)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--variant", nargs="*", default=None,
                    help="experiments: build exp/libqqa_<name>.so with -D defines, e.g. u8m3=QQA_GATHER_U=8,QQA_STEP_MIN_BLOCKS=3")
    a = ap.parse_args()
    if a.variant:
        for v in a.variant:
            name, _, defs = v.partition("=")
            print("built:", build_qqa(force=True, verbose=a.verbose, out=os.path.join(ROOT, "exp", f"libqqa_{name}.so"),
                                      defines=[d for d in defs.split(",") if d]))
    else:
        build_all(force=a.force, verbose=a.verbose)
        print("built:", LIB)
