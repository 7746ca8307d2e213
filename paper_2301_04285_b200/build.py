"""Build recipe: the CUDA engine (sm_100a) in-tree, plus the test oracles."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

from .abi import ENGINE_SO, PKG_DIR, REPO_DIR

SOURCES = [os.path.join(PKG_DIR, "csrc", "tp_engine.cu")]
DEPS = SOURCES + sorted(glob.glob(os.path.join(PKG_DIR, "csrc", "*.cuh"))) + \
    [os.path.join(REPO_DIR, "include", "taps_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # no FMA contraction: bit-exact with the CPU reference
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_engine(force: bool = False, verbose: bool = False) -> str:
    if force or _stale(ENGINE_SO, DEPS):
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, *NVCC_FLAGS, "-o", ENGINE_SO, *SOURCES]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return ENGINE_SO


def build_oracles(verbose: bool = False) -> None:
    """oracle/liboracle.so always; oracle/_ref/ only where /root/reference
    exists (this container) — the GPU box uses the prebuilt copy."""
    subprocess.run(["make", "-s", "-C", os.path.join(REPO_DIR, "oracle")], check=True,
                   stdout=None if verbose else subprocess.DEVNULL)


def build_devcheck() -> str:
    """Host compilation of tp_core.cuh for the CPU-side logic check."""
    src = os.path.join(REPO_DIR, "tests", "devcheck", "core_host.cpp")
    out = os.path.join(REPO_DIR, "tests", "devcheck", "libcore_host.so")
    if _stale(out, [src, os.path.join(PKG_DIR, "csrc", "tp_core.cuh"), os.path.join(PKG_DIR, "csrc", "tp_fast.cuh")]):
        subprocess.run([os.environ.get("CXX", "g++"), "-O2", "-std=c++17", "-fPIC", "-shared",
                        "-ffp-contract=off", "-o", out, src], check=True)
    return out


def build_all(verbose: bool = False) -> None:
    build_engine(verbose=verbose)
    build_oracles(verbose=verbose)
    build_devcheck()


if __name__ == "__main__":
    build_all(verbose=True)
