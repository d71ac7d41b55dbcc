"""Build libsteepgs.so in-tree with nvcc for sm_100a only (no JIT, no torch extension machinery).

Each .cu is compiled separately (-O3 -lineinfo, IEEE division/sqrt, no fast-math; the fp32 decision
chain of DESIGN.md §3.2 uses explicit round-to-nearest intrinsics, which are never contracted), then
linked into one shared library.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libsteepgs.so")
LIB_CHECKED = os.path.join(HERE, "libsteepgs_checked.so")   # -DSTEEPGS_CHECKS (tests/test_checked_build.py)
SOURCES = ["abi.cu", "project.cu", "sort.cu", "render.cu", "gauss_bwd.cu", "densify.cu", "optim.cu", "adc.cu", "sh.cu", "ssim.cu", "prune.cu"]
PER_FILE: dict = {}
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _flags(verbose_ptxas: bool = False):
    f = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
                "--expt-relaxed-constexpr"]
    if verbose_ptxas:
        f += ["-Xptxas", "-v"]
    return f


def build(force: bool = False, verbose_ptxas: bool = False, checked: bool = False) -> str:
    """checked=True: the debug-checked library (device-side invariant checks, SGS_CHECK in
    common.cuh) as libsteepgs_checked.so, built from the same sources with -DSTEEPGS_CHECKS."""
    build_dir = BUILD + ("_checked" if checked else "")
    lib_path = LIB_CHECKED if checked else LIB
    os.makedirs(build_dir, exist_ok=True)
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [os.path.join(CSRC, h) for h in ("common.cuh", "scan.cuh")] + [
        os.path.join(ROOT, "include", "steepgs.h")]
    newest = max(os.path.getmtime(d) for d in deps)
    if not force and os.path.exists(lib_path) and os.path.getmtime(lib_path) >= newest:
        return lib_path
    objs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(build_dir, s.replace(".cu", ".o"))
        cmd = [NVCC, "-c", src, "-o", obj] + _flags(verbose_ptxas) + PER_FILE.get(s, []) + (
            ["-DSTEEPGS_CHECKS=1"] if checked else [])
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose_ptxas:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    cmd = [NVCC, "-shared", "-o", lib_path] + objs + ARCH + ["-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    return lib_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv, checked="--checked" in sys.argv))
