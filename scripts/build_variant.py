"""Build the library with extra nvcc defines into _variants/<name>.so (git-ignored) for an A/B with
scripts/gpu_ab_libs.sh (STEEPGS_LIB=_variants/<name>.so).

usage: python scripts/build_variant.py NAME [-DMACRO=VALUE ...]
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_05587_b200 import build as b  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    out_dir = os.path.join(b.ROOT, "_variants", name + "_build")
    os.makedirs(out_dir, exist_ok=True)
    objs = []
    for s in b.SOURCES:
        obj = os.path.join(out_dir, s.replace(".cu", ".o"))
        subprocess.run([b.NVCC, "-c", os.path.join(b.CSRC, s), "-o", obj] + b._flags() + defs, check=True)
        objs.append(obj)
    lib = os.path.join(b.ROOT, "_variants", name + ".so")
    subprocess.run([b.NVCC, "-shared", "-o", lib] + objs + b.ARCH + ["-lcudart"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
