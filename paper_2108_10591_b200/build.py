"""Build libpbsafe.so in-tree for sm_100a (nvcc, no torch JIT cache).

    python -m paper_2108_10591_b200.build

-fmad=false keeps every product and sum separately rounded, the evaluation
order the reference's kernels use (kernels.py:95-137); the kernels are
HBM-bound, so FMA contraction would buy nothing but bit differences.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libpbsafe.so")
# one translation unit per part of the library, compiled in parallel
SOURCES = [os.path.join(CSRC, f) for f in ("core.cu", "solve.cu", "prod.cu", "pstab.cu", "dist.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("host.h", "common.cuh", "spmv.cuh", "sell.cuh", "vec.cuh", "finalize.cuh", "zmarch.cuh",
                                                  "ptx.cuh")] + [
    os.path.join(ROOT, "include", "pbsafe.h")]
OBJDIR = os.path.join(ROOT, "build", "pbsafe")


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def flags() -> list[str]:
    return [
        "-O3", "-std=c++17", "-lineinfo", "-fmad=false",
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-Xcompiler", "-fPIC,-fvisibility=hidden",
        "-Xptxas", "-v",
        "-I", os.path.join(ROOT, "include"),
    ]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    os.makedirs(OBJDIR, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJDIR, os.path.basename(src) + ".o")
        cmd = [nvcc(), *flags(), "-c", "-o", obj, src]
        return obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as pool:
        results = list(pool.map(compile_one, SOURCES))
    info = []
    for (obj, proc), src in zip(results, SOURCES):
        if proc.returncode != 0:
            sys.stderr.write(proc.stdout + proc.stderr)
            raise RuntimeError(f"nvcc failed compiling {os.path.basename(src)}")
        info.append(proc.stderr)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
           "-o", tmp, *[obj for obj, _ in results]]
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed linking libpbsafe.so")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as fh:
        fh.write("".join(info))
    if verbose:
        sys.stderr.write("".join(info))
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
