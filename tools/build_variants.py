"""Build alternative libpbsafe.so variants (extra -D flags) for A/B sweeps.

    python tools/build_variants.py NAME=-DFOO=1,-DBAR=2 ...

Writes paper_2108_10591_b200/variants/libpbsafe_NAME.so (git-ignored; travels
with the gpurun snapshot) and prints each variant's csr_pipe register/spill
lines.  Select one at run time with PBS_LIB=<path>.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2108_10591_b200 import build as B  # noqa: E402

OUT = os.path.join(B.HERE, "variants")


def one(spec):
    name, _, defs = spec.partition("=")
    out = os.path.join(OUT, f"libpbsafe_{name}.so")
    objdir = os.path.join(B.ROOT, "build", "variants", name)
    os.makedirs(objdir, exist_ok=True)
    extra = [d for d in defs.split(",") if d]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        return obj, subprocess.run([B.nvcc(), *B.flags(), *extra, "-c", "-o", obj, src], capture_output=True, text=True)

    with ThreadPoolExecutor(len(B.SOURCES)) as ex:
        res = list(ex.map(compile_one, B.SOURCES))
    for obj, p in res:
        if p.returncode:
            return name, "FAILED\n" + p.stderr[-2000:]
    p = subprocess.run([B.nvcc(), "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fPIC",
                        "-o", out, *[obj for obj, _ in res]], capture_output=True, text=True)
    if p.returncode:
        return name, "FAILED\n" + p.stderr[-2000:]
    lines, cur = [], None
    for ln in "".join(pp.stderr for _, pp in res).splitlines():
        if "Compiling entry function" in ln and ("csr_pipe" in ln or "sell_pipe" in ln):
            cur = subprocess.run(["c++filt", ln.split("'")[1]], capture_output=True, text=True).stdout.strip()[:60]
        elif cur and "spill" in ln:
            if " 0 bytes spill stores" not in ln:
                lines.append(f"  {cur:60s} {ln.split('info    :')[-1].strip()}")
            cur = None
    return name, out + "\n" + "\n".join(lines)


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    with ThreadPoolExecutor(1) as ex:
        for name, info in ex.map(one, sys.argv[1:]):
            print(name, info)
