"""Profiling driver: a fixed number of p-BiCGSafe iterations on a BASELINE config.

Launch sequence is deterministic (no graphs unless --graphs): 1 SpMV (b = A·1),
then setup (2 SpMV + finalize) and 4 kernels per iteration, so ncu's -s/-c
select exact kernels, e.g.

    ncu --metrics gpu__time_duration.sum -c 200 --csv python tools/prof_solve.py --iters 40
"""

import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--operator", default="csr", choices=("csr", "stencil", "devcsr"))
    ap.add_argument("--method", default="pbicgsafe")
    ap.add_argument("--graphs", action="store_true")
    ap.add_argument("--repeat", type=int, default=1)
    ap.add_argument("--timing", action="store_true", help="per-kernel CUDA-event breakdown")
    ap.add_argument("--reduce", default="tree", choices=("tree", "plan"))
    ap.add_argument("--workers", type=int, default=1)
    args = ap.parse_args()
    import torch

    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    torch.cuda.set_device(0)
    if problems.CONFIGS[args.config]["kind"] == "random":
        c = problems.CONFIGS[args.config]
        rp, ci, v, _ = problems.random_banded_csr(c["n"], seed=c["seed"], col_dtype=np.int32)
        dm = DeviceMatrix.from_csr((rp, ci, v))
    elif args.operator == "csr":
        st = problems.config_stencil(args.config)
        rp, ci, v = problems.stencil_csr(st, col_dtype=np.int32)
        dm = DeviceMatrix.from_csr((rp, ci, v))
    elif args.operator == "devcsr":  # CSR built on the device (config 4's 1.5e9 nonzeros)
        sm = DeviceMatrix.from_stencil(problems.config_stencil(args.config))
        dm = sm.to_csr()
        sm.free()
    else:
        dm = DeviceMatrix.from_stencil(problems.config_stencil(args.config))
    n = dm.n_rows
    ones = torch.ones(n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(ones)
    dm.spmv_dev(ones.data_ptr(), b.data_ptr())
    bh = b.cpu().numpy()
    cfg = pb.SolverConfig(tol=1e-30, max_iters=args.iters)
    for _ in range(args.repeat):
        out = pb.solve(dm, bh, method=args.method, config=cfg,
                       engine=pb.DeviceEngine(use_graphs=args.graphs, timing=args.timing,
                                              reduce=args.reduce, workers=args.workers))
    extra = ""
    if args.timing:
        kc = out.device["kernel_count"]
        extra = " | " + " ".join(f"{k}={v / max(kc[k], 1) * 1e3:.1f}us" for k, v in out.device["kernel_ms"].items() if kc[k])
    print(f"{args.config} {args.operator} {args.method}: {out.iterations} iterations, "
          f"{out.device['device_ms']:.3f} ms ({out.device['device_ms'] / max(out.iterations, 1) * 1e3:.1f} us/it), "
          f"launches {out.device['kernel_launches']}{extra}")


if __name__ == "__main__":
    main()
