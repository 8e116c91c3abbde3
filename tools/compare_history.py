"""Compare GPU solve histories (tree and plan order) with the CPU oracle on a config.

    python tools/compare_history.py --config c2 [--operator csr|stencil]

Prints iteration counts and the first iteration where the relative-residual
histories differ by more than 1e-6 relative (reduction-order drift).
"""

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def first_diverge(a, b, rtol=1e-6):
    m = min(len(a), len(b))
    d = np.abs(np.asarray(a[:m]) - np.asarray(b[:m])) / np.maximum(np.abs(np.asarray(b[:m])), 1e-300)
    idx = np.nonzero(d > rtol)[0]
    return int(idx[0]) if idx.size else m


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--operator", default="csr")
    ap.add_argument("--methods", default="pbicgsafe")
    ap.add_argument("--workers", type=int, default=16)
    args = ap.parse_args()
    import paper_2108_10591_b200 as pb
    from oracle import oracle as orc
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    st = problems.config_stencil(args.config)
    rp, ci, v = problems.stencil_csr(st)
    n = len(rp) - 1
    b = orc.spmv(rp, ci, v, np.ones(n))
    tol = problems.CONFIGS[args.config]["tol"]
    dm = DeviceMatrix.from_csr((rp, ci, v)) if args.operator == "csr" else DeviceMatrix.from_stencil(st)
    thr = os.cpu_count() or 1
    for method in args.methods.split(","):
        cfg = pb.SolverConfig(tol=tol, max_iters=3000)
        t = time.time()
        comp = orc.solve(rp, ci, v, b, method=method, tol=tol, max_iters=3000, workers=-1, threads=thr)
        tc = time.time() - t
        t = time.time()
        plan = orc.solve(rp, ci, v, b, method=method, tol=tol, max_iters=3000, workers=args.workers, threads=thr)
        tp = time.time() - t
        gtree = pb.solve(dm, b, method=method, config=cfg)
        gplan = pb.solve(dm, b, method=method, config=cfg,
                         engine=pb.DeviceEngine(reduce="plan", workers=args.workers))
        rt = [r.rel_res_recur for r in gtree.history]
        rpl = [r.rel_res_recur for r in gplan.history]
        print(f"{args.config} {args.operator} {method}: oracle compensated {comp['iterations']} ({tc:.1f}s), "
              f"oracle W={args.workers} {plan['iterations']} ({tp:.1f}s), gpu tree {gtree.iterations}, "
              f"gpu plan W={args.workers} {gplan.iterations}")
        print(f"  gpu plan == oracle plan bitwise: rel {np.array_equal(rpl, plan['rel'])} "
              f"x {np.array_equal(gplan.x, plan['x'])}")
        print(f"  tree vs compensated first divergence >1e-6 at iteration {first_diverge(rt, comp['rel'])}; "
              f"plan vs compensated at {first_diverge(plan['rel'], comp['rel'])}")
        for i in (0, 1, 2, 5, 10, 20, 50, 100, 200, 300):
            if i < min(len(rt), len(comp["rel"])):
                print(f"    it {i:4d}: tree {rt[i]:.6e} comp {comp['rel'][i]:.6e} plan {plan['rel'][i]:.6e}")
        true = np.linalg.norm(b - orc.spmv(rp, ci, v, gtree.x)) / gtree.r0_norm
        print(f"  tree true residual {true:.3e}")


if __name__ == "__main__":
    main()
