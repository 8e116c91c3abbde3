"""Small sliced-ELL runs for compute-sanitizer (memcheck / racecheck / synccheck):
every layout (pairs, value dictionary, f64) on a ragged-tail stencil CSR and a banded
matrix, plain SpMV plus a short fused solve and a 2-partition loopback solve."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2108_10591_b200 as pb
    from oracle import oracle as orc
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.distributed import LoopbackSystem
    from paper_2108_10591_b200.operators import DeviceMatrix

    for env in ({}, {"PBS_SELL_PAIR": "0"}, {"PBS_SELL_DICT": "0"}):
        os.environ.update(env)
        for spec in (problems.config_stencil("c2", k=11), problems.config_stencil("c4", k=9),
                     problems.config_stencil("c1", k=37)):
            rp, ci, v = problems.stencil_csr(spec)
            dm = DeviceMatrix.from_csr((rp, ci.astype(np.int32), v))
            b = orc.spmv(rp, ci, v, np.ones(spec.n))
            out = pb.solve(dm, b, config=pb.SolverConfig(tol=1e-10, max_iters=40))
            ref = orc.solve(rp, ci, v, b, tol=1e-10, max_iters=40, workers=-1)
            assert out.iterations == ref["iterations"], (env, spec.npts, out.iterations, ref["iterations"])
            out = pb.solve(dm, b, method="pbicgsafe-rr", config=pb.SolverConfig(tol=1e-10, max_iters=25, rr_epoch=10))
            out = pb.solve(dm, b, method="ssbicgsafe2", config=pb.SolverConfig(tol=1e-10, max_iters=25))
            print(env, spec.dim, spec.npts, dm.layout()["layout"], out.iterations, flush=True)
            dm.free()
        for k in env:
            os.environ.pop(k)
    spec = problems.config_stencil("c2", k=12)
    sysd = LoopbackSystem(2, spec=spec, operator="csr")
    try:
        b = sysd.spmv(np.ones(spec.n))
        out = sysd.solve(b, config=pb.SolverConfig(tol=1e-10, max_iters=30))
        print("loopback 2:", out.status, out.iterations, flush=True)
    finally:
        sysd.close()


if __name__ == "__main__":
    main()
