"""Which phase of solve(CsrMatrix, b) stalls: upload, solve on the fresh operator, or free."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2108_10591_b200 as pb
    from oracle import oracle as orc
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    torch.cuda.set_device(0)
    st = problems.config_stencil("c2")
    rp, ci, v = problems.stencil_csr(st)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    rp, ci, v = pin(rp), pin(ci), pin(v)
    n = len(rp) - 1
    A = pb.CsrMatrix(n, n, rp, ci, v)
    b = pin(orc.spmv(rp, ci, v, np.ones(n)))
    cfg = pb.SolverConfig(tol=1e-10, max_iters=2000)
    resident = DeviceMatrix.from_csr(A) if "--resident" in sys.argv else None
    if resident is not None:
        pb.solve(resident, b, config=cfg)
    rows = []
    for i in range(80):
        t0 = time.perf_counter()
        dm = DeviceMatrix.from_csr(A)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        o = pb.solve(dm, b, config=cfg)
        t3 = time.perf_counter()
        dm.free()
        t4 = time.perf_counter()
        rows.append([(t1 - t0) * 1e3, (t2 - t1) * 1e3, (t3 - t2) * 1e3, (t4 - t3) * 1e3, o.device["device_ms"]])
    r = np.array(rows[3:])
    print("median upload %.1f sync %.2f solve %.1f free %.2f device %.1f" % tuple(np.median(r, axis=0)))
    for i, row in enumerate(r):
        if row[:4].sum() > 52:
            print("  call %d: upload %.1f sync %.2f solve %.1f free %.2f device %.1f" % (i + 3, *row))


if __name__ == "__main__":
    main()
