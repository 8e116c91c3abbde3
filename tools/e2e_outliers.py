"""Hunt for sporadic slow solve(CsrMatrix, b) calls: 40 calls per setting, per-call wall times."""
import gc
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
    resident = DeviceMatrix.from_csr(A)  # like the bench: a resident copy with its own graphs
    pb.solve(resident, b, config=cfg)
    for name, pinned, nogc in (("pinned", True, False), ("pinned+nogc", True, True), ("pageable", False, False),
                               ("pageable+nogc", False, True)):
        eng = pb.DeviceEngine(pinned_result=pinned)
        for _ in range(3):
            out = pb.solve(A, b, config=cfg, engine=eng)
        if nogc:
            gc.disable()
        ts = []
        for _ in range(40):
            t0 = time.perf_counter()
            out = pb.solve(A, b, config=cfg, engine=eng)
            ts.append((time.perf_counter() - t0) * 1e3)
        gc.enable()
        ts = np.array(ts)
        print(f"{name:14s} median {np.median(ts):.1f} max {ts.max():.1f} outliers(>50ms) {[round(t, 1) for t in ts if t > 50]}",
              flush=True)
    del out


if __name__ == "__main__":
    main()
