"""Where the e2e time goes: upload, first solve on a fresh operator (workspace +
graph capture), repeat solve on a resident operator, full solve(CsrMatrix)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.linalg import check_finite
    from paper_2108_10591_b200.operators import DeviceMatrix

    torch.cuda.set_device(0)
    st = problems.config_stencil("c2")
    rp, ci, v = problems.stencil_csr(st)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    rp, ci, v = pin(rp), pin(ci), pin(v)
    n = len(rp) - 1
    A = pb.CsrMatrix(n, n, rp, ci, v)
    b = pin(rp[:0].astype(np.float64))
    from oracle import oracle as orc
    b = pin(orc.spmv(rp, ci, v, np.ones(n)))
    cfg = pb.SolverConfig(tol=1e-10, max_iters=2000)
    pb.solve(A, b, config=cfg)
    for _ in range(3):
        t0 = time.perf_counter()
        check_finite(b, "rhs")
        t1 = time.perf_counter()
        dm = DeviceMatrix.from_csr(A)
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        o1 = pb.solve(dm, b, config=cfg)
        t3 = time.perf_counter()
        o2 = pb.solve(dm, b, config=cfg)
        t4 = time.perf_counter()
        dm.free()
        t5 = time.perf_counter()
        o3 = pb.solve(A, b, config=cfg)
        t6 = time.perf_counter()
        print(f"check_finite {1e3*(t1-t0):.2f} ms | upload {1e3*(t2-t1):.1f} | first solve {1e3*(t3-t2):.1f} "
              f"(device {o1.device['device_ms']:.1f}) | resident solve {1e3*(t4-t3):.1f} (device "
              f"{o2.device['device_ms']:.1f}) | free {1e3*(t5-t4):.1f} | solve(CsrMatrix) {1e3*(t6-t5):.1f} "
              f"(device {o3.device['device_ms']:.1f}) its {o3.iterations}", flush=True)


if __name__ == "__main__":
    main()
