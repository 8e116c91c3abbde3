"""Time the e2e pieces: CSR upload (int64 / int32 col_idx), solve through the public API."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    torch.cuda.set_device(0)
    st = problems.config_stencil("c2")
    rp, ci, v = problems.stencil_csr(st)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    rp, ci, v = pin(rp), pin(ci), pin(v)
    n = len(rp) - 1
    for label, cols in (("int64", ci), ("int32", pin(ci.astype(np.int32)))):
        for _ in range(3):
            torch.cuda.synchronize()
            t = time.perf_counter()
            dm = DeviceMatrix.from_csr((rp, cols, v))
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            dm.free()
            t2 = time.perf_counter()
            print(f"upload {label}: {1e3 * (t1 - t):.1f} ms, free {1e3 * (t2 - t1):.1f} ms", flush=True)
    A = pb.CsrMatrix(n, n, rp, ci, v)
    b = pin(np.ones(n))
    for _ in range(3):
        t = time.perf_counter()
        out = pb.solve(A, b, config=pb.SolverConfig(tol=1e-10, max_iters=2000))
        print(f"solve(CsrMatrix): {1e3 * (time.perf_counter() - t):.1f} ms, device {out.device['device_ms']:.1f} ms, "
              f"{out.iterations} its", flush=True)


if __name__ == "__main__":
    main()
