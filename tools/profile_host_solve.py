"""cProfile of solve() on a resident config-2 operator: where the host time
between the device's time-to-tol and the wall clock goes."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix
    from oracle import oracle as orc

    torch.cuda.set_device(0)
    st = problems.config_stencil("c2")
    rp, ci, v = problems.stencil_csr(st)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    n = len(rp) - 1
    b = pin(orc.spmv(rp, ci, v, np.ones(n)))
    dm = DeviceMatrix.from_csr((pin(rp), pin(ci.astype(np.int32)), pin(v)))
    cfg = pb.SolverConfig(tol=1e-10, max_iters=2000)
    for _ in range(2):
        pb.solve(dm, b, config=cfg)
    for _ in range(3):
        t = time.perf_counter()
        o = pb.solve(dm, b, config=cfg)
        print(f"wall {1e3 * (time.perf_counter() - t):.2f} ms device {o.device['device_ms']:.2f} ms", flush=True)
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        pb.solve(dm, b, config=cfg)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
