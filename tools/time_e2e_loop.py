"""Per-call wall time of solve(CsrMatrix, b) from pinned host buffers (the bench's e2e step),
to see whether the freed operator's workspace and graphs are re-used by the next upload."""
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

    torch.cuda.set_device(0)
    st = problems.config_stencil("c2")
    rp, ci, v = problems.stencil_csr(st)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    rp, ci, v = pin(rp), pin(ci), pin(v)
    n = len(rp) - 1
    A = pb.CsrMatrix(n, n, rp, ci, v)
    b = pin(orc.spmv(rp, ci, v, np.ones(n)))
    cfg = pb.SolverConfig(tol=1e-10, max_iters=2000)
    eng = pb.DeviceEngine(pinned_result=True)
    ts = []
    for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 14):
        t0 = time.perf_counter()
        o = pb.solve(A, b, config=cfg, engine=eng)
        ts.append((time.perf_counter() - t0) * 1e3)
        print(f"call {i}: {ts[-1]:.1f} ms wall, device {o.device['device_ms']:.1f} ms, launches {o.device['kernel_launches']}",
              flush=True)
    print("median", float(np.median(ts[2:])))


if __name__ == "__main__":
    main()
