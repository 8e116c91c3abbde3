"""Compare pbs_spmv_dev with the oracle SpMV on a few matrices; print mismatching rows."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from oracle import oracle as orc
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    cases = {
        "c5s32": problems.stencil_csr(problems.convdiff_stencil(3, 32, (100.0, 50.0, 25.0))),
        "cd3d16": problems.stencil_csr(problems.convdiff_stencil(3, 16, (1.0, 0.5, 0.25))),
        "rand20k": problems.random_banded_csr(20000, seed=7, half_window=500)[:3],
        "c2": problems.stencil_csr(problems.config_stencil("c2")),
    }
    for name, (rp, ci, v) in cases.items():
        n = len(rp) - 1
        x = np.random.default_rng(1).standard_normal(n)
        ref = orc.spmv(rp, ci, v, x)
        dm = DeviceMatrix.from_csr((rp, ci, v))
        xd = torch.from_numpy(x).cuda()
        yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        bad = dm.spmv_dev(xd.data_ptr(), yd.data_ptr())
        torch.cuda.synchronize()
        y = yd.cpu().numpy()
        wrong = np.nonzero(~(y == ref))[0]
        print(name, "n", n, "nonfinite", bad, "wrong rows", wrong.size, wrong[:10], flush=True)
        if wrong.size:
            i = wrong[0]
            print("   row", i, "cols", ci[rp[i]:rp[i+1]] - i, "got", y[i], "ref", ref[i])
            blocks = np.unique(wrong // 256)
            print("   blocks", blocks[:20], "count", blocks.size, "of", (n + 255) // 256)
        dm.free()


if __name__ == "__main__":
    main()
