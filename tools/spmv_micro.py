"""Plain CSR SpMV (y = A x, EpiStore) on config 2, repeated: run under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:csr_pipe`
to time the bare engine (no epilogue inputs) against its 226 MB of algorithmic bytes."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    torch.cuda.set_device(0)
    rp, ci, v = problems.stencil_csr(problems.config_stencil("c2"))
    dm = DeviceMatrix.from_csr((rp, ci.astype(np.int32), v))
    n = len(rp) - 1
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 8):
        dm.spmv_dev(x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
