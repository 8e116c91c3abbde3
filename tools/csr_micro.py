"""Plain CSR SpMV (y = A x, EpiStore; the multi-GPU schedule's K1) repeated on
config 2 or 4 (config 4's CSR built on the device): time it under
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:csr`.

    python tools/csr_micro.py [c2|c4] [reps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    torch.cuda.set_device(0)
    st = problems.config_stencil(cfg)
    if cfg == "c2":
        rp, ci, v = problems.stencil_csr(st)
        dm = DeviceMatrix.from_csr((rp, ci.astype(np.int32), v))
    else:
        s = DeviceMatrix.from_stencil(st)
        dm = s.to_csr()
        s.free()
    x = torch.ones(st.n + 4, dtype=torch.float64, device="cuda")
    y = torch.empty(st.n, dtype=torch.float64, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        dm.spmv_dev(x.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        dm.spmv_dev(x.data_ptr(), y.data_ptr())
    e1.record()
    torch.cuda.synchronize()
    alg = 12 * dm.nnz + 8 * (st.n + 1) + 16 * st.n
    ms = e0.elapsed_time(e1) / reps
    print(f"{cfg} CSR plain SpMV ({os.environ.get('PBS_CSR_ENGINE', 'pipe')}): {ms * 1e3:.1f} us/call incl. x staging; "
          f"{alg / ms / 1e6:.0f} GB/s algorithmic")


if __name__ == "__main__":
    main()
