"""Plain stencil SpMV micro-benchmark (the engine spmv_launch picks): C2 or C4.

    python tools/zm_micro.py [c2|c4] [reps]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2108_10591_b200 import problems  # noqa: E402
from paper_2108_10591_b200.operators import DeviceMatrix  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
spec = problems.config_stencil(cfg)
dm = DeviceMatrix.from_stencil(spec)
x = torch.rand(spec.n + 4, dtype=torch.float64, device="cuda")
y = torch.empty(spec.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    dm.spmv_dev(x.data_ptr(), y.data_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    dm.spmv_dev(x.data_ptr(), y.data_ptr())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
gb = 2 * 8 * spec.n / 1e9
print(f"{cfg} stencil {spec.npts}pt plain SpMV: {ms * 1e3:.1f} us/call (incl. x staging copy), "
      f"{gb / ms * 1e3:.0f} GB/s on 2 vectors")
