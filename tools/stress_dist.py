"""Repeat a loopback partitioned solve and report the iteration counts seen
(a race shows as a spread).  python tools/stress_dist.py NPARTS REPS [operator]"""
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2108_10591_b200 as pb  # noqa: E402
from oracle import oracle as orc  # noqa: E402
from paper_2108_10591_b200 import problems  # noqa: E402
from paper_2108_10591_b200.distributed import LoopbackSystem  # noqa: E402

nparts = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
op = sys.argv[3] if len(sys.argv) > 3 else "csr"
spec = problems.convdiff_stencil(3, 32, (1.0, 0.5, 0.25))
rp, ci, v = problems.stencil_csr(spec)
b = orc.spmv(rp, ci, v, np.ones(spec.n))
cfg = pb.SolverConfig(tol=1e-10, max_iters=2000)
cnt = collections.Counter()
hist0 = None
bad = 0
for k in range(reps):
    g = LoopbackSystem(nparts, spec=spec, operator=op) if k % 5 == 0 or k == 0 else g
    out = g.solve(b, config=cfg)
    h = [r.rel_res_recur for r in out.history]
    if hist0 is None:
        hist0 = h
    elif h != hist0:
        bad += 1
        first = next(i for i, (a, c) in enumerate(zip(h, hist0)) if a != c) if len(h) == len(hist0) else -1
        print(f"rep {k}: differs (first at record {first}), iterations {out.iterations}", flush=True)
    cnt[out.iterations] += 1
    if k % 5 == 4:
        g.close()
print(f"nparts={nparts} op={op} env={ {k: v for k, v in os.environ.items() if k.startswith('PBS_')} } "
      f"iterations={dict(cnt)} histories differing={bad}/{reps}")
