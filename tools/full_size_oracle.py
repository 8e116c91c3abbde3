"""One-off oracle runs at full / large size for the GPU count checks.

Writes tests/golden/fullsize_counts.json: for config 5 at full size (256^3
7-point, Péclet 100, p-BiCGSafe-rr m = 100 to 1e-12) and config 4's operator
at k = 128 (27-point, 2.1M rows) to 1e-10, the oracle's iteration count and
true residual under the reference's default reduction order (W = 1) and
other PartitionPlan orders, plus the near-exact-dot run.  The oracle is the C
restatement of the reference (bitwise equal on the fixtures); these sizes are
too large to run it inside a test.

    python tools/full_size_oracle.py [--threads N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import oracle as orc  # noqa: E402
from paper_2108_10591_b200 import problems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
args = ap.parse_args()
out_path = os.path.join(ROOT, "tests", "golden", "fullsize_counts.json")
res = json.load(open(out_path)) if os.path.exists(out_path) else {}
cases = [
    ("c5_full_rr", problems.config_stencil("c5"), "pbicgsafe-rr", 1e-12, 4000, (1, 8, -1, 2, 3, 16, 64, 512, 4096)),
    ("c4_k128", problems.config_stencil("c4", k=128), "pbicgsafe", 1e-10, 4000, (1, 8, 64, -1)),
]
for name, spec, method, tol, max_iters, orders in cases:
    rp, ci, v = problems.stencil_csr(spec)
    n = spec.n
    b = orc.spmv(rp, ci, v, np.ones(n))
    entry = res.setdefault(name, {"n": n, "nnz": int(rp[-1]), "method": method, "tol": tol,
                                  "max_iters": max_iters, "runs": {}})
    for w in orders:
        key = str(w)
        if key in entry["runs"]:
            continue
        t0 = time.time()
        o = orc.solve(rp, ci, v, b, method=method, tol=tol, max_iters=max_iters, workers=w, threads=args.threads)
        true = float(np.linalg.norm(b - orc.spmv(rp, ci, v, o["x"])) / o["r0_norm"])
        entry["runs"][key] = {"status": o["status"], "iterations": o["iterations"], "true_rel": true,
                              "rel_first": [float(r) for r in o["rel"][:20]], "seconds": time.time() - t0}
        print(name, "W=%s" % key, o["status"], o["iterations"], "true %.3e" % true, "%.0f s" % (time.time() - t0),
              flush=True)
        with open(out_path, "w") as fh:
            json.dump(res, fh, indent=1)
