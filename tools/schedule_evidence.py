"""Device schedule evidence of the partitioned solve, in the reference's format.

Runs p-BiCGSafe and ssBiCGSafe2 on config 2 as loopback groups of N = 2 and
4 partitions on one GPU (and as the one-partition torchrun N = 1 path), with
%globaltimer stamps of every product and reduction, and writes per partition
the reference's EventLog JSONL (reduction.py:136-178 schema) plus an overlap
summary.  tests/test_evidence.py then runs the reference's own
verify_phase_order (reduction.py:486-563) on the committed logs.

    python tools/schedule_evidence.py OUTDIR
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2108_10591_b200 as pb  # noqa: E402
from paper_2108_10591_b200 import problems  # noqa: E402
from paper_2108_10591_b200.distributed import DistributedSystem, LoopbackSystem  # noqa: E402
from paper_2108_10591_b200.reduction import events_to_log, overlap_report, stamps_to_records  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/evidence"
os.makedirs(out, exist_ok=True)
spec = problems.config_stencil("c2")
summary = {}
for method, spine in (("pbicgsafe", "As"), ("ssbicgsafe2", "Ar")):
    for nparts in (1, 2, 4):
        if nparts == 1:
            sysd = DistributedSystem(spec=spec, operator="csr")
            b_own = np.zeros(spec.n)
            import torch

            ones = torch.ones(spec.n, dtype=torch.float64, device="cuda")
            bd = torch.empty(spec.n, dtype=torch.float64, device="cuda")
            sysd.spmv_dev(ones.data_ptr(), bd.data_ptr())
            b_own = bd.cpu().numpy()
            solve = lambda cfg, eng: sysd.solve(b_own, method=method, config=cfg, engine=eng)  # noqa: E731
        else:
            sysd = LoopbackSystem(nparts, spec=spec, operator="csr")
            b = sysd.spmv(np.ones(spec.n))
            solve = lambda cfg, eng: sysd.solve(b, method=method, config=cfg, engine=eng)  # noqa: E731
        try:
            o = solve(pb.SolverConfig(tol=1e-30, max_iters=100), pb.DeviceEngine(evidence=True))
        finally:
            sysd.close()
        stamps = o.device["stamps"]
        key = f"{method}_n{nparts}"
        summary[key] = {}
        for p in range(stamps.shape[0]):
            log = events_to_log(stamps_to_records(stamps[p], spine=spine))
            log.write_jsonl(os.path.join(out, f"eventlog_{key}_p{p}.jsonl"))
            rep = overlap_report(stamps[p])
            steady = [r for i, r in rep.items() if i >= 1]
            summary[key][f"p{p}"] = {
                "iterations": len(steady),
                "reduce_overlaps_spine_frac": sum(r["overlapped"] for r in steady) / max(len(steady), 1),
                "reduce_hidden_frac": sum(r["hidden"] for r in steady) / max(len(steady), 1),
                "reduce_us_median": float(np.median([r["reduce_us"] for r in steady])),
                "spine_us_median": float(np.median([r["as_us"] for r in steady])),
            }
        print(key, json.dumps(summary[key]))
with open(os.path.join(out, "overlap_summary.json"), "w") as fh:
    json.dump({"workload": "config 2 CSR, 100 iterations (tol 1e-30), loopback groups on one B200 "
                           "(sms/N SMs per partition) and the one-partition P2P path",
               "stamps": "device %globaltimer (csrc/dist.cu): spine product first-CTA start / last-CTA end, "
                         "publish of the check's record, finalize after every partition's flag",
               "results": summary}, fh, indent=1)
