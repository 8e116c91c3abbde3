"""Run BASELINE.json's five configurations on one B200 and report.

For each config and method: iterations to tolerance, status, time-to-tol
(device CUDA events, operator resident), iterations/s, per-iteration HBM
roofline fraction (algorithmic bytes of this schedule: 2*M_A + 32*8n for CSR,
32*8n matrix-free) and the true relative residual ||b - A x|| / ||r0||.

    python tools/run_configs.py [--configs c1,c2,c3,c4,c5] [--out profiles/r1_configs.json]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c1,c2,c3,c4,c5")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch

    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.operators import DeviceMatrix

    torch.cuda.set_device(0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rows = []

    def true_rel(dm, b_t, x, r0n):
        xt = torch.from_numpy(x).cuda()
        y = torch.empty_like(b_t)
        if dm.n_cols != dm.n_rows:
            raise ValueError
        dm.spmv_dev(xt.data_ptr(), y.data_ptr())
        return float(torch.linalg.norm(b_t - y).item()) / r0n

    def run(cfg_name, op_name, dm, b_t, methods, tol, max_iters=4000, extra=None):
        n = dm.n_rows
        m_a = 0 if dm.stencil else 12 * dm.nnz + 8 * (n + 1)
        b_h = b_t.cpu().numpy()
        for method in methods:
            cfg = pb.SolverConfig(tol=tol, max_iters=max_iters)
            pb.solve(dm, b_h, method=method, config=pb.SolverConfig(tol=tol, max_iters=3))  # warm
            out = pb.solve(dm, b_h, method=method, config=cfg)
            ms = out.device["device_ms"]
            its = max(out.iterations, 1)
            # vector passes of each method's device schedule
            passes = {"ssbicgsafe2": 26, "bicgstab": 17, "gpbicg": 35, "pbicgstab": 24}.get(method, 32)
            it_bytes = 2 * m_a + passes * 8 * n
            row = {
                "config": cfg_name, "operator": op_name, "method": method, "n": n, "nnz": dm.nnz,
                "status": out.status.value, "iterations": out.iterations, "time_to_tol_ms": ms,
                "it_per_s": its / (ms * 1e-3), "alg_bytes_per_iter": it_bytes,
                "hbm_frac": it_bytes * its / (ms * 1e-3) / 1e9 / peak,
                "final_rel_recur": out.final_rel_res_recur,
                "true_rel": true_rel(dm, b_t, out.x, out.r0_norm) if out.r0_norm > 0 else 0.0,
            }
            if extra:
                row.update(extra)
            rows.append(row)
            print(json.dumps(row), flush=True)

    cfgs = args.configs.split(",")
    for name in cfgs:
        c = problems.CONFIGS[name]
        t0 = time.time()
        if c["kind"] == "random":
            rp, ci, v, b = problems.random_banded_csr(c["n"], seed=c["seed"])
            dm = DeviceMatrix.from_csr((rp, ci.astype(np.int32), v))
            b_t = torch.from_numpy(b).cuda()
            gen_s = time.time() - t0
            run(name, "csr", dm, b_t, ["pbicgsafe", "pbicgsafe-rr", "ssbicgsafe2", "pbicgstab", "bicgstab", "gpbicg"], c["tol"],
                extra={"gen_s": gen_s})
            dm.free()
            continue
        st = problems.config_stencil(name)
        sm = DeviceMatrix.from_stencil(st)
        csr = sm.to_csr()  # device-built CSR, identical to problems.stencil_csr
        ones = torch.ones(sm.n_rows, dtype=torch.float64, device="cuda")
        b_t = torch.empty_like(ones)
        csr.spmv_dev(ones.data_ptr(), b_t.data_ptr())
        methods = ["pbicgsafe", "pbicgsafe-rr", "ssbicgsafe2", "pbicgstab", "bicgstab", "gpbicg"]
        run(name, "csr", csr, b_t, methods, c["tol"])
        run(name, "stencil", sm, b_t, methods, c["tol"])
        csr.free()
        sm.free()
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as fh:
            json.dump({"peak_hbm_gbs": peak, "rows": rows}, fh, indent=1)


if __name__ == "__main__":
    main()
