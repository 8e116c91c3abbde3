#!/usr/bin/env python
"""Benchmark: p-BiCGSafe iterations/s and time-to-tolerance on B200 (BASELINE.json metric).

One step = one full p-BiCGSafe solve of BASELINE config 2 (3D 7-point
convection-diffusion, 128^3, b = A·1, x0 = 0) to rel. residual 1e-10, with the
CSR operator resident in HBM.  ``value`` = iterations/s over the K timed
solves (CUDA events on the solver stream, max over ranks); ``e2e`` = the same
metric through the public API ``solve(CsrMatrix, b)`` from pinned host
buffers, CSR + b uploaded and x + history read back every step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

``--impl reference`` times the reference algorithm's CPU restatement
(oracle/, bitwise equal to the reference's numba path) on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "p-BiCGSafe iterations/s and time-to-tol; achieved HBM GB/s vs roofline"
WORKLOAD = ("BASELINE config 2: 3D 7-point convection-diffusion 128^3 (n=2,097,152, "
            "nnz=14,581,760), beta=(1,0.5,0.25)*h, b=A*1, x0=0, p-BiCGSafe to rel. residual 1e-10, "
            "fp64 CSR (int64 row_ptr, int32 col_idx)")


def peaks() -> tuple[float, str]:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def build_problem(cfg_name: str = "c2"):
    from paper_2108_10591_b200 import problems

    st = problems.config_stencil(cfg_name)
    rp, ci, v = problems.stencil_csr(st, col_dtype=np.int64)
    return st, rp, ci, v


def cpu_baseline(rp, ci, v, b, iters: int, threads: int) -> dict:
    """The reference algorithm on the host (oracle port): fixed-iteration window."""
    from oracle import oracle as orc

    n = len(rp) - 1
    orc.solve(rp, ci, v, b, tol=1e-30, max_iters=1, workers=threads, threads=threads)  # warm
    t0 = time.perf_counter()
    out = orc.solve(rp, ci, v, b, tol=1e-30, max_iters=iters, workers=threads, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": out["iterations"] / dt, "unit": "it/s", "cores": threads, "kind": "port",
            "sample": f"{iters}-iteration p-BiCGSafe window on config 2 (n={n}), tol=1e-30, "
                      f"PartitionPlan.balanced(n,{threads}) dot chains, {threads} OpenMP threads; "
                      f"{dt:.2f} s"}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import paper_2108_10591_b200  # noqa: F401  (generators only)

    st, rp, ci, v = build_problem()
    from oracle import oracle as orc

    n = len(rp) - 1
    threads = os.cpu_count() or 1
    b = orc.spmv(rp, ci, v, np.ones(n))
    window = 60  # iterations per reference step (~1 s on 16 host cores)
    for _ in range(args.warmup):
        orc.solve(rp, ci, v, b, tol=1e-30, max_iters=2, workers=threads, threads=threads)
    t0 = time.perf_counter()
    total = 0
    for _ in range(args.steps):
        out = orc.solve(rp, ci, v, b, tol=1e-30, max_iters=window, workers=threads, threads=threads)
        total += out["iterations"]
    dt = time.perf_counter() - t0
    val = total / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "step": f"{window}-iteration window (bounded CPU sample)",
                   "operator": "csr"},
        "cpu_baseline": {"value": val, "unit": "it/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} x {window}-iteration p-BiCGSafe windows on config 2, "
                                   f"tol=1e-30, oracle/ restatement (bitwise = reference numba path), "
                                   f"{threads} threads"},
        "e2e": {"value": val, "unit": "it/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import _lib
    from paper_2108_10591_b200.operators import DeviceMatrix

    dev = torch.cuda.current_device()
    ctx = _lib.context(dev)
    st, rp, ci, v = build_problem()
    n = len(rp) - 1
    nnz = int(rp[-1])
    if world > 1 or args.partitioned:
        # strong scaling: the global config-2 system row-partitioned over the ranks
        from paper_2108_10591_b200.distributed import DistributedSystem

        dsys = DistributedSystem(rp, ci.astype(np.int32), v, n)
        dm = dsys.matrix
        n_loc = dsys.n_own
        ones = torch.ones(dsys.slab.n_ext, dtype=torch.float64, device="cuda")
    else:
        dsys = None
        dm = DeviceMatrix.from_csr((rp, ci.astype(np.int32), v), ctx=ctx)
        n_loc = n
        ones = torch.ones(n, dtype=torch.float64, device="cuda")
    b_dev = torch.empty(n_loc, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    dm.spmv_dev(ones.data_ptr(), b_dev.data_ptr())  # b = A*1 (this rank's rows)
    x_dev = torch.empty(n_loc, dtype=torch.float64, device="cuda")
    cfgpb = pb.SolverConfig(tol=1e-10, max_iters=2000)

    import ctypes as C

    def solve_dev(timing=False, graphs=True, method="pbicgsafe", max_iters=None):
        cfg = _lib.Config()
        mi = max_iters or cfgpb.max_iters
        cfg.tol, cfg.max_iters, cfg.rr_epoch, cfg.rr_cutoff = cfgpb.tol, mi, 100, -1
        cfg.record_history, cfg.reduce_mode, cfg.plan_workers = 1, _lib.REDUCE_TREE, 1
        cfg.use_graphs, cfg.timing = int(graphs), int(timing)
        res = _lib.Result()
        rel = np.empty(mi + 1)
        rc = _lib.load().pbs_solve_dev(dm.handle, _lib.METHOD_IDS[method], C.c_void_p(b_dev.data_ptr()), None,
                                       C.byref(cfg), C.c_void_p(x_dev.data_ptr()),
                                       rel.ctypes.data_as(C.c_void_p), None, None, C.byref(res))
        _lib.check(rc, ctx.handle)
        if method == "pbicgsafe":
            assert res.status == 0, f"solve did not converge: status {res.status}"
        return res

    # warm-up (graph capture, occupancy queries, clocks)
    for _ in range(max(args.warmup, 3)):
        solve_dev()
    # timed region: K solves, HBM-resident inputs, CUDA events on the solver stream
    sampler = ClockSampler(dev)
    sampler.start()
    time.sleep(0.3)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    total_it, total_ms, launches = 0, 0.0, 0
    results = []
    for _ in range(args.steps):
        res = solve_dev()
        total_it += res.iterations
        total_ms += res.device_ms
        launches += res.kernel_launches
        results.append(res)
    torch.cuda.synchronize()
    # per-kernel durations, same workload, event-bracketed launches
    tres = [solve_dev(timing=True) for _ in range(args.steps)]
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms = float(t.item())
    iters_per_s = total_it / (total_ms / 1e3)  # iterations of the one global solve

    # roofline of the dominant kernel.  Matrix bytes at SURVEY 8(d)'s 12 B per
    # nonzero (f64 value + int32 column) + row_ptr; the staged engine actually
    # streams 10 B (u16 window-local columns), so `traffic` can sit below it.
    peak, peak_src = peaks()
    part = dsys is not None
    # bytes per rank: the row slab this GPU owns (the whole system at N = 1)
    nr, nz = (n_loc, int(dm.nnz)) if part else (n, nnz)
    m_a = 12 * nz + 8 * (nr + 1)
    if part:
        # multi-GPU schedule (csrc/pbsafe.cu dist_iter): K1 As = A s alone so the
        # all-gather overlaps it, K2 the row-local update, K3 with all nine dots
        k12_bytes = m_a + 2 * 8 * nr   # s gather, As write
        k2_bytes = 20 * 8 * nr         # r p u s t y As l g w z x reads, p u w t z y x r writes
        k3_bytes = m_a + 12 * 8 * nr   # w gather, As l g s y r r0s t reads, l g s writes
        it_bytes_fused = 2 * m_a + 34 * 8 * nr
    else:
        k3_bytes = m_a + 11 * 8 * nr    # w gather, As l g s y r r0s reads, l g s writes (+ dots a c d g)
        k12_bytes = m_a + 21 * 8 * nr   # s gather, r p u t y l g w z x r0s reads, As p u w t z y x r writes (+ b e f h r)
        it_bytes_fused = 2 * m_a + 32 * 8 * nr  # this schedule: K1+K2 fused (As not re-read)
    it_bytes = 2 * m_a + 34 * 8 * nr  # SURVEY 8(d) three-phase minimum (K1, K2, K3)
    kms = {name: sum(r.kernel_ms[j] for r in tres) for j, name in enumerate(_lib.KERNEL_KINDS)}
    kcnt = {name: sum(r.kernel_count[j] for r in tres) for j, name in enumerate(_lib.KERNEL_KINDS)}
    k3_avg = kms["K3_Aw_epilogue"] / max(kcnt["K3_Aw_epilogue"], 1)
    k3_gbs = k3_bytes / (k3_avg * 1e-3) / 1e9
    k12_avg = kms["K1_As"] / max(kcnt["K1_As"], 1)
    k12_gbs = k12_bytes / (k12_avg * 1e-3) / 1e9
    k1_label = ("K1 (As = A s on the halo-exchanged s; the all-gather overlaps it)" if part else
                "K12 (As CSR SpMV + fused p u w t z y x r updates + dots b e f h r)")
    if kms["K1_As"] > kms["K3_Aw_epilogue"]:  # dominant kernel = larger share of the step
        dom = (k1_label, k12_bytes, k12_avg, k12_gbs, "K1_As")
    else:
        dom = ("K3 (Aw CSR SpMV + l,g,s updates + all nine dots; all-gather + finalize follow)" if part else
               "K3 (Aw CSR SpMV + l,g,s updates + dots a c d g + fused check)", k3_bytes, k3_avg, k3_gbs,
               "K3_Aw_epilogue")
    tim_ms = sum(r.device_ms for r in tres)
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "dram_bytes.json")  # from the committed ncu --set full capture
    if os.path.exists(tr_path) and not part:  # the capture is of the single-GPU fused kernels
        try:
            traffic = json.load(open(tr_path)).get(dom[4], {}).get("dram_bytes_per_launch")
        except Exception:
            traffic = None
    kernels = {}
    per_kind = [("K1_As", k12_bytes), ("K3_Aw_epilogue", k3_bytes)] + ([("K2_update", k2_bytes)] if part else [])
    for name, byt in per_kind:
        if kcnt[name]:
            avg = kms[name] / kcnt[name]
            kernels[name] = {"avg_us": avg * 1e3, "alg_bytes": byt, "GBps": byt / (avg * 1e-3) / 1e9,
                             "frac": byt / (avg * 1e-3) / 1e9 / peak, "share_of_step": kms[name] / tim_ms}
    kernels["K1_As"]["name"] = k1_label
    if kcnt["F_finalize"]:
        fin = kms["F_finalize"] / kcnt["F_finalize"]
        kernels["F_finalize"] = {"avg_us": fin * 1e3, "share_of_step": kms["F_finalize"] / tim_ms}

    # BASELINE config 2's comparison (outside the timed region): every method
    # of the drop-in on the same resident operator and right-hand side
    comparators = None
    if dsys is None:
        comparators = {}
        for mname in ("pbicgsafe", "ssbicgsafe2", "pbicgstab", "bicgstab", "gpbicg"):
            solve_dev(method=mname, max_iters=4000)  # warm (graph capture)
            rr_ = solve_dev(method=mname, max_iters=4000)
            comparators[mname] = {"status": {0: "converged", 1: "max_iters", 2: "breakdown",
                                             3: "non_finite"}[rr_.status],
                                  "iterations": int(rr_.iterations), "time_to_tol_ms": rr_.device_ms,
                                  "it_per_s": rr_.iterations / (rr_.device_ms * 1e-3)}
        comparators["note"] = ("one device solve each to 1e-10, CSR resident; pbicgstab is the pipelined "
                               "BiCGStab of Cools & Vanroose BASELINE names (not in the reference; restated in "
                               "oracle/pbsafe_oracle.c solve_pstab, parity unpinned against reference outputs); "
                               "bicgstab is the reference's two-reduction BiCGStab (solvers.py:210-327)")

    # e2e through the public API, pinned host buffers, upload + solve + readback per step
    e2e = None
    if dsys is not None:
        # public API of the partitioned path: solve(b_own) from pinned host
        # memory (the slab stays resident), x_own + history read back
        b_own = torch.from_numpy(b_dev.cpu().numpy()).pin_memory().numpy()
        dsys.solve(b_own, config=cfgpb)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        e_it = 0
        for _ in range(args.steps):
            out = dsys.solve(b_own, config=cfgpb)
            e_it += out.iterations
        if world > 1:
            torch.distributed.barrier()
        dt = time.perf_counter() - t0
        e2e = {"value": e_it / dt, "unit": "it/s", "h2d_bytes_per_step": int(b_own.nbytes),
               "d2h_bytes_per_step": int(8 * n_loc + out.iterations * 41),
               "ms_per_step": dt / args.steps * 1e3,
               "note": "wall clock around DistributedSystem.solve(b_own) on every rank; slab resident"}
    elif world == 1:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
        A_host = pb.CsrMatrix(n, n, pin(rp), pin(ci), pin(v))
        b_host = pin(b_dev.cpu().numpy())
        # warm-up steps: graphs, the workspace cache and the two page-locked
        # result blocks the loop alternates between (x of step k is alive
        # while step k+1 allocates its own)
        for _ in range(max(2, args.warmup)):
            out = pb.solve(A_host, b_host, config=cfgpb)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e_it = 0
        for _ in range(args.steps):
            out = pb.solve(A_host, b_host, config=cfgpb)
            e_it += out.iterations
        dt = time.perf_counter() - t0
        h2d = rp.nbytes + ci.nbytes + v.nbytes + b_host.nbytes
        d2h = 8 * n + out.iterations * (8 + 1 + 32)
        e2e = {"value": e_it / dt, "unit": "it/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": dt / args.steps * 1e3,
               "note": "wall clock around solve(CsrMatrix, b): CSR (int64 col_idx) + b H2D, "
                       "int64->int32 narrowing, solve, x + history D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline: rank 0 at N = 1 only
        threads = os.cpu_count() or 1
        b_host_np = b_dev.cpu().numpy()
        cpu = cpu_baseline(rp, ci, v, b_host_np, iters=args.cpu_iters, threads=threads)

    if rank == 0:
        avg_it = total_it / args.steps
        line = {
            "metric": METRIC, "value": iters_per_s, "unit": "it/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "operator": "csr", "iterations_per_solve": avg_it,
                       "time_to_tol_ms": total_ms / args.steps,
                       "parallelism": (f"row partition x{world} (NCCL halo + compensated all-gather)"
                                       if part else "single GPU"),
                       "l2": "inputs larger than L2: CSR 192 MB + 18 workspace vectors 302 MB per solve "
                             "vs 126 MB L2",
                       "graphs": True},
            "roofline": {"bound": "hbm", "achieved": dom[3], "peak": peak, "unit": "GB/s",
                         "frac": dom[3] / peak, "traffic": traffic, "kernel": dom[0],
                         "alg_bytes_per_launch": dom[1], "avg_launch_us": dom[2] * 1e3,
                         "peak_source": peak_src},
            "iteration_roofline": {"alg_bytes_per_iter": it_bytes,
                                   "achieved_GBps": it_bytes * iters_per_s / world / 1e9,
                                   "frac": it_bytes * iters_per_s / world / 1e9 / peak,
                                   "note": ("per rank: B_iter = 2*(12 nnz + 8(n+1)) + 34*8n over the rank's "
                                            "row slab (SURVEY 8(d)); the multi-GPU schedule moves exactly that"
                                            if part else
                                            "B_iter = 2*(12 nnz + 8(n+1)) + 34*8n (SURVEY 8(d)); this "
                                            "schedule moves 2*(12 nnz+8(n+1)) + 32*8n (K1+K2 fused)"),
                                   "frac_own_schedule": it_bytes_fused * iters_per_s / world / 1e9 / peak},
            "kernels": kernels,
            "comparators": comparators,
            "timing_mode_it_per_s": sum(r.iterations for r in tres) / (tim_ms / 1e3),
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks,
        }
        emit(line)
    if dsys is not None:
        dsys.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


_JSON_OUT = None


def emit(line):
    """The one JSON line, on the process's original stdout.  Everything else
    native code prints (NCCL's version banner under NCCL_DEBUG, driver
    messages) goes to stderr, so stdout carries exactly one line."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)  # fd 1 -> stderr for native libraries and stray prints
    sys.stdout = sys.stderr
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--cpu-iters", type=int, default=600)  # ~10 s on a 16-core host
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--partitioned", action="store_true", help="use the multi-GPU schedule even at N=1")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
