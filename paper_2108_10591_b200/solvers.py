"""Drop-in solver entry points (pipesafe.solvers) running on the B200.

Same names, arguments, validation and return types as the reference
(solvers.py:44-114, 133-145, 742-803): ``solve(A, b, method, x0, config,
engine, trace_hook) -> SolveOutcome``.  The whole iteration loop runs on the
device (libpbsafe.so): SpMVs, fused updates, the packed 9-dot batch, the
coefficient step, convergence/breakdown checks and the history all stay in
HBM; the host sees the outcome once.  There is no CPU path: without the
library or a B200 these functions raise.

``engine`` accepts a :class:`DeviceEngine`, or a reference-style engine
exposing ``.plan`` (a balanced PartitionPlan), in which case the dot batch
follows that plan's chains and combine order and the solve is bitwise equal
to the reference driven by the same engine (small systems; it is a parity
mode, one thread per range).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .coefficients import BREAKDOWN_QUANTITIES, CoefficientSet
from .instrument import OpCounters, synthesize
from .linalg import CsrMatrix, NonFiniteVectorError, check_finite
from .operators import DeviceMatrix
from .reduction import PartitionPlan


class SolveStatus(Enum):
    CONVERGED = "converged"
    MAX_ITERS = "max_iters"
    BREAKDOWN = "breakdown"
    NON_FINITE = "non_finite"


_STATUS = {0: SolveStatus.CONVERGED, 1: SolveStatus.MAX_ITERS, 2: SolveStatus.BREAKDOWN,
           3: SolveStatus.NON_FINITE}


@dataclass
class SolverConfig:
    """Knobs shared by every method (solvers.py:51-78)."""

    tol: float = 1e-8
    max_iters: int = 10_000
    rr_epoch: int = 100
    rr_cutoff: int | None = None
    record_history: bool = True
    monitor_every: int = 0
    deterministic: bool = True

    def __post_init__(self):
        if not self.tol > 0.0:
            raise ValueError("tol must be positive")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")
        if self.rr_epoch < 1:
            raise ValueError("rr_epoch must be >= 1")
        if self.rr_cutoff is not None and not 0 <= self.rr_cutoff <= self.max_iters:
            raise ValueError("rr_cutoff must lie in [0, max_iters]")
        if self.monitor_every < 0:
            raise ValueError("monitor_every must be >= 0")


@dataclass
class IterationRecord:
    """State at the convergence check of one iteration (solvers.py:81-95)."""

    iter: int
    rel_res_recur: float
    rel_res_true: float | None = None
    replaced: bool = False
    coefficients: CoefficientSet | None = None


@dataclass
class SolveOutcome:
    """solvers.py:98-114, plus ``device``: timings/launch counts of the device run."""

    status: SolveStatus
    iterations: int
    x: np.ndarray
    history: list[IterationRecord]
    counters: OpCounters
    r0_norm: float
    final_rel_res_recur: float
    best_rel_res_recur: float
    breakdown_quantity: str | None = None
    failure_iter: int | None = None
    drift: list = field(default_factory=list)
    device: dict = field(default_factory=dict)

    @property
    def converged(self) -> bool:
        return self.status is SolveStatus.CONVERGED


def write_history_csv(path: str, history: list[IterationRecord]) -> None:
    """``iter,rel_res_recur,rel_res_true,replaced`` rows, %.17g (solvers.py:117-130)."""
    with open(path, "w", encoding="ascii") as fh:
        fh.write("iter,rel_res_recur,rel_res_true,replaced\n")
        for rec in history:
            true_s = "" if rec.rel_res_true is None else format(rec.rel_res_true, ".17g")
            fh.write(f"{rec.iter},{format(rec.rel_res_recur, '.17g')},{true_s},{int(rec.replaced)}\n")


@dataclass
class DeviceEngine:
    """Where and how a solve runs (stands in for the reference's ReductionEngine).

    reduce="tree": fixed-shape block-tree dot batch (deterministic, full speed).
    reduce="plan": the reference's PartitionPlan.balanced(n, workers) chains
    with a left-to-right combine — bitwise the reference's results.
    """

    device: int | None = None
    reduce: str = "tree"
    workers: int = 1
    use_graphs: bool = True
    timing: bool = False
    # return x in page-locked host memory (torch's caching host allocator): the
    # device->host copy runs at DMA speed with no page faults (~2.5 ms less per
    # config-2 solve), but every x the caller keeps pins its block and torch's
    # CUDA state is touched; off: a plain pageable ndarray
    pinned_result: bool = False
    evidence: bool = False  # multi-GPU schedule: device-clock stamps of every product and reduction

    def __post_init__(self):
        if self.reduce not in ("tree", "plan"):
            raise ValueError(f"unknown reduce mode {self.reduce!r}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


def _engine_params(engine, n: int) -> DeviceEngine:
    if engine is None:
        return DeviceEngine()
    if isinstance(engine, DeviceEngine):
        return engine
    plan = getattr(engine, "plan", None)
    if plan is not None and hasattr(plan, "ranges"):
        mine = PartitionPlan(plan.n, tuple(tuple(r) for r in plan.ranges))
        if mine.n != n:
            raise ValueError(f"plan covers {mine.n} rows, system has {n}")
        if not mine.is_balanced():
            raise ValueError("only PartitionPlan.balanced plans are supported on the device")
        return DeviceEngine(reduce="plan", workers=mine.worker_count)
    raise TypeError(f"unsupported engine {type(engine).__name__}")


def _prepare(A, b, x0):
    """solvers.py:133-145: shape/finite validation, x0 copied."""
    if A.n_rows != A.n_cols:
        raise ValueError(f"solver needs a square operator, got {A.shape}")
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (A.n_rows,):
        raise ValueError(f"rhs has shape {b.shape}, matrix is {A.shape}")
    check_finite(b, "right-hand side")
    if x0 is None:
        return np.ascontiguousarray(b), None
    x = np.array(x0, dtype=np.float64)
    if x.shape != (A.n_rows,):
        raise ValueError(f"x0 has shape {x.shape}, matrix is {A.shape}")
    check_finite(x, "initial guess")
    return np.ascontiguousarray(b), np.ascontiguousarray(x)


_TRACE_NAMES = ("x", "r", "p", "u", "o", "t", "w", "y", "z", "s", "q", "g", "l")
# the reference's trace_hook dicts of the product-type methods (solvers.py:315, 448)
_TRACE_NAMES_BY_METHOD = {"bicgstab": ("x", "r", "p", "t", "Ap", "At"),
                          "gpbicg": ("x", "r", "p", "u", "t", "w", "y", "z"),
                          "pbicgstab": ("x", "r", "p", "s", "z", "q", "y", "w", "t", "v")}


def _host_result(n, pinned: bool = False):
    """The returned x.  pinned (DeviceEngine(pinned_result=True)): page-locked
    host memory from torch's caching host allocator (reused once the caller
    drops an earlier result), so the device->host copy runs at DMA speed with
    no page faults; the array keeps its block alive and the caller owns it
    like any other ndarray.  Otherwise a plain pageable array."""
    if pinned:
        try:
            import torch

            if torch.cuda.is_available():
                return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        except Exception:  # pragma: no cover - pinned memory unavailable
            pass
    return np.empty(n)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _make_config(config: SolverConfig, eng: DeviceEngine, nparts: int = 1):
    """pbs_config for a solve (+ the host buffers its evidence outputs land in)."""
    cfg = _lib.Config()
    cfg.tol = config.tol
    cfg.max_iters = config.max_iters
    cfg.rr_epoch = config.rr_epoch
    cfg.rr_cutoff = -1 if config.rr_cutoff is None else config.rr_cutoff
    cfg.record_history = 1 if config.record_history else 0
    cfg.reduce_mode = _lib.REDUCE_PLAN if eng.reduce == "plan" else _lib.REDUCE_TREE
    cfg.plan_workers = eng.workers
    cfg.use_graphs = 1 if eng.use_graphs else 0
    cfg.timing = 1 if eng.timing else 0
    keep = {}
    if eng.evidence:
        # multi-GPU schedule: %globaltimer stamps per partition and iteration
        cap = config.max_iters + 2
        keep["stamps"] = np.full((nparts, cap, len(_lib.STAMP_WORDS)), -1.0)
        keep["stamps_count"] = C.c_int64(0)
        cfg.stamps_out = keep["stamps"].ctypes.data_as(C.c_void_p)
        cfg.stamps_cap = cap
        cfg.stamps_count = C.pointer(keep["stamps_count"])
    return cfg, keep


def _history_buffers(config: SolverConfig):
    slots = config.max_iters + 1
    return np.empty(slots), np.zeros(slots, dtype=np.uint8), np.empty((slots, 4))


def _raise_for(rc, res, ctx_handle):
    if rc == _lib.PBS_ERR_NONFINITE:
        tag = _lib.SPMV_TAGS.get(res.nonfinite_tag, "?")
        idx = int(res.nonfinite_index)
        raise NonFiniteVectorError(f"matvec {tag!r} output row has non-finite entry at index {idx}", idx)
    if rc == _lib.PBS_ERR_INVALID:
        raise ValueError(_lib.last_error(ctx_handle))
    _lib.check(rc, ctx_handle)


def _build_outcome(method, config, eng, res, x, rel, flags, coef, keep) -> SolveOutcome:
    k = int(res.n_records)
    history = []
    # plain Python floats / ints once (tolist), not a numpy scalar per field
    rel_l, flag_l, coef_l = rel[:k].tolist(), flags[:k].tolist(), coef[:k].tolist()
    omega_form = method in ("bicgstab", "pbicgstab")  # CoefficientSet(alpha, beta, omega) (solvers.py:309)
    for i in range(k):
        f = flag_l[i]
        cs = None
        if f & _lib.HIST_HAS_COEF:
            a, b_, z, e = coef_l[i]
            cs = CoefficientSet(a, b_, None, None, z) if omega_form else CoefficientSet(a, b_, z, e)
        history.append(IterationRecord(i, rel_l[i], None, bool(f & _lib.HIST_REPLACED), cs))
    status = _STATUS[res.status]
    iterations = int(res.iterations)
    stopped_in_loop = iterations < config.max_iters  # a loop check ended it
    replaced_at = set()
    if method == "pbicgsafe-rr":
        cutoff = config.rr_cutoff if config.rr_cutoff is not None else config.max_iters
        replaced_at = {i for i in range(1, iterations) if i % config.rr_epoch == 0 and i < cutoff}
    counters = synthesize(method, iterations, stopped_in_loop, replaced_at, stop_stage=int(res.stop_stage))
    best = min((r.rel_res_recur for r in history), default=math.inf)
    final = history[-1].rel_res_recur if history else math.inf
    device = {
        "device_ms": float(res.device_ms),
        "kernel_launches": int(res.kernel_launches),
        "n_spmv": int(res.n_spmv),
        "kernel_ms": {name: float(res.kernel_ms[j]) for j, name in enumerate(_lib.KERNEL_KINDS)},
        "kernel_count": {name: int(res.kernel_count[j]) for j, name in enumerate(_lib.KERNEL_KINDS)},
        "reduce": eng.reduce,
    }
    if "stamps" in keep:
        # as many iterations as the solve ran (+ the final check)
        device["stamps"] = keep["stamps"][:, : int(res.n_records) + 1].copy()
    return SolveOutcome(
        status=status,
        iterations=iterations,
        x=x,
        history=history,
        counters=counters,
        r0_norm=float(res.r0_norm),
        final_rel_res_recur=final,
        best_rel_res_recur=best,
        breakdown_quantity=BREAKDOWN_QUANTITIES.get(int(res.breakdown)) if status is SolveStatus.BREAKDOWN else None,
        failure_iter=None if res.failure_iter < 0 else int(res.failure_iter),
        device=device,
    )


def _solve_device(A, b, method, x0, config, engine, trace_hook) -> SolveOutcome:
    config = config or SolverConfig()
    b, x0 = _prepare(A, b, x0)
    n = A.n_rows
    if config.monitor_every > 0:
        raise NotImplementedError("monitor_every (DriftMonitor) is not available on the device path")
    eng = _engine_params(engine, n)
    own = not isinstance(A, DeviceMatrix)
    dm = DeviceMatrix.from_csr(A, device=eng.device) if own else A
    try:
        cfg, keep = _make_config(config, eng)
        cb_keep = None
        if trace_hook is not None:
            names = _TRACE_NAMES_BY_METHOD.get(method, _TRACE_NAMES)

            def _cb(i, vecs, _user):
                ws = {name: np.ctypeslib.as_array(vecs[k], shape=(n,))
                      for k, name in enumerate(names)}
                trace_hook(int(i), ws)
            cb_keep = _lib.TRACE_FN(_cb)
            cfg.trace_fn = cb_keep
        x = _host_result(n, eng.pinned_result)
        rel, flags, coef = _history_buffers(config)
        res = _lib.Result()
        rc = _lib.load().pbs_solve(dm.handle, _lib.METHOD_IDS[method], _ptr(b), _ptr(x0), C.byref(cfg),
                                   _ptr(x), _ptr(rel), _ptr(flags), _ptr(coef), C.byref(res))
    finally:
        if own:
            dm.free()
    _raise_for(rc, res, dm.ctx.handle)
    return _build_outcome(method, config, eng, res, x, rel, flags, coef, keep)


def solve_group(mats, b_ptrs, x_ptrs, method="pbicgsafe", x0_ptrs=None, config=None, engine=None) -> SolveOutcome:
    """A solve on a loopback group (include/pbsafe.h pbs_solve_group): mats are
    the partitions' DeviceMatrix objects, b_ptrs / x_ptrs / x0_ptrs device
    pointers to their own segments.  The outcome's x is None (the caller owns
    the segments)."""
    config = config or SolverConfig()
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}; choose from {sorted(METHODS)}")
    eng = engine if isinstance(engine, DeviceEngine) else DeviceEngine()
    n = len(mats)
    cfg, keep = _make_config(config, eng, nparts=n)
    rel, flags, coef = _history_buffers(config)
    res = _lib.Result()
    P = C.c_void_p * n
    hm = P(*[m.handle for m in mats])
    hb = P(*b_ptrs)
    hx = P(*x_ptrs)
    h0 = P(*x0_ptrs) if x0_ptrs is not None else None
    rc = _lib.load().pbs_solve_group(hm, n, _lib.METHOD_IDS[method], hb, h0, C.byref(cfg), hx, _ptr(rel),
                                     _ptr(flags), _ptr(coef), C.byref(res))
    _raise_for(rc, res, mats[0].ctx.handle)
    return _build_outcome(method, config, eng, res, None, rel, flags, coef, keep)


def solve_pbicgsafe(A, b, x0=None, config=None, engine=None, trace_hook=None) -> SolveOutcome:
    """Pipelined single-reduction solver (solvers.py:742-758) on the device."""
    return _solve_device(A, b, "pbicgsafe", x0, config, engine, trace_hook)


def solve_pbicgsafe_rr(A, b, x0=None, config=None, engine=None, trace_hook=None) -> SolveOutcome:
    """Pipelined solver with scheduled residual replacement (solvers.py:761-779)."""
    return _solve_device(A, b, "pbicgsafe-rr", x0, config, engine, trace_hook)


def solve_ssbicgsafe2(A, b, x0=None, config=None, engine=None, trace_hook=None) -> SolveOutcome:
    """Single-reduction comparator, batch after s = A r (solvers.py:485-592)."""
    return _solve_device(A, b, "ssbicgsafe2", x0, config, engine, trace_hook)


def solve_bicgstab(A, b, x0=None, config=None, engine=None, trace_hook=None) -> SolveOutcome:
    """Stabilized bi-conjugate gradients, two reduction phases per iteration
    (solvers.py:210-327) on the device: BASELINE config 2's BiCGStab comparator."""
    return _solve_device(A, b, "bicgstab", x0, config, engine, trace_hook)


def solve_gpbicg(A, b, x0=None, config=None, engine=None, trace_hook=None) -> SolveOutcome:
    """Generalized product-type solver, three reduction phases per iteration
    (solvers.py:330-460) on the device."""
    return _solve_device(A, b, "gpbicg", x0, config, engine, trace_hook)


def solve_pbicgstab(A, b, x0=None, config=None, engine=None, trace_hook=None) -> SolveOutcome:
    """Pipelined BiCGStab (Cools & Vanroose), the paper's p-BiCGStab comparator
     on the device.  The reference does not ship it
    (SPEC.md:13); this follows the restatement in oracle/pbsafe_oracle.c
    (solve_pstab) with the reference BiCGStab's conventions
    (solvers.py:210-327): same shadow residual, check order, guards and
    (alpha, beta, omega) records.  Two reduction phases per iteration, each
    overlappable with an independent SpMV (t = A w, v = A z)."""
    return _solve_device(A, b, "pbicgstab", x0, config, engine, trace_hook)


METHODS = {
    "bicgstab": solve_bicgstab,
    "pbicgstab": solve_pbicgstab,
    "gpbicg": solve_gpbicg,
    "ssbicgsafe2": solve_ssbicgsafe2,
    "pbicgsafe": solve_pbicgsafe,
    "pbicgsafe-rr": solve_pbicgsafe_rr,
}


def solve(A, b, method: str = "pbicgsafe", x0=None, config=None, engine=None, trace_hook=None) -> SolveOutcome:
    """Dispatch by name (solvers.py:791-803)."""
    if method not in METHODS:
        raise ValueError(f"unknown method {method!r}; choose from {sorted(METHODS)}")
    return METHODS[method](A, b, x0=x0, config=config, engine=engine, trace_hook=trace_hook)
