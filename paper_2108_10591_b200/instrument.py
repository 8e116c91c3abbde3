"""Operation counters of a device solve (drop-in subset of pipesafe.instrument).

The reference ticks ``OpCounters`` inside its loop (instrument.py:49-87,
solvers.py:613-733).  The device loop has no host in it, so the counters are
synthesised afterwards from what the device reports (iterations, stop check,
replacement schedule) with the reference's per-update tallies; the snapshot
sequence is the one the reference would have produced, so
``per_iteration_costs`` (instrument.py:118-171) applies unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field

# (#Ax, #dots, #reductions) a steady-state iteration must cost (instrument.py:28-32)
EXPECTED_PER_ITERATION = {
    "bicgstab": (2, 5, 2),
    "ssbicgsafe2": (2, 9, 1),
    "pbicgsafe": (2, 9, 1),
}
EXPECTED_WORKSPACE = {"bicgstab": 7, "ssbicgsafe2": 10, "pbicgsafe": 15, "pbicgsafe-rr": 15}

# per-update (scalar mults, vector adds) exactly as the reference tallies them
_PIPE_STEADY = (21, 22)   # solvers.py:679-724
_PIPE_REPLACE = (12, 13)  # solvers.py:679-706 with the replacement branch
_SS_ITER = (13, 14)       # solvers.py:563-580


class CounterAssertionError(AssertionError):
    """A steady-state per-iteration cost deviated from the cost model."""


@dataclass
class OpCounters:
    n_spmv: int = 0
    n_dots: int = 0
    n_reductions: int = 0
    n_scalar_mults: int = 0
    n_vec_adds: int = 0
    n_monitor_spmv: int = 0
    n_workspace_vectors: int = 0
    snapshots: list[tuple[int, int, int, int, int]] = field(default_factory=list)

    def spmv(self, k: int = 1) -> None:
        self.n_spmv += k

    def batch(self, n_dots: int) -> None:
        self.n_dots += n_dots
        self.n_reductions += 1

    def updates(self, mults: int, adds: int) -> None:
        self.n_scalar_mults += mults
        self.n_vec_adds += adds

    def snapshot(self) -> None:
        self.snapshots.append(
            (self.n_spmv, self.n_dots, self.n_reductions, self.n_scalar_mults, self.n_vec_adds)
        )

    def as_dict(self) -> dict:
        return {
            "n_spmv": self.n_spmv, "n_dots": self.n_dots, "n_reductions": self.n_reductions,
            "n_scalar_mults": self.n_scalar_mults, "n_vec_adds": self.n_vec_adds,
            "n_monitor_spmv": self.n_monitor_spmv, "n_workspace_vectors": self.n_workspace_vectors,
        }


# The product-type comparators tick in stages (solvers.py:239-317, 360-450);
# each stage is (spmv, dots-in-batch or 0, (mults, adds) updates...).  A
# stopping iteration runs the stages up to its stop stage (the device reports
# it: 1 alpha, 2 omega/zeta, 3 after the x/r update, 4 complete).
_PROD_STAGES = {
    "bicgstab": [
        [(0, 0, (2, 2)), (1, 1, None)],                      # p, Ap, (r0*, Ap)
        [(0, 0, (1, 1)), (1, 4, None)],                      # t, At, b e c d
        [(0, 0, (2, 2)), (0, 0, (1, 1))],                    # x, r
        [],                                                  # beta, record
    ],
    "gpbicg": [
        [(0, 0, (1, 2)), (1, 1, None)],                      # p, Ap, (r0*, Ap)
        [(0, 0, (2, 3)), (0, 0, (1, 2)), (0, 0, (1, 1)), (1, 5, None)],  # y u t, At, a..e
        [(0, 0, (2, 1)), (0, 0, (3, 2)), (0, 0, (1, 2)), (0, 0, (2, 2)), (0, 2, None)],  # u z x r, f rr
        [(0, 0, (1, 1))],                                    # w
    ],
    # p-BiCGStab (oracle solve_pstab; not in the reference): stage 1 alpha
    # (scalar), 2 omega, 3 after the x/r/w update, 4 complete
    "pbicgstab": [
        [],                                                  # alpha
        [(1, 0, None), (0, 0, (2, 2)), (0, 0, (2, 2)), (0, 0, (2, 2)), (0, 0, (1, 1)),
         (0, 0, (1, 1)), (0, 3, None), (1, 0, None)],        # t, p s z q y, b e d, v
        [(0, 0, (2, 2)), (0, 0, (1, 1)), (0, 0, (2, 2)), (0, 5, None)],  # x r w, f rr g sd zd
        [],                                                  # beta, record
    ],
}
_PROD_WORKSPACE = {"bicgstab": 7, "gpbicg": 11, "pbicgstab": 11}


def _prod_tick(c: OpCounters, method: str, stages: int) -> None:
    for stage in _PROD_STAGES[method][:stages]:
        for spmv_n, dots, upd in stage:
            if spmv_n:
                c.spmv(spmv_n)
            if dots:
                c.batch(dots)
            if upd:
                c.updates(*upd)


def synthesize(method: str, iterations: int, stopped_in_loop: bool, replaced_at,
               stop_stage: int = 0) -> OpCounters:
    """Counters the reference loop would have ticked for this outcome.

    ``iterations`` completed iterations; ``stopped_in_loop`` when a loop check
    (not the post-loop final record) ended the solve, in which case that
    iteration's batch and spine SpMV were still counted; ``replaced_at`` the
    set of completed iterations that ran residual replacement.
    """
    if method in _PROD_STAGES:
        c = OpCounters(n_workspace_vectors=_PROD_WORKSPACE[method])
        c.spmv()
        c.updates(0, 1)
        if method == "pbicgstab":  # w0 = A r0, then rr and (r0*, w0)
            c.spmv()
            c.batch(2)
        else:
            c.batch(1)
        c.snapshot()
        for _ in range(iterations):
            _prod_tick(c, method, 4)
            c.snapshot()
        if stopped_in_loop and stop_stage:
            _prod_tick(c, method, stop_stage)
        return c
    pipelined = method != "ssbicgsafe2"
    c = OpCounters(n_workspace_vectors=16 if pipelined else 11)
    c.spmv(2 if pipelined else 1)
    c.updates(0, 1)
    c.snapshot()
    # the same ticks as the reference loop, kept in locals: a snapshot per
    # iteration is what per_iteration_costs reads (this runs once per solve on
    # the host, 0.6 ms for 340 iterations when written with the tick methods)
    sp, dots, red, mul, add = c.n_spmv, c.n_dots, c.n_reductions, c.n_scalar_mults, c.n_vec_adds
    steady = _PIPE_STEADY if pipelined else _SS_ITER
    snaps = c.snapshots
    for i in range(iterations):
        dots += 5 if i == 0 else 9
        red += 1
        if pipelined and i in replaced_at:
            sp += 7
            mul += _PIPE_REPLACE[0]
            add += _PIPE_REPLACE[1]
        else:
            sp += 2
            mul += steady[0]
            add += steady[1]
        snaps.append((sp, dots, red, mul, add))
    c.n_spmv, c.n_dots, c.n_reductions, c.n_scalar_mults, c.n_vec_adds = sp, dots, red, mul, add
    if stopped_in_loop:
        c.batch(5 if iterations == 0 else 9)
        c.spmv()
    return c


@dataclass
class CostRow:
    method: str
    ax_per_iter: int
    dots_per_iter: int
    reductions_per_iter: int
    scalar_mults_per_iter: int
    vec_adds_per_iter: int
    workspace_vectors: int
    tabulated_workspace_vectors: int | None
    steady_iterations: int

    def as_dict(self) -> dict:
        return dict(self.__dict__)


def per_iteration_costs(counters: OpCounters, method: str) -> CostRow:
    """Steady-state per-iteration costs from snapshots (instrument.py:118-171)."""
    snaps = counters.snapshots
    if len(snaps) < 4:
        raise ValueError("need at least three completed iterations to measure steady state")
    deltas = [tuple(b[k] - a[k] for k in range(5)) for a, b in zip(snaps, snaps[1:])]
    steady = deltas[1:]
    if method in EXPECTED_PER_ITERATION:
        if any(d != steady[0] for d in steady):
            raise CounterAssertionError(f"{method}: steady-state deltas not constant: {sorted(set(steady))}")
        row = steady[0]
        for k, name in enumerate(("n_spmv", "n_dots", "n_reductions")):
            if row[k] != EXPECTED_PER_ITERATION[method][k]:
                raise CounterAssertionError(
                    f"{method}: {name} per iteration = {row[k]}, cost model says "
                    f"{EXPECTED_PER_ITERATION[method][k]}")
        rep, count = row, len(steady)
    else:
        tally: dict[tuple, int] = {}
        for d in steady:
            tally[d] = tally.get(d, 0) + 1
        rep = max(tally, key=tally.get)
        count = tally[rep]
    return CostRow(method, rep[0], rep[1], rep[2], rep[3], rep[4], counters.n_workspace_vectors,
                   EXPECTED_WORKSPACE.get(method), count)
