"""Multi-GPU schedule on the device, at world size 1 (this pool gives one GPU).

The partitioned path (halo exchange + compensated all-gather of the dot batch
on a separate stream + 1-CTA finalize) runs with NCCL communicators of one
rank: the schedule, the extended-space layout and the cross-stream ordering
are exercised; the history must equal the single-GPU fast path's (both
reduce the batch in compensated arithmetic) and the oracle's near-exact run.
"""

import os

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("method", ["pbicgsafe", "pbicgsafe-rr"])
def test_partitioned_world1_matches_single_gpu(method):
    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.distributed import DistributedSystem

    st = problems.convdiff_stencil(3, 32, (1.0, 0.5, 0.25))
    rp, ci, v = problems.stencil_csr(st)
    n = len(rp) - 1
    b = orc.spmv(rp, ci, v, np.ones(n))
    cfg = pb.SolverConfig(tol=1e-10, max_iters=2000, rr_epoch=20)
    ref = pb.solve(pb.CsrMatrix(n, n, rp, ci, v), b, method=method, config=cfg)
    sysd = DistributedSystem(rp, ci, v, n)
    try:
        out = sysd.solve(b, method=method, config=cfg)
    finally:
        sysd.close()
    assert out.status == ref.status
    assert abs(out.iterations - ref.iterations) <= 1
    m = min(len(out.history), len(ref.history), 40)
    np.testing.assert_allclose([r.rel_res_recur for r in out.history[:m]],
                               [r.rel_res_recur for r in ref.history[:m]], rtol=1e-12)
    true = np.linalg.norm(b - orc.spmv(rp, ci, v, out.x)) / out.r0_norm
    assert true <= 1e-8


def test_partitioned_nonfinite_raises():
    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.distributed import DistributedSystem

    rp, ci, v = problems.stencil_csr(problems.convdiff_stencil(2, 16, (1.0, 1.0)))
    v = v.copy()
    v[5] = np.inf
    n = len(rp) - 1
    sysd = DistributedSystem(rp, ci, v, n)
    try:
        with pytest.raises(pb.NonFiniteVectorError):
            sysd.solve(np.ones(n))
    finally:
        sysd.close()


def test_overlap_evidence_in_reference_event_format():
    """the schedule as the reference's EventLog, plus real overlap.

    Per iteration >= 1 the reference's verifier requires exactly one
    reduce_start and reduce_start before the end of the As product
    (reduction.py:486-563, test_acceptance.py:248-288).  CUDA-event times
    also show the all-gather + check interval intersecting the As interval.
    """
    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.distributed import DistributedSystem
    from paper_2108_10591_b200.reduction import REDUCE_START, SPMV_END, events_to_log, overlap_report

    st = problems.convdiff_stencil(3, 96, (1.0, 0.5, 0.25))
    rp, ci, v = problems.stencil_csr(st)
    n = len(rp) - 1
    b = orc.spmv(rp, ci, v, np.ones(n))
    sysd = DistributedSystem(rp, ci, v, n)
    try:
        out = sysd.solve(b, config=pb.SolverConfig(tol=1e-30, max_iters=40),
                         engine=pb.DeviceEngine(evidence=True))
    finally:
        sysd.close()
    recs = out.device["events"]
    log = events_to_log(recs)
    by_iter = {}
    for ev in log.events():
        by_iter.setdefault(ev.iter, []).append(ev)
    checked = 0
    for it, evs in sorted(by_iter.items()):
        starts = [e.seq for e in evs if e.kind == REDUCE_START]
        as_end = [e.seq for e in evs if e.kind == SPMV_END and e.tag == "As"]
        if not as_end:
            continue  # the final check has no As product
        assert len(starts) == 1, (it, starts)
        assert starts[0] < as_end[0], it
        checked += 1
    assert checked >= 39
    rep = overlap_report(recs)
    frac = sum(r["overlapped"] for r in rep.values()) / max(len(rep), 1)
    assert frac >= 0.5, rep


@pytest.mark.parametrize("method", ["pbicgsafe", "pbicgsafe-rr"])
def test_partitioned_split_schedule_world1(method, monkeypatch):
    """The interior/boundary split (halo exchange on its own stream while the
    interior rows of As and Aw compute, boundary rows after it lands; the
    K3 pieces' dot records stored one after another) exercised on one GPU by
    forcing 4 boundary blocks at each end of the slab: the history must equal
    the unsplit single-GPU fast path's."""
    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import problems
    from paper_2108_10591_b200.distributed import DistributedSystem

    monkeypatch.setenv("PBS_SPLIT_TEST", "4")
    st = problems.convdiff_stencil(3, 32, (1.0, 0.5, 0.25))
    rp, ci, v = problems.stencil_csr(st)
    n = len(rp) - 1
    b = orc.spmv(rp, ci, v, np.ones(n))
    cfg = pb.SolverConfig(tol=1e-10, max_iters=2000, rr_epoch=20)
    ref = pb.solve(pb.CsrMatrix(n, n, rp, ci, v), b, method=method, config=cfg)
    sysd = DistributedSystem(rp, ci, v, n)
    try:
        out = sysd.solve(b, method=method, config=cfg)
    finally:
        sysd.close()
    assert out.status == ref.status
    assert abs(out.iterations - ref.iterations) <= 1
    m = min(len(out.history), len(ref.history), 40)
    np.testing.assert_allclose([r.rel_res_recur for r in out.history[:m]],
                               [r.rel_res_recur for r in ref.history[:m]], rtol=1e-12)
    true = np.linalg.norm(b - orc.spmv(rp, ci, v, out.x)) / out.r0_norm
    assert true <= 1e-8
