"""Row-partitioned multi-GPU layout: slabs, remapped local CSR, halo plan.

The reference's only parallelism is a row partition: ``PartitionPlan``
contiguous ranges (reduction.py:55-87), partial dots per range combined in
range order (reduction.py:282-294) and row-range SpMV (linalg.py:164-172).
On B200 each range is a rank (one process per GPU):

* rank r owns rows ``[lo, hi)`` of ``PartitionPlan.balanced(n, N)`` (for the
  grid configs: whole axis-0 planes);
* its local CSR keeps its rows with columns remapped into an *extended* local
  index space ``[left halo | own | right halo]``: the left halo is the
  contiguous column range ``[cmin, lo)`` and the right halo ``[hi, cmax]``
  of the columns its rows touch outside its own range (exact for banded /
  stencil matrices, a superset otherwise);
* every SpMV input vector is held in that extended space; before an SpMV the
  halo is filled from the owners — the transfer list is the ``HaloPlan``
  (identical on every rank, derived from all ranks' halo widths);
* the per-iteration dot batch reduces to 9 compensated pairs per rank; ranks
  all-gather them and combine in rank order, so every rank computes the
  identical coefficients and stops at the identical check.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .reduction import PartitionPlan


@dataclass(frozen=True)
class Slab:
    rank: int
    nranks: int
    n: int       # global rows
    lo: int      # first owned row
    hi: int      # one past the last owned row
    hl: int      # left halo length  (columns [lo-hl, lo))
    hr: int      # right halo length (columns [hi, hi+hr))

    @property
    def pad(self) -> int:
        # one dummy element in front when hl is odd, so the own segment starts
        # at an even extended index (16-byte aligned for the bulk copies)
        return self.hl & 1

    @property
    def own_off(self) -> int:
        return self.pad + self.hl

    @property
    def n_own(self) -> int:
        return self.hi - self.lo

    @property
    def n_ext(self) -> int:
        return self.pad + self.hl + self.n_own + self.hr

    def to_ext(self, global_cols: np.ndarray) -> np.ndarray:
        """Global column -> extended local index."""
        return global_cols - (self.lo - self.hl) + self.pad


@dataclass
class HaloPlan:
    """Transfers that fill every rank's halo from the owners.

    sends[r] / recvs[r]: lists of (peer, offset, length); send offsets are
    relative to the sender's OWN segment, recv offsets are extended-space
    indices on the receiver.
    """

    sends: dict[int, list[tuple[int, int, int]]] = field(default_factory=dict)
    recvs: dict[int, list[tuple[int, int, int]]] = field(default_factory=dict)


def slab_bounds(n: int, nranks: int) -> list[tuple[int, int]]:
    plan = PartitionPlan.balanced(n, nranks)
    if plan.worker_count != nranks:
        raise ValueError(f"cannot split {n} rows over {nranks} ranks")
    return list(plan.ranges)


def local_csr(row_ptr, col_idx, values, n: int, rank: int, nranks: int):
    """Rows of ``rank``'s slab with columns remapped to the extended space.

    Returns (Slab, local_row_ptr int64, local_col_idx int32, local_values).
    """
    lo, hi = slab_bounds(n, nranks)[rank]
    rp = np.asarray(row_ptr, dtype=np.int64)
    s, e = int(rp[lo]), int(rp[hi])
    cols = np.asarray(col_idx[s:e], dtype=np.int64)
    vals = np.ascontiguousarray(values[s:e], dtype=np.float64)
    cmin = int(cols.min()) if cols.size else lo
    cmax = int(cols.max()) if cols.size else hi - 1
    hl = max(0, lo - cmin)
    hr = max(0, cmax + 1 - hi)
    slab = Slab(rank, nranks, n, lo, hi, hl, hr)
    lrp = rp[lo:hi + 1] - s
    lci = slab.to_ext(cols).astype(np.int32)
    return slab, lrp, lci, vals


def halo_plan(slabs: list[Slab]) -> HaloPlan:
    """Owner-to-halo transfers for every rank (pure function of all slabs)."""
    plan = HaloPlan({s.rank: [] for s in slabs}, {s.rank: [] for s in slabs})
    for dst in slabs:
        for g0, g1, base in ((dst.lo - dst.hl, dst.lo, dst.pad), (dst.hi, dst.hi + dst.hr, dst.own_off + dst.n_own)):
            if g1 <= g0:
                continue
            for src in slabs:
                a, b = max(g0, src.lo), min(g1, src.hi)
                if a >= b:
                    continue
                if src.rank == dst.rank:
                    raise AssertionError("a halo column owned by the same rank")
                plan.sends[src.rank].append((dst.rank, a - src.lo, b - a))
                plan.recvs[dst.rank].append((src.rank, base + (a - g0), b - a))
    # deterministic order: by peer, then offset
    for r in plan.sends:
        plan.sends[r].sort()
        plan.recvs[r].sort()
    return plan


def gather_slabs(slab: Slab, group=None) -> list[Slab]:
    """All ranks' slabs via torch.distributed (all_gather of 7 integers)."""
    import torch
    import torch.distributed as dist

    mine = torch.tensor([slab.rank, slab.nranks, slab.n, slab.lo, slab.hi, slab.hl, slab.hr], dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        mine = mine.cuda()
    out = [torch.zeros_like(mine) for _ in range(slab.nranks)]
    dist.all_gather(out, mine, group=group)
    return [Slab(*[int(v) for v in t.cpu().tolist()]) for t in out]


def exchange_halo_host(slab: Slab, plan: HaloPlan, x_ext: np.ndarray, group=None) -> None:
    """Fill x_ext's halo with torch.distributed send/recv (host arrays).

    The host reference of the device halo exchange: used by the gloo tests to
    check the plan, and never on the device path.
    """
    import torch
    import torch.distributed as dist

    reqs = []
    bufs = []
    for peer, off, ln in plan.recvs[slab.rank]:
        t = torch.empty(ln, dtype=torch.float64)
        bufs.append((t, off, ln))
        reqs.append(dist.irecv(t, src=peer, group=group))
    for peer, off, ln in plan.sends[slab.rank]:
        t = torch.from_numpy(np.ascontiguousarray(x_ext[slab.own_off + off: slab.own_off + off + ln]))
        reqs.append(dist.isend(t, dst=peer, group=group))
    for r in reqs:
        r.wait()
    for t, off, ln in bufs:
        x_ext[off:off + ln] = t.numpy()


def combine_pairs(pairs: np.ndarray) -> np.ndarray:
    """Rank-order combination of per-rank compensated dot pairs.

    pairs: [nranks, 9, 2] (p, s).  Mirrors the device finalize: TwoSum of the
    p parts, s parts added, rounded once (csrc/common.cuh dd_add).
    """
    acc_p = pairs[0, :, 0].copy()
    acc_s = pairs[0, :, 1].copy()
    for r in range(1, pairs.shape[0]):
        p = pairs[r, :, 0]
        s = acc_p + p
        bb = s - acc_p
        err = (acc_p - (s - bb)) + (p - bb)
        acc_s = (acc_s + pairs[r, :, 1]) + err
        acc_p = s
    return acc_p + acc_s


class DistributedSystem:
    """One rank's share of a row-partitioned system on its GPU.

    Every rank passes the same global CSR (or a callable returning it) and
    gets its slab uploaded with remapped columns, the halo plan attached and
    two NCCL communicators (halo exchange; dot all-gather) created from ids
    rank 0 generates and torch.distributed broadcasts.  ``solve`` takes and
    returns this rank's own segments; the history and status are identical
    on every rank.
    """

    def __init__(self, row_ptr, col_idx, values, n: int, group=None, device: int | None = None):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib
        from .operators import DeviceMatrix

        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        self.ctx = _lib.context(device)
        slab, lrp, lci, lv = local_csr(row_ptr, col_idx, values, n, self.rank, self.nranks)
        slabs = gather_slabs(slab, group) if self.nranks > 1 else [slab]
        plan = halo_plan(slabs)
        self.slab, self.plan = slab, plan
        self.matrix = DeviceMatrix.from_csr((lrp, lci, lv, slab.n_ext), ctx=self.ctx)
        ids = np.zeros(256, dtype=np.uint8)
        if self.rank == 0:
            for k in range(2):
                buf = (C.c_uint8 * 128)()
                _lib.check(_lib.load().pbs_nccl_unique_id(buf))
                ids[128 * k:128 * (k + 1)] = np.frombuffer(bytes(buf), dtype=np.uint8)
        if self.nranks > 1:
            t = torch.from_numpy(ids)
            if dist.get_backend(group) == "nccl":
                t = t.cuda()
            dist.broadcast(t, src=0, group=group)
            ids = t.cpu().numpy()
        h = C.c_void_p()
        idb = ids.ctypes.data_as(C.c_void_p)
        _lib.check(_lib.load().pbs_dist_init(self.ctx.handle, self.nranks, self.rank, idb,
                                             C.c_void_p(ids.ctypes.data + 128), C.byref(h)), self.ctx.handle)
        self.handle = h
        sends = np.array([v for t3 in plan.sends[self.rank] for v in t3], dtype=np.int64)
        recvs = np.array([v for t3 in plan.recvs[self.rank] for v in t3], dtype=np.int64)
        _lib.check(_lib.load().pbs_mat_set_partition(
            self.matrix.handle, h, n, slab.lo, slab.hl, slab.hr, len(plan.sends[self.rank]),
            sends.ctypes.data_as(C.c_void_p), len(plan.recvs[self.rank]), recvs.ctypes.data_as(C.c_void_p)),
            self.ctx.handle)
        self.n_own = slab.n_own
        # the solver sees the rank's square block of the global system
        self.matrix.n_cols = slab.n_own

    def solve(self, b_own, x0_own=None, method: str = "pbicgsafe", config=None, engine=None):
        from .solvers import solve

        return solve(self.matrix, b_own, method=method, x0=x0_own, config=config, engine=engine)

    def close(self):
        from . import _lib

        if getattr(self, "handle", None):
            self.matrix.free()
            _lib.load().pbs_dist_destroy(self.handle)
            self.handle = None
