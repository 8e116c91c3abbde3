"""Row-partitioned systems: slabs, extended-space operators, halo plans, groups.

The reference's only parallelism is a row partition: ``PartitionPlan``
contiguous ranges (reduction.py:55-87), partial dots per range combined in
range order (reduction.py:282-294) and row-range SpMV (linalg.py:164-172).
On B200 each range is a partition of the system on its own GPU:

* partition r owns rows ``[lo, hi)`` of ``PartitionPlan.balanced(n, N)`` (for
  the grid configs: whole axis-0 planes);
* its operator keeps its rows with columns in an *extended* local index
  space ``[pad | left halo | own | right halo]``: the left halo is the
  contiguous column range ``[lo - hl, lo)`` and the right halo
  ``[hi, hi + hr)`` of the columns its rows reach outside its own range.  A
  CSR slab is sliced from a host CSR (``local_csr``) or — for the generated
  grids, so no rank ever holds the global matrix — built on the device from
  the stencil (``pbs_stencil_slab``, then ``pbs_stencil_to_csr``); a
  matrix-free slab is the stencil slab itself;
* every SpMV input vector lives in that extended space; before an SpMV the
  halo is filled from the owners — the transfer list is the ``HaloPlan``
  (identical on every rank, derived from all ranks' halo widths);
* the per-iteration dot batch reduces to one record of 9 compensated pairs
  per partition; every partition combines all records in rank order, so all
  compute the identical coefficients and stop at the identical check.

Two ways to hold a partitioned system:

* ``DistributedSystem`` — one process per GPU (torch.distributed for the
  plumbing: slab sizes, IPC handles and barriers); the device transport is
  CUDA-IPC peer memory + copy engines + stream-memory-op flags (or NCCL);
* ``LoopbackSystem`` — all N partitions in this process on one device, with
  the same kernels, schedule and transport (each partition limited to
  sms / N SMs, like N smaller GPUs): the N-partition path on one B200.
"""

from __future__ import annotations

import ctypes as C
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

    sends[r]: (peer, offset in r's OWN segment, length, extended-space offset
    on the peer); recvs[r]: (peer, extended-space offset on r, length).
    """

    sends: dict[int, list[tuple[int, int, int, int]]] = field(default_factory=dict)
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


def _stencil_cols(spec, rows: np.ndarray, p: int) -> tuple[np.ndarray, np.ndarray]:
    """Columns of stencil point p for grid rows ``rows`` and whether they are
    in the grid (Dirichlet elimination), C-order grid (linalg.py:188)."""
    k, dim = spec.k, spec.dim
    coords = []
    rem = rows.copy()
    for a in range(dim):
        w = k ** (dim - 1 - a)
        coords.append(rem // w)
        rem = rem % w
    ok = np.ones(rows.shape, dtype=bool)
    for a in range(dim):
        c = coords[a] + spec.offsets[p][a]
        ok &= (c >= 0) & (c < k)
    return rows + spec.flat_offsets()[p], ok


def stencil_halo(spec, lo: int, hi: int) -> tuple[int, int]:
    """Exact halo widths of the rows [lo, hi) of a stencil operator: the
    columns its rows reach below lo and at or above hi (only rows within one
    stencil reach of either end can reach out)."""
    reach = max(abs(f) for f in spec.flat_offsets())
    hl = hr = 0
    left = np.arange(lo, min(hi, lo + reach + 1), dtype=np.int64)
    right = np.arange(max(lo, hi - reach - 1), hi, dtype=np.int64)
    for p in range(spec.npts):
        cols, ok = _stencil_cols(spec, left, p)
        if ok.any():
            hl = max(hl, lo - int(cols[ok].min()))
        cols, ok = _stencil_cols(spec, right, p)
        if ok.any():
            hr = max(hr, int(cols[ok].max()) + 1 - hi)
    return hl, hr


def stencil_slab(spec, rank: int, nranks: int) -> Slab:
    """``rank``'s slab of a stencil operator (no matrix needed)."""
    lo, hi = slab_bounds(spec.n, nranks)[rank]
    hl, hr = stencil_halo(spec, lo, hi)
    return Slab(rank, nranks, spec.n, lo, hi, hl, hr)


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
                plan.sends[src.rank].append((dst.rank, a - src.lo, b - a, base + (a - g0)))
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


def gather_blobs(blob: bytes, nranks: int, group=None) -> bytes:
    """Every rank's fixed-size partition blob (IPC handles), rank order."""
    import torch.distributed as dist

    out = [None] * nranks
    dist.all_gather_object(out, bytes(blob), group=group)
    if any(len(b) != len(blob) for b in out):
        raise RuntimeError("partition blobs differ in size across ranks")
    return b"".join(out)


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
    for peer, off, ln, _dst in plan.sends[slab.rank]:
        t = torch.from_numpy(np.ascontiguousarray(x_ext[slab.own_off + off: slab.own_off + off + ln]))
        reqs.append(dist.isend(t, dst=peer, group=group))
    for r in reqs:
        r.wait()
    for t, off, ln in bufs:
        x_ext[off:off + ln] = t.numpy()


def combine_pairs(pairs: np.ndarray) -> np.ndarray:
    """Rank-order combination of per-rank compensated dot pairs.

    pairs: [nranks, 9, 2] (p, s).  TwoSum of the p parts, s parts added,
    rounded once (csrc/common.cuh dd_add).
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


# ------------------------------------------------------------- device side

@dataclass(frozen=True)
class SystemSource:
    """The global system a partitioned solve works on: a host CSR (every rank
    slices its rows) or a stencil spec (every rank builds its slab on the
    device, matrix-free or as CSR)."""

    kind: str  # "csr" | "stencil"
    n: int
    csr: tuple | None = None
    spec: object | None = None

    @classmethod
    def from_csr(cls, row_ptr, col_idx, values, n: int) -> "SystemSource":
        return cls("csr", int(n), csr=(row_ptr, col_idx, values))

    @classmethod
    def from_stencil(cls, spec) -> "SystemSource":
        return cls("stencil", int(spec.n), spec=spec)

    def slab(self, rank: int, nranks: int) -> Slab:
        if self.kind == "stencil":
            return stencil_slab(self.spec, rank, nranks)
        rp, ci, v = self.csr
        return local_csr(rp, ci, v, self.n, rank, nranks)[0]


def partition_operator(source: SystemSource, slab: Slab, ctx, operator: str = "csr"):
    """The DeviceMatrix of one slab (extended-space columns)."""
    from . import _lib
    from .operators import DeviceMatrix

    if source.kind == "csr":
        if operator != "csr":
            raise ValueError("a host CSR source can only give CSR slabs")
        rp, ci, v = source.csr
        _, lrp, lci, lv = local_csr(rp, ci, v, source.n, slab.rank, slab.nranks)
        return DeviceMatrix.from_csr((lrp, lci, lv, slab.n_ext), ctx=ctx)
    if operator not in ("csr", "stencil"):
        raise ValueError(f"unknown operator {operator!r}")
    whole = DeviceMatrix.from_stencil(source.spec, ctx=ctx)
    try:
        h = C.c_void_p()
        _lib.check(_lib.load().pbs_stencil_slab(whole.handle, slab.lo, slab.hi, slab.hl, slab.hr, C.byref(h)),
                   ctx.handle)
        nr, nc, nnz, st = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        _lib.load().pbs_mat_info(h, C.byref(nr), C.byref(nc), C.byref(nnz), C.byref(st))
        sm = DeviceMatrix(h, ctx, nr.value, nc.value, nnz.value, True, whole.source + f"[{slab.lo}:{slab.hi}]")
    finally:
        whole.free()
    if operator == "stencil":
        return sm
    try:
        return sm.to_csr()
    finally:
        sm.free()


def _link(mat, slab: Slab, plan: HaloPlan, ctx, transport: str = "p2p", ids: bytes | None = None):
    """pbs_dist_init + pbs_mat_set_partition for one partition."""
    from . import _lib

    L = _lib.load()
    h = C.c_void_p()
    idh = idr = None
    if transport == "nccl":
        idh = C.c_char_p(ids[:128])
        idr = C.c_char_p(ids[128:256])
    _lib.check(L.pbs_dist_init(ctx.handle, slab.nranks, slab.rank, _lib.TRANSPORTS[transport], idh, idr,
                               C.byref(h)), ctx.handle)
    sends = np.array([v for t4 in plan.sends[slab.rank] for v in t4], dtype=np.int64)
    recvs = np.array([v for t3 in plan.recvs[slab.rank] for v in t3], dtype=np.int64)
    rc = L.pbs_mat_set_partition(mat.handle, h, slab.n, slab.lo, slab.hl, slab.hr, len(plan.sends[slab.rank]),
                                 sends.ctypes.data_as(C.c_void_p), len(plan.recvs[slab.rank]),
                                 recvs.ctypes.data_as(C.c_void_p))
    if rc != _lib.PBS_OK:
        msg = _lib.last_error(ctx.handle)
        L.pbs_dist_destroy(h)
        raise _lib.PbsError(rc, msg)
    return h


def _source_of(row_ptr, col_idx, values, n, spec, source):
    if source is not None:
        return source
    if spec is not None:
        return SystemSource.from_stencil(spec)
    if row_ptr is None or n is None:
        raise ValueError("need a CSR (row_ptr, col_idx, values, n), a stencil spec or a SystemSource")
    return SystemSource.from_csr(row_ptr, col_idx, values, n)


class DistributedSystem:
    """One rank's partition of a row-partitioned system on its GPU (one
    process per GPU, torch.distributed initialised).

    Every rank passes the same global system — a host CSR (``row_ptr,
    col_idx, values, n``), a stencil ``spec`` (slab built on the device) or a
    ``SystemSource`` — and gets its slab uploaded with extended-space
    columns, the halo plan attached and the peers mapped (CUDA IPC handles
    exchanged over torch.distributed; ``transport="nccl"`` creates two NCCL
    communicators instead).  ``solve`` takes and returns this rank's own
    segments; the history and status are identical on every rank.
    """

    def __init__(self, row_ptr=None, col_idx=None, values=None, n: int | None = None, group=None,
                 device: int | None = None, *, spec=None, source: SystemSource | None = None,
                 operator: str = "csr", transport: str = "p2p"):
        import torch.distributed as dist

        from . import _lib

        self.source = _source_of(row_ptr, col_idx, values, n, spec, source)
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        self.group = group
        self.ctx = _lib.context(device)
        slab = self.source.slab(self.rank, self.nranks)
        slabs = gather_slabs(slab, group) if self.nranks > 1 else [slab]
        self.slab, self.plan = slab, halo_plan(slabs)
        self.matrix = partition_operator(self.source, slab, self.ctx, operator)
        ids = None
        if transport == "nccl":
            ids = np.zeros(256, dtype=np.uint8)
            if self.rank == 0:
                for k in range(2):
                    buf = (C.c_uint8 * 128)()
                    _lib.check(_lib.load().pbs_nccl_unique_id(buf))
                    ids[128 * k:128 * (k + 1)] = np.frombuffer(bytes(buf), dtype=np.uint8)
            if self.nranks > 1:
                obj = [ids.tobytes()]
                dist.broadcast_object_list(obj, src=0, group=group)
                ids = np.frombuffer(obj[0], dtype=np.uint8)
            ids = ids.tobytes()
        self.handle = _link(self.matrix, slab, self.plan, self.ctx, transport, ids)
        L = _lib.load()
        blob = (C.c_uint8 * _lib.DIST_BLOB_BYTES)()
        _lib.check(L.pbs_dist_export(self.matrix.handle, blob), self.ctx.handle)
        blobs = gather_blobs(bytes(blob), self.nranks, group) if self.nranks > 1 else bytes(blob)
        _lib.check(L.pbs_dist_connect(self.matrix.handle, blobs), self.ctx.handle)
        if self.nranks > 1:
            dist.barrier(group=group)  # every rank mapped its peers before anyone pushes
        self.n_own = slab.n_own
        # the solver sees the rank's square block of the global system
        self.matrix.n_cols = slab.n_own

    def solve(self, b_own, x0_own=None, method: str = "pbicgsafe", config=None, engine=None):
        from .solvers import solve

        return solve(self.matrix, b_own, method=method, x0=x0_own, config=config, engine=engine)

    def spmv_dev(self, x_ptr: int, y_ptr: int) -> int:
        """y_own = (A x)_own on device pointers to own segments; returns the
        first non-finite local row or -1."""
        from . import _lib

        bad = (C.c_int64 * 1)()
        _lib.check(_lib.load().pbs_spmv_group((C.c_void_p * 1)(self.matrix.handle), 1,
                                              (C.c_void_p * 1)(x_ptr), (C.c_void_p * 1)(y_ptr), bad),
                   self.ctx.handle)
        return int(bad[0])

    def close(self):
        from . import _lib

        if getattr(self, "handle", None):
            self.matrix.free()
            _lib.load().pbs_dist_destroy(self.handle)
            self.handle = None


class LoopbackSystem:
    """All ``nparts`` partitions of a system in this process, on one device.

    The partitions run the multi-GPU schedule exactly — extended-space slabs,
    copy-engine halo pushes between the partitions' workspaces with stream
    memory-op flags, the published records and the rank-order combine — so
    the N-partition path is held to the oracle on one B200.  With
    ``emulate=True`` each partition may fill only sms // nparts SMs, as if
    it had a GPU of its own (so the reduction and the As SpMV of every
    partition can be resident at once).  Not a scaling measurement: the
    partitions share one HBM.
    """

    def __init__(self, nparts: int, row_ptr=None, col_idx=None, values=None, n: int | None = None, *,
                 spec=None, source: SystemSource | None = None, operator: str = "csr",
                 device: int | None = None, emulate: bool = True):
        from . import _lib

        self.source = _source_of(row_ptr, col_idx, values, n, spec, source)
        self.nparts = int(nparts)
        self.ctx = _lib.context(device)
        self.slabs = [self.source.slab(r, self.nparts) for r in range(self.nparts)]
        self.plan = halo_plan(self.slabs)
        self.mats, self.handles = [], []
        try:
            for sl in self.slabs:
                m = partition_operator(self.source, sl, self.ctx, operator)
                self.mats.append(m)
                self.handles.append(_link(m, sl, self.plan, self.ctx))
                m.n_cols = sl.n_own
            L = _lib.load()
            if emulate and self.nparts > 1:
                for h in self.handles:
                    _lib.check(L.pbs_dist_set_sm_limit(h, max(2, self.ctx.sm_count // self.nparts)),
                               self.ctx.handle)
            arr = (C.c_void_p * self.nparts)(*[m.handle for m in self.mats])
            _lib.check(L.pbs_dist_connect_local(arr, self.nparts), self.ctx.handle)
        except Exception:
            self.close()
            raise
        self.n = self.source.n

    def _device_segments(self, v):
        import torch

        dev = torch.device("cuda", self.ctx.device)
        out = []
        for sl in self.slabs:
            t = torch.empty(sl.n_own, dtype=torch.float64, device=dev)
            if v is not None:
                t.copy_(torch.from_numpy(np.ascontiguousarray(v[sl.lo:sl.hi], dtype=np.float64)))
            out.append(t)
        return out

    def solve(self, b, x0=None, method: str = "pbicgsafe", config=None, engine=None):
        """Solve with the global host b (and x0); the outcome's x is global."""
        import torch

        from .linalg import check_finite
        from .solvers import solve_group

        b = np.asarray(b, dtype=np.float64)
        if b.shape != (self.n,):
            raise ValueError(f"rhs has shape {b.shape}, system has {self.n} rows")
        check_finite(b, "right-hand side")
        if x0 is not None:
            x0 = np.asarray(x0, dtype=np.float64)
            if x0.shape != (self.n,):
                raise ValueError(f"x0 has shape {x0.shape}, system has {self.n} rows")
            check_finite(x0, "initial guess")
        bs = self._device_segments(b)
        xs = self._device_segments(None)
        x0s = self._device_segments(x0) if x0 is not None else None
        torch.cuda.synchronize(self.ctx.device)
        out = solve_group(self.mats, [t.data_ptr() for t in bs], [t.data_ptr() for t in xs], method=method,
                          x0_ptrs=None if x0s is None else [t.data_ptr() for t in x0s], config=config,
                          engine=engine)
        torch.cuda.synchronize(self.ctx.device)
        out.x = np.concatenate([t.cpu().numpy() for t in xs])
        return out

    def spmv(self, x) -> np.ndarray:
        """Global y = A x through the partitions (halo exchange included)."""
        import torch

        from . import _lib
        from .linalg import NonFiniteVectorError

        xs = self._device_segments(np.asarray(x, dtype=np.float64))
        ys = self._device_segments(None)
        torch.cuda.synchronize(self.ctx.device)
        n = self.nparts
        bad = (C.c_int64 * n)()
        P = C.c_void_p * n
        _lib.check(_lib.load().pbs_spmv_group(P(*[m.handle for m in self.mats]), n,
                                              P(*[t.data_ptr() for t in xs]), P(*[t.data_ptr() for t in ys]), bad),
                   self.ctx.handle)
        for sl, i in zip(self.slabs, bad):
            if i >= 0:
                idx = sl.lo + int(i)
                raise NonFiniteVectorError(f"matvec 'Ax' output row has non-finite entry at index {idx}", idx)
        return np.concatenate([t.cpu().numpy() for t in ys])

    def close(self):
        from . import _lib

        for m in getattr(self, "mats", []):
            m.free()
        for h in getattr(self, "handles", []):
            _lib.load().pbs_dist_destroy(h)
        self.mats, self.handles = [], []
