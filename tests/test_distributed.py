"""Row-partitioned multi-GPU host logic, exercised with gloo on CPU (world_size 2 and 3).

The device halo exchange and dot all-gather follow exactly these plans; here
each rank runs the oracle SpMV on its remapped local CSR after a gloo halo
exchange, and the result must equal the global SpMV rows bitwise.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2108_10591_b200 import distributed as D
from paper_2108_10591_b200 import problems


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _matrix(kind):
    if kind == "c5s12":
        return problems.stencil_csr(problems.convdiff_stencil(3, 12, (100.0, 50.0, 25.0)))
    if kind == "cd27":
        return problems.stencil_csr(problems.convdiff27_stencil(10, (1.0, 0.5, 0.25)))
    rp, ci, v, _ = problems.random_banded_csr(3000, seed=3, half_window=400)
    return rp, ci, v


def _worker(rank, world, port, kind, q):
    import torch.distributed as dist

    from oracle import oracle as orc

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rp, ci, v = _matrix(kind)
        n = len(rp) - 1
        x = np.random.default_rng(11).standard_normal(n)
        ref = orc.spmv(rp, ci, v, x)
        slab, lrp, lci, lv = D.local_csr(rp, ci, v, n, rank, world)
        slabs = D.gather_slabs(slab)
        plan = D.halo_plan(slabs)
        x_ext = np.full(slab.n_ext, np.nan)
        x_ext[slab.own_off:slab.own_off + slab.n_own] = x[slab.lo:slab.hi]
        D.exchange_halo_host(slab, plan, x_ext)
        if slab.pad:
            x_ext[0] = 0.0  # the alignment dummy is never referenced
        assert not np.isnan(x_ext).any(), "halo not fully filled"
        y = orc.spmv(lrp, lci.astype(np.int64), lv, x_ext)
        ok_spmv = np.array_equal(y, ref[slab.lo:slab.hi])
        # compensated dot pairs, combined in rank order == near-exact global dot
        a = x[slab.lo:slab.hi]
        b = ref[slab.lo:slab.hi]
        p, s = 0.0, 0.0
        for ai, bi in zip(a, b):
            h = ai * bi
            # exact product error via fma-free Dekker split (numpy has no fma)
            sp = 134217729.0
            ca, cb = sp * ai, sp * bi
            ah, bh = ca - (ca - ai), cb - (cb - bi)
            al, bl = ai - ah, bi - bh
            r = ((ah * bh - h) + ah * bl + al * bh) + al * bl
            t = p + h
            bb = t - p
            e = (p - (t - bb)) + (h - bb)
            p, s = t, s + (e + r)
        mine = np.zeros((9, 2))
        mine[0] = (p, s)
        import torch

        allp = [torch.zeros(18, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, torch.from_numpy(mine.reshape(-1)))
        pairs = np.stack([t.numpy().reshape(9, 2) for t in allp])
        combined = D.combine_pairs(pairs)[0]
        q.put((rank, ok_spmv, float(combined), slab))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("kind", ["c5s12", "cd27", "rand"])
def test_distributed_spmv_matches_global(world, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _, _ in res), res
    # every rank combined the same value, and it equals the near-exact dot
    vals = {c for _, _, c, _ in res}
    assert len(vals) == 1
    rp, ci, v = _matrix(kind)
    from oracle import oracle as orc

    n = len(rp) - 1
    x = np.random.default_rng(11).standard_normal(n)
    y = orc.spmv(rp, ci, v, x)
    assert vals.pop() == pytest.approx(float(np.dot(x, y)), rel=1e-14)
    # slabs tile [0, n) and every halo is within bounds
    slabs = [s for _, _, _, s in res]
    assert slabs[0].lo == 0 and slabs[-1].hi == n
    for a, b in zip(slabs, slabs[1:]):
        assert a.hi == b.lo


def test_halo_plan_for_grid_slabs():
    # 3D 7-point, k=8, 4 ranks: slabs are 2 planes; halos are exactly one plane
    k = 8
    rp, ci, v = problems.stencil_csr(problems.convdiff_stencil(3, k, (1.0, 0.5, 0.25)))
    n = k**3
    slabs = [D.local_csr(rp, ci, v, n, r, 4)[0] for r in range(4)]
    for s in slabs:
        assert s.n_own == 2 * k * k
        assert s.hl == (0 if s.rank == 0 else k * k)
        assert s.hr == (0 if s.rank == 3 else k * k)
    plan = D.halo_plan(slabs)
    assert all(s.pad == 0 for s in slabs)
    assert plan.recvs[1] == [(0, 0, k * k), (2, k * k + 2 * k * k, k * k)]
    # (peer, own offset, length, the peer's extended offset): rank 1's first
    # plane fills rank 0's right halo, its last plane rank 2's left halo
    assert plan.sends[1] == [(0, 0, k * k, 2 * k * k), (2, k * k, k * k, 0)]
    # every send lands exactly where the receiver expects it
    for src in slabs:
        for peer, off, ln, dst in plan.sends[src.rank]:
            assert (src.rank, dst, ln) in plan.recvs[peer]


@pytest.mark.parametrize("spec", [
    problems.convdiff_stencil(3, 12, (100.0, 50.0, 25.0)),
    problems.convdiff27_stencil(10, (1.0, 0.5, 0.25)),
    problems.convdiff_stencil(2, 7, (1.0, 1.0)),
    problems.convdiff27_stencil(9, (1.0, 0.5, 0.25)),
])
@pytest.mark.parametrize("nranks", [1, 2, 3, 4, 8])
def test_stencil_slab_halos_equal_the_csr_slab(spec, nranks):
    """stencil_slab (no matrix) gives exactly the slab local_csr measures on
    the stencil's CSR: the device builds slabs from the spec alone."""
    rp, ci, v = problems.stencil_csr(spec)
    for r in range(nranks):
        assert D.stencil_slab(spec, r, nranks) == D.local_csr(rp, ci, v, spec.n, r, nranks)[0]


def test_c4_slabs_are_planes_with_one_plane_halos():
    """Config 4 (384^3, 27-point) over 2, 4, 8 ranks: axis-0 plane slabs
    (48 planes at 8), one-plane halos, computed without the 1.5e9-nonzero CSR."""
    spec = problems.config_stencil("c4")
    k = spec.k
    for nranks in (2, 4, 8):
        for r in range(nranks):
            s = D.stencil_slab(spec, r, nranks)
            assert s.lo % (k * k) == 0 and s.n_own == (k // nranks) * k * k
            assert s.hl == (0 if r == 0 else k * k) and s.hr == (0 if r == nranks - 1 else k * k)


def _blob_worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blob = bytes([rank]) * 256
        q.put((rank, D.gather_blobs(blob, world)))
    finally:
        dist.destroy_process_group()


def test_partition_blobs_gather_in_rank_order():
    """The IPC-handle exchange of DistributedSystem: every rank gets every
    rank's 256-byte blob, concatenated in rank order (gloo, world 3)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_blob_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = b"".join(bytes([r]) * 256 for r in range(3))
    assert all(b == want for _, b in res)


def test_odd_halo_gets_an_alignment_pad():
    # 2D 5-point with k=7 over 2 ranks: hl = 7 (odd) -> pad 1, own at index 8
    rp, ci, v = problems.stencil_csr(problems.convdiff_stencil(2, 7, (1.0, 1.0)))
    s1 = D.local_csr(rp, ci, v, 49, 1, 2)
    slab, lrp, lci, lv = s1
    assert slab.hl == 7 and slab.pad == 1 and slab.own_off == 8 and slab.own_off % 2 == 0
    assert lci.min() >= 1 and lci.max() < slab.n_ext


def test_combine_pairs_rank_order_is_deterministic():
    rng = np.random.default_rng(0)
    pairs = rng.standard_normal((5, 9, 2)) * np.array([1.0, 1e-17])
    a = D.combine_pairs(pairs)
    b = D.combine_pairs(pairs.copy())
    assert np.array_equal(a, b)
