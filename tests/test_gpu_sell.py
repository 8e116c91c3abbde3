"""The sliced-ELL device layout (csrc/sell.cuh) against the oracle.

At upload a window-mode CSR operator whose rows have stencil-like lengths is
also laid out level-major per 256-row block (u8 row lengths, u16
window-local columns), with a u8 value dictionary when it holds at most 256
distinct f64 bit patterns.  The layout is an internal device form of the
reference's CsrMatrix (linalg.py:28-48): every row sum must stay bitwise
kernels.py:95-100's — ascending columns, rounded products and rounded adds —
including signed zeros and non-finite inputs, on ragged blocks, empty rows,
rows longer than one chunk of levels, and when the layout is refused
(too much padding, too many distinct values).
"""

import os

import numpy as np
import pytest

from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pb():
    import paper_2108_10591_b200 as pb
    from paper_2108_10591_b200 import _lib

    _lib.context(0)
    return pb


def _upload(rp, ci, v, **env):
    from paper_2108_10591_b200.operators import DeviceMatrix

    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(val) for k, val in env.items()})
    try:  # the layout decision is taken at upload
        return DeviceMatrix.from_csr((rp, ci.astype(np.int32), v))
    finally:
        for k, val in old.items():
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val


def _spmv_dev(dm, x, expect_bad=-1):
    import torch

    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    yd = torch.empty_like(xd)
    bad = dm.spmv_dev(xd.data_ptr(), yd.data_ptr())
    torch.cuda.synchronize()
    assert bad == expect_bad
    return yd.cpu().numpy()


def _bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def _banded(n, lens, width, rng, values):
    """Rows of the given lengths with columns inside [i - width, i + width]."""
    rows, cols = [], []
    for i in range(n):
        a, b = max(0, i - width), min(n - 1, i + width)
        k = min(int(lens[i]), b - a + 1)
        c = np.sort(rng.choice(np.arange(a, b + 1), size=k, replace=False)) if k else np.zeros(0, dtype=np.int64)
        rows.append(np.full(c.size, i))
        cols.append(c)
    c = np.concatenate(cols).astype(np.int64)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, np.concatenate(rows).astype(np.int64) + 1, 1)
    rp = np.cumsum(rp)
    return rp, c, values(c.size)


@pytest.mark.parametrize("n,length,ndistinct,want", [
    (5000, 12, 5, "sell-dict"),      # ragged last block, one chunk of levels + part of a second
    (4096, 20, 256, "sell-dict"),    # exactly the dictionary's capacity, three chunks per block
    (3000, 9, 257, "sell"),          # one value too many: f64 value stream
    (2500, 27, 0, "sell"),           # all values distinct, four chunks per block
])
def test_sell_spmv_bitwise(pb, n, length, ndistinct, want):
    rng = np.random.default_rng(n + length)
    lens = np.full(n, length)
    lens[rng.integers(0, n, n // 20)] -= rng.integers(1, 4, n // 20)  # a few shorter rows (padding entries)
    pool = rng.standard_normal(max(ndistinct, 1))
    values = (lambda m: pool[np.arange(m) % ndistinct]) if ndistinct else (lambda m: rng.standard_normal(m))
    rp, ci, v = _banded(n, lens, 40, rng, values)
    x = rng.standard_normal(n)
    ref = orc.spmv(rp, ci, v, x)
    dm = _upload(rp, ci, v, PBS_PLAIN_TPR=0)
    lay = dm.layout()
    assert lay["layout"] == want, lay
    lens_ = np.diff(rp)
    nblk = (n + 255) // 256
    padded = np.zeros(nblk * 256, dtype=np.int64)
    padded[:n] = lens_
    assert lay["entries"] == int(256 * padded.reshape(nblk, 256).max(axis=1).sum())  # each block padded to its longest row
    assert lay["max_row"] == int(lens_.max())
    if want == "sell-dict":
        assert lay["dict_entries"] == ndistinct
    assert np.array_equal(_bits(_spmv_dev(dm, x)), _bits(ref))
    csr = _upload(rp, ci, v, PBS_SELL=0)
    assert csr.layout()["layout"] == "csr-window"
    assert np.array_equal(_bits(_spmv_dev(csr, x)), _bits(ref))
    dm.free()
    csr.free()


@pytest.mark.parametrize("seed", range(12))
def test_sell_random_shapes_bitwise(pb, seed):
    """Seeded sweep over shapes the layout must handle: n around block
    multiples, row lengths from empty to several chunks of levels, narrow and
    wide bands, few / many distinct values, and constant-offset (stencil-like)
    columns that take the pair dictionary.  Whatever layout the upload picks,
    the row sums are the oracle's bit for bit."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.choice([1, 255, 256, 257, 700, 4096, 5000, 12345]))
    base = int(rng.integers(1, 40))
    lens = np.clip(base + rng.integers(-2, 1, n), 0, None)
    if seed % 3 == 0:
        lens[rng.integers(0, n, max(1, n // 50))] = 0
    width = int(rng.choice([base // 2 + 2, 60, 400]))
    nd = int(rng.choice([1, 3, 27, 256, 300, 0]))
    pool = rng.standard_normal(max(nd, 1))
    values = (lambda m: pool[rng.integers(0, nd, m)]) if nd else (lambda m: rng.standard_normal(m))
    if seed % 4 == 1:
        # constant offsets per level: every row holds the same (value, offset) pairs
        offs = np.sort(rng.choice(np.arange(-width, width + 1), size=min(base, 2 * width + 1), replace=False))
        vals = pool[np.arange(offs.size) % max(nd, 1)] if nd else rng.standard_normal(offs.size)
        rows, cols, vv = [], [], []
        for i in range(n):
            ok = (i + offs >= 0) & (i + offs < n)
            rows.append(np.full(int(ok.sum()), i))
            cols.append(i + offs[ok])
            vv.append(vals[ok])
        ci = np.concatenate(cols).astype(np.int64)
        rp = np.zeros(n + 1, dtype=np.int64)
        np.add.at(rp, np.concatenate(rows).astype(np.int64) + 1, 1)
        rp = np.cumsum(rp)
        v = np.concatenate(vv)
    else:
        rp, ci, v = _banded(n, lens, width, rng, values)
    if rp[-1] == 0:
        pytest.skip("empty matrix")
    x = rng.standard_normal(n)
    x[rng.integers(0, n, max(1, n // 10))] = 0.0
    ref = orc.spmv(rp, ci, v, x)
    dm = _upload(rp, ci, v)
    lay = dm.layout()
    got = _spmv_dev(dm, x)
    assert np.array_equal(_bits(got), _bits(ref)), (seed, lay)
    if seed % 4 == 1 and lay["layout"].startswith("sell"):
        assert lay["layout"] == "sell-pairs", lay
    dm.free()


def test_sell_signed_zeros_empty_rows_and_nonfinite(pb):
    """Padding entries are formed but never added: a row summing to -0.0
    keeps its sign, an empty row gives +0.0, and inf / NaN in x reach exactly
    the rows the reference's loop gives them to (0 * inf would otherwise make
    NaN out of padding)."""
    rng = np.random.default_rng(7)
    n = 1500
    lens = rng.integers(8, 11, n)
    lens[[0, 17, 300, 1499]] = 0           # empty rows
    lens[[5, 6, 700]] = 2                   # short rows: mostly padding
    pool = np.array([1.5, -2.0, 0.25, -0.0, 0.0, 3.0])
    rp, ci, v = _banded(n, lens, 30, rng, lambda m: pool[rng.integers(0, pool.size, m)])
    x = rng.standard_normal(n)
    x[::7] = 0.0
    x[3::11] = -0.0
    dm = _upload(rp, ci, v, PBS_PLAIN_TPR=0)
    assert dm.layout()["layout"] == "sell-dict"
    ref = orc.spmv(rp, ci, v, x)
    assert np.array_equal(_bits(_spmv_dev(dm, x)), _bits(ref))
    assert np.signbit(ref).any()  # the case holds negative zeros
    # all-negative-zero products: every non-empty row sums to -0.0 or +0.0 exactly as the reference
    xz = np.zeros(n)
    assert np.array_equal(_bits(_spmv_dev(dm, xz)), _bits(orc.spmv(rp, ci, v, xz)))
    # non-finite x: same rows, same payload class; the first bad row is reported like check_finite
    xi = x.copy()
    xi[40] = np.inf
    xi[900] = np.nan
    refi = orc.spmv(rp, ci, v, xi)
    first = int(np.flatnonzero(~np.isfinite(refi))[0])
    got = _spmv_dev(dm, xi, expect_bad=first)
    assert np.array_equal(np.isnan(got), np.isnan(refi))
    assert np.array_equal(_bits(got[np.isfinite(refi)]), _bits(refi[np.isfinite(refi)]))
    assert np.array_equal(got[np.isinf(refi)], refi[np.isinf(refi)])
    dm.free()


@pytest.mark.parametrize("cfg,k", [("c2", 20), ("c4", 14), ("c1", 70)])
def test_sell_pair_dictionary_on_stencil_csr(pb, cfg, k):
    """A constant-coefficient stencil's CSR repeats the same (value, column -
    row) pairs in every interior row: one u8 per nonzero.  Blocks whose x
    windows are clamped at the matrix start hold other relative columns; the
    row sums stay the reference's, bit for bit, signed zeros and non-finite x
    included."""
    from paper_2108_10591_b200 import problems

    spec = problems.config_stencil(cfg, k=k)
    rp, ci, v = problems.stencil_csr(spec)
    n = spec.n
    dm = _upload(rp, ci, v, PBS_PLAIN_TPR=0)
    lay = dm.layout()
    assert lay["layout"] == "sell-pairs", lay
    assert lay["bytes_per_entry"] == 1 and spec.npts <= lay["dict_entries"] <= 256
    rng = np.random.default_rng(k)
    x = rng.standard_normal(n)
    x[::5] = 0.0
    x[2::9] = -0.0
    assert np.array_equal(_bits(_spmv_dev(dm, x)), _bits(orc.spmv(rp, ci, v, x)))
    xz = -np.zeros(n)
    assert np.array_equal(_bits(_spmv_dev(dm, xz)), _bits(orc.spmv(rp, ci, v, xz)))
    xi = x.copy()
    xi[n // 3] = np.inf
    refi = orc.spmv(rp, ci, v, xi)
    first = int(np.flatnonzero(~np.isfinite(refi))[0])
    got = _spmv_dev(dm, xi, expect_bad=first)
    assert np.array_equal(np.isnan(got), np.isnan(refi))
    ok = np.isfinite(refi)
    assert np.array_equal(_bits(got[ok]), _bits(refi[ok]))
    two = _upload(rp, ci, v, PBS_SELL_PAIR=0, PBS_PLAIN_TPR=0)
    assert two.layout()["layout"] == "sell-dict"
    assert np.array_equal(_bits(_spmv_dev(two, x)), _bits(orc.spmv(rp, ci, v, x)))
    dm.free()
    two.free()


def test_sell_dictionary_refuses_its_own_marker(pb):
    """The value hash set marks free slots with one NaN bit pattern; an
    operator that holds exactly that pattern gets no dictionary (f64 value
    stream) and its products keep the reference's NaN placement."""
    rng = np.random.default_rng(11)
    n = 2000
    pool = np.array([1.0, -0.5, 2.0, np.float64(np.uint64(0x7ff8dead00000001).view(np.float64))])
    rp, ci, v = _banded(n, np.full(n, 9), 30, rng, lambda m: pool[np.arange(m) % 3])
    v[123] = pool[3]  # one entry with the marker pattern
    dm = _upload(rp, ci, v, PBS_PLAIN_TPR=0)
    assert dm.layout()["layout"] == "sell", dm.layout()
    x = rng.standard_normal(n)
    ref = orc.spmv(rp, ci, v, x)
    bad = int(np.flatnonzero(~np.isfinite(ref))[0])
    got = _spmv_dev(dm, x, expect_bad=bad)
    assert np.array_equal(np.isnan(got), np.isnan(ref))
    ok = np.isfinite(ref)
    assert np.array_equal(_bits(got[ok]), _bits(ref[ok]))
    dm.free()


def test_sell_pairs_rows_longer_than_one_chunk(pb):
    """45 constant offsets per row: the pair dictionary applies (45 pairs plus
    the clamped first block's) and a block's levels span two 32-level chunks."""
    rng = np.random.default_rng(45)
    n = 3000
    offs = np.sort(rng.choice(np.arange(-70, 71), size=45, replace=False))
    vals = rng.standard_normal(45)
    rows, cols, vv = [], [], []
    for i in range(n):
        ok = (i + offs >= 0) & (i + offs < n)
        rows.append(np.full(int(ok.sum()), i))
        cols.append(i + offs[ok])
        vv.append(vals[ok])
    ci = np.concatenate(cols).astype(np.int64)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, np.concatenate(rows).astype(np.int64) + 1, 1)
    rp = np.cumsum(rp)
    v = np.concatenate(vv)
    dm = _upload(rp, ci, v, PBS_SELL_PAD=50)
    lay = dm.layout()
    assert lay["layout"] == "sell-pairs" and lay["max_row"] == 45, lay
    x = rng.standard_normal(n)
    assert np.array_equal(_bits(_spmv_dev(dm, x)), _bits(orc.spmv(rp, ci, v, x)))
    dm.free()


def test_wide_random_matrix_gathers_x(pb):
    """Columns anywhere in the row: offsets occupy thousands of 256-wide bins
    (more than the upload reads back), no x window or band fits, and the CSR
    engine gathers x from L2 — still the reference's sums."""
    rng = np.random.default_rng(5)
    n = 400_000
    k = 6
    ci = np.sort(rng.integers(0, n, (n, k)), axis=1)
    ci[:, 0] = np.minimum(ci[:, 0], np.arange(n))  # keep rows sorted and mostly distinct
    ci = np.sort(ci, axis=1).reshape(-1).astype(np.int64)
    rp = np.arange(0, n * k + 1, k, dtype=np.int64)
    v = rng.uniform(-1, 1, n * k)
    dm = _upload(rp, ci, v)
    assert dm.layout()["layout"] == "csr-gather", dm.layout()
    x = rng.standard_normal(n)
    assert np.array_equal(_bits(_spmv_dev(dm, x)), _bits(orc.spmv(rp, ci, v, x)))
    dm.free()


def test_sell_refused_for_ragged_rows(pb):
    """Row lengths uniform in [5, 30] (config 3's shape) would pad each block
    to its longest row: the layout is refused and CSR order kept."""
    rng = np.random.default_rng(3)
    n = 6000
    rp, ci, v = _banded(n, rng.integers(5, 31, n), 60, rng, lambda m: rng.uniform(-1, 1, m))
    dm = _upload(rp, ci, v)
    assert dm.layout()["layout"] == "csr-window"
    x = rng.standard_normal(n)
    assert np.array_equal(_bits(_spmv_dev(dm, x)), _bits(orc.spmv(rp, ci, v, x)))
    forced = _upload(rp, ci, v, PBS_SELL_PAD=400, PBS_PLAIN_TPR=0)  # accept the padding: still the reference's sums
    assert forced.layout()["layout"] == "sell"
    assert np.array_equal(_bits(_spmv_dev(forced, x)), _bits(orc.spmv(rp, ci, v, x)))
    dm.free()
    forced.free()


@pytest.mark.parametrize("env", [{}, {"PBS_SELL_PAIR": 0}, {"PBS_SELL_DICT": 0}, {"PBS_SELL": 0}])
def test_sell_solve_equals_csr_order_solve(pb, env):
    """The same system solved through each layout: identical histories in
    plan order (bitwise the reference's) and on the fast path."""
    from paper_2108_10591_b200 import problems

    spec = problems.convdiff27_stencil(24, (1.0, 0.5, 0.25))
    rp, ci, v = problems.stencil_csr(spec)
    b = orc.spmv(rp, ci, v, np.ones(spec.n))
    ref = orc.solve(rp, ci, v, b, tol=1e-10, max_iters=500, workers=3)
    dm = _upload(rp, ci, v, **env)
    want = {(): "sell-pairs", ("PBS_SELL_PAIR",): "sell-dict", ("PBS_SELL_DICT",): "sell",
            ("PBS_SELL",): "csr-window"}[tuple(env)]
    assert dm.layout()["layout"] == want
    out = pb.solve(dm, b, config=pb.SolverConfig(tol=1e-10, max_iters=500),
                   engine=pb.DeviceEngine(reduce="plan", workers=3))
    assert out.iterations == ref["iterations"]
    assert np.array_equal(_bits([r.rel_res_recur for r in out.history]), _bits(ref["rel"][:len(out.history)]))
    assert np.array_equal(_bits(out.x), _bits(ref["x"]))
    fast = pb.solve(dm, b, config=pb.SolverConfig(tol=1e-10, max_iters=500))
    near = orc.solve(rp, ci, v, b, tol=1e-10, max_iters=500, workers=-1)
    assert fast.iterations == near["iterations"]
    dm.free()
