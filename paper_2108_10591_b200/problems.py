"""Synthetic systems of BASELINE.json's five configurations.

None of these problems is in the reference, which ships only the pure
Laplacian ``gen_poisson`` (linalg.py:175-209).  They are fixed here once and
fed, as identical canonical CSR arrays, to the GPU path, the CPU oracle and
the reference:

* grid ordering is C-order ``arange(n).reshape((k,)*dim)``, last axis fastest,
  as ``gen_poisson`` does (linalg.py:188), so a contiguous row range is a
  slab along axis 0;
* convection-diffusion ``-Δu + β·∇u`` by central differences scaled by h²,
  h = 1/(k+1), Dirichlet boundaries eliminated: diagonal 2·dim, neighbour
  along axis a at +1 is ``-1 + c_a/2`` and at -1 is ``-1 - c_a/2`` with
  ``c_a = β_a·h``;
* the 27-point operator is HPCG-like diffusion (26 on the diagonal, -1 to
  each of the 26 neighbours) plus the same central convection on the six
  face neighbours;
* the random operator has U{5..30} entries per row including the diagonal,
  off-diagonal columns drawn without replacement from ``[i-5000, i+5000]``,
  values U(-1,1), diagonal ``1.1·Σ|off-diagonal|``.

Rows are emitted in canonical form (strictly increasing columns, no
duplicates), i.e. exactly what ``csr_from_coo`` (linalg.py:110-139) returns
for the same triplets; tests/golden pins that against the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class StencilSpec:
    """Constant-coefficient stencil on a k^dim grid (matrix-free operator).

    ``offsets`` are (dz, dy, dx)-style tuples of length ``dim`` sorted so that
    the flattened column offset is ascending — the accumulation order of the
    CSR row — and ``coeffs`` the matching values.
    """

    dim: int
    k: int
    offsets: tuple[tuple[int, ...], ...]
    coeffs: tuple[float, ...]

    @property
    def n(self) -> int:
        return self.k**self.dim

    @property
    def npts(self) -> int:
        return len(self.offsets)

    def flat_offsets(self) -> list[int]:
        out = []
        for off in self.offsets:
            f = 0
            for a, d in enumerate(off):
                f += d * self.k ** (self.dim - 1 - a)
            out.append(f)
        return out


def _convdiff_coeffs(dim: int, k: int, beta) -> tuple[float, list[float], list[float]]:
    h = 1.0 / (k + 1)
    up, dn = [], []
    for a in range(dim):
        c = float(beta[a]) * h
        up.append(-1.0 + 0.5 * c)
        dn.append(-1.0 - 0.5 * c)
    return 2.0 * dim, up, dn


def convdiff_stencil(dim: int, k: int, beta) -> StencilSpec:
    """(2·dim+1)-point convection-diffusion stencil (configs 1, 2, 5)."""
    if dim not in (1, 2, 3):
        raise ValueError("dim must be 1, 2, or 3")
    if len(beta) != dim:
        raise ValueError("beta needs one entry per axis")
    diag, up, dn = _convdiff_coeffs(dim, k, beta)
    entries = []
    for a in range(dim):
        off = [0] * dim
        off[a] = -1
        entries.append((tuple(off), dn[a]))
        off = [0] * dim
        off[a] = +1
        entries.append((tuple(off), up[a]))
    entries.append((tuple([0] * dim), diag))
    entries.sort(key=lambda e: sum(d * k ** (dim - 1 - a) for a, d in enumerate(e[0])))
    return StencilSpec(dim, k, tuple(e[0] for e in entries), tuple(e[1] for e in entries))


def convdiff27_stencil(k: int, beta) -> StencilSpec:
    """27-point HPCG-like diffusion + central face convection (config 4)."""
    diag, up, dn = _convdiff_coeffs(3, k, beta)
    offsets, coeffs = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                off = (dz, dy, dx)
                nz = [a for a in range(3) if off[a] != 0]
                if not nz:
                    val = 26.0
                elif len(nz) == 1:
                    a = nz[0]
                    val = up[a] if off[a] > 0 else dn[a]
                else:
                    val = -1.0
                offsets.append(off)
                coeffs.append(val)
    return StencilSpec(3, k, tuple(offsets), tuple(coeffs))


def stencil_csr(spec: StencilSpec, col_dtype=np.int64):
    """Canonical CSR of a stencil, built row-ordered without a triplet sort."""
    dim, k = spec.dim, spec.k
    n = k**dim
    coords = np.indices((k,) * dim, dtype=np.int64).reshape(dim, n)
    masks = []
    for off in spec.offsets:
        m = np.ones(n, dtype=bool)
        for a, d in enumerate(off):
            if d < 0:
                m &= coords[a] >= -d
            elif d > 0:
                m &= coords[a] < k - d
        masks.append(m)
    counts = np.zeros(n, dtype=np.int64)
    for m in masks:
        counts += m
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col_idx = np.empty(nnz, dtype=col_dtype)
    values = np.empty(nnz, dtype=np.float64)
    cursor = row_ptr[:-1].copy()
    rows = np.arange(n, dtype=np.int64)
    for m, foff, val in zip(masks, spec.flat_offsets(), spec.coeffs):
        pos = cursor[m]
        col_idx[pos] = rows[m] + foff
        values[pos] = val
        cursor[m] += 1
    return row_ptr, col_idx, values


def random_banded_csr(n: int, seed: int = 2108, half_window: int = 5000, nnz_lo: int = 5,
                      nnz_hi: int = 30, col_dtype=np.int64, chunk: int = 1 << 18):
    """Config 3: random nonsymmetric, diagonally dominant, banded CSR.

    Per row i: m ~ U{nnz_lo-1 .. nnz_hi-1} off-diagonal columns drawn
    without replacement from [i-w, i+w] ∩ [0, n) minus {i} (candidates are
    drawn with replacement and the first m distinct ones kept, redrawing the
    rare row that runs short); values U(-1,1) assigned in ascending column
    order; diagonal 1.1·Σ|off-diagonal| summed in ascending column order.
    Returns (row_ptr, col_idx, values, b) with b ~ U(0,1).
    """
    if half_window < 1 or n < 2:
        raise ValueError("need n >= 2 and a positive window")
    rng = np.random.default_rng(seed)
    m_off = rng.integers(nnz_lo - 1, nnz_hi, size=n, dtype=np.int64)
    m_off = np.minimum(m_off, n - 1)
    b = rng.random(n)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(m_off + 1, out=row_ptr[1:])
    nnz = int(row_ptr[-1])
    col_idx = np.empty(nnz, dtype=col_dtype)
    values = np.empty(nnz, dtype=np.float64)
    big = np.iinfo(np.int64).max
    mmax = nnz_hi - 1
    ncand = nnz_hi + 16
    for lo in range(0, n, chunk):
        hi = min(n, lo + chunk)
        R = hi - lo
        rows = np.arange(lo, hi, dtype=np.int64)
        wlo = np.maximum(rows - half_window, 0)
        width = np.minimum(rows + half_window, n - 1) - wlo  # excludes the diagonal
        mm = m_off[lo:hi]
        chosen = np.full((R, mmax), big, dtype=np.int64)
        need = np.arange(R)
        while need.size:
            u = rng.random((need.size, ncand))
            cand = wlo[need, None] + np.floor(u * width[need, None]).astype(np.int64)
            cand += cand >= rows[need, None]
            order = np.argsort(cand, axis=1, kind="stable")
            sc = np.take_along_axis(cand, order, axis=1)
            dup_sorted = np.zeros(sc.shape, dtype=bool)
            dup_sorted[:, 1:] = sc[:, 1:] == sc[:, :-1]
            dup = np.zeros_like(dup_sorted)
            np.put_along_axis(dup, order, dup_sorted, axis=1)
            keep = ~dup
            rank = np.cumsum(keep, axis=1)
            ok = rank[:, -1] >= mm[need]
            sel = keep & (rank <= mm[need, None])
            picked = np.sort(np.where(sel, cand, big), axis=1)[:, :mmax]
            chosen[need[ok]] = picked[ok]
            need = need[~ok]
        slot = np.arange(mmax)[None, :]
        valid = slot < mm[:, None]
        v = rng.uniform(-1.0, 1.0, size=(R, mmax))
        v = np.where(valid, v, 0.0)
        diag = 1.1 * np.cumsum(np.abs(v), axis=1)[:, -1]
        cols = np.concatenate([chosen, rows[:, None]], axis=1)
        vals = np.concatenate([v, diag[:, None]], axis=1)
        order = np.argsort(cols, axis=1, kind="stable")
        cols = np.take_along_axis(cols, order, axis=1)
        vals = np.take_along_axis(vals, order, axis=1)
        mask = cols != big
        s, e = int(row_ptr[lo]), int(row_ptr[hi])
        col_idx[s:e] = cols[mask]
        values[s:e] = vals[mask]
    return row_ptr, col_idx, values, b


# BASELINE.json configs (SURVEY.md §8 notation C1..C5)
CONFIGS = {
    "c1": dict(kind="convdiff", dim=2, k=64, beta=(1.0, 1.0), tol=1e-10,
               label="2D 5-point convection-diffusion 64^2, beta=(1,1)*h"),
    "c2": dict(kind="convdiff", dim=3, k=128, beta=(1.0, 0.5, 0.25), tol=1e-10,
               label="3D 7-point convection-diffusion 128^3, beta=(1,0.5,0.25)*h"),
    "c3": dict(kind="random", n=4_000_000, seed=2108, tol=1e-10,
               label="random banded CSR n=4M, nnz/row U{5..30}, |i-j|<=5000"),
    "c4": dict(kind="convdiff27", dim=3, k=384, beta=(1.0, 0.5, 0.25), tol=1e-10,
               label="3D 27-point convection-diffusion 384^3"),
    "c5": dict(kind="convdiff", dim=3, k=256, beta=(100.0, 50.0, 25.0), tol=1e-12,
               label="3D 7-point convection-dominated 256^3, beta=(100,50,25)*h"),
}


def config_stencil(name: str, k: int | None = None) -> StencilSpec:
    cfg = CONFIGS[name]
    kk = cfg["k"] if k is None else k
    if cfg["kind"] == "convdiff":
        return convdiff_stencil(cfg["dim"], kk, cfg["beta"])
    if cfg["kind"] == "convdiff27":
        return convdiff27_stencil(kk, cfg["beta"])
    raise ValueError(f"config {name} is not a stencil problem")
