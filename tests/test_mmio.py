"""Matrix Market ingest (paper_2108_10591_b200.mmio) against the reference's loader.

tests/golden/mmio.npz holds, for each text, what the reference's
load_matrix_market (mmio.py:33-137) returned — the canonical CSR arrays — or
the line its MatrixMarketError named (make_golden.py, MM_TEXTS).  The GPU case
solves an ingested file on the device, bitwise against the oracle.
"""

import os

import numpy as np
import pytest

from paper_2108_10591_b200.linalg import csr_from_coo
from paper_2108_10591_b200.mmio import MatrixMarketError, load_matrix_market, write_matrix_market
from tests import golden_cases as gc

G = np.load(os.path.join(gc.GOLDEN, "mmio.npz"))
NAMES = sorted({k[: -len("_text")] for k in G.files if k.endswith("_text")})


def _write(tmp_path, text, name="m.mtx"):
    path = tmp_path / name
    path.write_text(text)
    return str(path)


@pytest.mark.parametrize("name", NAMES)
def test_loader_matches_reference(tmp_path, name):
    path = _write(tmp_path, str(G[f"{name}_text"]), f"{name}.mtx")
    if f"{name}_error_line" in G.files:
        with pytest.raises(MatrixMarketError) as exc:
            load_matrix_market(path)
        assert exc.value.line == int(G[f"{name}_error_line"])
        assert str(exc.value).split(": ", 1)[-1] == str(G[f"{name}_error"])
        assert f":{exc.value.line}:" in str(exc.value)
        return
    A, meta = load_matrix_market(path)
    assert np.array_equal(A.row_ptr, G[f"{name}_rp"])
    assert np.array_equal(A.col_idx, G[f"{name}_ci"])
    assert np.array_equal(A.values, G[f"{name}_v"])
    assert A.shape == tuple(G[f"{name}_shape"])
    assert meta.symmetric == bool(G[f"{name}_sym"])
    assert meta.name == name and meta.nnz == A.nnz


def test_symmetric_expansion_counts_mirrors(tmp_path):
    # test_mmio.py:42-55: two stored off-diagonals become four entries
    A, meta = load_matrix_market(_write(tmp_path, str(G["symmetric_text"])))
    assert meta.nnz == 6
    np.testing.assert_array_equal(A.to_dense(), [[2.0, -1.0, 0], [-1.0, 0.0, -1.0], [0, -1.0, 2.0]])


def test_missing_file_raises():
    with pytest.raises(FileNotFoundError):
        load_matrix_market("/no/such/dir/m.mtx")


def test_write_load_roundtrip_is_lossless(tmp_path):
    rng = np.random.default_rng(31)
    rows, cols = np.nonzero(rng.random((7, 5)) < 0.35)
    A = csr_from_coo(7, 5, rows, cols, rng.standard_normal(rows.size))
    path = str(tmp_path / "rt.mtx")
    write_matrix_market(path, A, comment="roundtrip check")
    B, _ = load_matrix_market(path)
    assert B.shape == A.shape
    for a, b in ((A.row_ptr, B.row_ptr), (A.col_idx, B.col_idx), (A.values, B.values)):
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_ingested_matrix_solves_bitwise_on_device(tmp_path):
    """Table 3's path (test_acceptance.py:74-147) with a generated file: write a
    convection-diffusion operator as Matrix Market, ingest it, solve on the
    B200 in plan order and compare with the oracle bitwise."""
    import paper_2108_10591_b200 as pb
    from oracle import oracle as orc
    from paper_2108_10591_b200 import problems

    rp, ci, v = problems.stencil_csr(problems.convdiff_stencil(2, 20, (1.0, 1.0)))
    n = len(rp) - 1
    path = str(tmp_path / "cd2d20.mtx")
    write_matrix_market(path, pb.CsrMatrix(n, n, rp, ci, v))
    A, meta = load_matrix_market(path)
    assert meta.nnz == len(v)
    b = orc.spmv(A.row_ptr, A.col_idx, A.values, np.ones(n))
    for method in ("pbicgsafe", "bicgstab"):
        ref = orc.solve(A.row_ptr, A.col_idx, A.values, b, method=method, tol=1e-10)
        out = pb.solve(A, b, method=method, config=pb.SolverConfig(tol=1e-10),
                       engine=pb.DeviceEngine(reduce="plan", workers=1))
        assert out.iterations == ref["iterations"]
        assert np.array_equal([r.rel_res_recur for r in out.history], ref["rel"])
        assert np.array_equal(out.x, ref["x"])
