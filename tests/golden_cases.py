"""Rebuild the systems behind tests/golden/*.npz from the repo's own generators.

The fixture records the SHA-256 of the CSR arrays the reference solved
(make_golden.py), so ``load_case`` fails loudly if a generator drifts.
Right-hand sides b = A·1 are recomputed with the oracle's sequential SpMV,
which equals the reference's (kernels.py:95-100) bitwise.
"""

from __future__ import annotations

import hashlib
import os

import numpy as np

from paper_2108_10591_b200 import problems
from paper_2108_10591_b200.linalg import CsrMatrix, csr_from_coo, gen_poisson

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _spec_module():
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden_specs", os.path.join(GOLDEN, "_cases.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def csr_sha(rp, ci, v) -> str:
    h = hashlib.sha256()
    for a, dt in ((rp, np.int64), (ci, np.int64), (v, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


def build_matrix(spec: dict) -> CsrMatrix:
    kind = spec["matrix"]
    if kind == "poisson":
        A, _ = gen_poisson(spec["dim"], spec["k"])
        return A
    if kind == "convdiff":
        rp, ci, v = problems.stencil_csr(problems.convdiff_stencil(spec["dim"], spec["k"], spec["beta"]))
    elif kind == "convdiff27":
        rp, ci, v = problems.stencil_csr(problems.convdiff27_stencil(spec["k"], spec["beta"]))
    elif kind == "random":
        rp, ci, v, _ = problems.random_banded_csr(spec["n"], seed=spec["seed"], half_window=spec["half_window"])
    elif kind == "identity":
        n = spec["n"]
        return csr_from_coo(n, n, np.arange(n), np.arange(n), np.ones(n))
    elif kind == "exchange":
        return csr_from_coo(2, 2, np.array([0, 1]), np.array([1, 0]), np.array([1.0, 1.0]))
    else:
        raise ValueError(kind)
    n = len(rp) - 1
    return CsrMatrix(n, n, rp, ci, v)


def build_rhs(spec: dict, A: CsrMatrix, spmv) -> np.ndarray:
    rhs = spec.get("rhs", "ones")
    n = A.n_rows
    if rhs == "ones":
        return spmv(A.row_ptr, A.col_idx, A.values, np.ones(n))
    if rhs == "zero":
        return np.zeros(n)
    if rhs == "e1":
        b = np.zeros(n)
        b[0] = 1.0
        return b
    if rhs.startswith("rng"):
        return np.random.default_rng(int(rhs[3:])).standard_normal(n)
    if rhs == "random_u01":
        return problems.random_banded_csr(spec["n"], seed=spec["seed"], half_window=spec["half_window"])[3]
    raise ValueError(rhs)


def build_x0(spec: dict, n: int):
    if "x0" not in spec:
        return None
    return np.random.default_rng(int(spec["x0"][3:])).standard_normal(n)


def load_case(name: str, spmv, trace: bool = False):
    """Return (spec, A, b, x0, golden dict) for a solve_/trace_ fixture."""
    mod = _spec_module()
    spec = (mod.TRACE_CASES if trace else mod.CASES)[name]
    g = dict(np.load(os.path.join(GOLDEN, f"{'trace' if trace else 'solve'}_{name}.npz")))
    A = build_matrix(spec)
    assert csr_sha(A.row_ptr, A.col_idx, A.values) == str(g["csr_sha"]), f"generator drift in {name}"
    b = build_rhs(spec, A, spmv)
    if "b" in g:
        assert np.array_equal(b, g["b"]), f"rhs drift in {name}"
    return spec, A, b, build_x0(spec, A.n_rows), g


def case_names(trace: bool = False):
    mod = _spec_module()
    return list((mod.TRACE_CASES if trace else mod.CASES).keys())


def case_spec(name: str, trace: bool = False) -> dict:
    mod = _spec_module()
    return (mod.TRACE_CASES if trace else mod.CASES)[name]
