"""Generate tests/golden/*.npz by running the REFERENCE (pipesafe) in this container.

Run from the repo root (needs /root/reference, which does not exist on the
GPU box — hence the committed fixtures):

    python tests/golden/make_golden.py

Everything is seeded; re-running reproduces the same files bitwise.  What is
recorded:

* kernels.npz   — the reference's numba kernels (kernels.py:95-137) on the
                  inputs of its own kernel tests (test_kernels.py seeds) and
                  on a few larger seeded cases;
* plans.npz     — PartitionPlan.balanced bounds (reduction.py:80-87);
* coeffs.npz    — compute_alpha_beta_safe / compute_zeta_eta_safe outputs and
                  breakdown quantities (coefficients.py:35-106);
* solve_<case>.npz — full solver outcomes (history, coefficients, flags,
                  status, x) of solve() (solvers.py:791-803) on the systems
                  listed in CASES, plus a SHA-256 of the CSR arrays so the
                  repo's generators are pinned to the matrices used here;
* trace_<case>.npz — per-iteration workspace vectors captured through
                  trace_hook (solvers.py:725-732) for single-step parity.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)

import pipesafe  # noqa: E402  (the reference, read-only)
from pipesafe import kernels as kn  # noqa: E402
from pipesafe.coefficients import (  # noqa: E402
    BreakdownError,
    compute_alpha_beta_safe,
    compute_zeta_eta_gpbicg,
    compute_zeta_eta_safe,
)
from pipesafe.linalg import NonFiniteVectorError, csr_from_coo, gen_poisson, spmv  # noqa: E402
from pipesafe.reduction import PartitionPlan, ReductionEngine  # noqa: E402
from pipesafe.solvers import SolverConfig, solve  # noqa: E402

from paper_2108_10591_b200 import problems  # noqa: E402


def csr_sha(rp, ci, v) -> str:
    h = hashlib.sha256()
    for a, dt in ((rp, np.int64), (ci, np.int64), (v, np.float64)):
        h.update(np.ascontiguousarray(a, dtype=dt).tobytes())
    return h.hexdigest()


# ---------------------------------------------------------------- matrices

def system(spec: dict):
    """Build (CsrMatrix, b, x0) for a case spec; the same spec is rebuilt by
    tests/golden_cases.py from the repo's own generators."""
    kind = spec["matrix"]
    if kind == "poisson":
        A, _ = gen_poisson(spec["dim"], spec["k"])
    elif kind == "convdiff":
        st = problems.convdiff_stencil(spec["dim"], spec["k"], spec["beta"])
        rp, ci, v = problems.stencil_csr(st)
        A = pipesafe.CsrMatrix(len(rp) - 1, len(rp) - 1, rp, ci, v)
    elif kind == "convdiff27":
        st = problems.convdiff27_stencil(spec["k"], spec["beta"])
        rp, ci, v = problems.stencil_csr(st)
        A = pipesafe.CsrMatrix(len(rp) - 1, len(rp) - 1, rp, ci, v)
    elif kind == "random":
        rp, ci, v, _ = problems.random_banded_csr(spec["n"], seed=spec["seed"],
                                                  half_window=spec["half_window"])
        A = pipesafe.CsrMatrix(len(rp) - 1, len(rp) - 1, rp, ci, v)
    elif kind == "identity":
        n = spec["n"]
        A = csr_from_coo(n, n, np.arange(n), np.arange(n), np.ones(n))
    elif kind == "exchange":
        A = csr_from_coo(2, 2, np.array([0, 1]), np.array([1, 0]), np.array([1.0, 1.0]))
    else:
        raise ValueError(kind)
    A.validate()
    rhs = spec.get("rhs", "ones")
    n = A.n_rows
    if rhs == "ones":
        b = spmv(A, np.ones(n))
    elif rhs == "zero":
        b = np.zeros(n)
    elif rhs == "e1":
        b = np.zeros(n)
        b[0] = 1.0
    elif rhs.startswith("rng"):
        b = np.random.default_rng(int(rhs[3:])).standard_normal(n)
    elif rhs == "random_u01":
        _, _, _, b = problems.random_banded_csr(spec["n"], seed=spec["seed"],
                                                half_window=spec["half_window"])
    else:
        raise ValueError(rhs)
    x0 = None
    if "x0" in spec:
        x0 = np.random.default_rng(int(spec["x0"][3:])).standard_normal(n)
    return A, b, x0


def canonical_check(A):
    """The repo generators must emit exactly what csr_from_coo returns."""
    rows, cols, vals = A.to_coo()
    perm = np.random.default_rng(0).permutation(rows.size)
    B = csr_from_coo(A.n_rows, A.n_cols, rows[perm], cols[perm], vals[perm])
    assert np.array_equal(A.row_ptr, B.row_ptr)
    assert np.array_equal(A.col_idx, B.col_idx)
    assert np.array_equal(A.values, B.values)


from _cases import CASES, TRACE_CASES  # noqa: E402


def run_case(spec, trace=False):
    A, b, x0 = system(spec)
    if spec["matrix"] in ("convdiff", "convdiff27", "random"):
        canonical_check(A)
    cfg = SolverConfig(tol=spec["tol"], max_iters=spec["max_iters"],
                       rr_epoch=spec.get("rr_epoch", 100), rr_cutoff=spec.get("rr_cutoff"))
    eng = ReductionEngine(PartitionPlan.balanced(A.n_rows, spec["workers"]), mode="inline")
    traces = {}

    def hook(i, ws):
        traces[i] = {k: v.copy() for k, v in ws.items()}

    out = solve(A, b, method=spec["method"], x0=x0, config=cfg, engine=eng,
                trace_hook=hook if trace else None)
    hist = out.history
    coef = np.full((len(hist), 4), np.nan)
    has = np.zeros(len(hist), dtype=bool)
    for j, rec in enumerate(hist):
        if rec.coefficients is not None:
            c = rec.coefficients
            # BiCGStab's CoefficientSet carries omega, stored in the zeta column
            coef[j] = (c.alpha, c.beta, c.omega if c.omega is not None else c.zeta, c.eta)
            has[j] = True
    payload = dict(
        csr_sha=np.array(csr_sha(A.row_ptr, A.col_idx, A.values)),
        n=np.int64(A.n_rows),
        nnz=np.int64(A.nnz),
        status=np.array(out.status.value),
        iterations=np.int64(out.iterations),
        r0_norm=np.float64(out.r0_norm),
        rel=np.array([r.rel_res_recur for r in hist]),
        iters=np.array([r.iter for r in hist], dtype=np.int64),
        replaced=np.array([r.replaced for r in hist], dtype=bool),
        coef=coef,
        has_coef=has,
        final_rel=np.float64(out.final_rel_res_recur),
        best_rel=np.float64(out.best_rel_res_recur),
        breakdown=np.array(out.breakdown_quantity or ""),
        failure_iter=np.int64(-1 if out.failure_iter is None else out.failure_iter),
        n_spmv=np.int64(out.counters.n_spmv),
        n_dots=np.int64(out.counters.n_dots),
        n_reductions=np.int64(out.counters.n_reductions),
        x=out.x,
        b=b,
    )
    if trace:
        for i, ws in traces.items():
            for k, v in ws.items():
                payload[f"it{i}_{k}"] = v
        payload["trace_iters"] = np.array(sorted(traces), dtype=np.int64)
    return payload


def kernels_fixture():
    kn.set_backend("numba")
    out = {}

    def random_csr(rng, n_rows, n_cols, density=0.2):
        mask = rng.random((n_rows, n_cols)) < density
        rows, cols = np.nonzero(mask)
        vals = rng.standard_normal(rows.size)
        return csr_from_coo(n_rows, n_cols, rows, cols, vals)

    # test_kernels.py:63-73, 76-85, 88-94 inputs
    for name, seed, n in (("spmv_a", 7, 40), ("spmv_b", 8, 30), ("spmv_c", 11, 80)):
        rng = np.random.default_rng(seed)
        A = random_csr(rng, n, n)
        x = rng.standard_normal(n)
        y = np.empty(n)
        kn.spmv_range(A.row_ptr, A.col_idx, A.values, x, y, 0, n)
        out.update({f"{name}_rp": A.row_ptr, f"{name}_ci": A.col_idx, f"{name}_v": A.values,
                    f"{name}_x": x, f"{name}_y": y})
    A = csr_from_coo(3, 3, np.array([1, 1]), np.array([0, 2]), np.array([2.0, 3.0]))
    y = np.full(3, 99.0)
    kn.spmv_range(A.row_ptr, A.col_idx, A.values, np.ones(3), y, 0, 3)
    out.update({"spmv_empty_rp": A.row_ptr, "spmv_empty_ci": A.col_idx,
                "spmv_empty_v": A.values, "spmv_empty_y": y})
    # a larger irregular case: rows 0..60 nnz, heavy cancellation
    rng = np.random.default_rng(2108)
    n = 3000
    counts = rng.integers(0, 61, size=n)
    rows = np.repeat(np.arange(n), counts)
    cols = rng.integers(0, n, size=rows.size)
    vals = rng.standard_normal(rows.size) * 10.0 ** rng.integers(-8, 9, size=rows.size)
    A = csr_from_coo(n, n, rows, cols, vals)
    x = rng.standard_normal(n)
    y = np.empty(n)
    kn.spmv_range(A.row_ptr, A.col_idx, A.values, x, y, 0, n)
    out.update({"spmv_big_rp": A.row_ptr, "spmv_big_ci": A.col_idx, "spmv_big_v": A.values,
                "spmv_big_x": x, "spmv_big_y": y})
    # dots and linear combinations (test_kernels.py:47-60, 97-160)
    rng = np.random.default_rng(42)
    x, y = rng.standard_normal(257), rng.standard_normal(257)
    out.update({"dot_x": x, "dot_y": y, "dot_full": np.float64(kn.dot_range(x, y, 0, 257)),
                "dot_sub": np.float64(kn.dot_range(x, y, 31, 200))})
    rng = np.random.default_rng(5)
    a, b, c, d = rng.standard_normal((4, 1000)) * 10.0 ** rng.integers(-5, 6, size=(4, 1000))
    out.update({"lc_a": a, "lc_b": b, "lc_c": c, "lc_d": d})
    o = np.empty(1000)
    kn.lincomb2(o, 2.0, a, -0.3, b)
    out["lc2"] = o.copy()
    kn.lincomb3(o, 1.5, a, -0.7, b, 0.25, c)
    out["lc3"] = o.copy()
    kn.lincomb4(o, 1.0, a, -1.0, b, -0.5, c, 0.3, d)
    out["lc4"] = o.copy()
    kn.lincomb_nested(o, 0.7, a, 0.3, b, -2.1, c)
    out["lcn"] = o.copy()
    kn.add_scaled_diff(o, a, 0.8, b, c)
    out["asd"] = o.copy()
    kn.add_scaled_damped_diff(o, a, 0.8, b, 0.3, c)
    out["asdd"] = o.copy()
    return out


def plans_fixture():
    ns, ws, bounds = [], [], []
    for n in (0, 1, 2, 7, 100, 4096, 12345, 2097152, 4000000, 16777216, 56623104):
        for w in (1, 2, 3, 4, 7, 8, 64, 148, 1000):
            p = PartitionPlan.balanced(n, w)
            ns.append(n)
            ws.append(w)
            bounds.append(np.array([lo for lo, _ in p.ranges] + [p.ranges[-1][1]]))
    flat = np.concatenate(bounds)
    lens = np.array([len(b) for b in bounds])
    return dict(n=np.array(ns), w=np.array(ws), lens=lens, bounds=flat)


def coeffs_fixture():
    rng = np.random.default_rng(4242)
    rows = []
    names = {"initial alpha denominator (r0*, s)": 1, "beta denominator zeta_prev * f_prev": 2,
             "alpha denominator g + beta*h": 3, "zeta denominator (s, s)": 4,
             "zeta/eta denominator a*b - c^2": 5}
    special = [
        (1.0, 1.0, 1.0, 1.0, 1.0, 1.0, 0),
        (2.0, 0.0, 4.0, 0.0, 0.0, 0.0, 1),
        (1.0, 0.0, 0.0, 0.0, 0.0, 0.0, 1),
        (1.0, 0.0, 1.0, 0.0, 1.0, 1.0, 0),
        (1.0, 1.0, 1.0, -1.0, 1.0, 1.0, 0),
        (np.nan, 1.0, 1.0, 1.0, 1.0, 1.0, 0),
    ]
    ab_in, ab_out = [], []
    for f, fp, g, h, ap, zp, first in special + [
        tuple(rng.standard_normal(6)) + (int(rng.random() < 0.1),) for _ in range(500)
    ]:
        try:
            a, bt = compute_alpha_beta_safe(f, fp, g, h, ap, zp, bool(first))
            q = 0
        except BreakdownError as e:
            a, bt, q = np.nan, np.nan, names[e.quantity]
        ab_in.append((f, fp, g, h, ap, zp, first))
        ab_out.append((q, a, bt))
    ze_in, ze_out = [], []
    special = [
        (1.0, 1.0, 0.0, 0.5, 0.25, 0),
        (4.0, 0.0, 0.0, 2.0, 0.0, 1),
        (2.0, 0.0, 0.0, 1.0, 0.0, 0),
        (1.0, 1.0, 1.0 - 1e-16, 0.5, 0.5, 0),
        (0.0, 0.0, 0.0, 1.0, 0.0, 1),
        (14.0, 56.0, 28.0, 4.0, 8.0, 0),
    ]
    rnd = []
    for _ in range(500):
        s, y, r = rng.standard_normal((3, 6))
        rnd.append((s @ s, y @ y, s @ y, s @ r, y @ r, int(rng.random() < 0.1)))
    for a, b, c, d, e, first in special + rnd:
        try:
            z, et = compute_zeta_eta_safe(a, b, c, d, e, bool(first))
            q = 0
        except BreakdownError as ex:
            z, et, q = np.nan, np.nan, names[ex.quantity]
        ze_in.append((a, b, c, d, e, first))
        ze_out.append((q, z, et))
    return dict(ab_in=np.array(ab_in, dtype=np.float64), ab_out=np.array(ab_out),
                ze_in=np.array(ze_in, dtype=np.float64), ze_out=np.array(ze_out))


def coeffs_gpbicg_fixture():
    """compute_zeta_eta_gpbicg (coefficients.py:109-135): the reference's own
    hand values (test_coefficients.py:53-63, 135-138, 187-194) plus seeded
    random normal-equation inputs."""
    rng = np.random.default_rng(4243)
    names = {"zeta denominator (At, At)": 10, "zeta/eta denominator e*a - d^2": 11}
    special = [
        (0.0, 3.0, 0.0, 0.0, 6.0, 1),
        (1.0, 4.0, 1.0, 0.0, 2.0, 0),
        (0.0, 3.0, 0.0, 0.0, 6.0, 0),
        (0.0, 0.0, 0.0, 0.0, 0.0, 1),
        (0.0, 1.0, 0.0, 0.0, 0.0, 0),
        (0.0, 1.0, 0.0, 0.0, 1e-320, 1),
        (1.0, 1.0, 1.0, 1.0, 1.0, 0),
        (4.0, 1.0, 2.0, 2.0, 1.0, 0),
        (np.nan, 1.0, 1.0, 1.0, 1.0, 0),
    ]
    rnd = []
    for _ in range(500):
        y, t, at = rng.standard_normal((3, 6))
        rnd.append((y @ y, at @ t, y @ t, at @ y, at @ at, int(rng.random() < 0.1)))
    gz_in, gz_out = [], []
    for a, b, c, d, e, first in special + rnd:
        try:
            z, et = compute_zeta_eta_gpbicg(a, b, c, d, e, bool(first))
            q = 0
        except BreakdownError as ex:
            z, et, q = np.nan, np.nan, names[ex.quantity]
        gz_in.append((a, b, c, d, e, first))
        gz_out.append((q, z, et))
    return dict(gz_in=np.array(gz_in, dtype=np.float64), gz_out=np.array(gz_out))


# Matrix Market texts the reference's loader (mmio.py:33-137) is run on;
# bad ones record the line number its error names
MM_TEXTS = {
    "general": "%%MatrixMarket matrix coordinate real general\n% c\n3 3 4\n1 1 2.0\n2 2 -1.5\n3 1 4.0\n3 3 0.5\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 4\n1 1 2.0\n2 1 -1.0\n3 2 -1.0\n3 3 2.0\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 1 3\n2 2 -4\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n1 1 2.5\n2 2 1.0\n",
    "blank_and_comments": "%%MatrixMarket matrix coordinate real general\n%x\n\n2 3 2\n% y\n1 3 1e-3\n\n2 1 -7\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n4 4 0\n",
    "bad_header": "%%NotMatrixMarket nope\n1 1 0\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n3 x 1\n1 1 1.0\n",
    "count_mismatch": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n2 2 1.0\n",
    "bad_entry": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 oops 1.0\n",
    "short_entry": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n3 1 1.0\n",
    "frac_index": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1.5 1 1.0\n",
    "sym_rect": "%%MatrixMarket matrix coordinate real symmetric\n2 3 1\n1 1 1.0\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n1 1 1\n1 1\n",
    "negative": "%%MatrixMarket matrix coordinate real general\n-1 2 0\n",
}


def mmio_fixture(tmpdir):
    from pipesafe.mmio import MatrixMarketError, load_matrix_market, write_matrix_market

    out = {}
    rng = np.random.default_rng(31)
    rows, cols = np.nonzero(rng.random((40, 30)) < 0.2)
    R = csr_from_coo(40, 30, rows, cols, rng.standard_normal(rows.size))
    path = os.path.join(tmpdir, "rt.mtx")
    write_matrix_market(path, R, comment="roundtrip\ncheck")
    with open(path) as fh:
        texts = dict(MM_TEXTS, roundtrip=fh.read())
    for name, text in texts.items():
        path = os.path.join(tmpdir, f"{name}.mtx")
        with open(path, "w") as fh:
            fh.write(text)
        out[f"{name}_text"] = np.array(text)
        try:
            A, meta = load_matrix_market(path)
            out[f"{name}_rp"] = A.row_ptr
            out[f"{name}_ci"] = A.col_idx
            out[f"{name}_v"] = A.values
            out[f"{name}_shape"] = np.array(A.shape, dtype=np.int64)
            out[f"{name}_sym"] = np.array(meta.symmetric)
        except MatrixMarketError as e:
            out[f"{name}_error_line"] = np.int64(-1 if e.line is None else e.line)
            out[f"{name}_error"] = np.array(str(e).split(": ", 1)[-1])
    return out


def main():
    # --only PREFIX regenerates just the solve/trace cases whose name starts with it
    only = sys.argv[sys.argv.index("--only") + 1] if "--only" in sys.argv else None
    if only is None or only == "gp_":
        np.savez_compressed(os.path.join(HERE, "coeffs_gpbicg.npz"), **coeffs_gpbicg_fixture())
    if only is None or only == "mmio":
        import tempfile

        with tempfile.TemporaryDirectory() as td:
            np.savez_compressed(os.path.join(HERE, "mmio.npz"), **mmio_fixture(td))
    if only is None:
        np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernels_fixture())
        np.savez_compressed(os.path.join(HERE, "plans.npz"), **plans_fixture())
        np.savez_compressed(os.path.join(HERE, "coeffs.npz"), **coeffs_fixture())
    for name, spec in CASES.items():
        if only is not None and not name.startswith(only):
            continue
        payload = run_case(spec)
        if payload["n"] > 5000:
            del payload["b"]  # rebuilt from the generator + pinned by csr_sha
        np.savez_compressed(os.path.join(HERE, f"solve_{name}.npz"), **payload)
        print(name, str(payload["status"]), int(payload["iterations"]))
    for name, spec in TRACE_CASES.items():
        if only is not None and not name.startswith(only):
            continue
        payload = run_case(spec, trace=True)
        np.savez_compressed(os.path.join(HERE, f"trace_{name}.npz"), **payload)
        print("trace", name, str(payload["status"]), int(payload["iterations"]))
    if only is not None:
        return
    # non-finite matrix raises (test_solvers.py:226-230)
    A = csr_from_coo(2, 2, np.array([0, 1]), np.array([0, 1]), np.array([1.0, 1.0]))
    A.values[0] = np.nan
    try:
        solve(A, np.ones(2), method="pbicgsafe")
        raise SystemExit("expected NonFiniteVectorError")
    except NonFiniteVectorError as e:
        np.savez_compressed(os.path.join(HERE, "nonfinite.npz"), index=np.int64(e.index),
                            message=np.array(str(e)))


if __name__ == "__main__":
    main()
