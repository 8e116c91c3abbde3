"""Pin the CPU oracle (oracle/) to the reference's own outputs (tests/golden/).

The oracle is only trusted as a parity checker once it reproduces the
reference BITWISE: kernels, plans, coefficients, and full solver histories
(every rel, every coefficient, flags, status, iteration count and x) on the
recorded systems, including a 3-range and an 8-range PartitionPlan.
"""

import os

import numpy as np
import pytest

from oracle import oracle as orc
from tests import golden_cases as gc

G = gc.GOLDEN


def test_oracle_builds_and_loads():
    orc.build()
    assert os.path.exists(orc.LIB_PATH)
    orc.lib()


def test_kernels_bitwise():
    k = np.load(os.path.join(G, "kernels.npz"))
    for name in ("spmv_a", "spmv_b", "spmv_c", "spmv_big"):
        y = orc.spmv(k[f"{name}_rp"], k[f"{name}_ci"], k[f"{name}_v"], k[f"{name}_x"])
        assert np.array_equal(y, k[f"{name}_y"]), name
    y = np.full(3, 99.0)
    orc.spmv_range(k["spmv_empty_rp"], k["spmv_empty_ci"], k["spmv_empty_v"], np.ones(3), y, 0, 3)
    assert np.array_equal(y, k["spmv_empty_y"])
    assert orc.dot_range(k["dot_x"], k["dot_y"], 0, 257) == k["dot_full"]
    assert orc.dot_range(k["dot_x"], k["dot_y"], 31, 200) == k["dot_sub"]
    a, b, c, d = k["lc_a"], k["lc_b"], k["lc_c"], k["lc_d"]
    o = np.empty(1000)
    orc.lincomb2(o, 2.0, a, -0.3, b)
    assert np.array_equal(o, k["lc2"])
    orc.lincomb3(o, 1.5, a, -0.7, b, 0.25, c)
    assert np.array_equal(o, k["lc3"])
    orc.lincomb4(o, 1.0, a, -1.0, b, -0.5, c, 0.3, d)
    assert np.array_equal(o, k["lc4"])
    orc.lincomb_nested(o, 0.7, a, 0.3, b, -2.1, c)
    assert np.array_equal(o, k["lcn"])
    orc.add_scaled_diff(o, a, 0.8, b, c)
    assert np.array_equal(o, k["asd"])
    orc.add_scaled_damped_diff(o, a, 0.8, b, 0.3, c)
    assert np.array_equal(o, k["asdd"])


def test_plans_match_reference():
    p = np.load(os.path.join(G, "plans.npz"))
    pos = 0
    for n, w, ln in zip(p["n"], p["w"], p["lens"]):
        ref = p["bounds"][pos:pos + ln]
        pos += ln
        assert np.array_equal(orc.plan_bounds(int(n), int(w)), ref), (n, w)


def _same(a, b):
    return (a == b) or (np.isnan(a) and np.isnan(b))


def test_coefficients_match_reference():
    c = np.load(os.path.join(G, "coeffs.npz"))
    for inp, out in zip(c["ab_in"], c["ab_out"]):
        q, a, bt = orc.alpha_beta_safe(*inp[:6], bool(inp[6]))
        assert q == int(out[0]), inp
        if q == 0:
            assert _same(a, out[1]) and _same(bt, out[2]), inp
    for inp, out in zip(c["ze_in"], c["ze_out"]):
        q, z, e = orc.zeta_eta_safe(*inp[:5], bool(inp[5]))
        assert q == int(out[0]), inp
        if q == 0:
            assert _same(z, out[1]) and _same(e, out[2]), inp


def test_gpbicg_coefficients_match_reference():
    c = np.load(os.path.join(G, "coeffs_gpbicg.npz"))
    for inp, out in zip(c["gz_in"], c["gz_out"]):
        q, z, e = orc.zeta_eta_gpbicg(*inp[:5], bool(inp[5]))
        assert q == int(out[0]), inp
        if q == 0:
            assert _same(z, out[1]) and _same(e, out[2]), inp


@pytest.mark.parametrize("name", gc.case_names())
def test_solver_history_bitwise(name):
    spec, A, b, x0, g = gc.load_case(name, orc.spmv)
    out = orc.solve(A.row_ptr, A.col_idx, A.values, b, x0=x0, method=spec["method"],
                    tol=spec["tol"], max_iters=spec["max_iters"],
                    rr_epoch=spec.get("rr_epoch", 100), rr_cutoff=spec.get("rr_cutoff"),
                    workers=spec["workers"])
    assert out["status"] == str(g["status"])
    assert out["iterations"] == int(g["iterations"])
    assert out["r0_norm"] == float(g["r0_norm"])
    assert np.array_equal(out["rel"], g["rel"])
    assert np.array_equal(out["replaced"], g["replaced"])
    assert np.array_equal(out["has_coef"], g["has_coef"])
    assert np.array_equal(out["coef"][out["has_coef"]], g["coef"][g["has_coef"]], equal_nan=True)
    assert (out["breakdown"] or "") == str(g["breakdown"])
    assert (-1 if out["failure_iter"] is None else out["failure_iter"]) == int(g["failure_iter"])
    assert out["n_spmv"] == int(g["n_spmv"])
    assert np.array_equal(out["x"], g["x"])


@pytest.mark.parametrize("name", gc.case_names(trace=True))
def test_trace_vectors_bitwise(name):
    spec, A, b, x0, g = gc.load_case(name, orc.spmv, trace=True)
    got = {}
    orc.solve(A.row_ptr, A.col_idx, A.values, b, x0=x0, method=spec["method"], tol=spec["tol"],
              max_iters=spec["max_iters"], rr_epoch=spec.get("rr_epoch", 100),
              workers=spec["workers"], trace=lambda i, v, s: got.__setitem__(i, v))
    assert sorted(got) == list(g["trace_iters"])
    for i in g["trace_iters"]:
        for name_v in orc.TRACE_NAMES_BY_METHOD.get(spec["method"], orc.TRACE_NAMES[:13]):
            assert np.array_equal(got[i][name_v], g[f"it{i}_{name_v}"]), (i, name_v)


def test_nonfinite_matrix_raises_like_reference():
    g = np.load(os.path.join(G, "nonfinite.npz"))
    out = orc.solve(np.array([0, 1, 2]), np.array([0, 1]), np.array([np.nan, 1.0]), np.ones(2))
    assert out["raised"] == "NonFiniteVectorError"
    assert out["index"] == int(g["index"])


def test_threads_do_not_change_bits():
    spec, A, b, x0, g = gc.load_case("cd3d16_w8", orc.spmv)
    outs = [orc.solve(A.row_ptr, A.col_idx, A.values, b, tol=spec["tol"], workers=8, threads=t)
            for t in (1, 3, 8)]
    for o in outs:
        assert np.array_equal(o["rel"], g["rel"]) and np.array_equal(o["x"], g["x"])
