"""ctypes front end of the CPU parity oracle (pbsafe_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package.  Every function restates a reference function (file:line cited in
pbsafe_oracle.c) with the reference's evaluation order, so the oracle run
with ``workers=W`` is bitwise equal to the reference solver driven by
``ReductionEngine(PartitionPlan.balanced(n, W))`` — pinned by
tests/test_oracle.py against tests/golden/.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

STATUS = {0: "converged", 1: "max_iters", 2: "breakdown", 3: "non_finite"}
METHOD_IDS = {"pbicgsafe": 0, "pbicgsafe-rr": 1, "ssbicgsafe2": 2, "bicgstab": 3, "gpbicg": 4,
              "pbicgstab": 5}
# coefficients.py:77, 80, 83, 102, 105
BREAKDOWN_QUANTITIES = {
    1: "initial alpha denominator (r0*, s)",
    2: "beta denominator zeta_prev * f_prev",
    3: "alpha denominator g + beta*h",
    4: "zeta denominator (s, s)",
    5: "zeta/eta denominator a*b - c^2",
    # solvers.py:275, 283, 302, 303 (BiCGStab), 434 (GPBi-CG); coefficients.py:130, 134
    6: "alpha denominator (r0*, Ap)",
    7: "omega denominator (At, At)",
    8: "beta denominator omega",
    9: "beta denominator (r0*, r)",
    10: "zeta denominator (At, At)",
    11: "zeta/eta denominator e*a - d^2",
    12: "beta denominator zeta",
    # p-BiCGStab (pbsafe_oracle.c solve_pstab; not in the reference)
    13: "alpha denominator (r0*, w) + beta*((r0*, s) - omega*(r0*, z))",
    14: "omega denominator (y, y)",
}
SPMV_TAGS = {1: "Ax", 2: "Ar", 3: "As", 4: "Aw", 5: "Ao", 6: "Au", 7: "At", 8: "Ay", 9: "Ap", 10: "Az"}
TRACE_NAMES = ("x", "r", "p", "u", "o", "t", "w", "y", "z", "s", "q", "g", "l", "r0s")
# trace_hook dicts of the product-type methods (solvers.py:315, 448)
TRACE_NAMES_BY_METHOD = {"bicgstab": ("x", "r", "p", "t", "Ap", "At"),
                         "gpbicg": ("x", "r", "p", "u", "t", "w", "y", "z"),
                         "pbicgstab": ("x", "r", "p", "s", "z", "q", "y", "w", "t", "v")}


class _Config(C.Structure):
    _fields_ = [("tol", C.c_double), ("max_iters", C.c_int64), ("rr_epoch", C.c_int64),
                ("rr_cutoff", C.c_int64), ("method", C.c_int32), ("workers", C.c_int32),
                ("threads", C.c_int32), ("pad", C.c_int32)]


class _Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("breakdown", C.c_int32), ("iterations", C.c_int64),
                ("failure_iter", C.c_int64), ("n_records", C.c_int64), ("r0_norm", C.c_double),
                ("nonfinite_tag", C.c_int32), ("pad", C.c_int32), ("nonfinite_index", C.c_int64),
                ("n_spmv", C.c_int64)]


_TRACE_FN = C.CFUNCTYPE(None, C.c_int64, C.POINTER(C.POINTER(C.c_double)),
                        C.POINTER(C.c_double), C.c_void_p)

_lib = None


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        d, i64, p = C.c_double, C.c_int64, C.c_void_p
        L.or_spmv_range.argtypes = [p, p, p, p, p, i64, i64]
        L.or_dot_range.argtypes = [p, p, i64, i64]
        L.or_dot_range.restype = d
        L.or_lincomb2.argtypes = [i64, p, d, p, d, p]
        L.or_lincomb3.argtypes = [i64, p, d, p, d, p, d, p]
        L.or_lincomb4.argtypes = [i64, p, d, p, d, p, d, p, d, p]
        L.or_lincomb_nested.argtypes = [i64, p, d, p, d, p, d, p]
        L.or_add_scaled_diff.argtypes = [i64, p, p, d, p, p]
        L.or_add_scaled_damped_diff.argtypes = [i64, p, p, d, p, d, p]
        L.or_plan_balanced.argtypes = [i64, i64, p]
        L.or_plan_balanced.restype = i64
        L.or_plan_dot.argtypes = [i64, i64, p, p]
        L.or_plan_dot.restype = d
        L.or_alpha_beta_safe.argtypes = [d, d, d, d, d, d, C.c_int, p]
        L.or_zeta_eta_safe.argtypes = [d, d, d, d, d, C.c_int, p]
        L.or_zeta_eta_gpbicg.argtypes = [d, d, d, d, d, C.c_int, p]
        L.or_solve.argtypes = [i64, p, p, p, p, p, C.POINTER(_Config), p, p, p, p, p,
                               C.POINTER(_Result), _TRACE_FN, p]
        L.or_solve.restype = C.c_int
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# -- kernels (kernels.py:95-137) ---------------------------------------------

def spmv_range(row_ptr, col_idx, values, x, out, lo, hi):
    rp, ci, v, xx = _i64(row_ptr), _i64(col_idx), _f64(values), _f64(x)
    lib().or_spmv_range(_ptr(rp), _ptr(ci), _ptr(v), _ptr(xx), _ptr(out), lo, hi)


def spmv(row_ptr, col_idx, values, x):
    n = len(row_ptr) - 1
    out = np.empty(n)
    spmv_range(row_ptr, col_idx, values, x, out, 0, n)
    return out


def dot_range(x, y, lo, hi):
    return lib().or_dot_range(_ptr(_f64(x)), _ptr(_f64(y)), lo, hi)


def lincomb2(out, sa, a, sb, b):
    lib().or_lincomb2(out.shape[0], _ptr(out), sa, _ptr(_f64(a)), sb, _ptr(_f64(b)))


def lincomb3(out, sa, a, sb, b, sc, c):
    lib().or_lincomb3(out.shape[0], _ptr(out), sa, _ptr(_f64(a)), sb, _ptr(_f64(b)), sc,
                      _ptr(_f64(c)))


def lincomb4(out, sa, a, sb, b, sc, c, sd, d):
    lib().or_lincomb4(out.shape[0], _ptr(out), sa, _ptr(_f64(a)), sb, _ptr(_f64(b)), sc,
                      _ptr(_f64(c)), sd, _ptr(_f64(d)))


def lincomb_nested(out, sa, a, sb, b, sc, c):
    lib().or_lincomb_nested(out.shape[0], _ptr(out), sa, _ptr(_f64(a)), sb, _ptr(_f64(b)), sc,
                            _ptr(_f64(c)))


def add_scaled_diff(out, base, s, a, b):
    lib().or_add_scaled_diff(out.shape[0], _ptr(out), _ptr(_f64(base)), s, _ptr(_f64(a)),
                             _ptr(_f64(b)))


def add_scaled_damped_diff(out, base, s, a, w, b):
    lib().or_add_scaled_damped_diff(out.shape[0], _ptr(out), _ptr(_f64(base)), s,
                                    _ptr(_f64(a)), w, _ptr(_f64(b)))


def plan_bounds(n, workers):
    b = np.zeros(workers + 2, dtype=np.int64)
    w = lib().or_plan_balanced(n, workers, _ptr(b))
    return b[: w + 1]


def plan_dot(x, y, workers=1):
    x, y = _f64(x), _f64(y)
    return lib().or_plan_dot(workers, x.shape[0], _ptr(x), _ptr(y))


def alpha_beta_safe(f, f_prev, g, h, alpha_prev, zeta_prev, first):
    out = np.zeros(2)
    q = lib().or_alpha_beta_safe(f, f_prev, g, h, alpha_prev, zeta_prev, int(first), _ptr(out))
    return q, float(out[0]), float(out[1])


def zeta_eta_safe(a, b, c, d, e, first):
    out = np.zeros(2)
    q = lib().or_zeta_eta_safe(a, b, c, d, e, int(first), _ptr(out))
    return q, float(out[0]), float(out[1])


def zeta_eta_gpbicg(a, b, c, d, e, first):
    out = np.zeros(2)
    q = lib().or_zeta_eta_gpbicg(a, b, c, d, e, int(first), _ptr(out))
    return q, float(out[0]), float(out[1])


# -- solver (solvers.py:210-460, 485-592, 595-779) ------------------------------------

def solve(row_ptr, col_idx, values, b, x0=None, method="pbicgsafe", tol=1e-8, max_iters=10_000,
          rr_epoch=100, rr_cutoff=None, workers=1, threads=0, trace=None):
    """Run one oracle solve; returns a dict mirroring SolveOutcome's fields.

    ``trace(i, vecs: dict[name -> array copy], scalars: array)`` is called
    after every completed iteration like the reference's trace_hook
    (solvers.py:725-732); scalars = alpha, beta, zeta, eta, f_prev, 9 dots
    (bicgstab / gpbicg: alpha, beta, omega|zeta, eta, f, rr).  The
    coefficient record of bicgstab carries omega in the zeta column.
    """
    rp, ci, v, bb = _i64(row_ptr), _i64(col_idx), _f64(values), _f64(b)
    n = rp.shape[0] - 1
    x0a = None if x0 is None else _f64(x0)
    cfg = _Config(tol, max_iters, rr_epoch, -1 if rr_cutoff is None else rr_cutoff,
                  METHOD_IDS[method], workers, threads, 0)
    x = np.zeros(n)
    rel = np.zeros(max_iters + 1)
    repl = np.zeros(max_iters + 1, dtype=np.uint8)
    coef = np.zeros((max_iters + 1, 4))
    has = np.zeros(max_iters + 1, dtype=np.uint8)
    res = _Result()

    if trace is not None:
        def _cb(i, vecs, scalars, _user):
            d = {name: np.ctypeslib.as_array(vecs[k], shape=(n,)).copy()
                 for k, name in enumerate(TRACE_NAMES_BY_METHOD.get(method, TRACE_NAMES))}
            trace(int(i), d, np.ctypeslib.as_array(scalars, shape=(14,)).copy())
        cb = _TRACE_FN(_cb)
    else:
        cb = _TRACE_FN()
    rc = lib().or_solve(n, _ptr(rp), _ptr(ci), _ptr(v), _ptr(bb), _ptr(x0a), C.byref(cfg),
                        _ptr(x), _ptr(rel), _ptr(repl), _ptr(coef), _ptr(has), C.byref(res),
                        cb, None)
    if rc != 0:
        return {"raised": "NonFiniteVectorError", "tag": SPMV_TAGS[res.nonfinite_tag],
                "index": int(res.nonfinite_index)}
    k = int(res.n_records)
    return {
        "status": STATUS[res.status],
        "iterations": int(res.iterations),
        "x": x,
        "rel": rel[:k].copy(),
        "replaced": repl[:k].astype(bool),
        "coef": coef[:k].copy(),
        "has_coef": has[:k].astype(bool),
        "r0_norm": float(res.r0_norm),
        "breakdown": BREAKDOWN_QUANTITIES.get(res.breakdown),
        "failure_iter": None if res.failure_iter < 0 else int(res.failure_iter),
        "n_spmv": int(res.n_spmv),
    }
