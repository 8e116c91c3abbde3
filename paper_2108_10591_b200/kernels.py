"""The "cuda" kernel backend table (drop-in for pipesafe.kernels' _TABLES).

The reference binds its kernels by name through ``set_backend``
(kernels.py:140-202) with these signatures (kernels.py:95-137)::

    spmv_range(row_ptr, col_idx, values, x, out, lo, hi)
    dot_range(x, y, lo, hi) -> float
    lincomb2(out, sa, a, sb, b)            lincomb3(out, sa, a, sb, b, sc, c)
    lincomb4(out, sa, a, sb, b, sc, c, sd, d)
    lincomb_nested(out, sa, a, sb, b, sc, c)
    add_scaled_diff(out, base, s, a, b)    add_scaled_damped_diff(out, base, s, a, w, b)

Each entry here runs the sm_100a kernel through the C-ABI with host arrays
(copy in, kernel, copy out).  This is the parity seam — registering it with
``register(pipesafe.kernels)`` makes the reference's own kernel tests run on
the GPU — not the performance path, which keeps everything in HBM.
SpMV and the linear combinations are bitwise the reference's; dot_range
reduces in a fixed tree (tolerance parity, like the reference's numpy twin).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

_NAMES = ("spmv_range", "dot_range", "lincomb2", "lincomb3", "lincomb4", "lincomb_nested",
          "add_scaled_diff", "add_scaled_damped_diff")


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ctx():
    return _lib.context().handle


def _out_ok(out):
    if not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous
            and out.flags.writeable):
        raise TypeError("out must be a writable C-contiguous float64 array")


def spmv_range(row_ptr, col_idx, values, x, out, lo, hi):
    _out_ok(out)
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    v = _f64(values)
    xx = _f64(x)
    ctx = _ctx()
    rc = _lib.load().pbs_k_spmv_range(ctx, rp.shape[0] - 1, xx.shape[0], _p(rp), _p(ci), _p(v), _p(xx),
                                      _p(out), int(lo), int(hi))
    if rc == _lib.PBS_ERR_INVALID:
        raise ValueError(_lib.last_error(ctx))
    _lib.check(rc, ctx)


def dot_range(x, y, lo, hi):
    xx, yy = _f64(x), _f64(y)
    r = C.c_double()
    ctx = _ctx()
    _lib.check(_lib.load().pbs_k_dot_range(ctx, _p(xx), _p(yy), int(lo), int(hi), C.byref(r)), ctx)
    return r.value


def _lincomb(kind, out, scalars, *vecs):
    _out_ok(out)
    sc = np.zeros(4)
    sc[: len(scalars)] = scalars
    arrs = [_f64(v) for v in vecs]
    for a in arrs:
        if a.shape != out.shape:
            raise ValueError("operands must match out's shape")
    ptrs = [_p(a) for a in arrs] + [None] * (4 - len(arrs))
    ctx = _ctx()
    _lib.check(_lib.load().pbs_k_lincomb(ctx, kind, out.shape[0], _p(out), _p(sc), *ptrs), ctx)


def lincomb2(out, sa, a, sb, b):
    _lincomb(2, out, (sa, sb), a, b)


def lincomb3(out, sa, a, sb, b, sc, c):
    _lincomb(3, out, (sa, sb, sc), a, b, c)


def lincomb4(out, sa, a, sb, b, sc, c, sd, d):
    _lincomb(4, out, (sa, sb, sc, sd), a, b, c, d)


def lincomb_nested(out, sa, a, sb, b, sc, c):
    _lincomb(5, out, (sa, sb, sc), a, b, c)


def add_scaled_diff(out, base, s, a, b):
    _lincomb(6, out, (s,), base, a, b)


def add_scaled_damped_diff(out, base, s, a, w, b):
    _lincomb(7, out, (s, w), base, a, b)


TABLE = {name: globals()[name] for name in _NAMES}


def register(kn_module, name: str = "cuda") -> None:
    """Add this table to a pipesafe-style ``kernels`` module's backend tables."""
    kn_module._TABLES[name] = dict(TABLE)
