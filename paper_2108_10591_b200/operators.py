"""Device-resident operators: CSR in HBM, or a matrix-free stencil.

``DeviceMatrix`` owns a libpbsafe ``pbs_mat`` (CSR with int64 row_ptr,
int32 col_idx, f64 values in HBM — SURVEY §8(a) a11 — or a
constant-coefficient stencil).  Solvers accept either a host ``CsrMatrix``
(uploaded per call, the reference's calling convention) or a DeviceMatrix
(uploaded once, reused across solves).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .linalg import CsrMatrix
from .problems import StencilSpec


class DeviceMatrix:
    def __init__(self, handle, ctx: _lib.Context, n_rows: int, n_cols: int, nnz: int, stencil: bool,
                 source: str = ""):
        self.handle = handle
        self.ctx = ctx
        self.n_rows = n_rows
        self.n_cols = n_cols
        self.nnz = nnz
        self.stencil = stencil
        self.source = source

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n_rows, self.n_cols)

    @classmethod
    def from_csr(cls, A: CsrMatrix | tuple, device: int | None = None, ctx=None) -> "DeviceMatrix":
        """Upload a CsrMatrix (or (row_ptr, col_idx, values[, n_cols]) arrays)."""
        if isinstance(A, CsrMatrix) or hasattr(A, "row_ptr"):  # ours or the reference's CsrMatrix
            rp, ci, v, n_rows, n_cols = A.row_ptr, A.col_idx, A.values, A.n_rows, A.n_cols
        else:
            rp, ci, v = A[:3]
            n_rows = len(rp) - 1
            n_cols = A[3] if len(A) > 3 else n_rows
        ctx = ctx or _lib.context(device)
        rp = np.ascontiguousarray(rp, dtype=np.int64)
        if ci.dtype == np.int32:
            ci = np.ascontiguousarray(ci)
            cb = 4
        else:
            ci = np.ascontiguousarray(ci, dtype=np.int64)
            cb = 8
        v = np.ascontiguousarray(v, dtype=np.float64)
        if rp.shape != (n_rows + 1,):
            raise ValueError("row_ptr length must be n_rows + 1")
        if ci.shape != v.shape:
            raise ValueError("row_ptr endpoints inconsistent with nnz arrays")
        h = C.c_void_p()
        rc = _lib.load().pbs_csr_upload(ctx.handle, n_rows, n_cols, v.shape[0],
                                         rp.ctypes.data_as(C.c_void_p), ci.ctypes.data_as(C.c_void_p),
                                         cb, v.ctypes.data_as(C.c_void_p), C.byref(h))
        if rc == _lib.PBS_ERR_INVALID:
            raise ValueError(_lib.last_error(ctx.handle))
        _lib.check(rc, ctx.handle)
        return cls(h, ctx, n_rows, n_cols, int(v.shape[0]), False, "csr")

    @classmethod
    def from_stencil(cls, spec: StencilSpec, device: int | None = None, ctx=None) -> "DeviceMatrix":
        ctx = ctx or _lib.context(device)
        offs = np.ascontiguousarray(np.array(spec.offsets, dtype=np.int32).reshape(-1))
        coefs = np.ascontiguousarray(np.array(spec.coeffs, dtype=np.float64))
        h = C.c_void_p()
        rc = _lib.load().pbs_stencil_create(ctx.handle, spec.dim, spec.k, spec.npts,
                                             offs.ctypes.data_as(C.c_void_p),
                                             coefs.ctypes.data_as(C.c_void_p), C.byref(h))
        if rc == _lib.PBS_ERR_INVALID:
            raise ValueError(_lib.last_error(ctx.handle))
        _lib.check(rc, ctx.handle)
        nr, nc, nnz, st = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int32()
        _lib.load().pbs_mat_info(h, C.byref(nr), C.byref(nc), C.byref(nnz), C.byref(st))
        return cls(h, ctx, nr.value, nc.value, nnz.value, True, f"stencil{spec.dim}d:{spec.npts}pt")

    def to_csr(self) -> "DeviceMatrix":
        """CSR of a stencil operator, built on the device (== problems.stencil_csr)."""
        if not self.stencil:
            raise ValueError("to_csr needs a stencil operator")
        h = C.c_void_p()
        _lib.check(_lib.load().pbs_stencil_to_csr(self.handle, C.byref(h)), self.ctx.handle)
        return DeviceMatrix(h, self.ctx, self.n_rows, self.n_cols, self.nnz, False, self.source + "->csr")

    def update_csr(self, row_ptr, col_idx, values) -> None:
        """Upload new arrays of the same shape into this CSR operator (its
        workspace and, for a partition slab, its halo plan and peer mappings
        stay): pbs_csr_update."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        if col_idx.dtype == np.int32:
            ci, cb = np.ascontiguousarray(col_idx), 4
        else:
            ci, cb = np.ascontiguousarray(col_idx, dtype=np.int64), 8
        v = np.ascontiguousarray(values, dtype=np.float64)
        if rp.shape != (self.n_rows + 1,) or ci.shape != (self.nnz,) or v.shape != (self.nnz,):
            raise ValueError("update_csr needs arrays of the operator's shape")
        rc = _lib.load().pbs_csr_update(self.handle, rp.ctypes.data_as(C.c_void_p), ci.ctypes.data_as(C.c_void_p),
                                         cb, v.ctypes.data_as(C.c_void_p))
        if rc == _lib.PBS_ERR_INVALID:
            raise ValueError(_lib.last_error(self.ctx.handle))
        _lib.check(rc, self.ctx.handle)

    def spmv_dev(self, x_ptr: int, y_ptr: int) -> int:
        """y = A x on device pointers; returns the first non-finite row or -1."""
        bad = C.c_int64()
        _lib.check(_lib.load().pbs_spmv_dev(self.handle, C.c_void_p(x_ptr), C.c_void_p(y_ptr),
                                            C.byref(bad)), self.ctx.handle)
        return bad.value

    LAYOUTS = {0: "csr-gather", 1: "csr-window", 2: "csr-band", 3: "sell", 4: "sell-dict", 5: "sell-pairs", 10: "stencil"}

    def layout(self) -> dict:
        """What the SpMV engines stream for this operator (pbs_mat_layout): the
        layout name, entries and bytes per product, dictionary size."""
        out = (C.c_int64 * 8)()
        _lib.check(_lib.load().pbs_mat_layout(self.handle, out), self.ctx.handle)
        return {"layout": self.LAYOUTS.get(int(out[0]), str(int(out[0]))), "entries": int(out[1]),
                "bytes_per_entry": int(out[2]), "bytes_per_row": int(out[3]), "dict_entries": int(out[4]),
                "max_row": int(out[5]), "x_windows": int(out[6]), "x_staged": int(out[7]),
                "matrix_bytes": int(out[1]) * int(out[2]) + int(out[3]) * self.n_rows}

    def free(self):
        if self.handle:
            _lib.load().pbs_mat_free(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover
        try:
            self.free()
        except Exception:
            pass
