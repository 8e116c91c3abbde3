"""ctypes binding of libpbsafe.so (include/pbsafe.h).

The library is built in-tree by ``paper_2108_10591_b200.build``; loading
never falls back to anything else: a missing or unloadable library, or a
machine without an sm_100 device, raises ``NativeUnavailable``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from . import build as _build

PBS_OK = 0
PBS_ERR_INVALID = -1
PBS_ERR_CUDA = -2
PBS_ERR_NONFINITE = -3
PBS_ERR_NOMEM = -4
PBS_ERR_NCCL = -5
PBS_ERR_UNSUPPORTED = -6

METHOD_IDS = {"pbicgsafe": 0, "pbicgsafe-rr": 1, "ssbicgsafe2": 2, "bicgstab": 3, "gpbicg": 4,
              "pbicgstab": 5}
REDUCE_TREE, REDUCE_PLAN = 0, 1
HIST_REPLACED, HIST_HAS_COEF = 1, 2
NUM_KERNEL_KINDS = 8
KERNEL_KINDS = ("K1_As", "K2_update", "K3_Aw_epilogue", "F_finalize", "R_rr_update",
                "RS_rr_spmv", "S_setup", "D_plan_dots")
# reduction.py:330/451 tags of the NonFiniteVectorError message
SPMV_TAGS = {1: "Ax", 2: "Ar", 3: "As", 4: "Aw", 5: "Ao", 6: "Au", 7: "At", 8: "Ay", 9: "Ap", 10: "Az"}

EXPORTS = (
    "pbs_init", "pbs_destroy", "pbs_last_error", "pbs_device_info", "pbs_set_stream",
    "pbs_csr_upload", "pbs_stencil_create", "pbs_mat_free", "pbs_mat_info", "pbs_spmv_dev",
    "pbs_solve", "pbs_solve_dev", "pbs_step_dev", "pbs_k_spmv_range", "pbs_k_dot_range",
    "pbs_k_lincomb", "pbs_dot_batch_dev", "pbs_nccl_unique_id", "pbs_dist_init", "pbs_dist_destroy",
    "pbs_mat_set_partition", "pbs_stencil_to_csr", "pbs_dist_set_sm_limit", "pbs_dist_export",
    "pbs_dist_connect", "pbs_dist_connect_local", "pbs_solve_group", "pbs_spmv_group", "pbs_stencil_slab",
    "pbs_csr_update", "pbs_mat_layout",
)
TRANSPORTS = {"p2p": 0, "nccl": 1}
DIST_BLOB_BYTES = 256
# schedule-evidence stamp words per iteration (pbs_config.stamps_out)
STAMP_WORDS = ("as_start", "as_end", "aw_start", "aw_end", "pub_start", "pub_end", "fin_start", "fin_end")


class NativeUnavailable(RuntimeError):
    """libpbsafe.so could not be loaded or has no usable B200 device."""


class PbsError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(f"libpbsafe error {code}: {message}")
        self.code = code


TRACE_FN = C.CFUNCTYPE(None, C.c_int64, C.POINTER(C.POINTER(C.c_double)), C.c_void_p)


class Config(C.Structure):
    _fields_ = [
        ("tol", C.c_double), ("max_iters", C.c_int64), ("rr_epoch", C.c_int64),
        ("rr_cutoff", C.c_int64), ("record_history", C.c_int32), ("reduce_mode", C.c_int32),
        ("plan_workers", C.c_int32), ("use_graphs", C.c_int32), ("timing", C.c_int32),
        ("pad", C.c_int32), ("trace_fn", TRACE_FN), ("trace_user", C.c_void_p),
        ("events_out", C.c_void_p), ("events_cap", C.c_int64), ("events_count", C.POINTER(C.c_int64)),
        ("stamps_out", C.c_void_p), ("stamps_cap", C.c_int64), ("stamps_count", C.POINTER(C.c_int64)),
    ]


class Result(C.Structure):
    _fields_ = [
        ("status", C.c_int32), ("breakdown", C.c_int32), ("iterations", C.c_int64),
        ("failure_iter", C.c_int64), ("n_records", C.c_int64), ("r0_norm", C.c_double),
        ("nonfinite_tag", C.c_int32), ("pad", C.c_int32), ("nonfinite_index", C.c_int64),
        ("n_spmv", C.c_int64), ("n_replacements", C.c_int64), ("stop_stage", C.c_int32),
        ("pad2", C.c_int32), ("device_ms", C.c_double),
        ("kernel_launches", C.c_int64), ("kernel_ms", C.c_double * NUM_KERNEL_KINDS),
        ("kernel_count", C.c_int64 * NUM_KERNEL_KINDS),
    ]


_lib = None
_lock = threading.Lock()


def lib_path() -> str:
    # PBS_LIB: an alternative build of the same library (engine sweeps)
    return os.environ.get("PBS_LIB") or _build.LIB


def load(build_if_missing: bool = True):
    """Load libpbsafe.so (building it first when absent and nvcc exists)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        # The multi-GPU schedule runs compute, halo and reduction streams per
        # partition; with the default 8 hardware queues streams alias and a
        # flag wait on one holds back a kernel on another.  Only effective
        # when set before the process creates its CUDA context.
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
        path = lib_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise NativeUnavailable(f"{path} is missing; run python -m paper_2108_10591_b200.build")
            _build.build()
        try:
            L = C.CDLL(path)
        except OSError as e:  # pragma: no cover
            raise NativeUnavailable(f"cannot load {path}: {e}") from e
        p, i32, i64, d = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        pp = C.POINTER(p)
        sig = {
            "pbs_init": ([C.c_int, pp], C.c_int),
            "pbs_destroy": ([p], C.c_int),
            "pbs_last_error": ([p], C.c_char_p),
            "pbs_device_info": ([p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)], C.c_int),
            "pbs_set_stream": ([p, C.c_size_t], C.c_int),
            "pbs_csr_upload": ([p, i64, i64, i64, p, p, i32, p, pp], C.c_int),
            "pbs_stencil_create": ([p, i32, i64, i32, p, p, pp], C.c_int),
            "pbs_mat_free": ([p], C.c_int),
            "pbs_mat_info": ([p, p, p, p, p], C.c_int),
            "pbs_mat_layout": ([p, p], C.c_int),
            "pbs_spmv_dev": ([p, p, p, C.POINTER(i64)], C.c_int),
            "pbs_solve": ([p, i32, p, p, C.POINTER(Config), p, p, p, p, C.POINTER(Result)], C.c_int),
            "pbs_solve_dev": ([p, i32, p, p, C.POINTER(Config), p, p, p, p, C.POINTER(Result)], C.c_int),
            "pbs_step_dev": ([p, p, p, i32, i32, p], C.c_int),
            "pbs_k_spmv_range": ([p, i64, i64, p, p, p, p, p, i64, i64], C.c_int),
            "pbs_k_dot_range": ([p, p, p, i64, i64, C.POINTER(d)], C.c_int),
            "pbs_k_lincomb": ([p, i32, i64, p, p, p, p, p, p], C.c_int),
            "pbs_dot_batch_dev": ([p, i64, p, p, p, p, p, i32, i32, p], C.c_int),
            "pbs_nccl_unique_id": ([p], C.c_int),
            "pbs_dist_init": ([p, i32, i32, i32, p, p, pp], C.c_int),
            "pbs_dist_set_sm_limit": ([p, i32], C.c_int),
            "pbs_dist_export": ([p, p], C.c_int),
            "pbs_dist_connect": ([p, p], C.c_int),
            "pbs_dist_connect_local": ([p, i32], C.c_int),
            "pbs_solve_group": ([p, i32, i32, p, p, C.POINTER(Config), p, p, p, p, C.POINTER(Result)], C.c_int),
            "pbs_spmv_group": ([p, i32, p, p, p], C.c_int),
            "pbs_stencil_slab": ([p, i64, i64, i64, i64, pp], C.c_int),
            "pbs_csr_update": ([p, p, p, i32, p], C.c_int),
            "pbs_dist_destroy": ([p], C.c_int),
            "pbs_mat_set_partition": ([p, p, i64, i64, i64, i64, i32, p, i32, p], C.c_int),
            "pbs_stencil_to_csr": ([p, pp], C.c_int),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
        return _lib


def last_error(ctx=None) -> str:
    msg = load().pbs_last_error(ctx)
    return msg.decode() if msg else ""


def check(code: int, ctx=None) -> None:
    if code != PBS_OK:
        raise PbsError(code, last_error(ctx))


class Context:
    """One libpbsafe context (one CUDA device, one stream)."""

    def __init__(self, device: int = 0):
        L = load()
        h = C.c_void_p()
        rc = L.pbs_init(device, C.byref(h))
        if rc != PBS_OK:
            raise NativeUnavailable(f"pbs_init({device}) failed: {last_error(None)}")
        self.handle = h
        self.device = device
        sms, ma, mi = C.c_int(), C.c_int(), C.c_int()
        check(L.pbs_device_info(h, C.byref(sms), C.byref(ma), C.byref(mi)), h)
        self.sm_count, self.cc = sms.value, (ma.value, mi.value)

    def close(self):
        if self.handle:
            load().pbs_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int | None = None) -> Context:
    """Process-wide context for a device (default: torch's current device or 0)."""
    if device is None:
        dev_env = os.environ.get("LOCAL_RANK")
        device = 0
        try:
            import torch

            if torch.cuda.is_available():
                device = torch.cuda.current_device()
        except Exception:  # pragma: no cover
            device = int(dev_env or 0)
    ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        _contexts[device] = ctx
    return ctx
