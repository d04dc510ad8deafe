"""ctypes binding of include/cavac_b200.h (libcavac_b200.so, built in-tree).

There is no fallback: if the shared library is missing or no sm_100 device is
present, loading / context creation raises.  The product never imports
anything under oracle/.
"""
from __future__ import annotations

import ctypes as C
import os
import re

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
# CVK_LIB_PATH: measurement builds of the same sources (tools/variant_build.sh)
LIB_PATH = os.environ.get("CVK_LIB_PATH") or os.path.join(PKG, "libcavac_b200.so")
HEADER = os.path.join(ROOT, "include", "cavac_b200.h")

CVK_OK = 0
ERRORS = {
    -1: "EINVAL", -2: "ECUDA", -3: "ENOMEM", -4: "EOVERFLOW", -5: "EZERODIAG",
    -6: "ESOLVER", -7: "ELOGIC", -8: "ETIMEOUT",
}
MODE_FAST, MODE_REF, MODE_REF_PAR = 0, 1, 2
# cvk_ctx_set_option keys (include/cavac_b200.h)
OPTIONS = {"phased_min_n": 1, "max_ctas": 2, "stream": 3, "stream_flavor": 4, "spmv_group": 5,
           "gmres_persistent": 6, "bicgl_persistent": 7, "ilu_hostloop": 8, "ddm_seq_min": 9,
           "rb_stream_min": 10, "bicg_fold": 11,
           "gmres_tiles": 12, "uniform_offdiag": 13}


class CvkOpts(C.Structure):
    _fields_ = [
        ("tol", C.c_double),
        ("max_iter", C.c_int64),
        ("l", C.c_int64),
        ("m", C.c_int64),
        ("record_history", C.c_int32),
        ("mode", C.c_int32),
        ("warm", C.c_int32),
        ("reserved", C.c_int32),
    ]


class CvkReport(C.Structure):
    _fields_ = [
        ("converged", C.c_int32),
        ("breakdown", C.c_int32),
        ("iterations", C.c_int64),
        ("final_relres", C.c_double),
        ("true_relres", C.c_double),
        ("wall_time_s", C.c_double),
        ("history", C.POINTER(C.c_double)),
        ("history_cap", C.c_int64),
        ("history_len", C.c_int64),
        ("device_time_s", C.c_double),
        ("kernel_launches", C.c_int64),
    ]


class CvkDdmReport(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_int64),
        ("converged", C.c_int32),
        ("inner_breakdown", C.c_int32),
        ("jump_history", C.POINTER(C.c_double)),
        ("jump_cap", C.c_int64),
        ("jump_len", C.c_int64),
        ("sub_reports", C.POINTER(CvkReport)),
        ("n_sub_reports", C.c_int64),
        ("total_inner_iterations", C.c_int64),
        ("device_time_s", C.c_double),
        ("wall_time_s", C.c_double),
        ("kernel_launches", C.c_int64),
    ]


class CvkError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{ERRORS.get(code, code)}] {msg}")
        self.code = code
        self.msg = msg


_lib = None
P = C.c_void_p


def declared_symbols() -> list[str]:
    """Function names declared in include/cavac_b200.h."""
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(cvk_[a-z_0-9]+)\s*\(", txt, re.M)))


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run python -m paper_2112_00087_b200.build")
    L = C.CDLL(LIB_PATH)
    i64, i32, dbl = C.c_int64, C.c_int, C.c_double
    sig = {
        "cvk_abi_version": ([], i32),
        "cvk_last_error": ([], C.c_char_p),
        "cvk_breakdown_name": ([i32], C.c_char_p),
        "cvk_solver_name": ([i32], C.c_char_p),
        "cvk_solver_from_name": ([C.c_char_p], i32),
        "cvk_ctx_create": ([i32, C.POINTER(P)], i32),
        "cvk_ctx_destroy": ([P], i32),
        "cvk_ctx_stream": ([P], P),
        "cvk_set_exec_mode": ([P, i32], i32),
        "cvk_get_exec_mode": ([P], i32),
        "cvk_ctx_set_option": ([P, i32, i64], i32),
        "cvk_ctx_get_option": ([P, i32, C.POINTER(i64)], i32),
        "cvk_csr_upload": ([P, i64, i64, i64, P, P, P, C.POINTER(P)], i32),
        "cvk_csr_set_values": ([P, P], i32),
        "cvk_csr_free": ([P], i32),
        "cvk_csr_nrows": ([P], i64),
        "cvk_csr_nnz": ([P], i64),
        "cvk_precond_jacobi": ([P, P, C.POINTER(P)], i32),
        "cvk_precond_identity": ([P, i64, C.POINTER(P)], i32),
        "cvk_precond_free": ([P], i32),
        "cvk_precond_get_diag": ([P, P], i32),
        "cvk_precond_ilu0": ([P, i32, C.POINTER(P)], i32),
        "cvk_precond_get_ilu0": ([P, P], i32),
        "cvk_precond_apply_device": ([P, P, P], i32),
        "cvk_precond_apply": ([P, P, P], i32),
        "cvk_solve": ([P, i32, P, P, C.POINTER(CvkOpts), P, P, C.POINTER(CvkReport)], i32),
        "cvk_solve_device": ([P, i32, P, P, C.POINTER(CvkOpts), P, P, C.POINTER(CvkReport)], i32),
        "cvk_spmv": ([P, P, P, i32], i32),
        "cvk_spmv_device": ([P, P, P, i32], i32),
        "cvk_spmv_bench": ([P, P, P, i32, i32, C.POINTER(dbl)], i32),
        "cvk_dot": ([P, i64, P, P, P, i32], i32),
        "cvk_norm2": ([P, i64, P, C.POINTER(dbl), i32], i32),
        "cvk_axpy": ([P, i64, P, P, P], i32),
        "cvk_xpay": ([P, i64, P, P, P], i32),
        "cvk_true_relres": ([P, P, P, C.POINTER(dbl), i32], i32),
    }
    for name, (args, res) in sig.items():
        if hasattr(L, name):
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
    _lib = L
    return L


def check(code: int) -> None:
    if code != CVK_OK:
        msg = load().cvk_last_error().decode(errors="replace")
        raise CvkError(code, msg)


def last_error() -> str:
    return load().cvk_last_error().decode(errors="replace")
