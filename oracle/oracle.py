"""ctypes front-end for the C restatement (liboracle.so) and the compiled
reference (oracle/_ref/libcavac_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py, always as the checker or
the timed CPU baseline -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libcavac_ref.so")

SOLVERS = {"bicgstab": 0, "bicgstab_l": 1, "tfqmr": 2, "gmres": 3, "cocg": 4}
BREAKDOWN = {
    0: None,
    1: "rho breakdown",
    2: "stagnation in <shadow, v>",
    3: "omega breakdown",
    4: "stagnation in <shadow, u>",
    5: "degenerate least-squares in MR step",
    6: "sigma breakdown",
    7: "arnoldi breakdown",
    8: "stagnation in <p, A p>",
}


class _Report(C.Structure):
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
    ]


class _Opts(C.Structure):
    _fields_ = [
        ("tol", C.c_double),
        ("max_iter", C.c_int64),
        ("l", C.c_int64),
        ("m", C.c_int64),
        ("record_history", C.c_int32),
        ("pad", C.c_int32),
    ]


class _Grid(C.Structure):
    _fields_ = [
        ("width", C.c_double), ("height", C.c_double), ("h", C.c_double),
        ("nx", C.c_int64), ("ny", C.c_int64),
        ("roof_begin", C.c_int64), ("roof_end", C.c_int64),
        ("adm_re", C.c_double), ("adm_im", C.c_double),
    ]


class _DdmReport(C.Structure):
    _fields_ = [
        ("outer_iterations", C.c_int64),
        ("converged", C.c_int32),
        ("inner_breakdown", C.c_int32),
        ("jump_history", C.POINTER(C.c_double)),
        ("jump_cap", C.c_int64),
        ("jump_len", C.c_int64),
        ("last_inner_iterations_total", C.c_int64),
    ]


@dataclass
class Report:
    converged: bool
    iterations: int
    final_relres: float
    true_relres: float
    wall_time: float
    breakdown: str | None
    residual_history: list = field(default_factory=list)


def build(force: bool = False) -> str:
    """Compile liboracle.so (gcc, no FMA contraction)."""
    src = os.path.join(HERE, "cavac_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
             "-o", LIB_PATH, src, "-lm"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        L = _lib
        P = C.c_void_p
        L.orc_solve.argtypes = [C.c_int, C.c_int64, P, P, P, P, P, C.POINTER(_Opts), P, C.POINTER(_Report)]
        L.orc_set_sum_mode.argtypes = [C.c_int]
        L.orc_solve.restype = C.c_int
        L.orc_jacobi_arrays.argtypes = [C.c_int64, P, P, P, P]
        L.orc_jacobi_arrays.restype = C.c_int64
        L.orc_spmv_arrays.argtypes = [C.c_int64, P, P, P, P, P]
        L.orc_true_relres_arrays.argtypes = [C.c_int64, P, P, P, P, P]
        L.orc_true_relres_arrays.restype = C.c_double
        L.orc_dot_out.argtypes = [C.c_int64, P, P, P]
        L.orc_norm2.argtypes = [C.c_int64, P]
        L.orc_norm2.restype = C.c_double
        L.orc_csr_from_triplets.argtypes = [C.c_int64, P, P, P, C.c_int64, C.c_int64, P, P, P]
        L.orc_csr_from_triplets.restype = C.c_int64
        L.orc_build_grid.argtypes = [C.c_double] * 7 + [C.POINTER(_Grid)]
        L.orc_build_grid.restype = C.c_int
        L.orc_assemble.argtypes = [C.POINTER(_Grid), C.c_double, C.c_double, P, P, P, P, P]
        L.orc_assemble.restype = C.c_int64
        L.orc_partition.argtypes = [C.c_int64, C.c_int64, P]
        L.orc_partition.restype = C.c_int
        L.orc_schwarz_solve.argtypes = [
            C.POINTER(_Grid), C.c_double, C.c_int64, P, P, P, P, C.c_int64, P,
            C.c_double, C.c_double, C.c_double, C.c_double, C.POINTER(_Opts), C.c_double, C.c_int64, C.c_int,
            P, C.POINTER(_DdmReport), P]
        L.orc_schwarz_solve.restype = C.c_int
        L.orc_cdiv.argtypes = [C.c_double] * 4 + [P]
        L.orc_ilu0_arrays.argtypes = [C.c_int64, P, P, P, P]
        L.orc_ilu0_arrays.restype = C.c_int64
        L.orc_ilu0_apply_arrays.argtypes = [C.c_int64, P, P, P, C.c_int64, P, P]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def _c128(a):
    return np.ascontiguousarray(a, dtype=np.complex128)


def _opts(tol=1e-9, max_iter=10000, l=8, m=30, record_history=False):
    return _Opts(tol, max_iter, l, m, 1 if record_history else 0, 0)


def _report(rep: _Report, hist) -> Report:
    h = list(hist[: min(rep.history_len, len(hist))]) if hist is not None else []
    return Report(bool(rep.converged), int(rep.iterations), rep.final_relres, rep.true_relres,
                  rep.wall_time_s, BREAKDOWN.get(rep.breakdown, "?"), h)


def jacobi(rp, ci, v):
    rp, ci, v = _i64(rp), _i64(ci), _c128(v)
    n = len(rp) - 1
    d = np.zeros(n, np.complex128)
    bad = lib().orc_jacobi_arrays(n, _p(rp), _p(ci), _p(v), _p(d))
    if bad >= 0:
        raise ValueError(f"jacobi: zero diagonal at row {bad}")
    return d


def solve(solver, rp, ci, v, b, dinv=None, tol=1e-9, max_iter=10000, l=8, m=30,
          record_history=False):
    """cavac::solve(SolverId, A, b, M, opts) restated; dinv=None -> jacobi(A)."""
    rp, ci, v, b = _i64(rp), _i64(ci), _c128(v), _c128(b)
    n = len(rp) - 1
    if dinv is None:
        dinv = jacobi(rp, ci, v)
    elif isinstance(dinv, str) and dinv == "identity":
        dinv = None
    x = np.zeros(n, np.complex128)
    rep = _Report()
    hist = None
    if record_history:
        cap = max(2 * max_iter + 16, 64)
        hist = np.zeros(cap, np.float64)
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_cap = cap
    o = _opts(tol, max_iter, l, m, record_history)
    sid = SOLVERS[solver] if isinstance(solver, str) else int(solver)
    rc = lib().orc_solve(sid, n, _p(rp), _p(ci), _p(v),
                         _p(dinv) if dinv is not None else None, _p(b), C.byref(o), _p(x),
                         C.byref(rep))
    if rc != 0:
        raise ValueError(f"orc_solve failed rc={rc}")
    return x, _report(rep, hist)


def ilu0(rp, ci, v):
    """Exact ILU(0) factor in A's value slots (cavac_oracle.c orc_ilu0_arrays;
    beyond the reference, which has only jacobi/identity, krylov.cpp:27-55)."""
    rp, ci, v = _i64(rp), _i64(ci), _c128(v)
    n = len(rp) - 1
    f = np.zeros(len(v), np.complex128)
    bad = lib().orc_ilu0_arrays(n, _p(rp), _p(ci), _p(v), _p(f))
    if bad >= 0:
        raise ValueError(f"ilu0: zero pivot at row {bad}")
    return f


def ilu0_apply(rp, ci, fac, sweeps, r):
    """z ~= U^-1 L^-1 r by `sweeps` Jacobi sweeps per triangle (orc_ilu0_apply_arrays)."""
    rp, ci, fac, r = _i64(rp), _i64(ci), _c128(fac), _c128(r)
    z = np.zeros(len(rp) - 1, np.complex128)
    lib().orc_ilu0_apply_arrays(len(rp) - 1, _p(rp), _p(ci), _p(fac), int(sweeps), _p(r), _p(z))
    return z


def spmv(rp, ci, v, x):
    rp, ci, v, x = _i64(rp), _i64(ci), _c128(v), _c128(x)
    y = np.zeros(len(rp) - 1, np.complex128)
    lib().orc_spmv_arrays(len(rp) - 1, _p(rp), _p(ci), _p(v), _p(x), _p(y))
    return y


def dot(x, y):
    x, y = _c128(x), _c128(y)
    out = np.zeros(2)
    lib().orc_dot_out(len(x), _p(x), _p(y), _p(out))
    return complex(out[0], out[1])


def norm2(x):
    x = _c128(x)
    return lib().orc_norm2(len(x), _p(x))


def true_relres(rp, ci, v, b, x):
    rp, ci, v, b, x = _i64(rp), _i64(ci), _c128(v), _c128(b), _c128(x)
    return lib().orc_true_relres_arrays(len(rp) - 1, _p(rp), _p(ci), _p(v), _p(b), _p(x))


def csr_from_triplets(rows, cols, vals, nrows, ncols):
    rows, cols, vals = _i64(rows), _i64(cols), _c128(vals)
    k = len(rows)
    rp = np.zeros(nrows + 1, np.int64)
    ci = np.zeros(max(k, 1), np.int64)
    v = np.zeros(max(k, 1), np.complex128)
    nnz = lib().orc_csr_from_triplets(k, _p(rows), _p(cols), _p(vals), nrows, ncols,
                                      _p(rp), _p(ci), _p(v))
    if nnz < 0:
        bad = -1 - nnz
        raise ValueError(f"csr_from_triplets: index out of range at ({rows[bad]}, {cols[bad]})")
    return rp, ci[:nnz].copy(), v[:nnz].copy()


def cdiv(a: complex, b: complex) -> complex:
    out = np.zeros(2)
    lib().orc_cdiv(a.real, a.imag, b.real, b.imag, _p(out))
    return complex(out[0], out[1])


class Grid:
    def __init__(self, g: _Grid):
        self._g = g
        for name, _ in _Grid._fields_:
            setattr(self, name, getattr(g, name))

    @property
    def size(self):
        return self.nx * self.ny

    @property
    def roof_size(self):
        return self.roof_end - self.roof_begin


def build_grid(width, height, h, roof_start, roof_end, admittance=0j):
    g = _Grid()
    rc = lib().orc_build_grid(width, height, h, roof_start, roof_end,
                              complex(admittance).real, complex(admittance).imag, C.byref(g))
    if rc != 0:
        raise ValueError(f"build_grid failed rc={rc}")
    return Grid(g)


def assemble(grid: Grid, omega, c, dirichlet):
    """helmholtz.cpp:59-115 restated; returns (rp, ci, v, b)."""
    dirichlet = _c128(dirichlet)
    if len(dirichlet) != grid.roof_size:
        raise ValueError("assemble: dirichlet length does not match roof span")
    n = grid.size
    rp = np.zeros(n + 1, np.int64)
    ci = np.zeros(5 * n, np.int64)
    v = np.zeros(5 * n, np.complex128)
    b = np.zeros(n, np.complex128)
    nnz = lib().orc_assemble(C.byref(grid._g), omega, c, _p(dirichlet), _p(rp), _p(ci), _p(v), _p(b))
    return rp, ci[:nnz].copy(), v[:nnz].copy(), b


def partition(nx, n_sub):
    cb = np.zeros(n_sub + 1, np.int64)
    rc = lib().orc_partition(nx, n_sub, _p(cb))
    if rc != 0:
        raise ValueError("partition: invalid n_sub")
    return cb


def schwarz_solve(grid: Grid, c, rp, ci, v, b, n_sub, s_left, s_right, tol=1e-9, max_iter=10000,
                  l=8, m=30, ddm_tol=1e-8, max_outer=200, inner_solver="bicgstab"):
    rp, ci, v, b = _i64(rp), _i64(ci), _c128(v), _c128(b)
    n = len(rp) - 1
    cb = partition(grid.nx, n_sub)
    x = np.zeros(n, np.complex128)
    rep = _DdmReport()
    hist = np.zeros(max_outer + 1, np.float64)
    rep.jump_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    rep.jump_cap = len(hist)
    o = _opts(tol, max_iter, l, m, False)
    subs = (_Report * n_sub)()
    rc = lib().orc_schwarz_solve(C.byref(grid._g), c, n, _p(rp), _p(ci), _p(v), _p(b), n_sub,
                                 _p(cb), complex(s_left).real, complex(s_left).imag,
                                 complex(s_right).real, complex(s_right).imag, C.byref(o), ddm_tol, max_outer,
                                 SOLVERS[inner_solver], _p(x), C.byref(rep), C.cast(subs, C.c_void_p))
    if rc != 0:
        raise RuntimeError(f"schwarz_solve failed rc={rc}")
    return x, {
        "outer_iterations": int(rep.outer_iterations),
        "converged": bool(rep.converged),
        "interface_residual_history": list(hist[: rep.jump_len]),
        "sub_iterations": [int(s.iterations) for s in subs],
    }


# ---------------------------------------------------------------- _ref ----

_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    """The unmodified reference core compiled by oracle/Makefile + ref_shim."""
    global _ref
    if _ref is None:
        _ref = C.CDLL(REF_PATH)
        R = _ref
        P = C.c_void_p
        R.ref_solve.argtypes = [C.c_int, C.c_int64, C.c_int64, P, P, P, P, C.c_double, C.c_int64,
                                C.c_int64, C.c_int, P, C.POINTER(_Report)]
        R.ref_solve.restype = C.c_int
        R.ref_set_exec_mode.argtypes = [C.c_int]
        R.ref_omp_threads.restype = C.c_int
        R.ref_spmv.argtypes = [C.c_int64, C.c_int64, P, P, P, P, P]
    return _ref


def ref_solve(solver, rp, ci, v, b, tol=1e-9, max_iter=10000, l=8, parallel=False,
              record_history=False):
    """cavac::jacobi + cavac::solve of the real reference (oracle/_ref)."""
    R = ref()
    rp, ci, v, b = _i64(rp), _i64(ci), _c128(v), _c128(b)
    n = len(rp) - 1
    x = np.zeros(n, np.complex128)
    rep = _Report()
    hist = None
    if record_history:
        cap = max(2 * max_iter + 16, 64)
        hist = np.zeros(cap, np.float64)
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_cap = cap
    R.ref_set_exec_mode(1 if parallel else 0)
    sid = SOLVERS[solver] if isinstance(solver, str) else int(solver)
    rc = R.ref_solve(sid, n, len(v), _p(rp), _p(ci), _p(v), _p(b), tol, max_iter, l,
                     1 if record_history else 0, _p(x), C.byref(rep))
    R.ref_set_exec_mode(0)
    if rc != 0:
        raise RuntimeError(f"ref_solve rc={rc}")
    return x, _report(rep, hist)


def ref_spmv(rp, ci, v, x, parallel=False):
    R = ref()
    rp, ci, v, x = _i64(rp), _i64(ci), _c128(v), _c128(x)
    y = np.zeros(len(rp) - 1, np.complex128)
    R.ref_set_exec_mode(1 if parallel else 0)
    R.ref_spmv(len(rp) - 1, len(v), _p(rp), _p(ci), _p(v), _p(x), _p(y))
    R.ref_set_exec_mode(0)
    return y


# ------------------------------------------------------------ file I/O ----

def read_matrix_market(path):
    """mmio.cpp:28-63 restated for the reference's own files."""
    with open(path) as f:
        header = f.readline()
        parts = header.split()
        if not header.startswith("%%MatrixMarket") or parts[1:5] != ["matrix", "coordinate", "complex", "general"]:
            raise ValueError(f"matrix market: unsupported header {header!r}")
        line = f.readline()
        while line and (not line.strip() or line.startswith("%")):
            line = f.readline()
        nrows, ncols, nnz = (int(t) for t in line.split())
        data = np.loadtxt(f, dtype=np.float64, ndmin=2, max_rows=nnz) if nnz else np.zeros((0, 4))
    rows = data[:, 0].astype(np.int64) - 1
    cols = data[:, 1].astype(np.int64) - 1
    vals = data[:, 2] + 1j * data[:, 3]
    return csr_from_triplets(rows, cols, vals, nrows, ncols)


def read_vector_csv(path):
    d = np.loadtxt(path, delimiter=",", skiprows=1, dtype=np.float64, ndmin=2)
    return d[:, 1] + 1j * d[:, 2]


def format_vector_csv(x) -> str:
    out = ["index,re,im\n"]
    for i, z in enumerate(x):
        out.append("%d,%.17g,%.17g\n" % (i, z.real, z.imag))
    return "".join(out)
