"""Python mirror of the reference's solver API (namespace cavac), backed by
the B200 kernels through the C ABI.  Names, argument meaning and error
behaviour follow the reference headers (paths relative to proj/core/):

  numkit.hpp:11-65    Complex/CVector (numpy complex128), CsrMatrix,
                      csr_from_triplets, csr_identity, spmv, dot_hermitian,
                      norm2, axpy, axpy_inplace, xpay_inplace, scale_inplace,
                      ExecMode / set_exec_mode / exec_mode
  krylov.hpp:13-69    SolverOptions, Preconditioner, SolveReport, SolveResult,
                      identity_preconditioner, jacobi, bicgstab, bicgstab_l,
                      tfqmr, SolverId, solver_from_name, solver_name, solve
                      (+ gmres, beyond the reference)

std::invalid_argument -> InvalidArgument (a ValueError), std::logic_error ->
LogicError, std::runtime_error -> RuntimeError.  Vectors live on the host as
numpy arrays (the reference's CVector); matrices are uploaded to the device
once and cached on the CsrMatrix.  The reference's two kernel modes
(numkit.hpp:14-18) both give its iterates bit for bit: ExecMode.Sequential
sums every dot in one device thread, ExecMode.Parallel forms the element terms
with a whole CTA and keeps one thread on the dependent adds.  ExecMode.Fast
(beyond the reference, the default of this module) is the product path:
double-double reductions and the streamed phase kernels.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import CvkError, CvkOpts, CvkReport, check


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class LogicError(RuntimeError):
    """std::logic_error in the reference."""


class ExecMode(enum.IntEnum):
    Sequential = 0
    Parallel = 1
    Fast = 2  # beyond the reference: the B200 product arithmetic


class SolverId(enum.IntEnum):
    BiCGStab = 0
    BiCGStabL = 1
    TfQmr = 2
    GMRES = 3  # beyond the reference
    COCG = 4  # beyond the reference: conjugate orthogonal CG (complex-symmetric A)


_NAMES = {SolverId.BiCGStab: "bicgstab", SolverId.BiCGStabL: "bicgstab_l",
          SolverId.TfQmr: "tfqmr", SolverId.GMRES: "gmres", SolverId.COCG: "cocg"}


def solver_name(sid: SolverId) -> str:
    return _NAMES[SolverId(sid)]


def solver_from_name(name: str) -> SolverId:
    """krylov.cpp:377-384: the reference's three names; "gmres" is rejected
    with the reference's message (test_krylov.cpp:35-46, test_config.cpp:37-46).
    The B200 extensions are reached through solver_id / gmres()."""
    for k in (SolverId.BiCGStab, SolverId.BiCGStabL, SolverId.TfQmr):
        if _NAMES[k] == name:
            return k
    raise InvalidArgument(f'unknown solver "{name}" (allowed: bicgstab, bicgstab_l, tfqmr)')


def solver_id(name: str) -> SolverId:
    """solver_from_name plus the B200 extensions ("gmres", "cocg")."""
    for k, v in _NAMES.items():
        if v == name:
            return k
    raise InvalidArgument(f'unknown solver "{name}" (allowed: bicgstab, bicgstab_l, tfqmr, gmres, cocg)')


# ------------------------------------------------------------- device ----

class Device:
    """One CUDA device context (cvk_ctx): stream, workspace, exec mode."""

    _default: Optional["Device"] = None

    def __init__(self, index: int = 0):
        L = _lib.load()
        h = C.c_void_p()
        check(L.cvk_ctx_create(index, C.byref(h)))
        self.handle = h
        self.index = index

    @classmethod
    def default(cls) -> "Device":
        if cls._default is None:
            cls._default = Device(0)
        return cls._default

    def close(self):
        if self.handle:
            _lib.load().cvk_ctx_destroy(self.handle)
            self.handle = None


_mode = ExecMode.Fast


def set_exec_mode(mode: ExecMode) -> None:
    global _mode
    _mode = ExecMode(mode)


def exec_mode() -> ExecMode:
    return _mode


def _dev_mode(mode: Optional[ExecMode] = None) -> int:
    m = _mode if mode is None else ExecMode(mode)
    return {ExecMode.Sequential: _lib.MODE_REF, ExecMode.Parallel: _lib.MODE_REF_PAR}.get(m, _lib.MODE_FAST)


class path_options:
    """Execution-path options of the default device context (cvk_ctx_set_option),
    restored on exit: ``with path_options(phased_min_n=0, stream=0): ...``.
    For path-parity tests and measurements; the defaults are the product's."""

    def __init__(self, **kw):
        self.kw = kw
        self.saved = {}

    def __enter__(self):
        L = _lib.load()
        h = Device.default().handle
        for k, v in self.kw.items():
            key = _lib.OPTIONS[k]
            old = C.c_int64()
            check(L.cvk_ctx_get_option(h, key, C.byref(old)))
            self.saved[key] = old.value
            check(L.cvk_ctx_set_option(h, key, int(v)))
        return self

    def __exit__(self, *exc):
        L = _lib.load()
        h = Device.default().handle
        for key, v in self.saved.items():
            L.cvk_ctx_set_option(h, key, v)
        return False


def option(name: str) -> int:
    """Current value of an execution-path option of the default context."""
    L = _lib.load()
    v = C.c_int64()
    check(L.cvk_ctx_get_option(Device.default().handle, _lib.OPTIONS[name], C.byref(v)))
    return int(v.value)


# ------------------------------------------------------------- numkit ----

def _cvec(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


class CsrMatrix:
    """Complex CSR (numkit.hpp:31-40); columns strictly increasing per row."""

    def __init__(self, nrows: int, ncols: int, row_offsets, col_indices, values):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.row_offsets = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        self.col_indices = np.ascontiguousarray(col_indices, dtype=np.uint64)
        self.values = _cvec(values)
        self._dev = {}

    def nnz(self) -> int:
        return len(self.values)

    def to_triplets(self):
        rows = np.repeat(np.arange(self.nrows, dtype=np.int64), np.diff(self.row_offsets.astype(np.int64)))
        return rows, self.col_indices.astype(np.int64), self.values.copy()

    def device(self, dev: Optional[Device] = None):
        """Upload once per device (cached); returns the cvk_csr handle."""
        dev = dev or Device.default()
        h = self._dev.get(dev.index)
        if h is None:
            if self.nrows != self.ncols:
                raise InvalidArgument("device matrices must be square")
            hh = C.c_void_p()
            check(_lib.load().cvk_csr_upload(dev.handle, self.nrows, self.ncols, self.nnz(),
                                             _ptr(self.row_offsets), _ptr(self.col_indices),
                                             _ptr(self.values), C.byref(hh)))
            h = hh
            self._dev[dev.index] = h
        return h

    def set_values(self, values) -> None:
        """New values on the same pattern (frequency sweeps); updates device copies."""
        v = _cvec(values)
        if len(v) != self.nnz():
            raise InvalidArgument("set_values: nnz mismatch")
        self.values = v
        for h in self._dev.values():
            check(_lib.load().cvk_csr_set_values(h, _ptr(self.values)))

    def __del__(self):
        try:
            L = _lib.load()
            for h in self._dev.values():
                L.cvk_csr_free(h)
        except Exception:
            pass


def csr_from_triplets(rows, cols, values, nrows: int, ncols: int) -> CsrMatrix:
    """numkit.cpp:41-75: range check, stable (row, col) sort, duplicates summed
    in input order.  Host-side setup (not on the device hot path)."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = _cvec(values)
    bad = np.nonzero((rows < 0) | (rows >= nrows) | (cols < 0) | (cols >= ncols))[0]
    if len(bad):
        k = bad[0]
        raise InvalidArgument(f"csr_from_triplets: index out of range at ({rows[k]}, {cols[k]})")
    order = np.lexsort((cols, rows))  # stable
    r, c, v = rows[order], cols[order], vals[order]
    if len(r):
        new = np.ones(len(r), dtype=bool)
        new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        starts = np.nonzero(new)[0]
        # sequential (left-to-right) duplicate sums, as the reference loop does
        if len(starts) == len(r):
            sv = v
        else:
            sv = v[starts].copy()
            ends = np.append(starts[1:], len(r))
            for j in np.nonzero(ends - starts > 1)[0]:
                s = v[starts[j]]
                for q in range(starts[j] + 1, ends[j]):
                    s = s + v[q]
                sv[j] = s
        ur, uc = r[starts], c[starts]
    else:
        ur, uc, sv = r, c, v
    rp = np.zeros(nrows + 1, dtype=np.uint64)
    np.add.at(rp, ur + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    return CsrMatrix(nrows, ncols, rp, uc, sv)


def csr_identity(n: int) -> CsrMatrix:
    return CsrMatrix(n, n, np.arange(n + 1), np.arange(n), np.ones(n, np.complex128))


def spmv(A: CsrMatrix, x, mode: Optional[ExecMode] = None) -> np.ndarray:
    """y = A x on the device (numkit.cpp:88-111)."""
    x = _cvec(x)
    if A.ncols != len(x):
        raise InvalidArgument("spmv: dimension mismatch")
    y = np.zeros(A.nrows, np.complex128)
    if A.nrows:
        check(_lib.load().cvk_spmv(A.device(), _ptr(x), _ptr(y), _dev_mode(mode)))
    return y


def dot_hermitian(x, y, mode: Optional[ExecMode] = None) -> complex:
    x, y = _cvec(x), _cvec(y)
    if len(x) != len(y):
        raise InvalidArgument("dot_hermitian: length mismatch")
    out = np.zeros(2)
    check(_lib.load().cvk_dot(Device.default().handle, len(x), _ptr(x), _ptr(y), _ptr(out), _dev_mode(mode)))
    return complex(out[0], out[1])


def norm2(x, mode: Optional[ExecMode] = None) -> float:
    x = _cvec(x)
    out = C.c_double()
    check(_lib.load().cvk_norm2(Device.default().handle, len(x), _ptr(x), C.byref(out), _dev_mode(mode)))
    return out.value


def axpy_inplace(alpha: complex, x, y: np.ndarray) -> None:
    """y += alpha x (device)."""
    x = _cvec(x)
    if len(x) != len(y):
        raise InvalidArgument("axpy: length mismatch")
    a = np.array([complex(alpha).real, complex(alpha).imag])
    yy = _cvec(y)
    check(_lib.load().cvk_axpy(Device.default().handle, len(x), _ptr(a), _ptr(x), _ptr(yy)))
    y[:] = yy


def axpy(alpha: complex, x, y) -> np.ndarray:
    """alpha x + y into a new vector (numkit.cpp:127-133)."""
    z = _cvec(y).copy()
    if len(_cvec(x)) != len(z):
        raise InvalidArgument("axpy: length mismatch")
    axpy_inplace(alpha, x, z)
    return z


def xpay_inplace(alpha: complex, x: np.ndarray, y) -> None:
    """x = alpha x + y (device)."""
    y = _cvec(y)
    if len(x) != len(y):
        raise InvalidArgument("xpay: length mismatch")
    a = np.array([complex(alpha).real, complex(alpha).imag])
    xx = _cvec(x)
    check(_lib.load().cvk_xpay(Device.default().handle, len(y), _ptr(a), _ptr(xx), _ptr(y)))
    x[:] = xx


def scale_inplace(alpha: complex, x: np.ndarray) -> None:
    """x *= alpha (numkit.cpp:161-163) as alpha*x + 0 on the device."""
    xpay_inplace(alpha, x, np.zeros(len(x), np.complex128))


# ------------------------------------------------------------- krylov ----

@dataclass
class SolverOptions:
    tol: float = 1e-9
    max_iter: int = 10000
    l: int = 8
    m: int = 30  # GMRES restart (beyond reference)
    record_history: bool = False


@dataclass
class SolveReport:
    converged: bool = False
    iterations: int = 0
    final_relres: float = 0.0
    true_relres: float = 0.0
    wall_time: float = 0.0
    residual_history: list = field(default_factory=list)
    breakdown: Optional[str] = None
    device_time: float = 0.0
    kernel_launches: int = 0


@dataclass
class SolveResult:
    x: np.ndarray
    report: SolveReport


class Preconditioner:
    """Left preconditioner x -> M^{-1} x held on the device (krylov.hpp:20-23).
    `inv_diag` is the Jacobi inverse diagonal (None for the identity)."""

    def __init__(self, kind: str, inv_diag: Optional[np.ndarray] = None, A: Optional[CsrMatrix] = None):
        self.kind = kind
        self.inv_diag = inv_diag
        self._A = A
        self._dev = {}

    def apply(self, v) -> np.ndarray:
        v = _cvec(v)
        if self.kind == "identity":
            return v.copy()
        if self.kind == "ilu0":  # device sweeps (cvk_ilu.cu)
            if len(v) != self._A.nrows:
                raise InvalidArgument("preconditioner: dimension mismatch")
            z = np.zeros_like(v)
            check(_lib.load().cvk_precond_apply(self.device(self._A), _ptr(v), _ptr(z)))
            return z
        # elementwise inv_diag[i] * v[i] with the reference rounding (no FMA)
        a, b = self.inv_diag.real, self.inv_diag.imag
        c, d = v.real, v.imag
        return (a * c - b * d) + 1j * (a * d + b * c)

    def device(self, A: CsrMatrix, dev: Optional[Device] = None):
        dev = dev or Device.default()
        key = (dev.index, A.nrows)
        h = self._dev.get(key)
        if h is None:
            hh = C.c_void_p()
            L = _lib.load()
            if self.kind == "identity":
                check(L.cvk_precond_identity(dev.handle, A.nrows, C.byref(hh)))
            elif self.kind == "ilu0":
                if A is not self._A:
                    raise InvalidArgument("ilu0: factor belongs to another matrix")
                code = L.cvk_precond_ilu0(A.device(dev), self.sweeps, C.byref(hh))
                if code == -5:
                    raise InvalidArgument(_lib.last_error())
                check(code)
            else:
                if len(self.inv_diag) != A.nrows:
                    raise InvalidArgument("preconditioner: dimension mismatch")
                check(L.cvk_precond_jacobi(A.device(dev), _ptr(self.inv_diag), C.byref(hh)))
            h = hh
            self._dev[key] = h
        return h

    def __del__(self):
        try:
            L = _lib.load()
            for h in self._dev.values():
                L.cvk_precond_free(h)
        except Exception:
            pass


def identity_preconditioner() -> Preconditioner:
    return Preconditioner("identity")


def jacobi(A: CsrMatrix) -> Preconditioner:
    """krylov.cpp:31-55: inverse diagonal computed by the device kernel with the
    reference's __divdc3 rounding; zero/missing diagonal -> InvalidArgument."""
    if A.nrows != A.ncols:
        raise InvalidArgument("jacobi: matrix must be square")
    L = _lib.load()
    hh = C.c_void_p()
    code = L.cvk_precond_jacobi(A.device(), None, C.byref(hh))
    if code == -5:
        raise InvalidArgument(_lib.last_error())
    check(code)
    d = np.zeros(A.nrows, np.complex128)
    if A.nrows:
        check(L.cvk_precond_get_diag(hh, _ptr(d)))
    M = Preconditioner("jacobi", d, A)
    M._dev[(Device.default().index, A.nrows)] = hh
    return M


def ilu0(A: CsrMatrix, sweeps: int = 2) -> Preconditioner:
    """ILU(0) (beyond the reference, which has jacobi / identity only,
    krylov.cpp:27-55): exact IKJ factor on A's pattern, applied on the device
    by `sweeps` Jacobi sweeps per triangle (cvk_ilu.cu).  Zero pivot ->
    InvalidArgument.  solve() accepts it for BiCGStab."""
    if A.nrows != A.ncols:
        raise InvalidArgument("ilu0: matrix must be square")
    if not 0 <= int(sweeps) <= 64:
        raise InvalidArgument("ilu0: sweeps must be in [0, 64]")
    M = Preconditioner("ilu0", None, A)
    M.sweeps = int(sweeps)
    M.device(A)  # factor now: a zero pivot raises here
    return M


def ilu0_factor(M: Preconditioner) -> np.ndarray:
    """The factor in A's value slots: L strict lower (unit diagonal implied), U on and above."""
    if M.kind != "ilu0":
        raise InvalidArgument("ilu0_factor: not an ILU(0) preconditioner")
    f = np.zeros(len(M._A.values), np.complex128)
    if len(f):
        check(_lib.load().cvk_precond_get_ilu0(M.device(M._A), _ptr(f)))
    return f


_BRK = {0: None, 1: "rho breakdown", 2: "stagnation in <shadow, v>", 3: "omega breakdown",
        4: "stagnation in <shadow, u>", 5: "degenerate least-squares in MR step",
        6: "sigma breakdown", 7: "arnoldi breakdown", 8: "stagnation in <p, A p>"}


def _opts(o: SolverOptions, mode: Optional[ExecMode]) -> CvkOpts:
    return CvkOpts(float(o.tol), int(o.max_iter), int(o.l), int(o.m),
                   1 if o.record_history else 0, _dev_mode(mode), 0, 0)


def _report(r: CvkReport, hist) -> SolveReport:
    h = [] if hist is None else list(hist[: min(r.history_len, len(hist))])
    return SolveReport(bool(r.converged), int(r.iterations), r.final_relres, r.true_relres,
                       r.wall_time_s, h, _BRK.get(r.breakdown, "unknown breakdown"),
                       r.device_time_s, int(r.kernel_launches))


def solve(sid: SolverId, A: CsrMatrix, b, M: Preconditioner, opts: SolverOptions = None,
          mode: Optional[ExecMode] = None) -> SolveResult:
    """krylov.cpp:395-403 dispatch; the whole solve is one device launch."""
    opts = opts or SolverOptions()
    sid = SolverId(sid)
    name = solver_name(sid)
    b = _cvec(b)
    if A.nrows != A.ncols or A.nrows != len(b):
        raise InvalidArgument(f"{name}: dimension mismatch")
    if sid == SolverId.BiCGStabL and opts.l < 1:
        raise InvalidArgument("bicgstab_l: l must be >= 1")
    x = np.zeros(len(b), np.complex128)
    rep = CvkReport()
    hist = None
    if opts.record_history:
        hist = np.zeros(2 * opts.max_iter + 8, np.float64)
        rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.history_cap = len(hist)
    o = _opts(opts, mode)
    L = _lib.load()
    dev = Device.default()
    code = L.cvk_solve(dev.handle, int(sid), A.device(dev), M.device(A, dev), C.byref(o),
                       _ptr(b), _ptr(x), C.byref(rep))
    if code in (-1, -6):
        raise InvalidArgument(_lib.last_error())
    check(code)
    return SolveResult(x, _report(rep, hist))


def bicgstab(A, b, M, opts=None, mode=None):
    return solve(SolverId.BiCGStab, A, b, M, opts, mode)


def bicgstab_l(A, b, M, opts=None, mode=None):
    return solve(SolverId.BiCGStabL, A, b, M, opts, mode)


def tfqmr(A, b, M, opts=None, mode=None):
    return solve(SolverId.TfQmr, A, b, M, opts, mode)


def gmres(A, b, M, opts=None, mode=None):
    return solve(SolverId.GMRES, A, b, M, opts, mode)


def cocg(A, b, M, opts=None, mode=None):
    """Conjugate orthogonal CG (beyond the reference; north_star's CG for the
    complex-symmetric Helmholtz operator A = A^T): one SpMV per iteration,
    the reference's conventions (x0 = 0, Jacobi, relres = ||M^-1 r|| / ||M^-1 b||)."""
    return solve(SolverId.COCG, A, b, M, opts, mode)


def true_relative_residual(A: CsrMatrix, b, x, mode: Optional[ExecMode] = None) -> float:
    b, x = _cvec(b), _cvec(x)
    out = C.c_double()
    check(_lib.load().cvk_true_relres(A.device(), _ptr(b), _ptr(x), C.byref(out), _dev_mode(mode)))
    return out.value
