"""Schwarz domain decomposition, reference API (schwarz.hpp:16-89) over the
device implementation (cvk_schwarz_solve, csrc/cvk_ddm.cu).

  partition               schwarz.cpp:93-109
  schwarz_solve           schwarz.cpp:111-238 (all strips' inner solves in one
                          batched cooperative launch per outer sweep)
  tune_parameters         schwarz.cpp:240-280
  default_candidate_grid  schwarz.cpp:282-301
  write_ddm_report_csv / write_tune_table_csv   schwarz.cpp:303-333
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .cavac import (Device, ExecMode, InvalidArgument, SolveReport, SolverId, SolverOptions,
                    _BRK, _dev_mode)
from .helmholtz import CavityGrid, HelmholtzProblem


class CvkGrid(C.Structure):
    _fields_ = [("width", C.c_double), ("height", C.c_double), ("h", C.c_double),
                ("nx", C.c_int64), ("ny", C.c_int64), ("roof_begin", C.c_int64),
                ("roof_end", C.c_int64), ("admittance_re", C.c_double), ("admittance_im", C.c_double)]


def _setup_lib():
    L = _lib.load()
    P = C.c_void_p
    L.cvk_partition.argtypes = [C.c_int64, C.c_int64, P]
    L.cvk_partition.restype = C.c_int
    L.cvk_schwarz_solve.argtypes = [P, C.POINTER(CvkGrid), C.c_double, C.c_int64, C.c_int64, P, P, P, P,
                                    C.c_int64, P, P, P, C.POINTER(_lib.CvkOpts), C.c_double, C.c_int64,
                                    C.c_int, P, C.POINTER(_lib.CvkDdmReport)]
    L.cvk_schwarz_solve.restype = C.c_int
    return L


@dataclass
class Partition:
    """Vertical strips of interior columns, leftovers to the left (schwarz.hpp:16-24)."""
    n_sub: int = 1
    col_begin: List[int] = field(default_factory=list)
    cut_columns: List[int] = field(default_factory=list)

    def strip_width(self, s: int) -> int:
        return self.col_begin[s + 1] - self.col_begin[s]


@dataclass
class TransmissionParams:
    """Robin coefficients: the subdomain left of a cut applies s_left on its
    right boundary, the one right of it s_right (schwarz.hpp:30-33)."""
    s_left: complex
    s_right: complex


@dataclass
class DdmReport:
    outer_iterations: int = 0
    interface_residual_history: List[float] = field(default_factory=list)
    converged: bool = False
    per_subdomain_solves: List[SolveReport] = field(default_factory=list)
    total_inner_iterations: int = 0
    device_time: float = 0.0
    wall_time: float = 0.0


@dataclass
class DdmResult:
    x: np.ndarray
    report: DdmReport


def partition(grid: CavityGrid, n_sub: int) -> Partition:
    if n_sub < 1:
        raise InvalidArgument("partition: n_sub must be >= 1")
    if n_sub > 1 and grid.nx // 3 < n_sub:
        raise InvalidArgument("partition: too many subdomains, each strip needs >= 3 columns")
    L = _setup_lib()
    cb = np.zeros(n_sub + 1, np.int64)
    rc = L.cvk_partition(grid.nx, n_sub, cb.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise InvalidArgument(_lib.last_error())
    return Partition(n_sub, [int(v) for v in cb], [int(v) for v in cb[1:-1]])


def _grid(g: CavityGrid) -> CvkGrid:
    a = complex(g.wall_admittance)
    return CvkGrid(g.width, g.height, g.h, g.nx, g.ny, g.roof_begin, g.roof_end, a.real, a.imag)


def schwarz_solve(problem: HelmholtzProblem, part: Partition, tp: TransmissionParams,
                  inner: SolverOptions, ddm_tol: float, max_outer: int,
                  inner_solver: SolverId = SolverId.BiCGStab,
                  mode: Optional[ExecMode] = None, warm_start: bool = False) -> DdmResult:
    """schwarz_solve (schwarz.cpp:111-238).  warm_start (beyond the reference,
    BiCGSTAB inner solver): each strip's inner solve starts from its
    previous-sweep solution instead of 0."""
    if warm_start and SolverId(inner_solver) != SolverId.BiCGStab:
        raise InvalidArgument("schwarz_solve: warm_start needs the bicgstab inner solver")
    L = _setup_lib()
    A = problem.A
    n = A.nrows
    b = np.ascontiguousarray(problem.b, np.complex128)
    x = np.zeros(n, np.complex128)
    hist = np.zeros(max_outer + 1, np.float64)
    subs = (_lib.CvkReport * max(1, part.n_sub))()
    rep = _lib.CvkDdmReport()
    rep.jump_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    rep.jump_cap = len(hist)
    rep.sub_reports = C.cast(subs, C.POINTER(_lib.CvkReport))
    rep.n_sub_reports = part.n_sub
    cb = np.asarray(part.col_begin, np.int64)
    sl = np.array([complex(tp.s_left).real, complex(tp.s_left).imag])
    sr = np.array([complex(tp.s_right).real, complex(tp.s_right).imag])
    o = _lib.CvkOpts(float(inner.tol), int(inner.max_iter), int(inner.l), int(inner.m), 0, _dev_mode(mode),
                     1 if warm_start else 0, 0)
    g = _grid(problem.grid)
    p = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    code = L.cvk_schwarz_solve(Device.default().handle, C.byref(g), float(problem.c), n, A.nnz(),
                               p(A.row_offsets), p(A.col_indices), p(A.values), p(b), part.n_sub, p(cb),
                               p(sl), p(sr), C.byref(o), float(ddm_tol), int(max_outer), int(inner_solver),
                               p(x), C.byref(rep))
    if code in (-1, -5, -6):
        raise InvalidArgument(_lib.last_error())
    _lib.check(code)
    reps = [SolveReport(bool(s.converged), int(s.iterations), s.final_relres, s.true_relres, 0.0, [],
                        _BRK.get(s.breakdown)) for s in subs[: part.n_sub]]
    r = DdmReport(int(rep.outer_iterations), list(hist[: min(rep.jump_len, len(hist))]), bool(rep.converged),
                  reps, int(rep.total_inner_iterations), rep.device_time_s, rep.wall_time_s)
    return DdmResult(x, r)


@dataclass
class TuneEntry:
    params: TransmissionParams
    outer_iterations: int
    total_inner_iterations: int
    converged: bool


@dataclass
class TuneResult:
    best: TransmissionParams
    table: List[TuneEntry]


def tune_entry(problem: HelmholtzProblem, part: Partition, tp: TransmissionParams, inner: SolverOptions,
               budget: int, mode: Optional[ExecMode] = None) -> TuneEntry:
    """One candidate of tune_parameters: schwarz_solve at ddm_tol 1e-6 within the budget."""
    r = schwarz_solve(problem, part, tp, inner, 1e-6, budget, mode=mode)
    return TuneEntry(tp, r.report.outer_iterations, r.report.total_inner_iterations, r.report.converged)


def select_best(table: List[TuneEntry]) -> TuneResult:
    """schwarz.cpp:258-279 over a complete table in candidate order."""
    best, key = None, None
    for e in table:
        if not e.converged:
            continue
        k = (e.outer_iterations, e.total_inner_iterations)
        if key is None or k < key:
            key, best = k, e.params
    if best is None:
        msg = "tune_parameters: all candidates diverged;" + "".join(
            f" ({e.params.s_left.real:f}+{e.params.s_left.imag:f}i / {e.params.s_right.real:f}+"
            f"{e.params.s_right.imag:f}i: {e.outer_iterations})" for e in table)
        raise RuntimeError(msg)
    return TuneResult(best, table)


def tune_parameters(problem: HelmholtzProblem, part: Partition, candidates: List[TransmissionParams],
                    inner: SolverOptions, budget: int, mode: Optional[ExecMode] = None) -> TuneResult:
    """schwarz.cpp:240-280: minimiser by outer iterations, ties by total inner
    iterations of the last sweep; RuntimeError when every candidate diverges.
    (ddm_dist.tune_parameters_distributed spreads the candidates over GPUs.)"""
    if not candidates:
        raise InvalidArgument("tune_parameters: empty candidate grid")
    return select_best([tune_entry(problem, part, tp, inner, budget, mode) for tp in candidates])


def default_candidate_grid(k: float) -> List[TransmissionParams]:
    """schwarz.cpp:282-301: i k baseline, 5 x 5 symmetric, 10 two-sided pairs."""
    out = [TransmissionParams(complex(0.0, k), complex(0.0, k))]
    re_scales = (0.25, 1.0, 4.0, 16.0, 64.0)
    im_scales = (0.0, 0.25, 1.0, 4.0, 16.0)
    for rs in re_scales:
        for is_ in im_scales:
            s = complex(rs * k, is_ * k)
            out.append(TransmissionParams(s, s))
    for rs in re_scales:
        s = complex(rs * k, k)
        out.append(TransmissionParams(s, 2.0 * s))
        out.append(TransmissionParams(2.0 * s, s))
    return out


def write_ddm_report_csv(path: str, part: Partition, tp: TransmissionParams, report: DdmReport) -> None:
    with open(path, "w") as f:
        f.write("n_sub,s_left_re,s_left_im,s_right_re,s_right_im,outer_iters,converged\n")
        f.write("%d,%.17g,%.17g,%.17g,%.17g,%d,%d\n" % (part.n_sub, tp.s_left.real, tp.s_left.imag,
                                                          tp.s_right.real, tp.s_right.imag,
                                                          report.outer_iterations, 1 if report.converged else 0))


def write_tune_table_csv(path: str, table: List[TuneEntry]) -> None:
    with open(path, "w") as f:
        f.write("s_left_re,s_left_im,s_right_re,s_right_im,outer_iters,total_inner_iters,converged\n")
        for e in table:
            f.write("%.17g,%.17g,%.17g,%.17g,%d,%d,%d\n" % (
                e.params.s_left.real, e.params.s_left.imag, e.params.s_right.real, e.params.s_right.imag,
                e.outer_iterations, e.total_inner_iterations, 1 if e.converged else 0))
