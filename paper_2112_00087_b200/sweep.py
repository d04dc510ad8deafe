"""Frequency-sweep driver: the cavity solved at a list of frequencies with
the matrix resident on the device (SURVEY.md 8(f) rank 1, config 2's
50-500 Hz sweep).

The reference solves one frequency per assemble() call (helmholtz.cpp:59-115)
and its only sweep driver, bench_solvers (pipeline.cpp:227-293), walks mesh
sizes: assemble -> jacobi -> solve, report rows of (solver, h, n, iterations,
converged, times), non-converged points reported rather than raised
(SPEC.md:562).  This driver keeps those conventions for a frequency axis:

  * the 5-point pattern is built and uploaded once (helmholtz.pattern);
  * per frequency, cvk_csr_assemble_cavity rewrites the values on the device
    (bitwise the reference's assemble(omega) values) and
    cvk_precond_jacobi_refresh recomputes the Jacobi inverse diagonal
    (krylov.cpp:31-55 rounding);
  * the rhs (k^2 x roof data) is frequency independent (built once);
  * each point is one device solve from x0 = 0 (cvk_solve).

Every point is parity-pinned by the reference's own assemble(omega) + solve
on the same grid (tests/test_gpu_sweep.py).
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Iterable, Optional

import numpy as np

from . import _lib
from .cavac import (CsrMatrix, Device, InvalidArgument, SolverId, SolverOptions, _dev_mode,
                    solver_id, solver_name)
from .helmholtz import CavityGrid, pattern, rhs
from .schwarz import CvkGrid, _grid  # noqa: F401

P = C.c_void_p


def _bind(L):
    if getattr(L, "_sweep_bound", False):
        return
    L.cvk_csr_assemble_cavity.argtypes = [P, C.POINTER(CvkGrid), C.c_double, C.c_double]
    L.cvk_csr_assemble_cavity.restype = C.c_int
    L.cvk_precond_jacobi_refresh.argtypes = [P, P]
    L.cvk_precond_jacobi_refresh.restype = C.c_int
    L.cvk_csr_get_values.argtypes = [P, P]
    L.cvk_csr_get_values.restype = C.c_int
    L._sweep_bound = True


@dataclass
class SweepRow:
    """One frequency point (bench_solvers' BenchRow, pipeline.hpp:37-44, with
    frequency in place of h)."""
    solver: str
    frequency_hz: float
    omega: float
    n: int
    iterations: int
    converged: bool
    final_relres: float
    true_relres: float
    breakdown: str
    device_time_s: float  # solve kernels (CUDA events)
    point_time_s: float   # assemble + jacobi + solve, wall clock


@dataclass
class SweepTable:
    rows: list = field(default_factory=list)
    solutions: dict = field(default_factory=dict)  # frequency -> x (if keep_solutions)


class CavitySweep:
    """Device-resident cavity operator re-evaluated per frequency."""

    def __init__(self, grid: CavityGrid, c: float, dirichlet, dev: Optional[Device] = None):
        dirichlet = np.asarray(dirichlet, np.complex128)
        if len(dirichlet) != grid.roof_size():
            raise InvalidArgument("assemble: dirichlet length does not match roof span")
        self.grid, self.c, self.dev = grid, float(c), dev or Device.default()
        rp, ci, _slot, _has = pattern(grid)
        n = grid.size()
        # values are filled on the device by the first set_frequency()
        self.A = CsrMatrix(n, n, rp, ci, np.zeros(len(ci), np.complex128))
        self.b = rhs(grid, c, dirichlet)
        self._hA = self.A.device(self.dev)
        self._g = _grid(grid)
        L = _lib.load()
        _bind(L)
        self._x = np.zeros(n, np.complex128)
        self._hM = None
        self.omega = None

    def set_frequency(self, f_hz: float) -> None:
        L = _lib.load()
        omega = 2.0 * math.pi * f_hz
        _lib.check(L.cvk_csr_assemble_cavity(self._hA, C.byref(self._g), omega, self.c))
        if self._hM is None:
            h = P()
            _lib.check(L.cvk_precond_jacobi(self._hA, None, C.byref(h)))
            self._hM = h
        else:
            _lib.check(L.cvk_precond_jacobi_refresh(self._hM, self._hA))
        self.omega = omega

    def values(self) -> np.ndarray:
        """Current device values (for parity checks)."""
        y = np.zeros(self.A.nnz(), np.complex128)
        _lib.check(_lib.load().cvk_csr_get_values(self._hA, y.ctypes.data_as(P)))
        return y

    def solve(self, solver=SolverId.BiCGStab, opts: Optional[SolverOptions] = None, mode=None):
        opts = opts or SolverOptions()
        sid = solver_id(solver) if isinstance(solver, str) else SolverId(solver)
        o = _lib.CvkOpts(opts.tol, opts.max_iter, opts.l, opts.m, 0, _dev_mode(mode), 0, 0)
        rep = _lib.CvkReport()
        L = _lib.load()
        # host b / x: 16 n bytes each way per point, ~1e-3 of a point's solve time
        _lib.check(L.cvk_solve(self.dev.handle, int(sid), self._hA, self._hM, C.byref(o),
                               self.b.ctypes.data_as(P), self._x.ctypes.data_as(P), C.byref(rep)))
        return rep

    def x(self) -> np.ndarray:
        return self._x.copy()

    def close(self):
        L = _lib.load()
        if self._hM is not None:
            L.cvk_precond_free(self._hM)
            self._hM = None


def frequency_sweep(grid: CavityGrid, c: float, dirichlet, freqs_hz: Iterable[float],
                    solver="bicgstab", opts: Optional[SolverOptions] = None, mode=None,
                    keep_solutions: bool = False, dev: Optional[Device] = None) -> SweepTable:
    """Solve the cavity at every frequency in freqs_hz; non-converged points
    are reported (converged=False), not raised, as bench_solvers does."""
    sw = CavitySweep(grid, c, dirichlet, dev)
    table = SweepTable()
    sname = solver if isinstance(solver, str) else solver_name(solver)
    try:
        for f in freqs_hz:
            t0 = time.perf_counter()
            sw.set_frequency(float(f))
            rep = sw.solve(sname, opts, mode)
            dt = time.perf_counter() - t0
            table.rows.append(SweepRow(sname, float(f), sw.omega, grid.size(), int(rep.iterations),
                                       bool(rep.converged), rep.final_relres, rep.true_relres,
                                       _lib.load().cvk_breakdown_name(rep.breakdown).decode(),
                                       rep.device_time_s, dt))
            if keep_solutions:
                table.solutions[float(f)] = sw.x()
    finally:
        sw.close()
    return table


def write_sweep_csv(path: str, table: SweepTable) -> None:
    """Schema in the style of write_bench_csv (pipeline.cpp:295-307)."""
    with open(path, "w") as f:
        f.write("solver,frequency_hz,n,iterations,converged,final_relres,true_relres,device_time_s,point_time_s\n")
        for r in table.rows:
            f.write(f"{r.solver},{r.frequency_hz:.17g},{r.n},{r.iterations},{int(r.converged)},"
                    f"{r.final_relres:.17g},{r.true_relres:.17g},{r.device_time_s:.9g},{r.point_time_s:.9g}\n")
