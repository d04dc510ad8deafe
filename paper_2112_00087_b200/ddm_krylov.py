"""Krylov-accelerated Schwarz interface iteration (
beyond the reference, whose schwarz_solve iterates the sweep as a fixed
point, schwarz.cpp:152-234).

One outer sweep of optimized Schwarz is an affine map of the interface
traces, g -> F(g) = T g + f: the strips' Robin problems are solved with the
current traces as data (k_ddm_rhs + the inner Krylov solves) and the traces
are updated from the local solutions (k_ddm_exchange).  The reference
iterates g <- F(g).  Here GMRES solves the interface equation

    (I - T) g = f,   f = F(0),   (I - T) g = g - (F(g) - f)

with one sweep per operator application, then one last sweep from the
converged traces yields the subdomain solutions.  The sweeps run on the
device through the rank plan (cvk_ddm_rank_*, csrc/cvk_ddm.cu); the GMRES
vectors (2 x cuts x ny complex) live on the host.  Parity is unpinned by the
reference: the solution is checked against the monodomain
solve, as the reference's own DDM = monodomain test does
(acceptance.cpp:277-291).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib
from .cavac import ExecMode, SolverId, SolverOptions
from .ddm_dist import DeviceRankEngine
from .helmholtz import HelmholtzProblem
from .schwarz import Partition, TransmissionParams

P = C.c_void_p


def _bind(L):
    if getattr(L, "_ddm_traces_bound", False):
        return
    L.cvk_ddm_rank_get_traces.argtypes = [P, P, P]
    L.cvk_ddm_rank_get_traces.restype = C.c_int
    L.cvk_ddm_rank_set_traces.argtypes = [P, P, P]
    L.cvk_ddm_rank_set_traces.restype = C.c_int
    L._ddm_traces_bound = True


@dataclass
class KrylovDdmReport:
    sweeps: int = 0                      # outer sweeps (operator applications + 2)
    gmres_iterations: int = 0
    converged: bool = False
    residual_history: List[float] = field(default_factory=list)  # ||(I - T) g - f|| / ||f||
    total_inner_iterations: int = 0
    device_time: float = 0.0


@dataclass
class KrylovDdmResult:
    x: np.ndarray
    report: KrylovDdmReport


class _Interface:
    """The interface map g -> F(g) on one device (every strip on one rank)."""

    def __init__(self, problem, part, tp, inner, inner_solver, mode):
        self.eng = DeviceRankEngine(problem, part, tp, inner, inner_solver, 0, part.n_sub, mode=mode)
        _bind(self.eng.L)
        self.ny = problem.grid.ny
        self.ns = part.n_sub
        self.slots = (self.ns + 1) * self.ny
        self._gl = np.zeros(self.slots, np.complex128)
        self._gr = np.zeros(self.slots, np.complex128)
        self.sweeps = 0
        self.inner = 0
        self.device_time = 0.0

    @property
    def size(self) -> int:  # internal cuts 1 .. ns-1, both traces
        return 2 * (self.ns - 1) * self.ny

    def apply(self, g: np.ndarray) -> np.ndarray:
        ny, L, h = self.ny, self.eng.L, self.eng.h
        m = (self.ns - 1) * ny
        self._gl[:] = 0
        self._gr[:] = 0
        self._gl[ny:ny + m] = g[:m]
        self._gr[ny:ny + m] = g[m:]
        p = lambda a: a.ctypes.data_as(P)  # noqa: E731
        _lib.check(L.cvk_ddm_rank_set_traces(h, p(self._gl), p(self._gr)))
        out = self.eng.sweep(None, None)
        self.sweeps += 1
        self.inner += out.inner_iterations
        self.device_time += out.device_time
        _lib.check(L.cvk_ddm_rank_get_traces(h, p(self._gl), p(self._gr)))
        return np.concatenate([self._gl[ny:ny + m], self._gr[ny:ny + m]])


def _gmres(op, f, tol, restart, max_it, hist):
    """Restarted GMRES (MGS, complex Givens) on the host; x0 = 0."""
    n = len(f)
    x = np.zeros(n, np.complex128)
    fn = np.linalg.norm(f)
    if fn == 0.0:
        return x, 0, True
    its = 0
    r = f.copy()
    while its < max_it:
        beta = np.linalg.norm(r)
        if beta / fn <= tol:
            return x, its, True
        V = np.zeros((restart + 1, n), np.complex128)
        H = np.zeros((restart + 1, restart), np.complex128)
        cs = np.zeros(restart)
        sn = np.zeros(restart, np.complex128)
        gv = np.zeros(restart + 1, np.complex128)
        gv[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(restart):
            w = op(V[j])
            its += 1
            for i in range(j + 1):
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):
                a0, a1 = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * a0 + sn[i] * a1
                H[i + 1, j] = -np.conj(sn[i]) * a0 + cs[i] * a1
            aa, hn = abs(H[j, j]), abs(H[j + 1, j])
            nu = np.hypot(aa, hn)
            if aa == 0:
                cs[j], sn[j] = 0.0, 1.0
            else:
                cs[j], sn[j] = aa / nu, (hn / nu) * (H[j, j] / aa)
            H[j, j] = nu * (H[j, j] / aa) if aa else hn
            H[j + 1, j] = 0
            gv[j + 1] = -np.conj(sn[j]) * gv[j]
            gv[j] = cs[j] * gv[j]
            k = j + 1
            rel = abs(gv[j + 1]) / fn
            hist.append(float(rel))
            if rel <= tol or its >= max_it or hn == 0:
                break
        y = np.linalg.solve(np.triu(H[:k, :k]), gv[:k])
        x = x + V[:k].T @ y
        r = f - op(x)
        its += 1
        if np.linalg.norm(r) / fn <= tol:
            return x, its, True
    return x, its, False


def schwarz_solve_krylov(problem: HelmholtzProblem, part: Partition, tp: TransmissionParams,
                         inner: SolverOptions, tol: float = 1e-8, max_sweeps: int = 300, restart: int = 40,
                         inner_solver: SolverId = SolverId.BiCGStab,
                         mode: Optional[ExecMode] = None) -> KrylovDdmResult:
    """Optimized Schwarz (the reference's subdomain problems, transmission
    conditions and trace update) with the interface equation solved by
    GMRES(restart) to ||(I - T) g - f|| <= tol ||f||, f = F(0)."""
    if part.n_sub < 2:
        raise ValueError("schwarz_solve_krylov: needs at least two strips")
    itf = _Interface(problem, part, tp, inner, inner_solver, mode)
    try:
        f = itf.apply(np.zeros(itf.size, np.complex128))
        hist: List[float] = []
        g, its, ok = _gmres(lambda v: v - (itf.apply(v) - f), f, tol, restart, max(1, max_sweeps - 2), hist)
        itf.apply(g)  # the subdomain solutions for the converged traces
        u = itf.eng.solution()
    finally:
        itf.eng.close()
    rep = KrylovDdmReport(itf.sweeps, its, ok, hist, itf.inner, itf.device_time)
    return KrylovDdmResult(u.reshape(-1), rep)
