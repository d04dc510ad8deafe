"""Schwarz DDM on algebraic subdomains -- FEM meshes partitioned METIS-style
(here RCB of the mesh points, rowblock.rcb_partition) -- over the C ABI
cvk_asm_* (csrc/cvk_asm.cu).  Beyond the reference, whose schwarz_solve
(schwarz.cpp:111-238) knows only the FD cavity's vertical strips.

Each subdomain owns its rows and solves on them grown by `overlap` graph
layers, with the couplings that leave that set folded into the diagonal by
the reference's Robin factor (1/h - s/2) / (1/h + s/2) (schwarz.cpp:43-50).
The outer iteration is the reference's additive fixed point (m = 0) or
FGMRES(m) preconditioned by the same sweep (m > 0, the default): one-level
Schwarz on Helmholtz with more than two subdomains does not converge as a
fixed point, the Krylov outer loop does.  At convergence the
solution is the monodomain one (b - A u = 0).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .cavac import CsrMatrix, Device, ExecMode, InvalidArgument, SolverId, SolverOptions, _dev_mode
from .schwarz import DdmReport, DdmResult

P = C.c_void_p


def _bind(L):
    if getattr(L, "_asm_bound", False):
        return
    i64 = C.c_int64
    L.cvk_asm_create.argtypes = [P, i64, i64, P, P, P, i64, P, i64, P, C.c_double, C.POINTER(_lib.CvkOpts),
                                 C.c_int, C.POINTER(P)]
    L.cvk_asm_solve.argtypes = [P, P, P, C.c_double, i64, i64, C.POINTER(_lib.CvkDdmReport)]
    L.cvk_asm_apply_device.argtypes = [P, P, P]
    L.cvk_asm_destroy.argtypes = [P]
    L.cvk_asm_n_parts.argtypes = [P]
    L.cvk_asm_n_parts.restype = i64
    L.cvk_asm_create_rank.argtypes = [P, i64, i64, P, P, P, i64, P, i64, P, C.c_double, C.POINTER(_lib.CvkOpts),
                                      C.c_int, C.c_int, C.c_int, C.POINTER(P)]
    L.cvk_asm_set_reducer.argtypes = [P, REDUCE_FN, P, P]
    for f in ("create", "create_rank", "solve", "apply_device", "destroy", "set_reducer"):
        getattr(L, "cvk_asm_" + f).restype = C.c_int
    L._asm_bound = True


# int (*)(void* user, double* z_dev, int64 n, int64* meta)
REDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_int64))


class SubdomainSchwarz:
    """The subdomain systems of A for a partition of its rows, resident on the
    device (cvk_asm_create); solve() runs the outer DDM iteration."""

    def __init__(self, A: CsrMatrix, part_of_row, s_robin: complex, h: float, inner: SolverOptions = None,
                 overlap: int = 1, inner_solver: SolverId = SolverId.BiCGStab, mode: Optional[ExecMode] = None,
                 group=None):
        """group: a torch.distributed group (one rank per GPU): rank r solves
        the subdomains q with q % world == r, one all-reduce per sweep
        completes the preconditioner (cvk_asm_create_rank)."""
        L = _lib.load()
        _bind(L)
        self.L = L
        inner = inner or SolverOptions(tol=1e-10)
        part = np.ascontiguousarray(part_of_row, np.int64)
        if len(part) != A.nrows:
            raise InvalidArgument("schwarz: part_of_row must have one entry per row")
        self.n_parts = int(part.max()) + 1 if len(part) else 0
        rp = np.ascontiguousarray(A.row_offsets, np.uint64)
        ci = np.ascontiguousarray(A.col_indices, np.uint64)
        v = np.ascontiguousarray(A.values, np.complex128)
        s = np.array([complex(s_robin).real, complex(s_robin).imag])
        o = _lib.CvkOpts(float(inner.tol), int(inner.max_iter), int(inner.l), int(inner.m), 0, _dev_mode(mode), 0, 0)
        h_ = P()
        p = lambda a: a.ctypes.data_as(P)  # noqa: E731
        rank, world = 0, 1
        if group is not None or _dist_initialized():
            import torch.distributed as dist
            rank, world = dist.get_rank(group), dist.get_world_size(group)
        code = L.cvk_asm_create_rank(Device.default().handle, A.nrows, len(v), p(rp), p(ci), p(v), self.n_parts,
                                     p(part), int(overlap), p(s), float(h), C.byref(o), int(inner_solver), rank, world,
                                     C.byref(h_))
        if code in (-1, -6):
            raise InvalidArgument(_lib.last_error())
        _lib.check(code)
        self.h = h_
        self.n = A.nrows
        self.rank, self.world = rank, world
        if world > 1:
            self._install_reducer(group)

    def _install_reducer(self, group):
        """Sum over ranks of each sweep's owned-row results (an all-reduce of
        n complex values on the rank's device, plus the sweep's counters)."""
        import torch
        import torch.distributed as dist
        dev = torch.device("cuda", torch.cuda.current_device())
        self._buf = torch.zeros(2 * self.n, dtype=torch.float64, device=dev)
        meta_t = torch.zeros(2, dtype=torch.int64)

        def reduce(user, z_dev, n, meta):
            try:
                dist.all_reduce(self._buf, group=group)
                meta_t[0], meta_t[1] = meta[0], meta[1]
                m0 = meta_t[:1].clone()
                m1 = meta_t[1:].clone()
                dist.all_reduce(m0, group=group)
                dist.all_reduce(m1, op=dist.ReduceOp.MAX, group=group)
                torch.cuda.synchronize(dev)
                meta[0], meta[1] = int(m0[0]), int(m1[0])
                return 0
            except Exception:  # the C side reports CVK_ECUDA
                return 1

        self._reduce_cb = REDUCE_FN(reduce)  # keep alive
        _lib.check(self.L.cvk_asm_set_reducer(self.h, self._reduce_cb, None, C.c_void_p(self._buf.data_ptr())))

    def solve(self, b, tol: float = 1e-8, max_outer: int = 300, m: int = 30) -> DdmResult:
        b = np.ascontiguousarray(b, np.complex128)
        x = np.zeros(self.n, np.complex128)
        hist = np.zeros(max_outer + 2, np.float64)
        rep = _lib.CvkDdmReport()
        rep.jump_history = hist.ctypes.data_as(C.POINTER(C.c_double))
        rep.jump_cap = len(hist)
        _lib.check(self.L.cvk_asm_solve(self.h, b.ctypes.data_as(P), x.ctypes.data_as(P), float(tol), int(max_outer),
                                        int(m), C.byref(rep)))
        r = DdmReport(outer_iterations=int(rep.outer_iterations),
                      interface_residual_history=list(hist[: min(rep.jump_len, len(hist))]),
                      converged=bool(rep.converged), total_inner_iterations=int(rep.total_inner_iterations),
                      device_time=rep.device_time_s, wall_time=rep.wall_time_s)
        return DdmResult(x, r)

    def close(self):
        if self.h:
            self.L.cvk_asm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dist_initialized() -> bool:
    try:
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1
    except Exception:
        return False


def schwarz_solve_subdomains(A: CsrMatrix, b, part_of_row, s_robin: complex, h: float,
                             inner: SolverOptions = None, ddm_tol: float = 1e-8, max_outer: int = 300,
                             m: int = 30, overlap: int = 1, inner_solver: SolverId = SolverId.BiCGStab,
                             mode: Optional[ExecMode] = None, group=None) -> DdmResult:
    """One call: build the subdomain systems, run the outer iteration, free.
    Under torch.distributed (or with `group`) the subdomains are split over
    the ranks, one GPU each."""
    S = SubdomainSchwarz(A, part_of_row, s_robin, h, inner, overlap, inner_solver, mode, group)
    try:
        return S.solve(b, ddm_tol, max_outer, m)
    finally:
        S.close()
