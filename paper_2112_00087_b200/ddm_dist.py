"""Multi-GPU Schwarz domain decomposition: one process per GPU, each owning a
contiguous block of the reference's vertical strips (SURVEY.md 8(e) mode 2).

The reference runs its subdomains sequentially in one address space
(schwarz.cpp:152-234).  Here rank r owns strips [s_r, s_{r+1}) on its device
(cvk_ddm_rank_*: local systems, batched inner solves, Robin trace update on
the rank's internal cuts).  Per outer sweep the only traffic between ranks is
the exchange step of the reference's own algorithm:

  * each external cut moves one interface trace (ny complex values) in each
    direction -- the new g computed from the local side's edge column
    (schwarz.cpp:194-206) goes to the neighbour that owns the other side;
  * the interface-jump terms (2 ny doubles per cut, zero where not owned) are
    sum-reduced and then summed sequentially in the reference's order (per
    cut, per row, left column then right, schwarz.cpp:211-220), so every rank
    sees bitwise the single-process jump and takes the same convergence
    decision;
  * the inner-breakdown flag (max) and the inner iteration total (sum).

Iterates are therefore bitwise those of the single-process solve for any
number of ranks (and, in REF mode, those of the reference).

The rank engine is pluggable: DeviceRankEngine (the product; needs the CUDA
library and a device) or, in tests/, an oracle-backed engine that lets the
N>1 host logic run on CPU under gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from .cavac import Device, ExecMode, SolverId, SolverOptions, _dev_mode
from .helmholtz import HelmholtzProblem
from .schwarz import DdmReport, DdmResult, Partition, TransmissionParams, _grid

P = C.c_void_p


class CvkDdmSweepInfo(C.Structure):
    _fields_ = [("inner_breakdown", C.c_int32), ("pad", C.c_int32), ("total_inner_iterations", C.c_int64),
                ("device_time_s", C.c_double), ("kernel_launches", C.c_int64)]


def _bind(L):
    if getattr(L, "_ddm_rank_bound", False):
        return
    from .schwarz import CvkGrid
    L.cvk_ddm_rank_create.argtypes = [P, C.POINTER(CvkGrid), C.c_double, C.c_int64, C.c_int64, P, P, P, P,
                                      C.c_int64, P, C.c_int64, C.c_int64, P, P, C.POINTER(_lib.CvkOpts),
                                      C.c_int, C.POINTER(P)]
    L.cvk_ddm_rank_create.restype = C.c_int
    L.cvk_ddm_rank_sweep.argtypes = [P, P, P, P, P, P, C.POINTER(CvkDdmSweepInfo)]
    L.cvk_ddm_rank_sweep.restype = C.c_int
    L.cvk_ddm_rank_solution.argtypes = [P, P]
    L.cvk_ddm_rank_solution.restype = C.c_int
    L.cvk_ddm_rank_destroy.argtypes = [P]
    L.cvk_ddm_rank_destroy.restype = C.c_int
    L._ddm_rank_bound = True


def strip_ranges(n_sub: int, world: int):
    """Contiguous strip blocks per rank (leftovers to the left, like partition)."""
    if n_sub < world:
        raise ValueError(f"distributed schwarz: {n_sub} strips cannot feed {world} ranks")
    base, rem = divmod(n_sub, world)
    out, s = [], 0
    for r in range(world):
        w = base + (1 if r < rem else 0)
        out.append((s, s + w))
        s += w
    return out


@dataclass
class SweepOut:
    g_out_left: np.ndarray   # ny complex (zeros if no left external cut)
    g_out_right: np.ndarray
    terms: np.ndarray        # (ns + 1, ny, 2) float64
    inner_breakdown: bool
    inner_iterations: int
    device_time: float


class DeviceRankEngine:
    """The rank's strips on its GPU through cvk_ddm_rank_* (csrc/cvk_ddm.cu)."""

    def __init__(self, problem: HelmholtzProblem, part: Partition, tp: TransmissionParams,
                 inner: SolverOptions, inner_solver: SolverId, s_begin: int, s_end: int,
                 mode: Optional[ExecMode] = None, dev: Optional[Device] = None):
        L = _lib.load()
        _bind(L)
        self.L = L
        dev = dev or Device.default()
        A = problem.A
        g = problem.grid
        self.ny = g.ny
        self.ns = s_end - s_begin
        self.ncols = part.col_begin[s_end] - part.col_begin[s_begin]
        self._g = _grid(g)
        cb = np.asarray(part.col_begin, np.int64)
        sl = np.array([complex(tp.s_left).real, complex(tp.s_left).imag])
        sr = np.array([complex(tp.s_right).real, complex(tp.s_right).imag])
        o = _lib.CvkOpts(float(inner.tol), int(inner.max_iter), int(inner.l), int(inner.m), 0, _dev_mode(mode))
        b = np.ascontiguousarray(problem.b, np.complex128)
        p = lambda a: a.ctypes.data_as(P)  # noqa: E731
        h = P()
        _lib.check(L.cvk_ddm_rank_create(dev.handle, C.byref(self._g), float(problem.c), A.nrows, A.nnz(),
                                         p(A.row_offsets), p(A.col_indices), p(A.values), p(b), part.n_sub,
                                         p(cb), s_begin, s_end, p(sl), p(sr), C.byref(o), int(inner_solver),
                                         C.byref(h)))
        self.h = h
        self._gol = np.zeros(self.ny, np.complex128)
        self._gor = np.zeros(self.ny, np.complex128)
        self._terms = np.zeros((self.ns + 1, self.ny, 2), np.float64)

    def sweep(self, g_in_left: Optional[np.ndarray], g_in_right: Optional[np.ndarray]) -> SweepOut:
        info = CvkDdmSweepInfo()
        gil = None if g_in_left is None else np.ascontiguousarray(g_in_left, np.complex128)
        gir = None if g_in_right is None else np.ascontiguousarray(g_in_right, np.complex128)
        p = lambda a: None if a is None else a.ctypes.data_as(P)  # noqa: E731
        _lib.check(self.L.cvk_ddm_rank_sweep(self.h, p(gil), p(gir), p(self._gol), p(self._gor), p(self._terms),
                                             C.byref(info)))
        return SweepOut(self._gol.copy(), self._gor.copy(), self._terms.copy(), bool(info.inner_breakdown),
                        int(info.total_inner_iterations), info.device_time_s)

    def solution(self) -> np.ndarray:
        x = np.zeros(self.ny * self.ncols, np.complex128)
        _lib.check(self.L.cvk_ddm_rank_solution(self.h, x.ctypes.data_as(P)))
        return x.reshape(self.ny, self.ncols)

    def close(self):
        if self.h:
            self.L.cvk_ddm_rank_destroy(self.h)
            self.h = None


class _Comm:
    """torch.distributed plumbing for numpy payloads (gloo: CPU tensors,
    nccl: tensors on the rank's current CUDA device)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")

    def _t(self, a: np.ndarray):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def _grank(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def exchange(self, to_left: Optional[np.ndarray], to_right: Optional[np.ndarray], ny: int):
        """Send to_left to rank-1 and to_right to rank+1; return what they sent us."""
        dist, torch = self.dist, self.torch
        ops, from_left, from_right = [], None, None
        if self.rank > 0:
            send_l = self._t(to_left.view(np.float64))
            from_left = torch.empty(2 * ny, dtype=torch.float64, device=self.device)
            ops += [dist.P2POp(dist.isend, send_l, self._grank(self.rank - 1), self.group),
                    dist.P2POp(dist.irecv, from_left, self._grank(self.rank - 1), self.group)]
        if self.rank + 1 < self.world:
            send_r = self._t(to_right.view(np.float64))
            from_right = torch.empty(2 * ny, dtype=torch.float64, device=self.device)
            ops += [dist.P2POp(dist.isend, send_r, self._grank(self.rank + 1), self.group),
                    dist.P2POp(dist.irecv, from_right, self._grank(self.rank + 1), self.group)]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        cv = lambda t: None if t is None else t.cpu().numpy().view(np.complex128).copy()  # noqa: E731
        return cv(from_left), cv(from_right)

    def allreduce(self, a: np.ndarray, op: str = "sum") -> np.ndarray:
        t = self._t(a)
        self.dist.all_reduce(t, op=getattr(self.dist.ReduceOp, op.upper()), group=self.group)
        return t.cpu().numpy()

    def allgather_obj(self, obj):
        out = [None] * self.world
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


EngineFactory = Callable[..., object]


def schwarz_solve_distributed(problem: HelmholtzProblem, part: Partition, tp: TransmissionParams,
                              inner: SolverOptions, ddm_tol: float, max_outer: int,
                              inner_solver: SolverId = SolverId.BiCGStab, mode: Optional[ExecMode] = None,
                              group=None, engine_factory: Optional[EngineFactory] = None,
                              gather_solution: bool = True) -> DdmResult:
    """schwarz_solve (schwarz.cpp:111-238) across the ranks of a
    torch.distributed group (initialised by the caller), strips split in
    contiguous blocks.  Every rank returns the same report; with
    gather_solution the full x (else only this rank's columns, x[:, c0:c1]
    flattened row-major in the report-free DdmResult.x)."""
    comm = _Comm(group)
    n_sub = part.n_sub
    if n_sub < 2:
        raise ValueError("distributed schwarz needs n_sub >= 2")
    ranges = strip_ranges(n_sub, comm.world)
    s0, s1 = ranges[comm.rank]
    ny = problem.grid.ny
    ncut = n_sub - 1
    factory = engine_factory or DeviceRankEngine
    eng = factory(problem, part, tp, inner, inner_solver, s0, s1, mode)
    rep = DdmReport()
    g_in_left = g_in_right = None
    res0 = -1.0
    try:
        for outer in range(1, max_outer + 1):
            out = eng.sweep(g_in_left, g_in_right)
            g_in_left, g_in_right = comm.exchange(out.g_out_left, out.g_out_right, ny)
            # jump terms onto the global (cut, row, side) grid; each entry is
            # owned by exactly one rank, so the sum-reduce is exact
            T = np.zeros((ncut, ny, 2), np.float64)
            for j in range(s1 - s0 + 1):
                q = s0 + j - 1
                if 0 <= q < ncut:
                    T[q] = out.terms[j]
            T = comm.allreduce(T, "sum")
            iters = comm.allreduce(np.array([out.inner_iterations], np.int64), "sum")
            mx = comm.allreduce(np.array([1.0 if out.inner_breakdown else 0.0, out.device_time], np.float64), "max")
            # sequential left-to-right sum in the reference's order
            jump2 = float(np.add.accumulate(T.ravel())[-1]) if T.size else 0.0
            jump = float(np.sqrt(jump2))
            rep.interface_residual_history.append(jump)
            rep.outer_iterations = outer
            rep.total_inner_iterations = int(iters[0])
            rep.device_time += float(mx[1])  # max over ranks per sweep
            if mx[0] > 0:
                rep.converged = False
                break
            if res0 < 0.0:
                res0 = jump
            if jump == 0.0 or jump <= ddm_tol * res0:
                rep.converged = True
                break
        mine = eng.solution()
    finally:
        eng.close()
    if not gather_solution:
        return DdmResult(mine.ravel(), rep)
    blocks = comm.allgather_obj((part.col_begin[s0], mine))
    x = np.zeros((ny, problem.grid.nx), np.complex128)
    for c0, blk in blocks:
        x[:, c0:c0 + blk.shape[1]] = blk
    return DdmResult(x.ravel(), rep)


def tune_parameters_distributed(problem: HelmholtzProblem, part: Partition, candidates, inner: SolverOptions,
                                budget: int, mode: Optional[ExecMode] = None, group=None, entry_fn=None):
    """tune_parameters (schwarz.cpp:240-280) with the candidates spread over the
    ranks of a torch.distributed group (candidate i on rank i % world, each a
    complete single-device schwarz_solve -- the sweep is embarrassingly
    parallel).  The table is gathered back into
    candidate order, so the minimiser, the tie-break and the all-diverged
    error are the reference's on every rank."""
    from .schwarz import InvalidArgument, select_best, tune_entry
    if not candidates:
        raise InvalidArgument("tune_parameters: empty candidate grid")
    comm = _Comm(group)
    fn = entry_fn or tune_entry
    mine = {i: fn(problem, part, tp, inner, budget, mode) for i, tp in enumerate(candidates)
            if i % comm.world == comm.rank}
    table = {}
    for part_table in comm.allgather_obj(mine):
        table.update(part_table)
    return select_best([table[i] for i in range(len(candidates))])
