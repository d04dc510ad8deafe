"""Row-block global Krylov: the global BiCGSTAB solve with the rows split over
ranks (SURVEY.md 8(e) mode 1).  Beyond the reference, whose solve()
(krylov.hpp:68-69, krylov.cpp:57-138) runs in one address space; the
iterates are bitwise those of a single-device FAST solve for any number of
blocks.

Each rank owns a contiguous block of rows [r0, r1) (nnz-balanced by
default).  Its local columns are its own rows first, then a halo: the
sorted rows of other ranks that its rows reference.  Per reduction phase of
BiCGSTAB there is one all-gather of a small exchange slot per rank carrying
the rank's double-double partial sums and the boundary values other ranks
read (r after the x/r update, p and v after the first SpMV phase); every
rank then folds the partials in rank order and runs the same scalar
recurrence (csrc/cvk_rowblock.cu).

Three ways to run the blocks:
  * solve_row_blocks     -- n blocks on one device, the all-gather done by
                            stream-ordered device copies (one C call);
  * solve_distributed    -- one block per rank of a torch.distributed group;
                            NCCL all-gathers on the library's stream (no host
                            round trip per phase), gloo staged through host;
  * RowBlockEngine       -- the per-rank engine both use; tests plug a numpy
                            engine into solve_distributed to run the N>1
                            host logic on CPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, List, Optional

import numpy as np

from . import _lib
from .cavac import (CsrMatrix, Device, InvalidArgument, Preconditioner, SolveReport, SolveResult, SolverId,
                    SolverOptions, _BRK, _cvec)

P = C.c_void_p
PH_INIT, PH_A, PH_B, PH_C, PH_X, PH_T = range(6)
ITER_PHASES = (PH_A, PH_B, PH_C)
ITERS_PER_POLL = 8  # iterations queued between reads of the device stop flag


class CvkRowblockDesc(C.Structure):
    _fields_ = [("n_own", C.c_int64), ("n_halo", C.c_int64), ("nnz", C.c_int64),
                ("row_offsets", P), ("col_local", P), ("values", P), ("inv_diag", P), ("b", P),
                ("n_send", C.c_int64), ("send_rows", P), ("n_ranks", C.c_int64), ("max_send", C.c_int64),
                ("halo_src", P), ("history_cap", C.c_int64)]


def _bind(L):
    if getattr(L, "_rb_bound", False):
        return
    i32, i64 = C.c_int, C.c_int64
    L.cvk_rowblock_create.argtypes = [P, C.POINTER(CvkRowblockDesc), i32, C.POINTER(_lib.CvkOpts), C.POINTER(P)]
    L.cvk_rowblock_exchange.argtypes = [P, C.POINTER(P), C.POINTER(P), C.POINTER(i64)]
    L.cvk_rowblock_local.argtypes = [P, i32]
    L.cvk_rowblock_post.argtypes = [P, i32]
    L.cvk_rowblock_exchange_local.argtypes = [C.POINTER(P), i32]
    L.cvk_rowblock_solve_local.argtypes = [C.POINTER(P), i32]
    L.cvk_rowblock_done.argtypes = [P, C.POINTER(i32)]
    L.cvk_rowblock_result.argtypes = [P, P, C.POINTER(_lib.CvkReport)]
    L.cvk_rowblock_destroy.argtypes = [P]
    L.cvk_nccl_unique_id.argtypes = [C.c_char_p]
    L.cvk_nccl_unique_id.restype = i32
    L.cvk_rowblock_attach_nccl.argtypes = [P, C.c_char_p, i32]
    L.cvk_rowblock_solve_nccl.argtypes = [P]
    L.cvk_rowblock_p2p_handle.argtypes = [P, P]
    L.cvk_rowblock_p2p_attach.argtypes = [P, C.c_char_p, i32]
    L.cvk_rowblock_p2p_attach_local.argtypes = [C.POINTER(P), i32]
    L.cvk_rowblock_solve_p2p.argtypes = [C.POINTER(P), i32]
    for f in ("create", "exchange", "local", "post", "exchange_local", "solve_local", "done", "result", "destroy",
              "attach_nccl", "solve_nccl", "p2p_handle", "p2p_attach", "p2p_attach_local", "solve_p2p"):
        getattr(L, "cvk_rowblock_" + f).restype = i32
    L._rb_bound = True


# ------------------------------------------------------------------ plan --

@dataclass
class RowBlockPlan:
    """One rank's block of the global system."""
    rank: int
    n_ranks: int
    r0: int
    r1: int
    row_offsets: np.ndarray   # int64 [n_own + 1], from 0
    col_local: np.ndarray     # int64 [nnz]: own rows 0..n_own-1, halo n_own + h
    values: np.ndarray        # complex128 [nnz]
    halo_cols: np.ndarray     # int64 [n_halo]: global rows of the halo entries (sorted)
    send_rows: np.ndarray     # int64 [n_send]: local rows other ranks read (sorted)
    max_send: int
    halo_src: np.ndarray      # int64 [n_halo]: owner * max_send + position in the owner's send list

    @property
    def n_own(self) -> int:
        return self.r1 - self.r0


def row_bounds(A: CsrMatrix, n_ranks: int, balance: str = "nnz") -> np.ndarray:
    """Contiguous row blocks: equal rows, or (default) equal nonzeros."""
    n = A.nrows
    if n_ranks < 1:
        raise InvalidArgument("row blocks: need at least one rank")
    if balance == "rows":
        return np.array([(q * n) // n_ranks for q in range(n_ranks + 1)], np.int64)
    if balance != "nnz":
        raise InvalidArgument(f'row blocks: unknown balance "{balance}" (allowed: nnz, rows)')
    rp = np.asarray(A.row_offsets, np.int64)
    targets = (np.arange(n_ranks + 1, dtype=np.float64) * rp[-1]) / n_ranks
    b = np.searchsorted(rp, targets, side="left").astype(np.int64)
    b[0], b[-1] = 0, n
    return np.maximum.accumulate(np.minimum(b, n))


def plan_row_blocks(A: CsrMatrix, n_ranks: int, bounds: Optional[np.ndarray] = None) -> List[RowBlockPlan]:
    """Every rank's block, halo and exchange lists (all ranks compute the
    same plan from the global pattern)."""
    if A.nrows != A.ncols:
        raise InvalidArgument("row blocks: matrix must be square")
    bounds = row_bounds(A, n_ranks) if bounds is None else np.asarray(bounds, np.int64)
    if len(bounds) != n_ranks + 1 or bounds[0] != 0 or bounds[-1] != A.nrows or np.any(np.diff(bounds) < 0):
        raise InvalidArgument("row blocks: bounds must run 0 .. n, non-decreasing")
    rp = np.asarray(A.row_offsets, np.int64)
    ci = np.asarray(A.col_indices, np.int64)
    vals = np.asarray(A.values, np.complex128)
    halos, cols = [], []
    for q in range(n_ranks):
        r0, r1 = int(bounds[q]), int(bounds[q + 1])
        c = ci[rp[r0]:rp[r1]]
        ext = (c < r0) | (c >= r1)
        halo = np.unique(c[ext])
        loc = c - r0
        loc[ext] = (r1 - r0) + np.searchsorted(halo, c[ext])
        halos.append(halo)
        cols.append(loc)
    owner_of = lambda g: np.searchsorted(bounds, g, side="right") - 1  # noqa: E731
    needed = [[] for _ in range(n_ranks)]
    for q in range(n_ranks):
        own = owner_of(halos[q])
        for o in np.unique(own):
            needed[int(o)].append(halos[q][own == o])
    sends = [np.unique(np.concatenate(v)) - bounds[o] if v else np.zeros(0, np.int64)
             for o, v in enumerate(needed)]
    max_send = max([len(s) for s in sends] + [0])
    plans = []
    for q in range(n_ranks):
        r0, r1 = int(bounds[q]), int(bounds[q + 1])
        own = owner_of(halos[q])
        src = np.zeros(len(halos[q]), np.int64)
        for o in np.unique(own):
            m = own == o
            src[m] = int(o) * max_send + np.searchsorted(sends[int(o)], halos[q][m] - bounds[o])
        plans.append(RowBlockPlan(q, n_ranks, r0, r1, rp[r0:r1 + 1] - rp[r0], cols[q], vals[rp[r0]:rp[r1]],
                                  halos[q], sends[q].astype(np.int64), max_send, src))
    return plans


def plan_local_block(rank: int, bounds, row_offsets, cols_global, values,
                     gather: Callable[[object], list]) -> RowBlockPlan:
    """This rank's plan from its own rows only (the distributed setup: no rank
    holds the global matrix).  Each rank derives its halo from its rows'
    columns; one all-gather of the halo lists (gather(obj) -> every rank's
    obj, e.g. torch.distributed.all_gather_object) tells every rank which of
    its rows the others read, and every owner's send list.  Bitwise the plan
    plan_row_blocks computes from the global pattern."""
    bounds = np.asarray(bounds, np.int64)
    n_ranks = len(bounds) - 1
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    c = np.asarray(cols_global, np.int64)
    ext = (c < r0) | (c >= r1)
    halo = np.unique(c[ext])
    loc = c - r0
    loc[ext] = (r1 - r0) + np.searchsorted(halo, c[ext])
    halos = gather(halo)
    owner_of = lambda g: np.searchsorted(bounds, g, side="right") - 1  # noqa: E731
    needed = [[] for _ in range(n_ranks)]
    for q in range(n_ranks):
        own = owner_of(halos[q])
        for o in np.unique(own):
            needed[int(o)].append(halos[q][own == o])
    sends = [np.unique(np.concatenate(v)) - bounds[o] if v else np.zeros(0, np.int64)
             for o, v in enumerate(needed)]
    max_send = max([len(x) for x in sends] + [0])
    own = owner_of(halo)
    src = np.zeros(len(halo), np.int64)
    for o in np.unique(own):
        m = own == o
        src[m] = int(o) * max_send + np.searchsorted(sends[int(o)], halo[m] - bounds[o])
    return RowBlockPlan(rank, n_ranks, r0, r1, np.asarray(row_offsets, np.int64), loc,
                        np.asarray(values, np.complex128), halo, sends[rank].astype(np.int64), max_send, src)


def local_jacobi(r0: int, row_offsets, cols_global, values) -> np.ndarray:
    """Inverse diagonal of a rank's own rows (jacobi, krylov.cpp:31-55: the
    first stored entry with col == row, inverted on the device with the
    reference's __divdc3 rounding); zero or missing -> InvalidArgument naming
    the global row, as the reference does."""
    rp = np.asarray(row_offsets, np.int64)
    c = np.asarray(cols_global, np.int64)
    v = np.asarray(values, np.complex128)
    n = len(rp) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    hit = np.nonzero(c == rows + r0)[0]
    first = np.full(n, -1, np.int64)
    first[rows[hit][::-1]] = hit[::-1]  # first col == row entry of each row
    d = np.zeros(n, np.complex128)
    ok = first >= 0
    d[ok] = v[first[ok]]
    ar = np.arange(n, dtype=np.uint64)
    D = CsrMatrix(n, n, np.arange(n + 1, dtype=np.uint64), ar, d)
    from .cavac import jacobi
    try:
        return jacobi(D).inv_diag
    except InvalidArgument as e:
        row = int(str(e).rsplit(" ", 1)[-1])
        raise InvalidArgument(f"jacobi: zero diagonal at row {row + r0}") from None


# ------------------------------------------------ geometric partitioning --

def rcb_partition(coords, n_parts: int) -> np.ndarray:
    """Recursive coordinate bisection (the geometric stand-in for METIS-style
    subdomains of an FEM mesh): split the point set along its longest extent
    at the count that gives each side its share of the parts, recursively.
    Returns the part id of every point; part sizes differ by at most one."""
    xyz = np.asarray(coords, np.float64)
    if xyz.ndim != 2 or n_parts < 1:
        raise InvalidArgument("rcb_partition: coords must be (n, d) and n_parts >= 1")
    part = np.zeros(len(xyz), np.int64)

    def split(idx, p0, k):
        if k == 1 or len(idx) == 0:
            part[idx] = p0
            return
        kl = k // 2
        nl = (len(idx) * kl) // k
        ext = xyz[idx].max(axis=0) - xyz[idx].min(axis=0)
        ax = int(np.argmax(ext))
        order = idx[np.lexsort((idx, xyz[idx, ax]))]  # ties broken by index: deterministic
        split(order[:nl], p0, kl)
        split(order[nl:], p0 + kl, k - kl)

    split(np.arange(len(xyz), dtype=np.int64), 0, n_parts)
    return part


def permute_system(A: CsrMatrix, perm: np.ndarray) -> CsrMatrix:
    """P A P^T with new row k = old row perm[k]; columns renumbered and
    sorted per row (values carried)."""
    perm = np.asarray(perm, np.int64)
    n = A.nrows
    if A.nrows != A.ncols or len(perm) != n or not np.array_equal(np.sort(perm), np.arange(n)):
        raise InvalidArgument("permute_system: perm must be a permutation of the rows of a square matrix")
    inv = np.empty(n, np.int64)
    inv[perm] = np.arange(n)
    rp = np.asarray(A.row_offsets, np.int64)
    ci = np.asarray(A.col_indices, np.int64)
    v = np.asarray(A.values, np.complex128)
    lens = np.diff(rp)[perm]
    nrp = np.zeros(n + 1, np.int64)
    nrp[1:] = np.cumsum(lens)
    src = np.repeat(rp[perm], lens) + (np.arange(nrp[-1]) - np.repeat(nrp[:-1], lens))
    rows = np.repeat(np.arange(n), lens)
    cols = inv[ci[src]]
    order = np.lexsort((cols, rows))
    return CsrMatrix(n, n, nrp.astype(np.uint64), cols[order].astype(np.uint64), v[src][order])


def rcb_order(coords, n_parts: int):
    """Permutation that makes every RCB part a contiguous block of rows
    (parts in id order, original order inside a part) and the block bounds."""
    part = rcb_partition(coords, n_parts)
    perm = np.lexsort((np.arange(len(part)), part))
    counts = np.bincount(part, minlength=n_parts)
    bounds = np.zeros(n_parts + 1, np.int64)
    bounds[1:] = np.cumsum(counts)
    return perm, bounds


# --------------------------------------------------------------- engines --

class RowBlockEngine:
    """One block on one device (cvk_rowblock_*, csrc/cvk_rowblock.cu)."""

    def __init__(self, plan: RowBlockPlan, b_own: np.ndarray, inv_diag_own: Optional[np.ndarray],
                 opts: SolverOptions, dev: Optional[Device] = None):
        L = _lib.load()
        _bind(L)
        self.L, self.plan = L, plan
        self.dev = dev or Device.default()
        self._keep = [np.ascontiguousarray(a) for a in
                      (plan.row_offsets, plan.col_local, plan.values, plan.send_rows, plan.halo_src)]
        self._b = _cvec(b_own)
        self._d = None if inv_diag_own is None else _cvec(inv_diag_own)
        self.hist_cap = 2 * opts.max_iter + 8 if opts.record_history else 0
        p = lambda a: None if a is None else a.ctypes.data_as(P)  # noqa: E731
        rp, ci, av, sr, hs = self._keep
        d = CvkRowblockDesc(plan.n_own, len(plan.halo_cols), len(ci), p(rp), p(ci), p(av), p(self._d), p(self._b),
                            len(sr), p(sr), plan.n_ranks, plan.max_send, p(hs), self.hist_cap)
        o = _lib.CvkOpts(float(opts.tol), int(opts.max_iter), int(opts.l), int(opts.m),
                         1 if opts.record_history else 0, _lib.MODE_FAST)
        h = P()
        code = L.cvk_rowblock_create(self.dev.handle, C.byref(d), int(SolverId.BiCGStab), C.byref(o), C.byref(h))
        if code in (-1, -6):
            raise InvalidArgument(_lib.last_error())
        _lib.check(code)
        self.h = h
        s, r, n = P(), P(), C.c_int64()
        _lib.check(L.cvk_rowblock_exchange(h, C.byref(s), C.byref(r), C.byref(n)))
        self.send_ptr, self.recv_ptr, self.slot = s.value, r.value, n.value
        self.stream = L.cvk_ctx_stream(self.dev.handle)

    def solve_nccl(self, group=None) -> None:
        """The whole phase loop in the library over its own NCCL communicator
        (bootstrapped through the torch.distributed group): ncclAllGather on
        the library's stream, captured in CUDA graphs with the kernels."""
        import torch.distributed as dist
        if getattr(self, "_nccl_attached", False):
            _lib.check(self.L.cvk_rowblock_solve_nccl(self.h))
            return
        rank = dist.get_rank(group)
        box = [None]
        if rank == 0:
            buf = C.create_string_buffer(128)
            _lib.check(self.L.cvk_nccl_unique_id(buf))
            box = [buf.raw]
        dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
        _lib.check(self.L.cvk_rowblock_attach_nccl(self.h, box[0], self.plan.rank))
        self._nccl_attached = True
        _lib.check(self.L.cvk_rowblock_solve_nccl(self.h))

    def solve_p2p(self, group=None) -> None:
        """The phase loop with the library's own peer-to-peer exchange: every
        rank's mailbox is mapped into every other rank through CUDA IPC
        (handles all-gathered over the torch.distributed group once), the
        pack kernels store into the peers' mailboxes and the post kernels
        wait on local flags -- no collective library on the data path."""
        import torch.distributed as dist
        if not getattr(self, "_p2p_attached", False):
            h = C.create_string_buffer(64)
            _lib.check(self.L.cvk_rowblock_p2p_handle(self.h, h))
            allh = [None] * dist.get_world_size(group)
            dist.all_gather_object(allh, h.raw, group=group)
            _lib.check(self.L.cvk_rowblock_p2p_attach(self.h, b"".join(allh), self.plan.rank))
            self._p2p_attached = True
            dist.barrier(group=group)
        arr = (P * 1)(self.h)
        _lib.check(self.L.cvk_rowblock_solve_p2p(arr, 1))

    def local(self, ph: int) -> None:
        _lib.check(self.L.cvk_rowblock_local(self.h, ph))

    def post(self, ph: int) -> None:
        _lib.check(self.L.cvk_rowblock_post(self.h, ph))

    def done(self) -> bool:
        v = C.c_int()
        _lib.check(self.L.cvk_rowblock_done(self.h, C.byref(v)))
        return bool(v.value)

    def result(self):
        x = np.zeros(self.plan.n_own, np.complex128)
        rep = _lib.CvkReport()
        hist = None
        if self.hist_cap:
            hist = np.zeros(self.hist_cap, np.float64)
            rep.history = hist.ctypes.data_as(C.POINTER(C.c_double))
            rep.history_cap = len(hist)
        _lib.check(self.L.cvk_rowblock_result(self.h, x.ctypes.data_as(P), C.byref(rep)))
        return x, _report(rep, hist)

    # exchange buffers as torch tensors over the library's device memory
    def tensors(self):
        import torch

        class _Cai:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                                 "version": 3}
        dev = torch.device("cuda", self.dev.index)
        send = torch.as_tensor(_Cai(self.send_ptr, self.slot), device=dev)
        recv = torch.as_tensor(_Cai(self.recv_ptr, self.slot * self.plan.n_ranks), device=dev)
        return send, recv

    def close(self):
        if self.h:
            self.L.cvk_rowblock_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _report(r, hist) -> SolveReport:
    h = [] if hist is None else list(hist[: min(r.history_len, len(hist))])
    return SolveReport(bool(r.converged), int(r.iterations), r.final_relres, r.true_relres, r.wall_time_s, h,
                       _BRK.get(r.breakdown, "unknown breakdown"), r.device_time_s, int(r.kernel_launches))


def _check_system(A: CsrMatrix, b, M: Preconditioner):
    b = _cvec(b)
    if A.nrows != A.ncols or A.nrows != len(b):
        raise InvalidArgument("bicgstab: dimension mismatch")
    d = None
    if M is not None and M.kind != "identity":
        d = _cvec(M.inv_diag)
        if len(d) != A.nrows:
            raise InvalidArgument("preconditioner: dimension mismatch")
    return b, d


def _rcb_system(A, b, d, coords, n_blocks):
    perm, bounds = rcb_order(coords, n_blocks)
    return permute_system(A, perm), b[perm], None if d is None else d[perm], perm, bounds


def _unpermute(res: SolveResult, perm) -> SolveResult:
    x = np.empty_like(res.x)
    x[perm] = res.x
    return SolveResult(x, res.report)


def solve_row_blocks(A: CsrMatrix, b, M: Preconditioner, opts: Optional[SolverOptions] = None, n_blocks: int = 2,
                     bounds: Optional[np.ndarray] = None, dev: Optional[Device] = None,
                     coords=None, p2p: bool = False) -> SolveResult:
    """BiCGSTAB over n_blocks row blocks on one device: every block runs the
    multi-rank kernels, the all-gather is a device copy (same stream).  With
    `coords` (one point per row, e.g. FemCavity.coords()) the blocks are RCB
    parts: the system is permuted so each part is contiguous, and x is
    returned in the original numbering."""
    opts = opts or SolverOptions()
    b, d = _check_system(A, b, M)
    if coords is not None:
        Ap, bp, dp, perm, bnd = _rcb_system(A, b, d, coords, n_blocks)
        Mp = Preconditioner("identity") if dp is None else Preconditioner("jacobi", dp)
        return _unpermute(solve_row_blocks(Ap, bp, Mp, opts, n_blocks, bnd, dev, p2p=p2p), perm)
    plans = plan_row_blocks(A, n_blocks, bounds)
    engines = [RowBlockEngine(pl, b[pl.r0:pl.r1], None if d is None else d[pl.r0:pl.r1], opts, dev) for pl in plans]
    try:
        L = engines[0].L
        arr = (P * n_blocks)(*[e.h for e in engines])
        if p2p:  # the mailbox exchange of the multi-GPU p2p path, blocks wired in-process
            _lib.check(L.cvk_rowblock_p2p_attach_local(arr, n_blocks))
            _lib.check(L.cvk_rowblock_solve_p2p(arr, n_blocks))
        else:
            _lib.check(L.cvk_rowblock_solve_local(arr, n_blocks))
        xs, reps = zip(*[e.result() for e in engines])
    finally:
        for e in engines:
            e.close()
    rep = reps[0]
    rep.kernel_launches = sum(r.kernel_launches for r in reps)
    return SolveResult(np.concatenate(xs) if xs else np.zeros(0, np.complex128), rep)


# ---------------------------------------------------------- distributed --

class _Exchange:
    """The per-phase all-gather of the ranks' exchange slots."""

    def __init__(self, engine, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.engine = engine
        self.backend = dist.get_backend(group)
        if isinstance(engine, RowBlockEngine):
            self.send, self.recv = engine.tensors()
            self.stream = torch.cuda.ExternalStream(engine.stream, device=self.send.device)
        else:  # host engine: numpy buffers shared with CPU tensors
            self.send, self.recv = torch.from_numpy(engine.send), torch.from_numpy(engine.recv)
            self.stream = None

    def __call__(self) -> None:
        torch, dist = self.torch, self.dist
        if self.stream is not None and self.backend == "nccl":
            # NCCL orders itself after the library's stream and the stream after it
            with torch.cuda.stream(self.stream):
                dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
            return
        if self.stream is not None:  # gloo with device buffers: stage through host
            with torch.cuda.stream(self.stream):
                host = self.send.cpu()
            parts = [torch.empty_like(host) for _ in range(dist.get_world_size(self.group))]
            dist.all_gather(parts, host, group=self.group)
            with torch.cuda.stream(self.stream):
                self.recv.copy_(torch.cat(parts))
            return
        parts = [torch.empty_like(self.send) for _ in range(dist.get_world_size(self.group))]
        dist.all_gather(parts, self.send, group=self.group)
        self.recv.copy_(torch.cat(parts))


EngineFactory = Callable[[RowBlockPlan, np.ndarray, Optional[np.ndarray], SolverOptions], object]


def solve_distributed(A: CsrMatrix, b, M: Preconditioner, opts: Optional[SolverOptions] = None, group=None,
                      bounds: Optional[np.ndarray] = None, engine_factory: Optional[EngineFactory] = None,
                      gather_solution: bool = True, use_library_nccl: bool = True, coords=None,
                      exchange: str = "collective") -> SolveResult:
    """BiCGSTAB (krylov.cpp:57-138) with one row block per rank of a
    torch.distributed group (initialised by the caller).  With device engines
    on an NCCL group the library runs the whole loop over its own NCCL
    communicator (use_library_nccl; otherwise the phases are issued from here
    with torch's NCCL all-gather on the library's stream); gloo stages the
    exchange through host.  exchange="p2p" replaces the collective with the
    library's mailbox exchange over CUDA IPC peer mappings (device engines;
    one GPU per rank).  Every rank returns the same report; x is the full
    solution (gather_solution) or the rank's own rows.  `coords` makes the
    ranks' blocks RCB parts (as in solve_row_blocks; x is then always the full
    solution in the original numbering)."""
    import torch.distributed as dist
    opts = opts or SolverOptions()
    b, d = _check_system(A, b, M)
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if coords is not None:
        Ap, bp, dp, perm, bnd = _rcb_system(A, b, d, coords, world)
        Mp = Preconditioner("identity") if dp is None else Preconditioner("jacobi", dp)
        res = solve_distributed(Ap, bp, Mp, opts, group, bnd, engine_factory, True, use_library_nccl,
                                exchange=exchange)
        return _unpermute(res, perm)
    plan = plan_row_blocks(A, world, bounds)[rank]
    factory = engine_factory or (lambda pl, bo, do, o: RowBlockEngine(pl, bo, do, o))
    eng = factory(plan, b[plan.r0:plan.r1], None if d is None else d[plan.r0:plan.r1], opts)
    try:
        if isinstance(eng, RowBlockEngine) and exchange == "p2p":
            eng.solve_p2p(group)
        elif isinstance(eng, RowBlockEngine) and dist.get_backend(group) == "nccl" and use_library_nccl:
            eng.solve_nccl(group)
        else:
            xchg = _Exchange(eng, group)

            def phase(ph):
                eng.local(ph)
                xchg()
                eng.post(ph)

            phase(PH_INIT)
            while not eng.done():
                for _ in range(ITERS_PER_POLL):
                    for ph in ITER_PHASES:
                        phase(ph)
            phase(PH_X)
            phase(PH_T)
        x_own, rep = eng.result()
    finally:
        if hasattr(eng, "close"):
            eng.close()
    if not gather_solution:
        return SolveResult(x_own, rep)
    parts = [None] * world
    dist.all_gather_object(parts, x_own, group=group)
    return SolveResult(np.concatenate(parts), rep)
