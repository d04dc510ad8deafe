"""Multi-rank Schwarz host logic (ddm_dist.schwarz_solve_distributed) on CPU:
world_size 2 and 3 over gloo, each rank's strips solved by the oracle-backed
engine (tests/ddm_oracle_engine.py).  The distributed run must reproduce the
single-process oracle schwarz_solve (schwarz.cpp:111-238 restated) bit for
bit: solution, interface-jump history and outer iteration count."""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case():
    from oracle import oracle as O
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.schwarz import Partition
    g = H.build_grid(2.4, 1.2, 0.1, 0.4, 0.65, 0.01)
    d = np.array([1.0 + 0.05 * i + 0.2j for i in range(g.roof_size())])
    prob = H.assemble(g, 2 * np.pi * 13.0, 340.0, d)
    return O, g, prob, Partition


def _worker(rank, world, port, n_sub, solver, q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from ddm_oracle_engine import OracleRankEngine
        from paper_2112_00087_b200 import SolverId, SolverOptions
        from paper_2112_00087_b200.ddm_dist import schwarz_solve_distributed
        from paper_2112_00087_b200.schwarz import TransmissionParams
        O, g, prob, Partition = _case()
        cb = [int(v) for v in O.partition(g.nx, n_sub)]
        part = Partition(n_sub, cb, cb[1:-1])
        k = prob.omega / prob.c
        tp = TransmissionParams(complex(2.0, k), complex(2.0, k))
        r = schwarz_solve_distributed(prob, part, tp, SolverOptions(tol=1e-10), 1e-8, 300,
                                      SolverId(["bicgstab", "bicgstab_l", "tfqmr"].index(solver)),
                                      engine_factory=OracleRankEngine)
        q.put((rank, r.x, r.report.outer_iterations, list(r.report.interface_residual_history),
               r.report.converged, r.report.total_inner_iterations))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_sub,solver", [(2, 3, "bicgstab"), (3, 4, "tfqmr"), (2, 2, "bicgstab_l")])
def test_distributed_schwarz_matches_single_process(world, n_sub, solver):
    import multiprocessing as mp
    O, g, prob, _ = _case()
    O.build()
    A = prob.A
    k = prob.omega / prob.c
    x_ref, rep_ref, hist_ref = _oracle_single(O, g, prob, n_sub, solver, k)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_sub, solver, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, x, outer, hist, conv, inner_total in outs:
        assert outer == rep_ref["outer"], (rank, outer, rep_ref)
        assert conv == rep_ref["converged"]
        assert np.array_equal(np.asarray(hist).view(np.uint64), np.asarray(hist_ref).view(np.uint64))
        assert np.array_equal(x.view(np.uint64), x_ref.view(np.uint64)), rank
        assert inner_total == rep_ref["inner_total"]
    assert A.nrows == g.size()


def _oracle_single(O, g, prob, n_sub, solver, k):
    import ctypes as C
    og = O.build_grid(2.4, 1.2, 0.1, 0.4, 0.65, 0.01)
    A = prob.A
    rp, ci, v = A.row_offsets.astype(np.int64), A.col_indices.astype(np.int64), np.asarray(A.values)
    n = A.nrows
    cb = O.partition(g.nx, n_sub)
    x = np.zeros(n, np.complex128)
    rep = O._DdmReport()
    hist = np.zeros(400)
    rep.jump_history = hist.ctypes.data_as(C.POINTER(C.c_double))
    rep.jump_cap = len(hist)
    o = O._opts(1e-10, 10000, 8, 30, False)
    rc = O.lib().orc_schwarz_solve(C.byref(og._g), prob.c, n, O._p(rp), O._p(ci), O._p(v), O._p(prob.b), n_sub,
                                   O._p(cb), 2.0, k, 2.0, k, C.byref(o), 1e-8, 300, O.SOLVERS[solver],
                                   O._p(x), C.byref(rep), None)
    assert rc == 0
    return x, {"outer": rep.outer_iterations, "converged": bool(rep.converged),
               "inner_total": rep.last_inner_iterations_total}, hist[: rep.jump_len]


def test_strip_ranges():
    from paper_2112_00087_b200.ddm_dist import strip_ranges
    assert strip_ranges(8, 8) == [(i, i + 1) for i in range(8)]
    assert strip_ranges(5, 2) == [(0, 3), (3, 5)]
    assert strip_ranges(7, 3) == [(0, 3), (3, 5), (5, 7)]
    with pytest.raises(ValueError):
        strip_ranges(2, 3)


def _tune_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2112_00087_b200 import SolverOptions
        from paper_2112_00087_b200.ddm_dist import tune_parameters_distributed
        from paper_2112_00087_b200.schwarz import default_candidate_grid
        O, g, prob, Partition = _case()
        cb = [int(v) for v in O.partition(g.nx, 3)]
        part = Partition(3, cb, cb[1:-1])
        cands = default_candidate_grid(prob.omega / prob.c)[:12]
        r = tune_parameters_distributed(prob, part, cands, SolverOptions(tol=1e-10), 150,
                                        entry_fn=_oracle_entry)
        q.put((rank, r.best, [(e.outer_iterations, e.total_inner_iterations, e.converged) for e in r.table]))
    finally:
        dist.destroy_process_group()


def _oracle_entry(problem, part, tp, inner, budget, mode=None):
    """tune_entry with the oracle's schwarz_solve (test infrastructure)."""
    from oracle import oracle as O
    from paper_2112_00087_b200.schwarz import TuneEntry
    g = problem.grid
    og = O.build_grid(2.4, 1.2, g.h, 0.4, 0.65, g.wall_admittance)
    A = problem.A
    x, rep = O.schwarz_solve(og, problem.c, A.row_offsets, A.col_indices, A.values, problem.b, part.n_sub,
                             tp.s_left, tp.s_right, tol=inner.tol, ddm_tol=1e-6, max_outer=budget)
    return TuneEntry(tp, rep["outer_iterations"], sum(rep["sub_iterations"]), rep["converged"])


def test_distributed_tuning_matches_serial():
    """Candidates spread over 3 gloo ranks: the gathered table and the
    minimiser equal the serial tune loop (schwarz.cpp:240-280)."""
    import multiprocessing as mp
    from paper_2112_00087_b200 import SolverOptions
    from paper_2112_00087_b200.schwarz import default_candidate_grid, select_best
    O, g, prob, Partition = _case()
    O.build()
    cb = [int(v) for v in O.partition(g.nx, 3)]
    part = Partition(3, cb, cb[1:-1])
    cands = default_candidate_grid(prob.omega / prob.c)[:12]
    serial = select_best([_oracle_entry(prob, part, tp, SolverOptions(tol=1e-10), 150) for tp in cands])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tune_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [(e.outer_iterations, e.total_inner_iterations, e.converged) for e in serial.table]
    for rank, best, table in outs:
        assert table == want
        assert best == serial.best
