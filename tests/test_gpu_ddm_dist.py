"""Multi-rank Schwarz on the device (ddm_dist with DeviceRankEngine /
cvk_ddm_rank_*): 2 and 3 ranks sharing cuda:0 over gloo (one GPU on the
test box).  Must equal the single-device cvk_schwarz_solve bit for bit (FAST
reductions are order independent, so the batched inner solves do not care
how strips are grouped), and in REF mode the reference's schwarz_solve."""
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from paper_2112_00087_b200 import helmholtz as H
    g = H.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, 0.01)
    d = np.array([1.0 + 0.05 * i + 0.2j for i in range(g.roof_size())])
    return H.assemble(g, 2 * np.pi * 13.0, 340.0, d)


def _worker(rank, world, port, n_sub, mode, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2112_00087_b200 as P
        from paper_2112_00087_b200.ddm_dist import schwarz_solve_distributed
        from paper_2112_00087_b200.schwarz import TransmissionParams, partition
        prob = _problem()
        part = partition(prob.grid, n_sub)
        k = prob.omega / prob.c
        r = schwarz_solve_distributed(prob, part, TransmissionParams(complex(2.0, k), complex(2.0, k)),
                                      P.SolverOptions(tol=1e-10), 1e-8, 300, P.SolverId.BiCGStab,
                                      mode=P.ExecMode(mode))
        q.put((rank, r.x, r.report.outer_iterations, list(r.report.interface_residual_history)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_sub,mode", [(2, 4, 1), (3, 4, 1), (2, 3, 0)])
def test_device_ranks_match_single_device(cvk, oracle, world, n_sub, mode):
    import multiprocessing as mp

    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200.schwarz import TransmissionParams, partition, schwarz_solve
    prob = _problem()
    part = partition(prob.grid, n_sub)
    k = prob.omega / prob.c
    tp = TransmissionParams(complex(2.0, k), complex(2.0, k))
    ref = schwarz_solve(prob, part, tp, P.SolverOptions(tol=1e-10), 1e-8, 300, mode=P.ExecMode(mode))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_sub, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, x, outer, hist in outs:
        assert outer == ref.report.outer_iterations, (rank, outer)
        assert np.array_equal(np.asarray(hist), np.asarray(ref.report.interface_residual_history))
        assert np.array_equal(x.view(np.uint64), ref.x.view(np.uint64)), rank
    if mode == 0:  # Sequential: the reference's own iterates
        A = prob.A
        x_o, rep_o = oracle.schwarz_solve(oracle.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, 0.01), 340.0,
                                          A.row_offsets, A.col_indices, A.values, prob.b, n_sub,
                                          complex(2.0, k), complex(2.0, k), tol=1e-10, ddm_tol=1e-8,
                                          max_outer=300)
        assert np.array_equal(outs[0][1].view(np.uint64), x_o.view(np.uint64))


def _tune_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2112_00087_b200 as P
        from paper_2112_00087_b200.ddm_dist import tune_parameters_distributed
        from paper_2112_00087_b200.schwarz import default_candidate_grid, partition
        prob = _problem()
        part = partition(prob.grid, 2)
        k = prob.omega / prob.c
        cands = default_candidate_grid(k)
        t = tune_parameters_distributed(prob, part, cands, P.SolverOptions(tol=1e-10), 300,
                                        mode=P.ExecMode.Fast)
        q.put((rank, t.best, [(e.outer_iterations, e.total_inner_iterations, e.converged) for e in t.table]))
    finally:
        dist.destroy_process_group()


def test_distributed_tuner_on_device(cvk):
    """tune_parameters (schwarz.cpp:240-301) with the 36 candidates split over
    2 ranks sharing cuda:0, every candidate a device schwarz_solve: the same
    table and minimiser as the single-process device tuner."""
    import torch.multiprocessing as mp
    from paper_2112_00087_b200.schwarz import default_candidate_grid, partition, tune_parameters
    P = cvk
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tune_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    got = [q.get(timeout=900) for _ in procs]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    prob = _problem()
    part = partition(prob.grid, 2)
    k = prob.omega / prob.c
    t = tune_parameters(prob, part, default_candidate_grid(k), P.SolverOptions(tol=1e-10), 300,
                        mode=P.ExecMode.Fast)
    want = [(e.outer_iterations, e.total_inner_iterations, e.converged) for e in t.table]
    for rank, best, table in got:
        assert best == t.best
        assert table == want
