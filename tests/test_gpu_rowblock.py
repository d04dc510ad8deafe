"""Row-block global BiCGSTAB on the device (csrc/cvk_rowblock.cu, SURVEY.md
8(e) mode 1): n row blocks on one device, and two processes sharing the
device over gloo, must reproduce the single-device FAST solve bit for bit
(solution, iteration count, residual history) -- the reductions are
double-double and every per-row / per-element rounding is the same."""
import math
import os
import socket
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    return np.ascontiguousarray(a, np.complex128).view(np.uint64)


def cavity(h, f=60.0, adm=0.01 + 0j):
    from paper_2112_00087_b200 import helmholtz as H
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
    d = np.array([1.0 + 0.05 * i + 0.2j for i in range(g.roof_size())])
    p = H.assemble(g, 2 * np.pi * f, 340.0, d)
    return p.A, np.asarray(p.b, np.complex128)


def _same(a, b):
    assert a.report.converged == b.report.converged
    assert a.report.iterations == b.report.iterations
    assert a.report.breakdown == b.report.breakdown
    assert np.array_equal(bits(a.x), bits(b.x))
    assert a.report.residual_history == b.report.residual_history
    assert a.report.final_relres == b.report.final_relres


@pytest.mark.parametrize("h", [0.05, 0.0075, 0.004])
@pytest.mark.parametrize("n_blocks", [1, 2, 3, 5])
def test_row_blocks_bitwise_single_device(cvk, h, n_blocks):
    """50k- and 180k-DOF cavities (the latter on the streamed phase kernels
    single-device) and the golden-size system."""
    from paper_2112_00087_b200.rowblock import solve_row_blocks
    P = cvk
    A, b = cavity(h)
    M = P.jacobi(A)
    o = P.SolverOptions(tol=1e-9, record_history=True, max_iter=20000)
    ref = P.solve(P.SolverId.BiCGStab, A, b, M, o)
    got = solve_row_blocks(A, b, M, o, n_blocks=n_blocks)
    assert ref.report.converged
    _same(got, ref)
    assert got.report.true_relres == pytest.approx(ref.report.true_relres, rel=1e-12)
    assert got.report.kernel_launches > 0 and got.report.device_time > 0


def test_row_blocks_edge_cases(cvk):
    from paper_2112_00087_b200.rowblock import solve_row_blocks
    P = cvk
    A, b = cavity(0.05)
    M = P.jacobi(A)
    # identity preconditioner, rows-balanced bounds with an empty block
    I = P.identity_preconditioner()
    o = P.SolverOptions(tol=1e-8, record_history=True)
    ref = P.solve(P.SolverId.BiCGStab, A, b, I, o)
    bounds = np.array([0, 0, 400, A.nrows], np.int64)
    _same(solve_row_blocks(A, b, I, o, n_blocks=3, bounds=bounds), ref)
    # zero rhs: converged in 0 iterations, true relres left at 0
    z = solve_row_blocks(A, np.zeros_like(b), M, P.SolverOptions(), n_blocks=2)
    assert z.report.converged and z.report.iterations == 0 and z.report.true_relres == 0.0
    assert not np.any(z.x)
    # max_iter exhausted: not converged, iterations = max_iter
    e = solve_row_blocks(A, b, M, P.SolverOptions(max_iter=3), n_blocks=2)
    r = P.solve(P.SolverId.BiCGStab, A, b, M, P.SolverOptions(max_iter=3))
    assert not e.report.converged and e.report.iterations == 3
    assert np.array_equal(bits(e.x), bits(r.x))
    with pytest.raises(P.InvalidArgument):
        solve_row_blocks(A, b[:-1], M, n_blocks=2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q, h):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2112_00087_b200 as P
        from paper_2112_00087_b200.rowblock import solve_distributed
        A, b = cavity(h)
        M = P.jacobi(A)
        r = solve_distributed(A, b, M, P.SolverOptions(tol=1e-9, record_history=True, max_iter=20000))
        q.put((rank, r.x, r.report.iterations, list(r.report.residual_history), r.report.converged))
    finally:
        dist.destroy_process_group()


def test_distributed_two_processes_one_device(cvk):
    """The multi-process path (RowBlockEngine + torch.distributed exchange,
    gloo staged through host) with both ranks on device 0."""
    import multiprocessing as mp
    P = cvk
    h = 0.0075
    A, b = cavity(h)
    ref = P.solve(P.SolverId.BiCGStab, A, b, P.jacobi(A), P.SolverOptions(tol=1e-9, record_history=True,
                                                                           max_iter=20000))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, h)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=900) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, x, it, hist, conv in outs:
        assert conv and it == ref.report.iterations
        assert hist == ref.report.residual_history
        assert np.array_equal(bits(x), bits(ref.x)), rank
    assert math.isfinite(ref.report.true_relres)


def _nccl_worker(port, q, h, lib_nccl):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_2112_00087_b200 as P
        from paper_2112_00087_b200.rowblock import solve_distributed
        A, b = cavity(h)
        r = solve_distributed(A, b, P.jacobi(A), P.SolverOptions(tol=1e-9, record_history=True, max_iter=20000),
                              use_library_nccl=lib_nccl)
        q.put((r.x, r.report.iterations, list(r.report.residual_history)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("lib_nccl", [True, False])
def test_distributed_nccl_plumbing_one_rank(cvk, lib_nccl):
    """NCCL on one rank, so the plumbing runs on the one GPU this suite has:
    the library's own communicator with the graph-captured phase loop
    (cvk_rowblock_solve_nccl), or torch's all-gather on the library's stream
    over tensors wrapping the exchange buffers."""
    import multiprocessing as mp
    P = cvk
    h = 0.004
    A, b = cavity(h)
    ref = P.solve(P.SolverId.BiCGStab, A, b, P.jacobi(A), P.SolverOptions(tol=1e-9, record_history=True,
                                                                           max_iter=20000))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_nccl_worker, args=(_free_port(), q, h, lib_nccl))
    p.start()
    x, it, hist = q.get(timeout=900)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert it == ref.report.iterations and hist == ref.report.residual_history
    assert np.array_equal(bits(x), bits(ref.x))


def test_rcb_blocks_on_renumbered_fem_mesh(cvk):
    """FEM-3D box with a random node numbering, 4 RCB blocks (the system is
    permuted so each part is contiguous, x returned in the original
    numbering): same solution as the single-device solve on the original
    system (the permutation changes the per-row summation order, so not bit
    for bit)."""
    from paper_2112_00087_b200 import fem3d as F
    from paper_2112_00087_b200.rowblock import permute_system, solve_row_blocks
    P = cvk
    cav = F.build_cavity(10)
    A0 = P.CsrMatrix(cav.n, cav.n, cav.rp.astype(np.uint64), cav.ci.astype(np.uint64), cav.values(2 * np.pi * 60.0))
    shuffle = np.random.default_rng(3).permutation(cav.n)
    A = permute_system(A0, shuffle)
    b = np.asarray(cav.b, np.complex128)[shuffle]
    xyz = cav.coords()[shuffle]
    o = P.SolverOptions(tol=1e-11, max_iter=20000)
    ref = P.solve(P.SolverId.BiCGStab, A0, cav.b, P.jacobi(A0), o)
    got = solve_row_blocks(A, b, P.jacobi(A), o, n_blocks=4, coords=xyz)
    assert ref.report.converged and got.report.converged
    assert abs(got.report.iterations - ref.report.iterations) <= max(3, 0.15 * ref.report.iterations)
    x = got.x[np.argsort(shuffle)]
    assert np.linalg.norm(x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)


@pytest.mark.parametrize("n_blocks", [1, 2, 3, 5])
def test_p2p_mailbox_exchange_bitwise(cvk, n_blocks):
    """The peer-to-peer mailbox exchange (pack kernels store every rank's slot
    into all mailboxes and raise flags, post kernels wait on them) with the
    blocks wired in-process on one device: bitwise the single-device solve."""
    from paper_2112_00087_b200.rowblock import solve_row_blocks
    P = cvk
    for h in (0.05, 0.004):
        A, b = cavity(h)
        M = P.jacobi(A)
        o = P.SolverOptions(tol=1e-9, record_history=True, max_iter=20000)
        ref = P.solve(P.SolverId.BiCGStab, A, b, M, o)
        _same(solve_row_blocks(A, b, M, o, n_blocks=n_blocks, p2p=True), ref)


def _p2p_worker(port, q, h):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        import paper_2112_00087_b200 as P
        from paper_2112_00087_b200.rowblock import solve_distributed
        A, b = cavity(h)
        o = P.SolverOptions(tol=1e-9, record_history=True, max_iter=20000)
        r = solve_distributed(A, b, P.jacobi(A), o, exchange="p2p")
        q.put((r.x, r.report.iterations, list(r.report.residual_history)))
    finally:
        dist.destroy_process_group()


def test_distributed_p2p_plumbing_one_rank(cvk):
    """solve_distributed(exchange="p2p"): IPC handle export, the all-gather of
    handles over the group and attach, then the graph-captured mailbox loop;
    one rank here (one GPU)."""
    import multiprocessing as mp
    P = cvk
    h = 0.0075
    A, b = cavity(h)
    ref = P.solve(P.SolverId.BiCGStab, A, b, P.jacobi(A), P.SolverOptions(tol=1e-9, record_history=True,
                                                                           max_iter=20000))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_p2p_worker, args=(_free_port(), q, h))
    p.start()
    x, it, hist = q.get(timeout=900)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert it == ref.report.iterations and hist == ref.report.residual_history
    assert np.array_equal(bits(x), bits(ref.x))


def test_p2p_edge_cases(cvk):
    """p2p exchange with an empty block, the identity preconditioner, zero
    rhs and an exhausted iteration budget; and RCB blocks with p2p."""
    from paper_2112_00087_b200.rowblock import solve_row_blocks
    P = cvk
    A, b = cavity(0.05)
    M = P.jacobi(A)
    I = P.identity_preconditioner()
    o = P.SolverOptions(tol=1e-8, record_history=True)
    _same(solve_row_blocks(A, b, I, o, n_blocks=3, bounds=np.array([0, 0, 500, A.nrows]), p2p=True),
          P.solve(P.SolverId.BiCGStab, A, b, I, o))
    z = solve_row_blocks(A, np.zeros_like(b), M, P.SolverOptions(), n_blocks=2, p2p=True)
    assert z.report.converged and z.report.iterations == 0 and not np.any(z.x)
    e = solve_row_blocks(A, b, M, P.SolverOptions(max_iter=3), n_blocks=4, p2p=True)
    r = P.solve(P.SolverId.BiCGStab, A, b, M, P.SolverOptions(max_iter=3))
    assert not e.report.converged and e.report.iterations == 3
    assert np.array_equal(bits(e.x), bits(r.x))
    g = np.stack(np.meshgrid(np.arange(47.0), np.arange(23.0), indexing="xy"), -1).reshape(-1, 2)
    q = solve_row_blocks(A, b, M, P.SolverOptions(tol=1e-11), n_blocks=4, coords=g, p2p=True)
    ref = P.solve(P.SolverId.BiCGStab, A, b, M, P.SolverOptions(tol=1e-11))
    assert q.report.converged
    assert np.linalg.norm(q.x - ref.x) <= 1e-8 * np.linalg.norm(ref.x)
