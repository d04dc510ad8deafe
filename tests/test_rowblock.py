"""Row-block global BiCGSTAB host logic (rowblock.py, SURVEY.md 8(e) mode 1)
on CPU: the block plan / halo / exchange lists, and solve_distributed on 2
and 3 gloo ranks with the numpy engine (tests/rowblock_numpy_engine.py),
which must reproduce the one-block run bit for bit -- solution, iteration
count and residual history -- and the oracle's solution."""
import math
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


def _system(h=0.1, f=60.0, adm=0.01 + 0j):
    from paper_2112_00087_b200 import helmholtz as H
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
    d = np.array([1.0 + 0.05 * i + 0.2j for i in range(g.roof_size())])
    p = H.assemble(g, 2 * np.pi * f, 340.0, d)
    return p.A, np.asarray(p.b, np.complex128)


def _inv_diag(A):
    from paper_2112_00087_b200.helmholtz import cdiv
    rp, ci, v = A.row_offsets, A.col_indices, A.values
    out = np.zeros(A.nrows, np.complex128)
    for i in range(A.nrows):
        k = rp[i] + int(np.nonzero(ci[rp[i]:rp[i + 1]] == i)[0][0])
        out[i] = cdiv(1 + 0j, complex(v[k]))
    return out


def _random_csr(n, seed, per_row=6):
    from paper_2112_00087_b200.cavac import CsrMatrix
    rng = np.random.default_rng(seed)
    rp, ci = [0], []
    for i in range(n):
        cols = np.unique(np.concatenate([[i], rng.integers(0, n, per_row)]))
        ci.extend(cols)
        rp.append(len(ci))
    v = rng.standard_normal(len(ci)) + 1j * rng.standard_normal(len(ci))
    return CsrMatrix(n, n, np.array(rp, np.uint64), np.array(ci, np.uint64), v)


@pytest.mark.parametrize("n_ranks,balance", [(1, "nnz"), (2, "nnz"), (3, "rows"), (5, "nnz")])
def test_plan_halo_reproduces_global_spmv(n_ranks, balance):
    """Each block's local SpMV over [own | halo] equals the global SpMV rows:
    the halo of every block is filled from the owners' send lists exactly as
    the exchange slot layout maps it (halo_src = owner * max_send + k)."""
    from paper_2112_00087_b200.rowblock import plan_row_blocks, row_bounds
    A = _random_csr(97, 5)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(A.nrows) + 1j * rng.standard_normal(A.nrows)
    rp, ci, v = (np.asarray(a) for a in (A.row_offsets, A.col_indices, A.values))
    ref = np.array([np.sum(v[rp[i]:rp[i + 1]] * x[ci[rp[i]:rp[i + 1]].astype(np.int64)]) for i in range(A.nrows)])
    bounds = row_bounds(A, n_ranks, balance)
    plans = plan_row_blocks(A, n_ranks, bounds)
    ms = plans[0].max_send
    slots = np.zeros((n_ranks, max(1, ms)), np.complex128)
    for pl in plans:
        assert pl.max_send == ms and len(pl.send_rows) <= ms
        assert np.all(np.diff(pl.send_rows) > 0)
        slots[pl.rank, :len(pl.send_rows)] = x[pl.r0 + pl.send_rows]
    y = np.zeros(A.nrows, np.complex128)
    for pl in plans:
        q, k = np.divmod(pl.halo_src, max(1, ms))
        xl = np.concatenate([x[pl.r0:pl.r1], slots[q, k]])
        assert np.array_equal(xl[pl.n_own:], x[pl.halo_cols])
        for i in range(pl.n_own):
            a, b = pl.row_offsets[i], pl.row_offsets[i + 1]
            y[pl.r0 + i] = np.sum(pl.values[a:b] * xl[pl.col_local[a:b]])
    assert np.array_equal(y, ref)
    assert sum(pl.n_own for pl in plans) == A.nrows
    if balance == "nnz" and n_ranks > 1:
        nnz = [pl.row_offsets[-1] for pl in plans]
        assert max(nnz) - min(nnz) <= 2 * 7


def test_plan_rejects_bad_bounds():
    from paper_2112_00087_b200.cavac import InvalidArgument
    from paper_2112_00087_b200.rowblock import plan_row_blocks, row_bounds
    A = _random_csr(20, 2)
    with pytest.raises(InvalidArgument):
        plan_row_blocks(A, 2, np.array([0, 15, 10]))
    with pytest.raises(InvalidArgument):
        row_bounds(A, 0)
    with pytest.raises(InvalidArgument):
        row_bounds(A, 2, "cols")


def _worker(rank, world, port, q, kw):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from rowblock_numpy_engine import NumpyRowBlockEngine
        from paper_2112_00087_b200.cavac import Preconditioner, SolverOptions
        from paper_2112_00087_b200.rowblock import solve_distributed
        A, b = _system(**kw)
        M = Preconditioner("jacobi", _inv_diag(A))
        r = solve_distributed(A, b, M, SolverOptions(tol=1e-10, record_history=True),
                              engine_factory=NumpyRowBlockEngine)
        q.put((rank, r.x, r.report.iterations, list(r.report.residual_history), r.report.converged,
               r.report.true_relres))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_rowblock_matches_one_block(world, oracle):
    import multiprocessing as mp
    from rowblock_numpy_engine import run_serial
    from paper_2112_00087_b200.cavac import SolverOptions
    kw = dict(h=0.1, f=60.0)
    A, b = _system(**kw)
    x1, rep1 = run_serial(A, b, _inv_diag(A), SolverOptions(tol=1e-10, record_history=True))
    assert rep1.converged
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, kw)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, x, it, hist, conv, trr in outs:
        assert conv and it == rep1.iterations, (rank, it, rep1.iterations)
        assert np.array_equal(np.asarray(hist).view(np.uint64), np.asarray(rep1.residual_history).view(np.uint64))
        assert np.array_equal(x.view(np.uint64), x1.view(np.uint64)), rank
        assert trr == rep1.true_relres
    # the reference algorithm (sequential sums) on the same system: same solution
    rp, ci, v = A.row_offsets.astype(np.int64), A.col_indices.astype(np.int64), np.asarray(A.values)
    xo, ro = oracle.solve("bicgstab", rp, ci, v, b, tol=1e-10)
    assert abs(ro.iterations - rep1.iterations) <= max(2, 0.15 * ro.iterations)
    assert np.linalg.norm(x1 - xo) <= 1e-7 * np.linalg.norm(xo)
    assert math.isfinite(rep1.true_relres) and rep1.true_relres < 1e-8


def test_rcb_partition_balanced_and_compact():
    """RCB parts of the FEM box: sizes within one, and on a randomly
    renumbered mesh the parts' halos are as small as the natural slabs'
    (contiguous blocks of the shuffled numbering have halos near the whole
    mesh)."""
    from paper_2112_00087_b200 import fem3d as F
    from paper_2112_00087_b200.cavac import CsrMatrix
    from paper_2112_00087_b200.rowblock import permute_system, plan_row_blocks, rcb_order, rcb_partition
    cav = F.build_cavity(6)
    xyz = cav.coords()
    A = CsrMatrix(cav.n, cav.n, cav.rp.astype(np.uint64), cav.ci.astype(np.uint64), cav.values(300.0))
    for k in (1, 2, 3, 5, 8):
        part = rcb_partition(xyz, k)
        sizes = np.bincount(part, minlength=k)
        assert sizes.max() - sizes.min() <= 1 and sizes.sum() == cav.n
    rng = np.random.default_rng(0)
    shuffle = rng.permutation(cav.n)
    As = permute_system(A, shuffle)
    xs = xyz[shuffle]
    halo = lambda plans: sum(len(p.halo_cols) for p in plans)  # noqa: E731
    natural = halo(plan_row_blocks(A, 4, np.array([(q * cav.n) // 4 for q in range(5)])))
    naive = halo(plan_row_blocks(As, 4, np.array([(q * cav.n) // 4 for q in range(5)])))
    perm, bounds = rcb_order(xs, 4)
    rcb = halo(plan_row_blocks(permute_system(As, perm), 4, bounds))
    assert naive > 2.5 * natural
    assert rcb <= 1.5 * natural


def test_permute_system_is_similarity():
    from paper_2112_00087_b200.rowblock import permute_system
    A = _random_csr(60, 3)
    perm = np.random.default_rng(4).permutation(60)
    Ap = permute_system(A, perm)
    D = np.zeros((60, 60), np.complex128)
    rp, ci, v = (np.asarray(a) for a in (A.row_offsets, A.col_indices, A.values))
    for i in range(60):
        D[i, ci[rp[i]:rp[i + 1]].astype(np.int64)] = v[rp[i]:rp[i + 1]]
    Dp = np.zeros_like(D)
    rp2, ci2, v2 = (np.asarray(a) for a in (Ap.row_offsets, Ap.col_indices, Ap.values))
    for i in range(60):
        c = ci2[rp2[i]:rp2[i + 1]].astype(np.int64)
        assert np.all(np.diff(c) > 0)
        Dp[i, c] = v2[rp2[i]:rp2[i + 1]]
    assert np.array_equal(Dp, D[np.ix_(perm, perm)])


def _local_plan_worker(rank, world, port, h, out_dir):
    """One rank of the bench's rank-local setup (bench.py run_rowblock): its
    own rows of the cavity, its plan from one gloo all-gather of halo lists."""
    import pickle

    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.rowblock import plan_local_block
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
    n = g.size()
    bounds = np.array([(q * n) // world for q in range(world + 1)], np.int64)
    d = np.ones(g.roof_size(), np.complex128)
    rp, cols, vals, b = H.assemble_rows(g, 2 * np.pi * 100.0, 340.0, d, int(bounds[rank]), int(bounds[rank + 1]))

    def gather(obj):
        res = [None] * world
        dist.all_gather_object(res, obj)
        return res

    plan = plan_local_block(rank, bounds, rp, cols, vals, gather)
    with open(os.path.join(out_dir, f"plan{rank}.pkl"), "wb") as f:
        pickle.dump((plan, b), f)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_local_setup_matches_global_plan(tmp_path, world):
    """bench.py's N > 1 setup on gloo ranks: every rank assembles only its own
    rows and plans its halo from an all-gather of halo lists; the plans and
    right-hand sides equal the global assemble + plan_row_blocks bit for bit."""
    import pickle

    import torch.multiprocessing as mp
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.rowblock import plan_row_blocks
    h = 0.05
    mp.spawn(_local_plan_worker, args=(world, _free_port(), h, str(tmp_path)), nprocs=world, join=True)
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
    p = H.assemble(g, 2 * np.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
    n = g.size()
    bounds = np.array([(q * n) // world for q in range(world + 1)], np.int64)
    ref = plan_row_blocks(p.A, world, bounds)
    for q in range(world):
        plan, b = pickle.load(open(tmp_path / f"plan{q}.pkl", "rb"))
        r = ref[q]
        assert (plan.r0, plan.r1, plan.max_send) == (r.r0, r.r1, r.max_send)
        for f in ("row_offsets", "col_local", "halo_cols", "send_rows", "halo_src"):
            assert np.array_equal(getattr(plan, f), getattr(r, f)), f
        assert np.array_equal(plan.values.view(np.uint64), r.values.view(np.uint64))
        assert np.array_equal(b.view(np.uint64), np.asarray(p.b[r.r0:r.r1]).view(np.uint64))
