"""Device Schwarz DDM against the oracle (restating schwarz.cpp:111-238) and
the reference's own schwarz tests (test_schwarz.cpp, acceptance.cpp:263-313)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

OMEGA = 2 * math.pi * 13.0


def bits(a):
    return np.ascontiguousarray(a, np.complex128).view(np.uint64)


@pytest.fixture(scope="module")
def ddm(cvk):
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200 import schwarz as S
    return H, S


def cavity_problem(H, h, roof=lambda i: complex(1.0 + 0.1 * i, 0.3)):
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65)
    data = np.array([roof(i) for i in range(g.roof_size())], np.complex128)
    return H.assemble(g, OMEGA, 340.0, data)


def oracle_grid(oracle, p):
    return oracle.build_grid(2.4, 1.2, p.grid.h, 0.4, 0.65, complex(p.grid.wall_admittance))


def test_partition_layouts(cvk, ddm):
    H, S = ddm
    g = H.build_grid(1.1, 0.5, 0.1, 0.3, 0.7)
    assert g.nx == 10
    even = S.partition(g, 2)
    assert even.strip_width(0) == 5 and even.strip_width(1) == 5 and even.cut_columns == [5]
    odd = S.partition(g, 3)
    assert odd.col_begin == [0, 4, 7, 10]
    with pytest.raises(cvk.InvalidArgument):
        S.partition(g, 4)
    with pytest.raises(cvk.InvalidArgument):
        S.partition(g, 0)


@pytest.mark.parametrize("ns", [2, 3, 4])
def test_ref_mode_ddm_bitwise_vs_oracle(cvk, oracle, ddm, ns):
    """REF mode: outer sweeps, interface history and x bitwise = restatement."""
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.1)
    k = p.omega / p.c
    part = S.partition(p.grid, ns)
    tp = S.TransmissionParams(complex(2.0, k), complex(2.0, k))
    inner = P.SolverOptions(tol=1e-10)
    r = S.schwarz_solve(p, part, tp, inner, 1e-8, 300, mode=P.ExecMode.Sequential)
    A = p.A
    xo, do = oracle.schwarz_solve(oracle_grid(oracle, p), 340.0, A.row_offsets.astype(np.int64),
                                  A.col_indices.astype(np.int64), A.values, p.b, ns, tp.s_left, tp.s_right,
                                  tol=1e-10, ddm_tol=1e-8, max_outer=300)
    assert r.report.converged == do["converged"]
    assert r.report.outer_iterations == do["outer_iterations"]
    assert r.report.interface_residual_history == do["interface_residual_history"]
    assert np.array_equal(bits(r.x), bits(xo))


@pytest.mark.parametrize("ns", [2, 3])
def test_fast_ddm_matches_monodomain(cvk, ddm, ns):
    """test_schwarz.cpp:101-114 on the device (FAST mode)."""
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.1)
    mono = P.bicgstab(p.A, p.b, P.jacobi(p.A), P.SolverOptions(tol=1e-10))
    assert mono.report.converged
    k = p.omega / p.c
    r = S.schwarz_solve(p, S.partition(p.grid, ns), S.TransmissionParams(complex(2.0, k), complex(2.0, k)),
                        P.SolverOptions(tol=1e-10), 1e-8, 300)
    assert r.report.converged
    assert np.linalg.norm(r.x - mono.x) / np.linalg.norm(mono.x) <= 1e-6


def test_two_sided_and_acceptance_h005(cvk, ddm):
    """test_schwarz.cpp:116-127 and acceptance.cpp:263-291 (h=0.05, 2 and 4 strips)."""
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.1)
    mono = P.bicgstab(p.A, p.b, P.jacobi(p.A), P.SolverOptions(tol=1e-10)).x
    k = p.omega / p.c
    r = S.schwarz_solve(p, S.partition(p.grid, 2), S.TransmissionParams(complex(1.5, k), complex(3.0, k)),
                        P.SolverOptions(tol=1e-10), 1e-8, 300)
    assert r.report.converged and np.linalg.norm(r.x - mono) / np.linalg.norm(mono) <= 1e-6
    pa = cavity_problem(H, 0.05, roof=lambda i: complex(1.0 + 0.05 * i, 0.2))
    monoa = P.bicgstab(pa.A, pa.b, P.jacobi(pa.A), P.SolverOptions(tol=1e-10)).x
    for ns in (2, 4):
        ra = S.schwarz_solve(pa, S.partition(pa.grid, ns), S.TransmissionParams(complex(2.0, k), complex(2.0, k)),
                             P.SolverOptions(tol=1e-10), 1e-8, 300)
        assert ra.report.converged
        assert np.linalg.norm(ra.x - monoa) / np.linalg.norm(monoa) <= 1e-6


def test_single_subdomain_is_plain_solve(cvk, ddm):
    """test_schwarz.cpp:76-87: n_sub = 1 is bitwise the plain Jacobi solve."""
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.1)
    for mode in (P.ExecMode.Sequential, P.ExecMode.Parallel, P.ExecMode.Fast):
        r = S.schwarz_solve(p, S.partition(p.grid, 1), S.TransmissionParams(1j, 1j), P.SolverOptions(), 1e-8, 50,
                            mode=mode)
        d = P.bicgstab(p.A, p.b, P.jacobi(p.A), P.SolverOptions(), mode=mode)
        assert r.report.converged and r.report.outer_iterations == 1
        assert np.array_equal(bits(r.x), bits(d.x))


def test_zero_data_and_divergence(cvk, ddm):
    """test_schwarz.cpp:89-99 and 144-156."""
    H, S = ddm
    P = cvk
    g = H.build_grid(2.4, 1.2, 0.1, 0.4, 0.65)
    z = H.assemble(g, OMEGA, 340.0, np.zeros(g.roof_size(), np.complex128))
    r = S.schwarz_solve(z, S.partition(g, 3), S.TransmissionParams(complex(2, 0.24), complex(2, 0.24)),
                        P.SolverOptions(), 1e-8, 50)
    assert r.report.converged and r.report.outer_iterations == 1 and np.linalg.norm(r.x) <= 1e-12
    p = cavity_problem(H, 0.1)
    d = S.schwarz_solve(p, S.partition(p.grid, 2), S.TransmissionParams(0.24j, 0.24j), P.SolverOptions(), 1e-8, 12)
    assert not d.report.converged and d.report.outer_iterations == 12
    assert len(d.report.interface_residual_history) == 12
    assert all(np.isfinite(d.report.interface_residual_history))


def test_scaling_invariance(cvk, ddm):
    """test_schwarz.cpp:129-142: outer count invariant under data scaling."""
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.1)
    q = cavity_problem(H, 0.1)
    q.b = q.b * complex(5.0, -2.0)
    tp = S.TransmissionParams(complex(2.0, 0.24), complex(2.0, 0.24))
    part = S.partition(p.grid, 2)
    a = S.schwarz_solve(p, part, tp, P.SolverOptions(tol=1e-10), 1e-8, 300)
    b = S.schwarz_solve(q, part, tp, P.SolverOptions(tol=1e-10), 1e-8, 300)
    assert a.report.converged and b.report.converged
    assert a.report.outer_iterations == b.report.outer_iterations


def test_tune_parameters(cvk, ddm):
    """test_schwarz.cpp:158-212 and acceptance.cpp:293-311 (tuned beats i k)."""
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.1)
    k = p.omega / p.c
    grid = S.default_candidate_grid(k)
    assert len(grid) == 36 and grid[0].s_left == complex(0, k)
    part = S.partition(p.grid, 2)
    t = S.tune_parameters(p, part, grid, P.SolverOptions(tol=1e-10), 120)
    conv = [e for e in t.table if e.converged]
    assert conv
    best = min((e.outer_iterations, e.total_inner_iterations) for e in conv)
    chosen = [e for e in t.table if e.params == t.best][0]
    assert (chosen.outer_iterations, chosen.total_inner_iterations) == best
    with pytest.raises(cvk.InvalidArgument):
        S.tune_parameters(p, part, [], P.SolverOptions(), 10)


@pytest.mark.parametrize("solver", ["bicgstab", "tfqmr", "gmres"])
def test_sequential_strip_solves_bitwise_batched(cvk, ddm, knobs, solver):
    """FAST DDM with the strips' inner solves run one after another on the
    single-system path (used when every strip has >= CVK_OPT_DDM_SEQ_MIN rows;
    forced here) = the batched persistent launch, bit for bit: the inner
    reductions are double-double on both paths."""
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.05)
    k = p.omega / p.c
    part = S.partition(p.grid, 3)
    tp = S.TransmissionParams(complex(2.0, k), complex(2.0, k))
    sid = P.solver_id(solver)
    out = {}
    for path, thr in (("batched", "1000000000"), ("sequential", "0")):
        knobs(ddm_seq_min=int(thr), phased_min_n=0 if path == "sequential" else 1000000000)
        out[path] = S.schwarz_solve(p, part, tp, P.SolverOptions(tol=1e-10, m=20), 1e-8, 40, inner_solver=sid)
    a, b = out["batched"], out["sequential"]
    assert a.report.outer_iterations == b.report.outer_iterations
    assert a.report.interface_residual_history == b.report.interface_residual_history
    assert a.report.total_inner_iterations == b.report.total_inner_iterations
    assert np.array_equal(bits(a.x), bits(b.x))


@pytest.mark.parametrize("ns", [2, 4, 8])
def test_krylov_interface_iteration(cvk, ddm, ns):
    """GMRES on the interface equation (ddm_krylov.py): the same subdomain
    problems and trace update as the reference's fixed-point sweep, far fewer
    sweeps, and the monodomain solution (acceptance.cpp:277-291 tolerance)."""
    from paper_2112_00087_b200.ddm_krylov import schwarz_solve_krylov
    H, S = ddm
    P = cvk
    p = cavity_problem(H, 0.05)
    k = p.omega / p.c
    part = S.partition(p.grid, ns)
    tp = S.TransmissionParams(complex(2.0, k), complex(2.0, k))
    inner = P.SolverOptions(tol=1e-12)
    fixed = S.schwarz_solve(p, part, tp, inner, 1e-8, 600)
    kr = schwarz_solve_krylov(p, part, tp, inner, tol=1e-9, max_sweeps=300)
    mono = P.bicgstab(p.A, p.b, P.jacobi(p.A), P.SolverOptions(tol=1e-12))
    assert fixed.report.converged and kr.report.converged
    assert kr.report.sweeps < fixed.report.outer_iterations / 2, (kr.report.sweeps, fixed.report.outer_iterations)
    err = np.linalg.norm(kr.x - mono.x) / np.linalg.norm(mono.x)
    assert err <= 1e-6, err
    assert kr.report.residual_history[-1] <= 1e-9


def test_warm_started_inner_solves(cvk, ddm, knobs):
    """Warm-started inner BiCGSTAB (beyond the reference): the same DDM
    solution as the reference's cold starts (monodomain tolerance) with fewer
    inner iterations, bitwise the same on the batched persistent and the
    sequential phase-kernel paths; and a warm start from x0 = 0 is bitwise a
    cold solve on both single-system paths."""
    H, S = ddm
    P = cvk
    from paper_2112_00087_b200 import _lib
    import ctypes as C
    p = cavity_problem(H, 0.05)
    k = p.omega / p.c
    part = S.partition(p.grid, 4)
    tp = S.TransmissionParams(complex(2.0, k), complex(2.0, k))
    inner = P.SolverOptions(tol=1e-10)
    cold = S.schwarz_solve(p, part, tp, inner, 1e-8, 300)
    warm = S.schwarz_solve(p, part, tp, inner, 1e-8, 300, warm_start=True)
    mono = P.bicgstab(p.A, p.b, P.jacobi(p.A), P.SolverOptions(tol=1e-12))
    assert cold.report.converged and warm.report.converged
    tot = lambda r: sum(s.iterations for s in r.report.per_subdomain_solves)  # noqa: E731
    assert tot(warm) < tot(cold), (tot(warm), tot(cold))
    assert np.linalg.norm(warm.x - mono.x) <= 1e-6 * np.linalg.norm(mono.x)
    knobs(ddm_seq_min=0, phased_min_n=0)
    seq = S.schwarz_solve(p, part, tp, inner, 1e-8, 300, warm_start=True)
    assert seq.report.outer_iterations == warm.report.outer_iterations
    assert np.array_equal(bits(seq.x), bits(warm.x))
    # warm from zero = cold, on the persistent and the phase-kernel path
    L = _lib.load()
    L.cvk_solve_device_warm.argtypes = [C.c_void_p] * 6 + [C.POINTER(_lib.CvkReport)]
    import torch
    A = p.A
    M = P.jacobi(A)
    dev = P.Device.default()
    for min_n in ("1000000000", "0"):
        knobs(phased_min_n=int(min_n))
        r = P.solve(P.SolverId.BiCGStab, A, p.b, M, P.SolverOptions(tol=1e-10))
        bd = torch.from_numpy(np.asarray(p.b, np.complex128).view(np.float64).copy()).cuda()
        xd = torch.zeros_like(bd)
        o = P.cavac._opts(P.SolverOptions(tol=1e-10), None)
        rep = _lib.CvkReport()
        _lib.check(L.cvk_solve_device_warm(dev.handle, A.device(dev), M.device(A, dev), C.byref(o),
                                           C.c_void_p(bd.data_ptr()), C.c_void_p(xd.data_ptr()), C.byref(rep)))
        assert rep.iterations == r.report.iterations
        assert np.array_equal(bits(xd.cpu().numpy().view(np.complex128)), bits(r.x))
        # from the converged solution: done at once
        rep2 = _lib.CvkReport()
        _lib.check(L.cvk_solve_device_warm(dev.handle, A.device(dev), M.device(A, dev), C.byref(o),
                                           C.c_void_p(bd.data_ptr()), C.c_void_p(xd.data_ptr()), C.byref(rep2)))
        assert rep2.converged and rep2.iterations <= 1
