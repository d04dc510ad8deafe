"""ILU(0) preconditioner on the device (beyond the reference, which has only
jacobi / identity_preconditioner, krylov.cpp:27-55).

Parity for ILU(0) itself is UNPINNED against the reference (it has none):
the factor and the sweep apply are checked BITWISE against the C
restatement (oracle/cavac_oracle.c orc_ilu0_arrays / orc_ilu0_apply_arrays),
the solves by solution-only checks against the reference algorithm's
Jacobi solve at tol 1e-12 (oracle orc_bicgstab).
"""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.complex128).view(np.uint64)


def cavity(O, h, f=100.0, adm=0.01 + 0j):
    g = O.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
    return O.assemble(g, 2 * math.pi * f, 343.0, np.full(g.roof_size, 1.0 + 0j))


def rand_csr(O, n, nnz, rng):
    rows = np.concatenate([rng.integers(0, n, nnz), np.arange(n)])
    cols = np.concatenate([rng.integers(0, n, nnz), np.arange(n)])
    vals = np.concatenate([rng.uniform(-1, 1, nnz) + 1j * rng.uniform(-1, 1, nnz),
                           8.0 + rng.uniform(-1, 1, n) + 1j])
    return O.csr_from_triplets(rows, cols, vals, n, n)


def systems(O):
    rng = np.random.default_rng(7)
    out = [cavity(O, 0.03)[:3], cavity(O, 0.012, f=250.0)[:3]]
    for n in (1, 7, 300, 2049):
        out.append(rand_csr(O, n, 6 * n, rng))
    return out


def test_factor_bitwise(cvk, oracle):
    P = cvk
    for rp, ci, v in systems(oracle):
        n = len(rp) - 1
        A = P.CsrMatrix(n, n, rp, ci, v)
        M = P.ilu0(A)
        assert np.array_equal(bits(P.ilu0_factor(M)), bits(oracle.ilu0(rp, ci, v)))


@pytest.mark.parametrize("sweeps", [0, 1, 2, 3, 6])
def test_apply_bitwise(cvk, oracle, sweeps):
    P = cvk
    rng = np.random.default_rng(sweeps)
    for rp, ci, v in systems(oracle):
        n = len(rp) - 1
        A = P.CsrMatrix(n, n, rp, ci, v)
        M = P.ilu0(A, sweeps)
        f = oracle.ilu0(rp, ci, v)
        r = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
        assert np.array_equal(bits(M.apply(r)), bits(oracle.ilu0_apply(rp, ci, f, sweeps, r)))


def test_apply_converges_to_exact_triangular_solves(cvk, oracle):
    P = cvk
    rp, ci, v = cavity(oracle, 0.05)[:3]
    n = len(rp) - 1
    A = P.CsrMatrix(n, n, rp, ci, v)
    f = oracle.ilu0(rp, ci, v)
    # exact forward / backward substitution (dense, small n)
    F = np.zeros((n, n), complex)
    for i in range(n):
        F[i, ci[rp[i]:rp[i + 1]]] = f[rp[i]:rp[i + 1]]
    L = np.tril(F, -1) + np.eye(n)
    U = np.triu(F)
    r = np.random.default_rng(3).standard_normal(n) + 0j
    want = np.linalg.solve(U, np.linalg.solve(L, r))
    # Jacobi sweeps on a triangular system are exact after n sweeps; 64 is plenty here
    got = P.ilu0(A, 64).apply(r)
    assert np.linalg.norm(got - want) <= 1e-10 * np.linalg.norm(want)


@pytest.mark.parametrize("h,f", [(0.012, 100.0), (0.008, 250.0)])
def test_bicgstab_ilu0_solution(cvk, oracle, h, f):
    P = cvk
    rp, ci, v, b = cavity(oracle, h, f)
    n = len(rp) - 1
    xr, rr = oracle.solve("bicgstab", rp, ci, v, b, tol=1e-12, max_iter=200000)
    assert rr.converged
    A = P.CsrMatrix(n, n, rp, ci, v)
    opts = P.SolverOptions(tol=1e-10, max_iter=100000, record_history=True)
    jac = P.solve(P.SolverId.BiCGStab, A, b, P.jacobi(A), opts)
    for s in (1, 2, 4):
        res = P.solve(P.SolverId.BiCGStab, A, b, P.ilu0(A, s), opts)
        rep = res.report
        assert rep.converged and rep.breakdown is None
        assert rep.final_relres <= 1e-10
        assert rep.true_relres <= 1e-8
        assert np.linalg.norm(res.x - xr) <= 1e-7 * np.linalg.norm(xr)
        assert len(rep.residual_history) == rep.iterations
        # the point of ILU(0): far fewer iterations than Jacobi
        assert rep.iterations * 2 <= jac.report.iterations, (s, rep.iterations, jac.report.iterations)


def test_ilu0_errors(cvk, oracle):
    P = cvk
    rp, ci, v, b = cavity(oracle, 0.05)
    n = len(rp) - 1
    A = P.CsrMatrix(n, n, rp, ci, v)
    M = P.ilu0(A)
    for sid in (P.SolverId.BiCGStabL, P.SolverId.TfQmr, P.SolverId.GMRES):
        with pytest.raises(P.InvalidArgument):
            P.solve(sid, A, b, M)
    with pytest.raises(P.InvalidArgument):
        P.ilu0(A, -1)
    # zero pivot: row 1 of [[1, 1], [1, 1]] eliminates to 0
    Z = P.CsrMatrix(2, 2, np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.ones(4, complex))
    with pytest.raises(P.InvalidArgument):
        P.ilu0(Z)
    with pytest.raises(ValueError):
        oracle.ilu0(np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.ones(4, complex))
    # zero rhs: converged at once, x = 0
    res = P.solve(P.SolverId.BiCGStab, A, np.zeros(n, complex), M)
    assert res.report.converged and res.report.iterations == 0 and not res.x.any()


def test_graph_chain_matches_host_loop(cvk, oracle, knobs):
    """FAST mode runs the device-scalar phase chain (cvk_ilu.cu, CUDA graph);
    CVK_OPT_ILU_HOSTLOOP forces the host loop of the same kernels' arithmetic.
    Same reduction kernels' sums, so the same iterations and a matching x."""
    P = cvk
    rp, ci, v, b = cavity(oracle, 0.008, 250.0)
    n = len(rp) - 1
    A = P.CsrMatrix(n, n, rp, ci, v)
    opts = P.SolverOptions(tol=1e-9, max_iter=100000, record_history=True)
    for s in (0, 2, 3):
        M = P.ilu0(A, s)
        chain = P.solve(P.SolverId.BiCGStab, A, b, M, opts)
        knobs(ilu_hostloop=1)
        host = P.solve(P.SolverId.BiCGStab, A, b, M, opts)
        knobs(ilu_hostloop=0)
        assert chain.report.converged and host.report.converged
        assert abs(chain.report.iterations - host.report.iterations) <= 1
        assert len(chain.report.residual_history) == chain.report.iterations
        assert np.linalg.norm(chain.x - host.x) <= 1e-9 * np.linalg.norm(host.x)
        assert chain.report.true_relres <= 1e-8


def test_chain_max_iter_and_zero_rhs(cvk, oracle):
    P = cvk
    rp, ci, v, b = cavity(oracle, 0.012)
    n = len(rp) - 1
    A = P.CsrMatrix(n, n, rp, ci, v)
    M = P.ilu0(A, 2)
    for k in (0, 1, 5, 13):
        r = P.solve(P.SolverId.BiCGStab, A, b, M, P.SolverOptions(tol=1e-30, max_iter=k)).report
        assert not r.converged and r.iterations == k
    r = P.solve(P.SolverId.BiCGStab, A, np.zeros(n, complex), M).report
    assert r.converged and r.iterations == 0
