"""COCG (conjugate orthogonal CG) for the complex-symmetric Helmholtz operator
-- north_star's "CG" row, beyond the reference (krylov.cpp:377-384 has no CG;
A = A^T is complex symmetric, not Hermitian, so plain CG does not apply).
Oracle: orc_cocg (oracle/cavac_oracle.c), written in the reference's
conventions.  Parity is pinned through the solution: the reference's own
tight solve of the same system."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def cavity(O, h, f=13.0, adm=0.0):
    g = O.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
    return O.assemble(g, 2 * math.pi * f, 340.0, np.ones(g.roof_size, np.complex128))


@pytest.mark.parametrize("mode", ["Sequential", "Parallel"])
def test_cocg_reference_modes_bitwise_oracle(cvk, oracle, golden, mode):
    P = cvk
    rp, ci, v, b = golden["rp"], golden["ci"], golden["v"], golden["b"]
    A = P.CsrMatrix(len(rp) - 1, len(rp) - 1, rp, ci, v)
    r = P.cocg(A, b, P.jacobi(A), P.SolverOptions(record_history=True), mode=P.ExecMode[mode])
    xo, ro = oracle.solve("cocg", rp, ci, v, b, record_history=True)
    assert (r.report.iterations, r.report.converged) == (ro.iterations, ro.converged)
    assert r.report.residual_history == ro.residual_history
    assert np.array_equal(bits(r.x), bits(xo))
    assert r.report.true_relres == ro.true_relres


@pytest.mark.parametrize("path", ["persistent", "phased", "streamed"])
def test_cocg_fast_matches_reference_solution(cvk, oracle, knobs, path):
    """FAST COCG on each device path against the reference's own tfQMR at
    tol 1e-13 (oracle/_ref when built, else the bitwise restatement), on a
    damped cavity large enough to stream; the paths agree bit for bit."""
    P = cvk
    knobs(phased_min_n=1 << 30 if path == "persistent" else 0, stream=0 if path == "phased" else 1)
    rp, ci, v, b = cavity(oracle, 0.02, f=60.0, adm=0.01)
    n = len(rp) - 1
    A = P.CsrMatrix(n, n, rp, ci, v)
    M = P.jacobi(A)
    solve_ref = oracle.ref_solve if oracle.ref_available() else oracle.solve
    x_tight, _ = solve_ref("tfqmr", rp, ci, v, b, tol=1e-13, max_iter=20000)
    r = P.cocg(A, b, M, P.SolverOptions(tol=1e-12, max_iter=20000, record_history=True))
    assert r.report.converged and r.report.final_relres <= 1e-12
    assert np.linalg.norm(r.x - x_tight) / np.linalg.norm(x_tight) <= 1e-10
    assert len(r.report.residual_history) == r.report.iterations
    _, ro = oracle.solve("cocg", rp, ci, v, b, tol=1e-9, max_iter=20000)
    r9 = P.cocg(A, b, M, P.SolverOptions(tol=1e-9, max_iter=20000))
    assert abs(r9.report.iterations - ro.iterations) <= max(2, 0.15 * ro.iterations)
    e = P.cocg(A, b, M, P.SolverOptions(max_iter=3))
    assert not e.report.converged and e.report.iterations == 3
    z = P.cocg(A, np.zeros_like(b), M)
    assert z.report.converged and z.report.iterations == 0 and z.report.true_relres == 0.0
    test_cocg_fast_matches_reference_solution.out[path] = (r.report.iterations, bits(r.x))
    out = test_cocg_fast_matches_reference_solution.out
    if len(out) == 3:
        its = {k: v[0] for k, v in out.items()}
        assert len(set(its.values())) == 1, its
        assert all(np.array_equal(v[1], out["persistent"][1]) for v in out.values())


test_cocg_fast_matches_reference_solution.out = {}


def test_cocg_one_spmv_per_iteration(cvk, oracle, knobs):
    """Two launches per iteration on the phase-kernel path (SpMV phase +
    elementwise phase), against BiCGSTAB's three."""
    P = cvk
    knobs(phased_min_n=0)
    rp, ci, v, b = cavity(oracle, 0.02, f=60.0, adm=0.01)
    n = len(rp) - 1
    A = P.CsrMatrix(n, n, rp, ci, v)
    r = P.cocg(A, b, P.jacobi(A), P.SolverOptions(tol=1e-10, max_iter=20000))
    graphs = r.report.kernel_launches
    assert graphs <= 2 * (r.report.iterations + 16) + 4, (graphs, r.report.iterations)
