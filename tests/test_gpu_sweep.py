"""Frequency sweeps with the operator assembled on the device
(cvk_csr_assemble_cavity): every point pinned by the reference's own
assemble(omega) (helmholtz.cpp:59-115, oracle restatement) and solve."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FREQS = (13.0, 50.0, 100.0, 250.0, 500.0)


def bits(a):
    return np.ascontiguousarray(a, np.complex128).view(np.uint64)


@pytest.mark.parametrize("adm", [0j, 0.01 + 0j, 0.02 + 0.005j])
def test_device_values_bitwise_reference(cvk, oracle, adm):
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.sweep import CavitySweep
    g = H.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, adm)
    og = oracle.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, adm)
    d = np.full(g.roof_size(), 1.0 + 0.25j)
    sw = CavitySweep(g, 340.0, d)
    try:
        for f in FREQS:
            omega = 2.0 * math.pi * f
            sw.set_frequency(f)
            rp, ci, v, b = oracle.assemble(og, omega, 340.0, d)
            assert np.array_equal(sw.A.row_offsets, rp) and np.array_equal(sw.A.col_indices, ci)
            assert np.array_equal(bits(sw.values()), bits(v)), f
            assert np.array_equal(bits(sw.b), bits(b))
    finally:
        sw.close()


def test_sweep_ref_mode_bitwise_reference(cvk, oracle):
    """Sequential mode on the device-assembled operator = the reference's
    assemble(omega) + jacobi + bicgstab, bit for bit, at every point."""
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.sweep import frequency_sweep
    g = H.build_grid(2.4, 1.2, 0.1, 0.4, 0.65, 0.01)
    og = oracle.build_grid(2.4, 1.2, 0.1, 0.4, 0.65, 0.01)
    d = np.ones(g.roof_size(), np.complex128)
    t = frequency_sweep(g, 340.0, d, (50.0, 200.0), "bicgstab", P.SolverOptions(tol=1e-9),
                        mode=P.ExecMode.Sequential, keep_solutions=True)
    for row in t.rows:
        rp, ci, v, b = oracle.assemble(og, row.omega, 340.0, d)
        x, rep = oracle.solve("bicgstab", rp, ci, v, b, tol=1e-9)
        assert row.iterations == rep.iterations and row.converged == rep.converged
        assert np.array_equal(bits(t.solutions[row.frequency_hz]), bits(x))


@pytest.mark.parametrize("solver", ["bicgstab", "tfqmr", "bicgstab_l", "gmres"])
def test_sweep_fast_matches_reference(cvk, oracle, solver):
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.sweep import frequency_sweep, write_sweep_csv
    g = H.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, 0.01)
    og = oracle.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, 0.01)
    d = np.ones(g.roof_size(), np.complex128)
    t = frequency_sweep(g, 340.0, d, FREQS, solver, P.SolverOptions(tol=1e-12, max_iter=20000),
                        keep_solutions=True)
    assert len(t.rows) == len(FREQS)
    for row in t.rows:
        rp, ci, v, b = oracle.assemble(og, row.omega, 340.0, d)
        _, rep = oracle.solve(solver, rp, ci, v, b, tol=1e-12, max_iter=20000)
        if not rep.converged:
            # the reference itself breaks down here (BiCGSTAB(8) at 500 Hz:
            # "degenerate least-squares in MR step"); the point is reported
            continue
        assert row.converged, row
        # pinned against the exact solution of the reference's assembled system
        n = len(rp) - 1
        Ad = np.zeros((n, n), np.complex128)
        for i in range(n):
            Ad[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
        x_ref = np.linalg.solve(Ad, b)
        x = t.solutions[row.frequency_hz]
        assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-10, row
        assert row.true_relres <= 1e-10
    write_sweep_csv("/tmp/sweep_test.csv", t)
    assert open("/tmp/sweep_test.csv").readline().startswith("solver,frequency_hz,n,iterations")


def test_sweep_reports_nonconvergence(cvk):
    """bench_solvers reports non-converged points instead of raising."""
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.sweep import frequency_sweep
    g = H.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, 0.01)
    t = frequency_sweep(g, 340.0, np.ones(g.roof_size()), (100.0, 300.0), "bicgstab",
                        P.SolverOptions(tol=1e-12, max_iter=5))
    assert all(not r.converged and r.iterations <= 5 for r in t.rows)


def test_assemble_rejects_foreign_pattern(cvk):
    import ctypes as C

    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import _lib
    from paper_2112_00087_b200 import helmholtz as H
    from paper_2112_00087_b200.schwarz import _grid
    from paper_2112_00087_b200.sweep import _bind
    g = H.build_grid(2.4, 1.2, 0.1, 0.4, 0.65, 0j)
    n = g.size()
    A = P.csr_identity(n)
    L = _lib.load()
    _bind(L)
    gg = _grid(g)
    code = L.cvk_csr_assemble_cavity(A.device(), C.byref(gg), 100.0, 340.0)
    assert code == -1 and "5-point pattern" in L.cvk_last_error().decode()
