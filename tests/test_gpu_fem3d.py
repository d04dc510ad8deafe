"""FEM cavity on the device (fem3d.FemOperator, cvk_fem_*): A(omega) values
written on the device bitwise equal to the host arithmetic, and solves pinned
to the dense / oracle solution of the same CSR (beyond the reference: no
reference FEM exists)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_device_values_bitwise(cvk):
    from paper_2112_00087_b200 import fem3d as F
    cav = F.build_cavity(4)
    op = F.FemOperator(cav)
    try:
        for f in (50.0, 123.0, 500.0):
            om = 2 * math.pi * f
            op.set_omega(om)
            assert np.array_equal(op.values().view(np.uint64), cav.values(om).view(np.uint64))
    finally:
        op.close()


@pytest.mark.parametrize("solver", ["bicgstab", "tfqmr", "gmres", "bicgstab_l"])
def test_fem_sweep_matches_dense(cvk, oracle, solver):
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import fem3d as F
    cav = F.build_cavity(4)          # 9 x 5 x 5 nodes, small enough for a dense check
    freqs = (60.0, 180.0, 333.0)
    t = F.fem_frequency_sweep(cav, freqs, solver, P.SolverOptions(tol=1e-12, max_iter=20000), keep_solutions=True)
    n = cav.n
    rows = np.repeat(np.arange(n), np.diff(cav.rp))
    for row in t.rows:
        Ad = np.zeros((n, n), np.complex128)
        Ad[rows, cav.ci] = cav.values(row.omega)
        x_ref = np.linalg.solve(Ad, cav.b)
        _, rep = oracle.solve(solver, cav.rp, cav.ci, cav.values(row.omega), cav.b, tol=1e-12, max_iter=20000)
        if not rep.converged:
            # the algorithm itself stagnates here (restarted GMRES(30) at 333 Hz
            # stalls near 1.5e-11 in the oracle too); the point is reported
            continue
        assert row.converged, row
        x = t.solutions[row.frequency_hz]
        assert np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref) <= 1e-9, row


def test_fem_streamed_path_matches_oracle(cvk, oracle, knobs):
    """A 14-entries-per-row operator on the phase-kernel (TMA-streamed) path,
    against the oracle's BiCGSTAB on the same CSR at tight tolerance."""
    import paper_2112_00087_b200 as P
    from paper_2112_00087_b200 import fem3d as F
    knobs(phased_min_n=0)
    cav = F.build_cavity(9)          # 19 x 10 x 10 = 1900 DOF, several 224-row chunks
    om = 2 * math.pi * 140.0
    A = cav.matrix(om)
    for s in ("bicgstab", "tfqmr"):
        r = P.solve(P.solver_id(s), A, cav.b, P.jacobi(A), P.SolverOptions(tol=1e-12, max_iter=20000))
        x_o, rep = oracle.solve(s, cav.rp, cav.ci, cav.values(om), cav.b, tol=1e-12, max_iter=20000)
        assert r.report.converged and rep.converged
        assert np.linalg.norm(r.x - x_o) / np.linalg.norm(x_o) <= 1e-9
        # tfQMR's quasi-residual under-reports (hard part 6): the
        # oracle stops at the same point with true relres ~3e-9
        assert r.report.true_relres <= max(1e-10, 10 * rep.true_relres)
