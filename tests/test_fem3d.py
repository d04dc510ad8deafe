"""Synthetic P1 FEM cavity (fem3d.py, beyond the reference): self-checks of
the assembled operators on CPU (the device path is tests/test_gpu_fem3d.py)."""
import numpy as np
import pytest

from paper_2112_00087_b200 import fem3d as F


@pytest.mark.parametrize("N", [2, 5])
def test_operators_self_checks(N):
    cav = F.build_cavity(N)
    n = cav.n
    assert n == (2 * N + 1) * (N + 1) ** 2
    rows = np.repeat(np.arange(n), np.diff(cav.rp))
    # columns sorted per row, pattern symmetric
    for i in range(n):
        c = cav.ci[cav.rp[i]:cav.rp[i + 1]]
        assert np.all(np.diff(c) > 0)
    key = set(zip(rows.tolist(), cav.ci.tolist()))
    assert all((c, r) in key for r, c in key)
    # K 1 = 0, K symmetric positive semidefinite (constant null space)
    K1 = np.zeros(n)
    np.add.at(K1, rows, cav.K)
    assert np.abs(K1).max() <= 1e-12 * np.abs(cav.K).max()
    Kd = np.zeros((n, n))
    Kd[rows, cav.ci] = cav.K
    assert np.allclose(Kd, Kd.T, rtol=0, atol=1e-12 * np.abs(cav.K).max())
    ev = np.linalg.eigvalsh(Kd)
    assert ev.min() >= -1e-9 * ev.max()
    # sum M = volume; sum C = c beta area of the absorbing face
    assert cav.M.sum() == pytest.approx(2.4 * 1.2 * 1.2, rel=1e-12)
    assert cav.Cd.sum() == pytest.approx(340.0 * 0.01 * 2.4 * 1.2, rel=1e-12)
    # A(omega) arithmetic: re = K - (omega omega) M, im = omega C
    om = 2 * np.pi * 120.0
    v = cav.values(om)
    assert np.array_equal(v.real, cav.K - (om * om) * cav.M) and np.array_equal(v.imag, om * cav.Cd)


def test_survey_sizes():
    # FEM-3D N=29 -> 53,100 DOF (config 1)
    assert (2 * 29 + 1) * 30 ** 2 == 53100
    cav = F.build_cavity(8)
    assert cav.n == 17 * 81 and 12.5 < len(cav.ci) / cav.n < 15.0
