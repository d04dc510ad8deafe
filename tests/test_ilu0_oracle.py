"""ILU(0) restatement (oracle/cavac_oracle.c, TEST INFRASTRUCTURE) on CPU:
L U reproduces A on its pattern, the sweep apply converges to the exact
triangular solves, a zero pivot is reported.  Beyond the reference (it has
jacobi / identity only, krylov.cpp:27-55): parity unpinned."""
import math

import numpy as np


def test_oracle_ilu0_pattern_and_apply(oracle):
    O = oracle
    g = O.build_grid(2.4, 1.2, 0.05, 0.4, 0.65, 0.01 + 0j)
    rp, ci, v, _ = O.assemble(g, 2 * math.pi * 100.0, 343.0, np.full(g.roof_size, 1.0 + 0j))
    n = len(rp) - 1
    f = O.ilu0(rp, ci, v)
    F = np.zeros((n, n), complex)
    A = np.zeros((n, n), complex)
    for i in range(n):
        F[i, ci[rp[i]:rp[i + 1]]] = f[rp[i]:rp[i + 1]]
        A[i, ci[rp[i]:rp[i + 1]]] = v[rp[i]:rp[i + 1]]
    L = np.tril(F, -1) + np.eye(n)
    U = np.triu(F)
    on = A != 0
    assert np.abs((L @ U - A)[on]).max() <= 1e-13 * np.abs(A).max()
    r = np.random.default_rng(0).standard_normal(n) + 1j
    want = np.linalg.solve(U, np.linalg.solve(L, r))
    errs = [np.linalg.norm(O.ilu0_apply(rp, ci, f, s, r) - want) for s in (0, 2, 8, 64)]
    assert errs[1] < errs[0] and errs[2] < errs[1]
    assert errs[3] <= 1e-10 * np.linalg.norm(want)
    # sweeps = 0 is d .* r with d = 1 / u_ii
    assert np.allclose(O.ilu0_apply(rp, ci, f, 0, r), r / np.diag(U), rtol=1e-15, atol=0)


def test_oracle_ilu0_zero_pivot(oracle):
    import pytest
    with pytest.raises(ValueError):
        oracle.ilu0(np.array([0, 2, 4]), np.array([0, 1, 0, 1]), np.ones(4, complex))
    with pytest.raises(ValueError):  # missing diagonal
        oracle.ilu0(np.array([0, 1, 2]), np.array([1, 0]), np.ones(2, complex))
