"""Host assembly input (helmholtz.py) against the golden system and the
oracle restatement of helmholtz.cpp, bitwise. CPU only."""
import math

import numpy as np
import pytest


def bits(a):
    return np.ascontiguousarray(a, np.complex128).view(np.uint64)


def test_build_grid_counts():
    """test_helmholtz.cpp:34-43."""
    from paper_2112_00087_b200 import helmholtz as H
    g = H.build_grid(2.4, 1.2, 0.133425, 0.4, 0.65)
    assert (g.nx, g.ny) == (17, 8)
    g = H.build_grid(2.4, 1.2, 0.05, 0.4, 0.65)
    assert (g.nx, g.ny, g.size()) == (47, 23, 1081)
    with pytest.raises(ValueError):
        H.build_grid(2.4, 1.2, 1.0, 0.4, 0.65)


def test_assemble_matches_golden_system(golden):
    from paper_2112_00087_b200 import helmholtz as H
    g = H.build_grid(2.4, 1.2, 0.05, 0.4, 0.65)
    p = H.assemble(g, 2 * math.pi * 74.21875, 340.0, np.zeros(g.roof_size(), np.complex128))
    assert np.array_equal(p.A.row_offsets.astype(np.int64), golden["rp"])
    assert np.array_equal(p.A.col_indices.astype(np.int64), golden["ci"])
    assert np.array_equal(bits(p.A.values), bits(golden["v"]))


@pytest.mark.parametrize("adm", [0j, 0.01 + 0j, 0.02 - 0.005j])
def test_assemble_matches_oracle(oracle, adm):
    from paper_2112_00087_b200 import helmholtz as H
    for h, f in ((0.1, 13.0), (0.033289, 250.0)):
        g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
        rng = np.random.default_rng(3)
        d = rng.uniform(-1, 1, g.roof_size()) + 1j * rng.uniform(-1, 1, g.roof_size())
        p = H.assemble(g, 2 * math.pi * f, 340.0, d)
        og = oracle.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
        rp, ci, v, b = oracle.assemble(og, 2 * math.pi * f, 340.0, d)
        assert np.array_equal(p.A.row_offsets.astype(np.int64), rp)
        assert np.array_equal(p.A.col_indices.astype(np.int64), ci)
        assert np.array_equal(bits(p.A.values), bits(v))
        assert np.array_equal(bits(p.b), bits(b))


def test_csr_from_triplets_mirror():
    """test_numkit.cpp:46-83 on the host mirror."""
    import paper_2112_00087_b200 as P
    A = P.csr_from_triplets([0, 0], [0, 0], [1.0, 2.0], 1, 1)
    assert A.nnz() == 1 and A.values[0] == 3.0
    A = P.csr_from_triplets([0, 0, 0], [3, 1, 2], [1.0, 2.0, 3.0], 1, 4)
    assert list(A.col_indices) == [1, 2, 3]
    with pytest.raises(P.InvalidArgument):
        P.csr_from_triplets([2], [0], [1.0], 2, 2)
    E = P.csr_from_triplets([], [], [], 2, 2)
    assert E.nnz() == 0 and list(E.row_offsets) == [0, 0, 0]
