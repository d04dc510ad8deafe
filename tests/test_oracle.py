"""The CPU oracle (oracle/cavac_oracle.c) pinned against the reference's own
golden vectors and known answers, and -- when oracle/_ref was built -- against
the unmodified reference itself, bit for bit.  CPU only."""
import math
import os

import numpy as np
import pytest

from conftest import FIXTURES, GOLDEN

H_GOLDEN = 0.05
OMEGA_GOLDEN = 2.0 * math.pi * 74.21875  # proj/tests/golden/dominant.csv:2


def cavity(O, h, f=13.0, roof=1.0 + 0j, adm=0j, c=340.0):
    g = O.build_grid(2.4, 1.2, h, 0.4, 0.65, adm)
    rp, ci, v, b = O.assemble(g, 2.0 * math.pi * f, c, np.full(g.roof_size, roof, np.complex128))
    return g, rp, ci, v, b


def test_golden_solution_byte_identical(oracle, golden):
    """proj/tests/golden/{solution,report}.csv: 246 iterations, relres bits."""
    x, rep = oracle.solve("bicgstab", golden["rp"], golden["ci"], golden["v"], golden["b"], tol=1e-9)
    assert rep.converged and rep.iterations == 246
    assert "%.17g" % rep.final_relres == "8.9265369265007959e-10"
    assert "%.17g" % rep.true_relres == "8.5608367217167752e-10"
    assert oracle.format_vector_csv(x) == golden["solution_csv"]


def test_golden_matrix_from_assemble(oracle, golden):
    g, rp, ci, v, b = cavity(oracle, H_GOLDEN)
    rp2, ci2, v2, _ = oracle.assemble(g, OMEGA_GOLDEN, 340.0, np.zeros(g.roof_size, np.complex128))
    assert np.array_equal(rp2, golden["rp"]) and np.array_equal(ci2, golden["ci"])
    assert np.array_equal(v2.view(np.uint64), golden["v"].view(np.uint64))


def test_known_iteration_counts(oracle, golden):
    """SURVEY.md 7 hard part 1 (reference run): BiCGSTAB(8) 25, tfQMR 207."""
    _, r1 = oracle.solve("bicgstab_l", golden["rp"], golden["ci"], golden["v"], golden["b"])
    _, r2 = oracle.solve("tfqmr", golden["rp"], golden["ci"], golden["v"], golden["b"])
    assert (r1.iterations, r2.iterations) == (25, 207)


def test_identity_and_diagonal_kats(oracle):
    """test_krylov.cpp:80-121."""
    rng = np.random.default_rng(777001)
    n = 10
    rp, ci = np.arange(n + 1), np.arange(n)
    b = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    for s in ("bicgstab", "bicgstab_l", "tfqmr", "gmres"):
        x, rep = oracle.solve(s, rp, ci, np.ones(n, np.complex128), b, dinv="identity")
        assert rep.converged and rep.iterations <= 1
        assert np.abs(x - b).max() <= 1e-12
    n = 12
    d = np.array([complex(1.0 + i, 0.5 * i) for i in range(n)])
    b = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    for s in ("bicgstab", "bicgstab_l", "tfqmr", "gmres"):
        x, rep = oracle.solve(s, np.arange(n + 1), np.arange(n), d, b)
        assert rep.converged and rep.iterations == 1 and rep.true_relres <= 1e-12
    x, rep = oracle.solve("bicgstab", [0, 1, 2], [0, 1], [1 + 1j, 2 - 1j], [1 + 1j, 2 - 1j])
    assert rep.iterations == 1 and np.abs(x - 1).max() <= 1e-12


def test_jacobi_zero_diagonal(oracle):
    rp, ci, v = oracle.csr_from_triplets([0, 1], [0, 0], [1.0, 1.0], 2, 2)
    with pytest.raises(ValueError, match="row 1"):
        oracle.jacobi(rp, ci, v)


def test_ladder_monotone(oracle):
    """acceptance.cpp:241-257 with the measured counts of SURVEY.md 8(c)."""
    want = {"bicgstab": [55, 115, 239], "bicgstab_l": [7, 14, 29], "tfqmr": [57, 125, 248]}
    for s, counts in want.items():
        got = []
        for h in (0.133425, 0.066604, 0.033289):
            _, rp, ci, v, b = cavity(oracle, h)
            _, rep = oracle.solve(s, rp, ci, v, b)
            assert rep.converged
            got.append(rep.iterations)
        assert got == counts, (s, got)


def test_csr_from_triplets_semantics(oracle):
    """test_numkit.cpp:46-83: duplicates summed, columns sorted, range check."""
    rp, ci, v = oracle.csr_from_triplets([0, 0], [0, 0], [1.0, 2.0], 1, 1)
    assert list(rp) == [0, 1] and v[0] == 3.0
    rp, ci, v = oracle.csr_from_triplets([0, 0, 0], [3, 1, 2], [1.0, 2.0, 3.0], 1, 4)
    assert list(ci) == [1, 2, 3]
    with pytest.raises(ValueError):
        oracle.csr_from_triplets([2], [0], [1.0], 2, 2)


def test_schwarz_matches_monodomain(oracle):
    """acceptance.cpp:263-291 at h=0.1 (2 and 3 strips, s = 2 + ik)."""
    g = oracle.build_grid(2.4, 1.2, 0.1, 0.4, 0.65)
    roof = np.array([complex(1.0 + 0.1 * i, 0.3) for i in range(g.roof_size)])
    omega = 2 * math.pi * 13.0
    rp, ci, v, b = oracle.assemble(g, omega, 340.0, roof)
    mono, rep = oracle.solve("bicgstab", rp, ci, v, b, tol=1e-10)
    assert rep.converged
    k = omega / 340.0
    for ns in (2, 3):
        x, dr = oracle.schwarz_solve(g, 340.0, rp, ci, v, b, ns, complex(2, k), complex(2, k),
                                     tol=1e-10, ddm_tol=1e-8, max_outer=300)
        assert dr["converged"]
        assert np.linalg.norm(x - mono) / np.linalg.norm(mono) <= 1e-6


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLDEN), "..", "oracle", "_ref",
                                                    "libcavac_ref.so")), reason="oracle/_ref not built")
def test_restatement_equals_reference_bitwise(oracle, golden):
    """The C restatement against the unmodified reference (oracle/_ref)."""
    for s in ("bicgstab", "bicgstab_l", "tfqmr"):
        xo, ro = oracle.solve(s, golden["rp"], golden["ci"], golden["v"], golden["b"], record_history=True)
        xr, rr = oracle.ref_solve(s, golden["rp"], golden["ci"], golden["v"], golden["b"], record_history=True)
        assert ro.iterations == rr.iterations
        assert np.array_equal(xo.view(np.uint64), xr.view(np.uint64))
        assert ro.residual_history == rr.residual_history
    _, rp, ci, v, b = cavity(oracle, 0.066604, f=100.0, adm=0.01)
    for s in ("bicgstab", "tfqmr"):
        xo, ro = oracle.solve(s, rp, ci, v, b)
        xr, rr = oracle.ref_solve(s, rp, ci, v, b)
        assert np.array_equal(xo.view(np.uint64), xr.view(np.uint64))


def test_breakdown_fixture_pinned(oracle):
    """tests/golden/breakdowns.json: the C restatement (and, where it is
    built, the reference itself) reproduces every recorded breakdown."""
    import hashlib
    import json
    cases = json.load(open(os.path.join(FIXTURES, "breakdowns.json")))
    assert {c["breakdown"] for c in cases.values()} == {
        "rho breakdown", "stagnation in <shadow, v>", "omega breakdown", "stagnation in <shadow, u>",
        "degenerate least-squares in MR step", "sigma breakdown"}
    for c in cases.values():
        v = np.array([complex(a, b) for a, b in c["v"]])
        b = np.array([complex(a, b_) for a, b_ in c["b"]])
        runs = [oracle.solve(c["solver"], c["rp"], c["ci"], v, b, tol=c["tol"], max_iter=c["max_iter"], l=c["l"])]
        if oracle.ref_available():
            runs.append(oracle.ref_solve(c["solver"], c["rp"], c["ci"], v, b, tol=c["tol"],
                                         max_iter=c["max_iter"], l=c["l"]))
        for x, rep in runs:
            assert rep.breakdown == c["breakdown"] and rep.iterations == c["iterations"]
            assert rep.final_relres.hex() == c["final_relres"]
            assert hashlib.sha256(np.ascontiguousarray(x).view(np.uint8)).hexdigest() == c["x_sha256"]


@pytest.mark.parametrize("m", [30, 7])
def test_gmres_dcgs2_solution(oracle, m):
    """GMRES(m) with delayed reorthogonalisation (orc_gmres, beyond the
    reference): on a damped cavity it converges to the reference's BiCGSTAB
    solution at tight tolerance, and its relative residual estimate tracks the
    true residual (the basis stays orthonormal to working accuracy)."""
    _, rp, ci, v, b = cavity(oracle, 0.05, adm=0.02)
    xt, rt = oracle.solve("bicgstab", rp, ci, v, b, tol=1e-13, max_iter=100000)
    x, r = oracle.solve("gmres", rp, ci, v, b, tol=1e-11, m=m, max_iter=20000)
    assert r.converged and r.breakdown is None
    assert np.linalg.norm(x - xt) / np.linalg.norm(xt) <= 1e-9
    # final_relres is GMRES's estimate (left-preconditioned); true_relres is
    # recomputed from x: they agree to the conditioning of the preconditioner
    assert r.true_relres <= 10 * r.final_relres
