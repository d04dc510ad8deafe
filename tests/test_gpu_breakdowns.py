"""Every breakdown the reference reports (krylov.cpp:83-87, 99-103, 117-121,
179-194, 232-236, 321-324, 355-358), on tiny systems where the reference's
own arithmetic hits an exact cancellation (tests/fixtures/breakdowns.json,
found by tools/find_breakdowns.py and confirmed on the reference itself).

Both reference-order modes must reproduce the reference's report and x bit
for bit; FAST must report the same reason with the same iteration accounting
(converged flag, iterations), on the persistent and the phase-kernel path."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import FIXTURES

pytestmark = pytest.mark.gpu

CASES = json.load(open(os.path.join(FIXTURES, "breakdowns.json")))


def system(P, c):
    v = np.array([complex(a, b) for a, b in c["v"]])
    b = np.array([complex(a, b_) for a, b_ in c["b"]])
    A = P.CsrMatrix(c["n"], c["n"], c["rp"], c["ci"], v)
    return A, b


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).view(np.uint8)).hexdigest()


@pytest.mark.parametrize("mode", ["Sequential", "Parallel"])
@pytest.mark.parametrize("key", sorted(CASES))
def test_reference_modes_reproduce_breakdown(cvk, key, mode):
    P = cvk
    c = CASES[key]
    A, b = system(P, c)
    r = P.solve(P.solver_id(c["solver"]), A, b, P.jacobi(A),
                P.SolverOptions(tol=c["tol"], max_iter=c["max_iter"], l=c["l"]), mode=P.ExecMode[mode])
    assert r.report.breakdown == c["breakdown"]
    assert (r.report.iterations, r.report.converged) == (c["iterations"], c["converged"])
    assert r.report.final_relres.hex() == c["final_relres"]
    assert r.report.true_relres.hex() == c["true_relres"]
    assert sha(r.x) == c["x_sha256"]


@pytest.mark.parametrize("path", ["persistent", "phased"])
@pytest.mark.parametrize("key", sorted(CASES))
def test_fast_reports_same_breakdown(cvk, knobs, key, path):
    P = cvk
    c = CASES[key]
    knobs(phased_min_n=0 if path == "phased" else 1 << 30)
    A, b = system(P, c)
    r = P.solve(P.solver_id(c["solver"]), A, b, P.jacobi(A),
                P.SolverOptions(tol=c["tol"], max_iter=c["max_iter"], l=c["l"]), mode=P.ExecMode.Fast)
    assert r.report.breakdown == c["breakdown"], r.report
    assert (r.report.iterations, r.report.converged) == (c["iterations"], c["converged"])
    assert np.all(np.isfinite(r.x))
