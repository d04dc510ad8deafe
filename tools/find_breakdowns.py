"""Search small systems on which the reference's solvers break down, one per
breakdown reason (krylov.cpp:83-87, 99-103, 117-121, 179-194, 232-236,
321-324, 355-358), and record them as tests/fixtures/breakdowns.json
(TEST INFRASTRUCTURE: the fixture of tests/test_gpu_breakdowns.py).  For each
reason the case with the earliest breakdown is kept: an exact cancellation a
few steps in is structural, so the double-double FAST sums meet it too, where
a late one depends on the rounding history.

Candidates are tiny CSR systems with small-integer complex entries, where
exact cancellations make <shadow, r>, <shadow, v>, |t|^2, ... vanish.  The
search runs on the C restatement (oracle/cavac_oracle.c); every recorded case
is then re-run on the reference itself (oracle/_ref) with the Jacobi
preconditioner, and only cases whose reports agree are kept.

    python tools/find_breakdowns.py
"""
from __future__ import annotations

import hashlib
import itertools
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "fixtures", "breakdowns.json")
WANT = {
    "bicgstab": ["rho breakdown", "stagnation in <shadow, v>", "omega breakdown"],
    "bicgstab_l": ["rho breakdown", "stagnation in <shadow, u>", "degenerate least-squares in MR step"],
    "tfqmr": ["rho breakdown", "sigma breakdown"],
}
VALS = [0, 1, -1, 2, 1j, -1j, 1 + 1j, 3]


def csr(dense):
    n = dense.shape[0]
    rp, ci, v = [0], [], []
    for i in range(n):
        for j in range(n):
            if dense[i, j] != 0 or i == j:
                ci.append(j)
                v.append(dense[i, j])
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int64), np.array(v, np.complex128)


def sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).view(np.uint8)).hexdigest()


def main():
    rng = np.random.default_rng(1234)
    found = {}
    todo = {(s, r) for s, rs in WANT.items() for r in rs}
    best = {}  # key -> iterations of the kept case: prefer the earliest breakdown
    for trial in range(60000):
        n = int(rng.integers(2, 5))
        dense = np.array([[VALS[k] for k in rng.integers(0, len(VALS), n)] for _ in range(n)], np.complex128)
        density = rng.uniform(0.3, 1.0)
        mask = rng.uniform(size=(n, n)) < density
        dense = np.where(mask | np.eye(n, dtype=bool), dense, 0)
        if np.any(np.diag(dense) == 0):
            continue
        b = np.array([VALS[k] for k in rng.integers(0, len(VALS), n)], np.complex128)
        if not b.any():
            continue
        rp, ci, v = csr(dense)
        for solver, l in (("bicgstab", 8), ("bicgstab_l", 2), ("bicgstab_l", 1), ("tfqmr", 8)):
            x, rep = O.solve(solver, rp, ci, v, b, tol=1e-12, max_iter=50, l=l)
            key = (solver, rep.breakdown)
            if key in todo and rep.iterations < best.get(key, 1 << 30) and np.all(np.isfinite(x)):
                # the same breakdown, at the same step, with near-exact sums
                O.lib().orc_set_sum_mode(1)
                _, rd = O.solve(solver, rp, ci, v, b, tol=1e-12, max_iter=50, l=l)
                O.lib().orc_set_sum_mode(0)
                if (rd.breakdown, rd.iterations, rd.converged) != (rep.breakdown, rep.iterations, rep.converged):
                    continue
                # the reference itself must agree (Sequential mode, Jacobi)
                xr, rr = O.ref_solve(solver, rp, ci, v, b, tol=1e-12, max_iter=50, l=l)
                if (rr.breakdown, rr.iterations, rr.converged) != (rep.breakdown, rep.iterations, rep.converged) \
                        or sha(xr) != sha(x):
                    continue
                best[key] = rep.iterations
                found[f"{solver}:{rep.breakdown}"] = {
                    "solver": solver, "l": l, "n": n, "rp": rp.tolist(), "ci": ci.tolist(),
                    "v": [[z.real, z.imag] for z in v], "b": [[z.real, z.imag] for z in b],
                    "tol": 1e-12, "max_iter": 50, "breakdown": rep.breakdown,
                    "iterations": rep.iterations, "converged": rep.converged,
                    "final_relres": rep.final_relres.hex(), "true_relres": rep.true_relres.hex(),
                    "x_sha256": sha(x), "trial": trial,
                }
                print(solver, rep.breakdown, "n", n, "trial", trial, "iterations", rep.iterations, flush=True)
    print("missing:", sorted(todo - set(best)))
    with open(OUT, "w") as f:
        json.dump(found, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
