"""Per-iteration device time of the solvers on the BASELINE configs' systems
(REF-2D cavity and the FEM-3D box), fixed iteration counts (tol 1e-30)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import fem3d as F
from paper_2112_00087_b200 import helmholtz as H


def ref2d(h, f=100.0):
    g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
    prob = H.assemble(g, 2 * math.pi * f, 340.0, np.ones(g.roof_size(), np.complex128))
    return prob.A, prob.b


def fem(N, f=100.0):
    cav = F.build_cavity(N)
    return cav.matrix(2 * math.pi * f), cav.b


cases = os.environ.get("PROBE_CASES", "ref2d:0.0075,fem:29,ref2d:0.0017,fem:79").split(",")
solvers = os.environ.get("PROBE_SOLVERS", "bicgstab,tfqmr,gmres,bicgstab_l").split(",")
maxit = int(os.environ.get("PROBE_MAXIT", "60"))
for case in cases:
    kind, arg = case.split(":")
    A, b = ref2d(float(arg)) if kind == "ref2d" else fem(int(arg))
    M = P.jacobi(A)
    n, nnz = A.nrows, A.nnz()
    for s in solvers:
        opts = P.SolverOptions(tol=1e-30, max_iter=maxit)
        P.solve(P.solver_id(s), A, b, M, opts)
        r = P.solve(P.solver_id(s), A, b, M, opts)
        it = max(1, r.report.iterations)
        per = r.report.device_time / it
        spmv_b = 20 * nnz + 4 * (n + 1) + 32 * n
        print(f"{case:14s} n={n:8d} nnz/row={nnz / n:5.2f} {s:10s} iters {it:5d} {per * 1e6:9.1f} us/it "
              f"({per / (spmv_b / 6.55e12):5.1f} SpMV-at-peak equivalents)", flush=True)
