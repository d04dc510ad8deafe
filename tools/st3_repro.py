"""Streamed BiCGSTAB on a small cavity (phase kernels forced): debugging aid
for ring-depth variants (CVK_LIB_PATH=_variants/st3/libcavac_b200.so)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as H  # noqa: E402

g = H.build_grid(2.4, 1.2, float(os.environ.get("ST_H", "0.01")), 0.4, 0.65, 0.01)
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
M = P.jacobi(prob.A)
for s in os.environ.get("ST_SOLVERS", "bicgstab,tfqmr,cocg").split(","):
    with P.path_options(phased_min_n=0, bicg_fold=int(os.environ.get("ST_FOLD", "1"))):
        r = P.solve(P.solver_id(s), prob.A, prob.b, M, P.SolverOptions(tol=1e-8, max_iter=int(os.environ.get("ST_IT", "50"))))
    print(s, prob.A.nrows, r.report.iterations, r.report.final_relres)
