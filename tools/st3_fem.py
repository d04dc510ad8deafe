"""FEM-3D (N=79) streamed solves with a ring-depth variant library: debugging
aid (CVK_LIB_PATH=_variants/st3/...); ST_FOLD, ST_SOLVERS, ST_IT."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import fem3d as F  # noqa: E402

cav = F.build_cavity(int(os.environ.get("ST_N", "79")))
A = cav.matrix(2 * math.pi * 100.0)
M = P.jacobi(A)
for s in os.environ.get("ST_SOLVERS", "bicgstab,cocg,tfqmr").split(","):
    with P.path_options(bicg_fold=int(os.environ.get("ST_FOLD", "1"))):
        r = P.solve(P.solver_id(s), A, cav.b, M, P.SolverOptions(tol=1e-30, max_iter=int(os.environ.get("ST_IT", "200"))))
    print(s, A.nrows, r.report.iterations, r.report.final_relres, flush=True)
