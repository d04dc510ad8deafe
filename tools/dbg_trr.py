import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_00087_b200 as P
from oracle import oracle as O
gold = "tests/golden"
rp, ci, v = O.read_matrix_market(gold + "/system.mtx")
b = O.read_vector_csv(gold + "/rhs.csv")
n = len(rp) - 1
for ctas in ("1", "2", "0"):
    if ctas == "0":
        os.environ.pop("CVK_MAX_CTAS", None)
    else:
        os.environ["CVK_MAX_CTAS"] = ctas
    A = P.CsrMatrix(n, n, rp, ci, v)
    M = P.jacobi(A)
    for mode in (P.ExecMode.Sequential, P.ExecMode.Parallel):
        r = P.bicgstab(A, b, M, P.SolverOptions(), mode=mode)
        t_api = P.true_relative_residual(A, b, r.x, mode=mode)
        t_orc = O.true_relres(rp, ci, v, b, r.x)
        print(ctas, mode.name, r.report.iterations, "%.17g %.17g %.17g" % (r.report.true_relres, t_api, t_orc), flush=True)
    for s in ("tfqmr", "bicgstab_l", "gmres"):
        r = P.solve(P.solver_id(s), A, b, M, P.SolverOptions(max_iter=300), mode=P.ExecMode.Sequential)
        print(ctas, s, r.report.iterations, "%.17g %.17g" % (r.report.true_relres, O.true_relres(rp, ci, v, b, r.x)), flush=True)
