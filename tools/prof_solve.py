"""Fixed-iteration 1M-DOF solve for ncu (max_iter small)."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import helmholtz as H
h = float(os.environ.get("PROBE_H", "0.0017"))
g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A = prob.A
M = P.jacobi(A)
for solver in os.environ.get("PROBE_SOLVERS", "bicgstab").split(","):
    r = P.solve(P.solver_id(solver), A, prob.b, M, P.SolverOptions(tol=1e-8, max_iter=int(os.environ.get("PROBE_MAXIT", "20"))))
    print(solver, r.report.iterations, r.report.device_time)
