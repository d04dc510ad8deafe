"""8 BiCGSTAB+ILU(0) iterations on the 1M-DOF bench system (for ncu launch lists)."""
import math, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as Hm  # noqa: E402
g = Hm.build_grid(2.4, 1.2, 0.0017, 0.4, 0.65, 0.01)
pr = Hm.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
M = P.ilu0(pr.A, int(sys.argv[1]) if len(sys.argv) > 1 else 3)
r = P.solve(P.SolverId.BiCGStab, pr.A, pr.b, M, P.SolverOptions(tol=1e-30, max_iter=8)).report
print(r.iterations, r.device_time)
