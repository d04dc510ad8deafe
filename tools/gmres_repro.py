"""GMRES(m) phase kernels on a REF-2D cavity: a short run for debugging
(compute-sanitizer) -- GMRES_H (mesh width), GMRES_IT (Arnoldi steps)."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as H  # noqa: E402

h = float(os.environ.get("GMRES_H", "0.0017"))
g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
M = P.jacobi(prob.A)
with P.path_options(gmres_tiles=int(os.environ.get("GMRES_TILES", "1"))):
    r = P.gmres(prob.A, prob.b, M, P.SolverOptions(tol=1e-30, m=int(os.environ.get("GMRES_M", "30")),
                                                    max_iter=int(os.environ.get("GMRES_IT", "40"))))
print(prob.A.nrows, r.report)
