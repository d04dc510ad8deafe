"""One BiCGSTAB(8) run on the 1M-DOF bench system for profiling the step
kernel (ncu wraps this script): PROBE_CYCLES cycles, FAST mode."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as H  # noqa: E402

g = H.build_grid(2.4, 1.2, float(os.environ.get("PROBE_H", "0.0017")), 0.4, 0.65, 0.01)
p = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
M = P.jacobi(p.A)
cyc = int(os.environ.get("PROBE_CYCLES", "3"))
for _ in range(int(os.environ.get("PROBE_REPS", "1"))):
    r = P.bicgstab_l(p.A, p.b, M, P.SolverOptions(tol=1e-30, l=8, max_iter=cyc))
    print("cycles", r.report.iterations, "device ms", r.report.device_time * 1e3,
          "ms/cycle", r.report.device_time * 1e3 / max(1, r.report.iterations), flush=True)
