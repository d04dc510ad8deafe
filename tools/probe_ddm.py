"""Outer-sweep cost of the device Schwarz DDM (cvk_ddm.cu) on the config-3
cavity: REF-2D, n_sub strips on one GPU, s = 2 + ik (the acceptance default),
inner BiCGSTAB tol 1e-10; PROBE_OUTER sweeps, device time per sweep and inner
iterations per strip."""
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as H  # noqa: E402
from paper_2112_00087_b200 import schwarz as S  # noqa: E402

h = float(os.environ.get("PROBE_H", "0.00076"))
nsub = int(os.environ.get("PROBE_NSUB", "8"))
outer = int(os.environ.get("PROBE_OUTER", "3"))
f = float(os.environ.get("PROBE_F", "100"))
g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01 + 0j)
prob = H.assemble(g, 2 * math.pi * f, 340.0, np.ones(g.roof_size(), np.complex128))
part = S.partition(g, nsub)
k = prob.omega / prob.c
tp = S.TransmissionParams(complex(2.0, k), complex(2.0, k))
t0 = time.perf_counter()
r = S.schwarz_solve(prob, part, tp, P.SolverOptions(tol=1e-10, max_iter=20000), 1e-8, outer)
t1 = time.perf_counter()
rep = r.report
print(f"n={g.size()} nsub={nsub} outer={rep.outer_iterations} wall={t1 - t0:.2f}s "
      f"device={getattr(rep, 'device_time', float('nan')):.3f}s "
      f"inner_total_last={getattr(rep, 'total_inner_iterations', None)} "
      f"sub_its={[s.iterations for s in rep.per_subdomain_solves][:8]}")
