"""Per-iteration time of the phased BiCGSTAB / tfQMR at 1M DOF under launcher
knobs (grid cap, PDL) -- CUDA-event device time of fixed-iteration solves."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import helmholtz as H

h = float(os.environ.get("PROBE_H", "0.0017"))
g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A = prob.A
M = P.jacobi(A)
maxit = int(os.environ.get("PROBE_MAXIT", "400"))
n, nnz = A.nrows, A.nnz()
iter_bytes = 40 * nnz + 344 * n
configs = [c for c in os.environ.get("PROBE_CONFIGS", "default").split(";")]
for solver in os.environ.get("PROBE_SOLVERS", "bicgstab").split(","):
    for cfg in configs:
        saved = dict(os.environ)
        if cfg != "default":
            for kv in cfg.split(","):
                k, v = kv.split("=")
                os.environ[k] = v
        sid = P.solver_id(solver)
        opts = P.SolverOptions(tol=1e-30, max_iter=maxit)
        P.solve(sid, A, prob.b, M, opts)  # warm (graph capture)
        ts = []
        for _ in range(3):
            r = P.solve(sid, A, prob.b, M, opts)
            ts.append(r.report.device_time)
        t = min(ts)
        it = r.report.iterations
        print(f"{solver:9s} {cfg:40s} iters {it:5d} dev {t*1e3:8.3f} ms  "
              f"{t/it*1e6:7.1f} us/it  {iter_bytes/(t/it)/1e9:7.1f} GB/s", flush=True)
        os.environ.clear()
        os.environ.update(saved)
