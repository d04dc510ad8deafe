"""ILU(0)-preconditioned BiCGSTAB vs the Jacobi product path on the bench
system (config 2, 1M DOF) and a smaller cavity: iterations, device time,
time per iteration.  Usage: python tools/probe_ilu0.py [h ...]"""
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as Hm  # noqa: E402


def run(h, f=100.0, tol=1e-8):
    if str(h).startswith("fem:"):  # 3-D P1 FEM cavity, N cells per edge (fem3d.py)
        from paper_2112_00087_b200 import fem3d as F
        cav = F.build_cavity(int(str(h)[4:]))
        A, b = cav.matrix(2 * math.pi * f), cav.b
    else:
        h = float(h)
        g = Hm.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
        pr = Hm.assemble(g, 2 * math.pi * f, 340.0, np.ones(g.roof_size(), np.complex128))
        A, b = pr.A, pr.b
    opts = P.SolverOptions(tol=tol, max_iter=200000)
    out = {"h": h, "dof": A.nrows, "nnz": A.nnz()}
    for name, mk in [("jacobi", lambda: P.jacobi(A))] + [
            (f"ilu0_s{s}", (lambda s=s: P.ilu0(A, s))) for s in (1, 2, 3, 4)]:
        M = mk()
        P.solve(P.SolverId.BiCGStab, A, b, M, P.SolverOptions(tol=tol, max_iter=5))  # warm-up
        r = P.solve(P.SolverId.BiCGStab, A, b, M, opts).report
        out[name] = {"iters": r.iterations, "converged": r.converged, "true_relres": r.true_relres,
                     "device_s": r.device_time, "wall_s": r.wall_time,
                     "us_per_iter": 1e6 * r.device_time / max(1, r.iterations),
                     "launches": r.kernel_launches}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for h in (sys.argv[1:] or ["0.008", "0.0017"]):
        run(h)
