"""Schwarz DDM on RCB subdomains of the FEM cavity (csrc/cvk_asm.cu): sweeps,
device time and the error against a tight monodomain solve, per size and
subdomain count.  Writes profiles/r02_asm_probe.json.

    PROBE_N=10,29,79 PROBE_PARTS=2,4,8 python tools/asm_probe.py
"""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import fem3d as F  # noqa: E402
from paper_2112_00087_b200.ddm_fem import SubdomainSchwarz  # noqa: E402
from paper_2112_00087_b200.rowblock import rcb_partition  # noqa: E402

out = []
for N in [int(v) for v in os.environ.get("PROBE_N", "10,29").split(",")]:
    cav = F.build_cavity(N)
    om = 2 * math.pi * float(os.environ.get("PROBE_F", "100"))
    A = cav.matrix(om)
    M = P.jacobi(A)
    mono = P.tfqmr(A, cav.b, M, P.SolverOptions(tol=1e-12, max_iter=100000))
    bicg = P.bicgstab(A, cav.b, M, P.SolverOptions(tol=1e-8, max_iter=100000))
    for nparts in [int(v) for v in os.environ.get("PROBE_PARTS", "2,4,8").split(",")]:
        part = rcb_partition(cav.coords(), nparts)
        k = om / 340.0
        t = time.time()
        S = SubdomainSchwarz(A, part, complex(2.0, k), cav.lx / cav.nx, P.SolverOptions(tol=1e-10))
        setup = time.time() - t
        for m in (30, 0):
            r = S.solve(cav.b, tol=1e-8, max_outer=300 if m else 60, m=m)
            row = {"N": N, "dof": A.nrows, "parts": nparts, "outer": "fgmres(30)" if m else "fixed point",
                   "converged": r.report.converged, "sweeps": r.report.outer_iterations,
                   "device_s": r.report.device_time, "wall_s": r.report.wall_time, "setup_s": setup,
                   "last_sweep_inner_iterations": r.report.total_inner_iterations,
                   "rel_err_vs_monodomain": float(np.linalg.norm(r.x - mono.x) / np.linalg.norm(mono.x)),
                   "final_residual": r.report.interface_residual_history[-1] if r.report.interface_residual_history else None,
                   "monodomain_bicgstab_1e-8_s": bicg.report.device_time}
            out.append(row)
            print(json.dumps(row), flush=True)
        S.close()
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_asm_probe.json"), "w"), indent=1)
