"""Run the unmodified reference (oracle/_ref, ExecMode::Parallel, all host
cores) to convergence on the bench system (h=0.0017, 994,755 DOF, admittance
0.01, 100 Hz, BiCGSTAB + Jacobi, tol 1e-8), the system built by the oracle's
restatement of build_grid/assemble (bitwise the reference's).  Validates the
bench's bounded CPU sample x iteration count (REF_ITERS) on the host it runs
on.  This container (8 threads): 6952 iterations, 524.5 s.  Writes
profiles/r02_ref_full_solve.json."""
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402

g = O.build_grid(2.4, 1.2, 0.0017, 0.4, 0.65, 0.01)
rp, ci, v, b = O.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size, np.complex128))
t = time.time()
sample = int(os.environ.get("REF_SAMPLE_ITERS", "40"))
_, rs = O.ref_solve("bicgstab", rp, ci, v, b, tol=1e-8, max_iter=sample, parallel=True)
t_sample = time.time() - t
t = time.time()
x, rep = O.ref_solve("bicgstab", rp, ci, v, b, tol=1e-8, max_iter=20000, parallel=True)
wall = time.time() - t
out = {"iterations": rep.iterations, "converged": rep.converged, "final_relres": rep.final_relres,
       "true_relres": rep.true_relres, "wall_s": wall, "threads": int(O.ref().ref_omp_threads()),
       "sample_iterations": sample, "sample_wall_s": t_sample,
       "extrapolated_s": t_sample / sample * rep.iterations,
       "host": os.uname().nodename}
print(json.dumps(out), flush=True)
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_ref_full_solve.json"), "w"), indent=1)
