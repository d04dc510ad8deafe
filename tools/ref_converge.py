"""Run the unmodified reference (oracle/_ref, ExecMode::Parallel) to convergence
on the bench system (h=0.0017, 994,755 DOF, admittance 0.01, 100 Hz, BiCGSTAB +
Jacobi, tol 1e-8).  Measured here (8-core Xeon): 6952 iterations, final relres
1.0609e-9, true relres 1.0604e-9, 688 s.  bench.py uses the iteration count
to extrapolate its bounded CPU sample (REF_ITERS)."""
import sys, math, time
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import oracle as O
from paper_2112_00087_b200 import helmholtz as Hm
g = Hm.build_grid(2.4, 1.2, 0.0017, 0.4, 0.65, 0.01)
prob = Hm.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A = prob.A
t = time.time()
x, rep = O.ref_solve("bicgstab", A.row_offsets.astype(np.int64), A.col_indices.astype(np.int64), A.values, prob.b, tol=1e-8, max_iter=20000, parallel=True)
print("iters", rep.iterations, "conv", rep.converged, "final", rep.final_relres, "true", rep.true_relres, "wall", time.time() - t, flush=True)
