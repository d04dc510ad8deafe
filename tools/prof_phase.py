"""ncu target: standalone SpMV + a short phased BiCGSTAB at 1M DOF."""
import ctypes as C, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import helmholtz as H, _lib
import torch
g = H.build_grid(2.4, 1.2, 0.0017, 0.4, 0.65, 0.01)
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A = prob.A
x = torch.randn(A.nrows, dtype=torch.complex128, device="cuda"); y = torch.empty_like(x)
out = C.c_double()
_lib.check(_lib.load().cvk_spmv_bench(A.device(), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 0, 3, C.byref(out)))
M = P.jacobi(A)
r = P.bicgstab(A, prob.b, M, P.SolverOptions(tol=1e-8, max_iter=int(os.environ.get("PROBE_MAXIT", "16"))))
print("iters", r.report.iterations, "dev", r.report.device_time, "launches", r.report.kernel_launches)
