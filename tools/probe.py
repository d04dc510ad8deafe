"""Scratch GPU probe: SpMV group-width sweep and a 1M-DOF solve."""
import math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes as C
import numpy as np
import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import helmholtz as H, _lib

def spmv_gbs(A, reps=50):
    import torch
    n = A.nrows
    x = torch.randn(n, dtype=torch.complex128, device="cuda")
    y = torch.empty_like(x)
    out = C.c_double()
    _lib.check(_lib.load().cvk_spmv_bench(A.device(), C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()), 0, reps, C.byref(out)))
    byts = 20 * A.nnz() + 4 * (n + 1) + 32 * n
    return out.value, byts / out.value / 1e9

h = float(os.environ.get("PROBE_H", "0.0017"))
g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01)
t = time.time()
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
print(f"n={g.size()} nnz={prob.A.nnz()} assemble {time.time()-t:.2f}s", flush=True)
A = P.CsrMatrix(prob.A.nrows, prob.A.ncols, prob.A.row_offsets, prob.A.col_indices, prob.A.values)
tt, gbs = spmv_gbs(A)
print(f"spmv tiled: {tt*1e6:.1f} us  {gbs:.0f} GB/s", flush=True)
os.environ["CVK_SPMV_ROWS"] = "1"
for S in (1, 2, 4):
    os.environ["CVK_SPMV_GROUP"] = str(S)
    A = P.CsrMatrix(prob.A.nrows, prob.A.ncols, prob.A.row_offsets, prob.A.col_indices, prob.A.values)
    tt, gbs = spmv_gbs(A)
    print(f"spmv rows S={S}: {tt*1e6:.1f} us  {gbs:.0f} GB/s", flush=True)
del os.environ["CVK_SPMV_ROWS"]
for S in (int(s) for s in os.environ.get("PROBE_SOLVE_S", "4").split(",")):
    os.environ["CVK_SPMV_GROUP"] = str(S)
    A = P.CsrMatrix(prob.A.nrows, prob.A.ncols, prob.A.row_offsets, prob.A.col_indices, prob.A.values)
    M = P.jacobi(A)
    for solver in os.environ.get("PROBE_SOLVERS", "bicgstab").split(","):
        r = P.solve(P.solver_id(solver), A, prob.b, M, P.SolverOptions(tol=1e-8, max_iter=int(os.environ.get("PROBE_MAXIT", "3000"))))
        rep = r.report
        it = max(rep.iterations, 1)
        print(f"S={S} {solver}: it={rep.iterations} conv={rep.converged} relres={rep.final_relres:.2e} true={rep.true_relres:.2e} "
              f"dev={rep.device_time:.3f}s wall={rep.wall_time:.3f}s per-it={rep.device_time/it*1e6:.1f}us "
              f"GB/s(bicgstab model)={(40*A.nnz()+344*A.nrows)*it/rep.device_time/1e9:.0f}", flush=True)
