"""Per-iteration device time of the row-block BiCGSTAB (csrc/cvk_rowblock.cu)
with n blocks on one device, against the single-device phase kernels, on the
config-2 cavity (h = 0.0017, 994,755 DOF), fixed iteration count."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import helmholtz as H  # noqa: E402
from paper_2112_00087_b200.rowblock import solve_row_blocks  # noqa: E402

h = float(os.environ.get("PROBE_H", "0.0017"))
it = int(os.environ.get("PROBE_MAXIT", "200"))
g = H.build_grid(2.4, 1.2, h, 0.4, 0.65, 0.01 + 0j)
p = H.assemble(g, 2 * np.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A, b = p.A, np.asarray(p.b, np.complex128)
M = P.jacobi(A)
o = P.SolverOptions(tol=1e-30, max_iter=it)
for _ in range(2):
    r = P.solve(P.SolverId.BiCGStab, A, b, M, o)
print(f"single-device  n={A.nrows} iters={r.report.iterations} {r.report.device_time / it * 1e6:8.1f} us/it "
      f"launches={r.report.kernel_launches}")
for nb in [int(v) for v in os.environ.get("PROBE_BLOCKS", "1,2,4,8").split(",")]:
    for _ in range(2):
        q = solve_row_blocks(A, b, M, o, n_blocks=nb)
    same = np.array_equal(q.x.view(np.uint64), r.x.view(np.uint64))
    print(f"row blocks {nb:2d}  iters={q.report.iterations} {q.report.device_time / it * 1e6:8.1f} us/it "
          f"launches={q.report.kernel_launches} bitwise={same}")
