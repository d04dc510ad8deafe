"""Phase boundaries of the persistent streamed BiCGSTAB (CVK_TRACE build):
    CVK_LIB_PATH=_variants/trace/libcavac_b200.so python tools/trace_streamk.py"""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import _lib
from paper_2112_00087_b200 import helmholtz as H

g = H.build_grid(2.4, 1.2, 0.0017, 0.4, 0.65, 0.01)
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A = prob.A
M = P.jacobi(A)
r = P.bicgstab(A, prob.b, M, P.SolverOptions(tol=1e-30, max_iter=40))
print("iters", r.report.iterations, "us/it", r.report.device_time / r.report.iterations * 1e6)
L = _lib.load()
buf = (C.c_ulonglong * 16)()
assert L.cvk_streamk_trace_read(buf) == 16
t = np.array(buf, dtype=np.float64).reshape(2, 8)
names = ["A stream", "A reduce", "B stream", "B reduce", "C elems", "C reduce"]
for cta in range(2):
    d = np.diff(t[cta, :7]) / 1e3
    print(f"CTA {cta}: " + ", ".join(f"{nm} {v:.2f}" for nm, v in zip(names, d)) + f" | total {d.sum():.2f} us")
