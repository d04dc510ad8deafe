"""Where the end-to-end time of a reference-style call goes (GPU box):
upload of A, Jacobi, solve (host b / x), free -- timed through the C ABI on
the bench system, each step repeated."""
import ctypes as C
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2112_00087_b200 as P  # noqa: E402
from paper_2112_00087_b200 import _lib, helmholtz as H  # noqa: E402

g = H.build_grid(2.4, 1.2, 0.0017, 0.4, 0.65, 0.01)
p = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A = p.A
L = _lib.load()
dev = P.Device.default()
rp = np.ascontiguousarray(A.row_offsets, np.uint64)
ci = np.ascontiguousarray(A.col_indices, np.uint64)
v = np.ascontiguousarray(A.values)
b = np.ascontiguousarray(p.b)
x = np.zeros_like(b)
d = P.jacobi(A).inv_diag
ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
opts = _lib.CvkOpts(1e-8, 20000, 8, 30, 0, _lib.MODE_FAST, 0, 0)
for rep in range(4):
    t = [time.perf_counter()]
    h = C.c_void_p()
    _lib.check(L.cvk_csr_upload(dev.handle, A.nrows, A.ncols, len(v), ptr(rp), ptr(ci), ptr(v), C.byref(h)))
    t.append(time.perf_counter())
    m = C.c_void_p()
    _lib.check(L.cvk_precond_jacobi(h, ptr(d), C.byref(m)))
    t.append(time.perf_counter())
    r = _lib.CvkReport()
    _lib.check(L.cvk_solve(dev.handle, 0, h, m, C.byref(opts), ptr(b), ptr(x), C.byref(r)))
    t.append(time.perf_counter())
    L.cvk_precond_free(m)
    L.cvk_csr_free(h)
    t.append(time.perf_counter())
    dt = np.diff(t) * 1e3
    print(f"rep {rep}: upload {dt[0]:.1f} ms, jacobi {dt[1]:.1f} ms, solve {dt[2]:.1f} ms "
          f"(device {r.device_time_s * 1e3:.1f} ms), free {dt[3]:.1f} ms", flush=True)
