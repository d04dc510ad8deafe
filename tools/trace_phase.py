"""Phase-kernel timeline from a CVK_TRACE build (tools/variant_build.sh trace -DCVK_TRACE):
    CVK_LIB_PATH=_variants/trace/libcavac_b200.so python tools/trace_phase.py
Per BiCGSTAB iteration: for k_bi_a_s / k_bi_b_s / k_bi_c the first CTA entry,
median / max 'main loop done', max 'partial published', the last CTA's fold
end, and the gap to the next kernel's first entry (all in microseconds)."""
import ctypes as C
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2112_00087_b200 as P
from paper_2112_00087_b200 import _lib
from paper_2112_00087_b200 import helmholtz as H

KT, IT, CTA = 4, 16, 1024
g = H.build_grid(2.4, 1.2, float(os.environ.get("PROBE_H", "0.0017")), 0.4, 0.65, 0.01)
prob = H.assemble(g, 2 * math.pi * 100.0, 340.0, np.ones(g.roof_size(), np.complex128))
A = prob.A
M = P.jacobi(A)
maxit = 40
P.bicgstab(A, prob.b, M, P.SolverOptions(tol=1e-30, max_iter=maxit))
r = P.bicgstab(A, prob.b, M, P.SolverOptions(tol=1e-30, max_iter=maxit))
L = _lib.load()
L.cvk_trace_read.restype = C.c_int
buf = np.zeros(KT * IT * CTA * 4 + KT * CTA * 4, np.uint64)
got = L.cvk_trace_read(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))
assert got > 0, "not a CVK_TRACE build"
t = buf[:KT * IT * CTA * 4].reshape(KT, IT, CTA, 4).astype(np.float64)
sp = buf[KT * IT * CTA * 4:].reshape(KT, CTA, 4).astype(np.float64)
names = {1: "k_bi_a_s", 2: "k_bi_b_s", 0: "k_bi_c"}
order = [1, 2, 0]
rows = []
for it in range(maxit - 12, maxit):
    for k in order:
        blk = t[k, it % IT]
        ent = blk[:, 0]
        used = ent > 0
        if not used.any():
            continue
        e = ent[used]
        l1 = blk[used, 1]
        l2 = blk[used, 2]
        f = blk[used, 3]
        f = f[f > 0]
        rows.append((it, names[k], e.min(), e.max(), np.median(l1), l1.max(), l2.max(), f.max() if len(f) else np.nan,
                     int(used.sum())))
t0 = rows[0][2]
print(f"{'it':>3} {'kernel':9} {'first_in':>9} {'last_in':>8} {'loop_med':>8} {'loop_max':>8} {'pub_max':>8} "
      f"{'fold':>8} {'span':>7} {'gap_prev':>8} ctas")
prev_end = None
for (it, nm, emin, emax, l1m, l1x, l2x, fe, nc) in rows:
    gap = (emin - prev_end) / 1e3 if prev_end is not None else float("nan")
    print(f"{it:3d} {nm:9} {(emin - t0) / 1e3:9.2f} {(emax - emin) / 1e3:8.2f} {(l1m - emin) / 1e3:8.2f} "
          f"{(l1x - emin) / 1e3:8.2f} {(l2x - emin) / 1e3:8.2f} {(fe - emin) / 1e3:8.2f} {(fe - emin) / 1e3:7.2f} "
          f"{gap:8.2f} {nc}")
    prev_end = fe

# per-CTA main-loop time distribution (last recorded iteration)
it = maxit - 1
for k in order:
    blk = t[k, it % IT]
    used = blk[:, 0] > 0
    d = (blk[used, 1] - blk[used, 0]) / 1e3
    ids = np.nonzero(used)[0]
    slow = ids[np.argsort(-d)[:8]]
    print(f"{names[k]:9} loop us: p10 {np.percentile(d, 10):.2f} p50 {np.median(d):.2f} "
          f"p90 {np.percentile(d, 90):.2f} max {d.max():.2f}; slowest CTAs {list(slow)}")

# streamed-kernel pipeline balance (last launch of each kernel, clock cycles per CTA)
for k in (1, 2):
    blk = sp[k, :148]
    print(f"{names[k]:9} producer waits for free stage {np.median(blk[:, 0]) / 1965:.2f} us, consumer waits for "
          f"full stage {np.median(blk[:, 1]) / 1965:.2f} us, consumer body {np.median(blk[:, 2]) / 1965:.2f} us, "
          f"chunks/group {np.median(blk[:, 3]):.0f} (medians over CTAs)")
