"""Host (numpy) row-block engine for the multi-rank BiCGSTAB host logic on CPU
(TEST INFRASTRUCTURE: the product engine is rowblock.RowBlockEngine).

Implements the engine contract of rowblock.solve_distributed (local / post /
done / result over `send` / `recv` exchange slots) with the same phase
schedule, exchange layout and scalar recurrence as csrc/cvk_rowblock.cu
(krylov.cpp:57-138).  Rank partial sums are exact-residual pairs
(hi = fsum(terms), lo = fsum(terms - hi)) folded across ranks with fsum, the
host analogue of the device's double-double reductions: the reduced scalars
do not depend on the row split, so runs on 1, 2 or 3 gloo ranks agree bit
for bit."""
import math

import numpy as np

from paper_2112_00087_b200.helmholtz import cdiv, cmul
from paper_2112_00087_b200.rowblock import PH_A, PH_B, PH_C, PH_INIT, PH_T, PH_X

HDR = 16


def vmul(a, b):
    """elementwise (ac - bd, ad + bc) -- the device's complex multiply"""
    a = np.asarray(a, np.complex128)
    b = np.asarray(b, np.complex128)
    out = np.empty(np.broadcast(a, b).shape, np.complex128)
    out.real = a.real * b.real - a.imag * b.imag
    out.imag = a.real * b.imag + a.imag * b.real
    return out


def vconjmul(x, y):
    """conj(x) * y term by term (dot_hermitian, numkit.cpp:113-119)"""
    return vmul(np.conj(x), y)


def _pair(terms):
    t = [float(v) for v in terms]
    hi = math.fsum(t)
    return hi, math.fsum(t + [-hi])


class NumpyRowBlockEngine:
    def __init__(self, plan, b_own, inv_diag_own, opts):
        self.plan = plan
        n, nh = plan.n_own, len(plan.halo_cols)
        self.n, self.nh = n, nh
        self.b = np.asarray(b_own, np.complex128)
        self.d = None if inv_diag_own is None else np.asarray(inv_diag_own, np.complex128)
        rp = plan.row_offsets
        lens = np.diff(rp)
        self.width = int(lens.max()) if n else 0
        self.cols = np.zeros((n, max(1, self.width)), np.int64)
        self.vals = np.zeros((n, max(1, self.width)), np.complex128)
        self.mask = np.zeros((n, max(1, self.width)), bool)
        for k in range(self.width):
            m = lens > k
            idx = rp[:-1][m] + k
            self.cols[m, k] = plan.col_local[idx]
            self.vals[m, k] = plan.values[idx]
            self.mask[m, k] = True
        z = lambda: np.zeros(n + nh, np.complex128)  # noqa: E731
        self.x, self.r, self.sh, self.s, self.t = z(), z(), z(), z(), z()
        self.p, self.v = [z(), z()], [z(), z()]
        self.slot = HDR + 4 * max(1, plan.max_send)
        self.send = np.zeros(self.slot, np.float64)
        self.recv = np.zeros(self.slot * plan.n_ranks, np.float64)
        self.tol, self.max_iter = opts.tol, max(0, opts.max_iter)
        self.record = bool(opts.record_history)
        self.hist = []
        self.done_ = False
        self.conv = False
        self.brk = None
        self.iters = 0
        self.final = 0.0
        self.true = 0.0
        self.skip_true = False
        self.cur = 0
        self.first = True
        self.it = 0

    # ---- kernels
    def _spmv(self, xv):
        acc = np.zeros(self.n, np.complex128)
        for k in range(self.width):
            m = self.mask[:, k]
            acc[m] = acc[m] + vmul(self.vals[m, k], xv[self.cols[m, k]])
        return acc

    def _prec(self, y):
        return y if self.d is None else vmul(self.d, y)

    def _totals(self, *sums):
        for k, z in enumerate(sums):
            hx, lx = _pair(np.real(z))
            hy, ly = _pair(np.imag(z))
            self.send[4 * k:4 * k + 4] = (hx, hy, lx, ly)

    def _fold(self, k):
        sl = self.recv.reshape(self.plan.n_ranks, self.slot)[:, 4 * k:4 * k + 4]
        return complex(math.fsum(list(sl[:, 0]) + list(sl[:, 2])), math.fsum(list(sl[:, 1]) + list(sl[:, 3])))

    def _vecs(self, ph):
        if ph in (PH_INIT, PH_C):
            return [self.r]
        if ph == PH_A:
            return [self.p[1 - self.cur], self.v[1 - self.cur]]
        if ph == PH_X:
            return [self.x]
        return []

    def local(self, ph):
        n = self.n
        if ph not in (PH_INIT, PH_X, PH_T) and self.done_:
            return
        if ph == PH_INIT:
            r = self._prec(self.b)
            self.r[:n], self.sh[:n], self.x[:n] = r, r, 0
            self._totals(r.real * r.real + r.imag * r.imag, vconjmul(r, r))
        elif ph == PH_A:
            pc, vc = self.p[self.cur], self.v[self.cur]
            pfull = self.r.copy() if self.first else vmul(self.beta, pc + vmul(-self.omega, vc)) + self.r
            vn = self._prec(self._spmv(pfull))
            self.p[1 - self.cur][:n] = pfull[:n]
            self.v[1 - self.cur][:n] = vn
            self._totals(vconjmul(self.sh[:n], vn))
        elif ph == PH_B:
            vn = self.v[1 - self.cur]
            sfull = self.r + vmul(-self.alpha, vn)
            t = self._prec(self._spmv(sfull))
            s = sfull[:n]
            self.s[:n], self.t[:n] = s, t
            self.x[:n] = self.x[:n] + vmul(self.alpha, self.p[1 - self.cur][:n])
            self._totals(s.real * s.real + s.imag * s.imag, vconjmul(t, t), vconjmul(t, s))
        elif ph == PH_C:
            s, t = self.s[:n], self.t[:n]
            self.x[:n] = self.x[:n] + vmul(self.omega, s)
            r = s + vmul(-self.omega, t)
            self.r[:n] = r
            self._totals(r.real * r.real + r.imag * r.imag, vconjmul(self.sh[:n], r))
        elif ph == PH_T:
            if self.skip_true:
                self._totals(np.zeros(0), np.zeros(0))
            else:
                dlt = self.b - self._spmv(self.x)
                self._totals(self.b.real ** 2 + self.b.imag ** 2, dlt.real ** 2 + dlt.imag ** 2)
        vs = self._vecs(ph)
        out = self.send[HDR:].view(np.complex128)
        for k, row in enumerate(self.plan.send_rows):
            for j, vec in enumerate(vs):
                out[k * len(vs) + j] = vec[row]

    def post(self, ph):
        if ph not in (PH_X, PH_T) and self.done_:
            return
        vs = self._vecs(ph)
        ms = max(1, self.plan.max_send)
        slots = self.recv.reshape(self.plan.n_ranks, self.slot)
        for h, src in enumerate(self.plan.halo_src):
            q, k = divmod(int(src), ms)
            data = slots[q, HDR:].view(np.complex128)
            for j, vec in enumerate(vs):
                vec[self.n + h] = data[k * len(vs) + j]
        if ph == PH_INIT:
            bn = math.sqrt(self._fold(0).real)
            self.bnorm = bn
            if bn == 0.0:
                self.done_, self.conv, self.iters, self.skip_true = True, True, 0, True
                return
            self.brk_thr = 1e-30 * bn * bn
            self.rho_new = self._fold(1)
            self.rho = self.alpha = self.omega = 1 + 0j
            self.it, self.first, self.cur = 1, True, 0
            self._top()
        elif ph == PH_A:
            sv = self._fold(0)
            if abs(sv) < self.brk_thr:
                self.done_, self.brk, self.iters = True, "stagnation in <shadow, v>", self.it - 1
                return
            self.alpha = cdiv(self.rho, sv)
        elif ph == PH_B:
            ss, tt, ts = self._fold(0), self._fold(1), self._fold(2)
            rel = math.sqrt(ss.real) / self.bnorm
            if rel <= self.tol:
                self.done_, self.conv, self.iters, self.final = True, True, self.it, rel
                self._hist(rel)
                return
            if abs(tt) < self.brk_thr:
                self.done_, self.brk, self.iters = True, "omega breakdown", self.it
                return
            self.omega = cdiv(ts, tt)
        elif ph == PH_C:
            rn, shr = self._fold(0), self._fold(1)
            rel = math.sqrt(rn.real) / self.bnorm
            self.final, self.iters = rel, self.it
            self._hist(rel)
            if rel <= self.tol:
                self.done_, self.conv = True, True
                return
            self.rho_new = shr
            self.cur ^= 1
            self.first = False
            self.it += 1
            self._top()
        elif ph == PH_T and not self.skip_true:
            bn, rn = math.sqrt(self._fold(0).real), math.sqrt(self._fold(1).real)
            self.true = rn / bn if bn > 0 else rn

    def _hist(self, v):
        if self.record:
            self.hist.append(v)

    def _top(self):
        if self.it > self.max_iter:
            self.done_ = True
            return
        if abs(self.rho_new) < self.brk_thr:
            self.done_, self.brk, self.iters = True, "rho breakdown", self.it - 1
            return
        if not self.first:
            self.beta = cmul(cdiv(self.rho_new, self.rho), cdiv(self.alpha, self.omega))
        self.rho = self.rho_new

    def done(self):
        return self.done_

    def result(self):
        from paper_2112_00087_b200.cavac import SolveReport
        return self.x[:self.n].copy(), SolveReport(self.conv, self.iters, self.final, self.true, 0.0,
                                                   list(self.hist), self.brk)


def run_serial(A, b, inv_diag, opts):
    """The same engine on one block with recv = send (no torch.distributed)."""
    from paper_2112_00087_b200.rowblock import ITER_PHASES, ITERS_PER_POLL, plan_row_blocks
    e = NumpyRowBlockEngine(plan_row_blocks(A, 1)[0], b, inv_diag, opts)

    def phase(ph):
        e.local(ph)
        e.recv[:] = e.send
        e.post(ph)
    phase(PH_INIT)
    while not e.done():
        for _ in range(ITERS_PER_POLL):
            for ph in ITER_PHASES:
                phase(ph)
    phase(PH_X)
    phase(PH_T)
    return e.result()
