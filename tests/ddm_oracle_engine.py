"""Oracle-backed rank engine for the multi-rank Schwarz host logic on CPU
(TEST INFRASTRUCTURE: the product engine is ddm_dist.DeviceRankEngine).

Implements the DeviceRankEngine contract for the strips [s_begin, s_end) with
the oracle's C restatement of build_local / the inner solvers
(oracle/cavac_oracle.c, schwarz.cpp:29-89, krylov.cpp) and the reference's
rhs / exchange / jump arithmetic (schwarz.cpp:160-220) in Python complex
floats with libgcc __divdc3 division -- so ranks on gloo reproduce the
single-process oracle schwarz_solve bit for bit."""
import ctypes as C

import numpy as np

from oracle import oracle as O
from paper_2112_00087_b200.ddm_dist import SweepOut
from paper_2112_00087_b200.helmholtz import cdiv, cmul

SOLVERS = {0: "bicgstab", 1: "bicgstab_l", 2: "tfqmr", 3: "gmres", 4: "cocg"}


def _local_system(problem, c0, c1, hl, hr, tp):
    L = O.lib()
    P = C.c_void_p
    L.orc_local_system.argtypes = [C.POINTER(O._Grid), C.c_double, C.c_int64, P, P, P, C.c_int64, C.c_int64,
                                   C.c_int, C.c_int, C.c_double, C.c_double, C.c_double, C.c_double, P, P, P, P, P]
    L.orc_local_system.restype = C.c_int64
    g = problem.grid
    og = O.build_grid(g.width, g.height, g.h, 0.0, 1.0, g.wall_admittance)
    og._g.nx, og._g.ny = g.nx, g.ny
    og._g.roof_begin, og._g.roof_end = g.roof_begin, g.roof_end
    A = problem.A
    rp, ci, v = A.row_offsets.astype(np.int64), A.col_indices.astype(np.int64), np.asarray(A.values)
    nl = (c1 - c0) * g.ny
    lrp = np.zeros(nl + 1, np.int64)
    lci = np.zeros(6 * nl + 1, np.int64)
    lv = np.zeros(6 * nl + 1, np.complex128)
    dinv = np.zeros(nl, np.complex128)
    w = np.zeros(2, np.complex128)
    sl, sr = complex(tp.s_left), complex(tp.s_right)
    p = lambda a: a.ctypes.data_as(P)  # noqa: E731
    nnz = L.orc_local_system(C.byref(og._g), problem.c, A.nrows, p(rp), p(ci), p(v), c0, c1, int(hl), int(hr),
                             sl.real, sl.imag, sr.real, sr.imag, p(lrp), p(lci), p(lv), p(dinv), p(w))
    assert nnz >= 0, nnz
    return lrp, lci[:nnz].copy(), lv[:nnz].copy(), dinv, complex(w[0]), complex(w[1])


class OracleRankEngine:
    def __init__(self, problem, part, tp, inner, inner_solver, s_begin, s_end, mode=None):
        g = problem.grid
        self.ny, self.nx = g.ny, g.nx
        self.s0, self.s1, self.ns = s_begin, s_end, s_end - s_begin
        self.n_sub = part.n_sub
        self.cb = list(part.col_begin)
        self.b = np.asarray(problem.b, np.complex128)
        self.inner, self.solver = inner, SOLVERS[int(inner_solver)]
        self.loc = []
        for s in range(s_begin, s_end):
            self.loc.append(_local_system(problem, self.cb[s], self.cb[s + 1], s > 0, s + 1 < part.n_sub, tp))
        h = g.h
        sl, sr = complex(tp.s_left), complex(tp.s_right)
        self.a_l = complex(1.0 / h) + complex(0.5 * sl.real, 0.5 * sl.imag)
        self.b_l = complex(-1.0 / h) + complex(0.5 * sl.real, 0.5 * sl.imag)
        self.a_r = complex(1.0 / h) + complex(0.5 * sr.real, 0.5 * sr.imag)
        self.b_r = complex(-1.0 / h) + complex(0.5 * sr.real, 0.5 * sr.imag)
        ss = sl + sr
        self.half = complex(ss.real * 0.5, ss.imag * 0.5)
        ny, ns = self.ny, self.ns
        self.gl = np.zeros((ns + 1, ny), np.complex128)
        self.gr = np.zeros((ns + 1, ny), np.complex128)
        self.prev = np.zeros((ns + 1, ny, 2), np.complex128)
        self.u = [None] * ns

    def _exists(self, j):
        q = self.s0 + j
        return 0 < q < self.n_sub

    def sweep(self, g_in_left, g_in_right):
        ny, ns = self.ny, self.ns
        if g_in_left is not None and self._exists(0):
            self.gr[0] = g_in_left
        if g_in_right is not None and self._exists(ns):
            self.gl[ns] = g_in_right
        brk, iters = False, 0
        for j in range(ns):
            s = self.s0 + j
            c0, c1 = self.cb[s], self.cb[s + 1]
            w = c1 - c0
            lrp, lci, lv, dinv, wl, wr = self.loc[j]
            rhs = self.b.reshape(self.ny, self.nx)[:, c0:c1].copy()
            if self._exists(j):
                for iy in range(ny):
                    rhs[iy, 0] = rhs[iy, 0] + cmul(wl, self.gr[j, iy])
            if self._exists(j + 1):
                for iy in range(ny):
                    rhs[iy, w - 1] = rhs[iy, w - 1] + cmul(wr, self.gl[j + 1, iy])
            x, rep = O.solve(self.solver, lrp, lci, lv, rhs.ravel(), dinv=dinv, tol=self.inner.tol,
                             max_iter=self.inner.max_iter, l=self.inner.l, m=self.inner.m)
            brk = brk or bool(rep.breakdown)
            iters += rep.iterations
            self.u[j] = x.reshape(ny, w)
        out_l = np.zeros(ny, np.complex128)
        out_r = np.zeros(ny, np.complex128)
        terms = np.zeros((ns + 1, ny, 2))
        for j in range(ns + 1):
            if not self._exists(j):
                continue
            for iy in range(ny):
                glv, grv = self.gl[j, iy], self.gr[j, iy]
                if j >= 1:
                    el = self.u[j - 1][iy, -1]
                    gho = cdiv(glv - cmul(self.b_l, el), self.a_l)
                    grn = -glv + cmul(self.half, gho + el)
                    if j == ns:
                        out_r[iy] = grn
                    else:
                        self.gr[j, iy] = grn
                    d = el - self.prev[j, iy, 0]
                    terms[j, iy, 0] = d.real * d.real + d.imag * d.imag
                    self.prev[j, iy, 0] = el
                if j < ns:
                    er = self.u[j][iy, 0]
                    gho = cdiv(grv - cmul(self.b_r, er), self.a_r)
                    gln = -grv + cmul(self.half, gho + er)
                    if j == 0:
                        out_l[iy] = gln
                    else:
                        self.gl[j, iy] = gln
                    d = er - self.prev[j, iy, 1]
                    terms[j, iy, 1] = d.real * d.real + d.imag * d.imag
                    self.prev[j, iy, 1] = er
        return SweepOut(out_l, out_r, terms, brk, iters, 0.0)

    def solution(self):
        return np.concatenate(self.u, axis=1)

    def close(self):
        pass
