"""Synthetic 3-D FEM cavity: P1 tetrahedra on a box,
the input family the north star's configs name ("car-compartment-like cavity
mesh", K - omega^2 M + i omega C) beside the reference's 2-D FD cavity.

Beyond the reference (its helmholtz.cpp is a 2-D 5-point FD grid), so parity
is pinned by FEM self-checks and by solution uniqueness:
  * K 1 = 0 (constant fields have no gradient), sum(M) = volume,
    sum(C) = beta x absorbing area (tests/test_fem3d.py);
  * the device solve of A(omega) against the oracle solve of the same CSR at
    tight tolerance (tests/test_gpu_fem3d.py).

Mesh: Lx x Ly x Lz box, nx x ny x nz hexahedra, each split into the 6 Kuhn
tetrahedra along the main diagonal (conforming), vertices numbered
i + (nx+1) (j + (ny+1) k).  Operators (per element e, P1 basis phi):
  K_e = c^2 vol grad(phi) grad(phi)^T      stiffness
  M_e = vol / 20 (1 + delta_ij)            mass
  C_e = c beta area / 12 (1 + delta_ij)    absorbing-wall (impedance) damping on
                                           the faces listed in `absorbing`
A(omega) = K - omega^2 M + i omega C on one CSR pattern (the union of the
three); the device re-evaluates it per frequency (cvk_fem_set_omega).
Source: b = M f with a smooth Gaussian f centred near one corner (real).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .cavac import CsrMatrix, Device

P = C.c_void_p

# the 6 Kuhn tetrahedra of the unit cube (corners as bit masks x=1, y=2, z=4)
_KUHN = np.array([[0, 1, 3, 7], [0, 1, 5, 7], [0, 2, 3, 7], [0, 2, 6, 7], [0, 4, 5, 7], [0, 4, 6, 7]], np.int64)
_FACES = ("x0", "x1", "y0", "y1", "z0", "z1")


@dataclass
class FemCavity:
    nx: int
    ny: int
    nz: int
    lx: float
    ly: float
    lz: float
    c: float
    beta: float
    rp: np.ndarray
    ci: np.ndarray
    K: np.ndarray      # real, on the CSR pattern
    M: np.ndarray
    Cd: np.ndarray
    b: np.ndarray      # complex rhs
    volume: float
    absorbing_area: float

    @property
    def n(self) -> int:
        return len(self.rp) - 1

    def values(self, omega: float) -> np.ndarray:
        """Host A(omega) = K - omega^2 M + i omega C, the device's rounding
        (re = K - (omega*omega) M, im = omega C)."""
        om2 = omega * omega
        v = np.empty(len(self.K), np.complex128)
        v.real = self.K - om2 * self.M
        v.imag = omega * self.Cd
        return v

    def matrix(self, omega: float) -> CsrMatrix:
        return CsrMatrix(self.n, self.n, self.rp, self.ci, self.values(omega))

    def coords(self) -> np.ndarray:
        """Vertex coordinates (n, 3) in DOF order (for geometric partitioning)."""
        return _vertices(self.nx, self.ny, self.nz, self.lx, self.ly, self.lz)


def _vertices(nx, ny, nz, lx, ly, lz):
    i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    idx = (i + (nx + 1) * (j + (ny + 1) * k)).ravel()
    xyz = np.zeros(((nx + 1) * (ny + 1) * (nz + 1), 3))
    xyz[idx, 0] = (i * lx / nx).ravel()
    xyz[idx, 1] = (j * ly / ny).ravel()
    xyz[idx, 2] = (k * lz / nz).ravel()
    return xyz


def _tets(nx, ny, nz):
    i, j, k = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    corners = []
    for m in range(8):
        dx, dy, dz = m & 1, (m >> 1) & 1, (m >> 2) & 1
        corners.append((i + dx) + (nx + 1) * ((j + dy) + (ny + 1) * (k + dz)))
    corners = np.stack(corners, axis=1)  # (ncells, 8)
    return corners[:, _KUHN].reshape(-1, 4)  # (6 ncells, 4)


def _boundary_triangles(nx, ny, nz, face):
    """Triangles of one box face (2 per boundary quad, consistent with the Kuhn split)."""
    def vid(i, j, k):
        return i + (nx + 1) * (j + (ny + 1) * k)
    if face[0] == "x":
        a, b_ = np.meshgrid(np.arange(ny), np.arange(nz), indexing="ij")
        i = 0 if face == "x0" else nx
        q = [vid(i, a, b_), vid(i, a + 1, b_), vid(i, a + 1, b_ + 1), vid(i, a, b_ + 1)]
    elif face[0] == "y":
        a, b_ = np.meshgrid(np.arange(nx), np.arange(nz), indexing="ij")
        j = 0 if face == "y0" else ny
        q = [vid(a, j, b_), vid(a + 1, j, b_), vid(a + 1, j, b_ + 1), vid(a, j, b_ + 1)]
    else:
        a, b_ = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
        k = 0 if face == "z0" else nz
        q = [vid(a, b_, k), vid(a + 1, b_, k), vid(a + 1, b_ + 1, k), vid(a, b_ + 1, k)]
    q = [x.ravel() for x in q]
    return np.concatenate([np.stack([q[0], q[1], q[2]], 1), np.stack([q[0], q[2], q[3]], 1)])


def build_cavity(N: int, lx: float = 2.4, ly: float = 1.2, lz: float = 1.2, c: float = 340.0, beta: float = 0.01,
                 absorbing=("y1",), source=(0.3, 0.3, 0.3), width: float = 0.15,
                 shape: Optional[tuple] = None) -> FemCavity:
    """The survey's 2N x N x N box of hexes: (2N+1)(N+1)^2
    DOF -- N=29 -> 53,100 (config 1), N=79 -> 1,017,600 (config 2), N=135 ->
    5.0M, N=215 -> 20.1M.  shape=(nx, ny, nz) overrides."""
    nx, ny, nz = shape if shape is not None else (2 * N, N, N)
    xyz = _vertices(nx, ny, nz, lx, ly, lz)
    n = len(xyz)
    T = _tets(nx, ny, nz)
    X = xyz[T]                                   # (ne, 4, 3)
    D = X[:, 1:, :] - X[:, :1, :]                # edge matrix rows
    det = np.linalg.det(D)
    vol = np.abs(det) / 6.0
    # grad(phi_1..3) = inv(D) columns; grad(phi_0) = -sum
    Dinv = np.linalg.inv(D)                      # (ne, 3, 3): grad phi_{k+1} = Dinv[:, :, k]
    G = np.concatenate([-Dinv.sum(axis=2, keepdims=True), Dinv], axis=2)  # (ne, 3, 4)
    Ke = (c * c) * vol[:, None, None] * np.einsum("eai,eaj->eij", G, G)
    Me = (vol / 20.0)[:, None, None] * (np.ones((4, 4)) + np.eye(4))[None]
    rows = np.repeat(T, 4, axis=1).ravel()
    cols = np.tile(T, (1, 4)).ravel()
    # absorbing faces
    tri = [_boundary_triangles(nx, ny, nz, f) for f in absorbing]
    area_tot = 0.0
    if tri:
        Tb = np.concatenate(tri)
        Xb = xyz[Tb]
        area = 0.5 * np.linalg.norm(np.cross(Xb[:, 1] - Xb[:, 0], Xb[:, 2] - Xb[:, 0]), axis=1)
        area_tot = float(area.sum())
        Ce = (c * beta * area / 12.0)[:, None, None] * (np.ones((3, 3)) + np.eye(3))[None]
        brow = np.repeat(Tb, 3, axis=1).ravel()
        bcol = np.tile(Tb, (1, 3)).ravel()
    else:
        Ce = np.zeros((0, 3, 3))
        brow = bcol = np.zeros(0, np.int64)
    # CSR pattern = union; duplicates summed (order of summation: np.add.at)
    key = np.concatenate([rows, brow]) * n + np.concatenate([cols, bcol])
    ukey, inv = np.unique(key, return_inverse=True)
    nk = len(rows)
    K = np.zeros(len(ukey))
    M = np.zeros(len(ukey))
    Cd = np.zeros(len(ukey))
    np.add.at(K, inv[:nk], Ke.ravel())
    np.add.at(M, inv[:nk], Me.ravel())
    if len(brow):
        np.add.at(Cd, inv[nk:], Ce.ravel())
    r = ukey // n
    ci = ukey % n
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp)
    # source: b = M f
    d2 = ((xyz - np.asarray(source)) ** 2).sum(axis=1)
    f = np.exp(-d2 / (2 * width * width))
    Mf = np.zeros(n)
    np.add.at(Mf, r, M * f[ci])
    return FemCavity(nx, ny, nz, lx, ly, lz, c, beta, rp, ci.astype(np.int64), K, M, Cd,
                     Mf.astype(np.complex128), float(vol.sum()), area_tot)


def _bind(L):
    if getattr(L, "_fem_bound", False):
        return
    L.cvk_fem_create.argtypes = [P, P, P, P, C.POINTER(P)]
    L.cvk_fem_create.restype = C.c_int
    L.cvk_fem_set_omega.argtypes = [P, C.c_double]
    L.cvk_fem_set_omega.restype = C.c_int
    L.cvk_fem_free.argtypes = [P]
    L.cvk_fem_free.restype = C.c_int
    L._fem_bound = True


class FemOperator:
    """K, M, C resident on the device on A's pattern; set_omega rewrites A's
    values (and a Jacobi refresh) without any host traffic."""

    def __init__(self, cav: FemCavity, dev: Optional[Device] = None, omega: float = 0.0):
        L = _lib.load()
        _bind(L)
        from .sweep import _bind as _sbind
        _sbind(L)
        self.L, self.cav = L, cav
        self.A = cav.matrix(omega)
        self.hA = self.A.device(dev or Device.default())
        h = P()
        p = lambda a: np.ascontiguousarray(a, np.float64).ctypes.data_as(P)  # noqa: E731
        self._keep = [np.ascontiguousarray(a, np.float64) for a in (cav.K, cav.M, cav.Cd)]
        _lib.check(L.cvk_fem_create(self.hA, p(self._keep[0]), p(self._keep[1]), p(self._keep[2]), C.byref(h)))
        self.h = h
        self.hM = None

    def set_omega(self, omega: float):
        _lib.check(self.L.cvk_fem_set_omega(self.h, omega))
        if self.hM is None:
            hm = P()
            _lib.check(self.L.cvk_precond_jacobi(self.hA, None, C.byref(hm)))
            self.hM = hm
        else:
            _lib.check(self.L.cvk_precond_jacobi_refresh(self.hM, self.hA))

    def values(self) -> np.ndarray:
        y = np.zeros(len(self.cav.K), np.complex128)
        _lib.check(self.L.cvk_csr_get_values(self.hA, y.ctypes.data_as(P)))
        return y

    def close(self):
        if self.h:
            self.L.cvk_fem_free(self.h)
            self.h = None
        if self.hM is not None:
            self.L.cvk_precond_free(self.hM)
            self.hM = None


def fem_frequency_sweep(cav: FemCavity, freqs_hz, solver="bicgstab", opts=None, mode=None, keep_solutions=False):
    """The sweep driver of sweep.py on the FEM operator (K, M, C resident)."""
    from .cavac import SolverOptions, _dev_mode, solver_id
    from .sweep import SweepRow, SweepTable
    import time
    op = FemOperator(cav)
    opts = opts or SolverOptions()
    table = SweepTable()
    x = np.zeros(cav.n, np.complex128)
    b = np.ascontiguousarray(cav.b)
    try:
        for f in freqs_hz:
            t0 = time.perf_counter()
            omega = 2.0 * math.pi * float(f)
            op.set_omega(omega)
            o = _lib.CvkOpts(opts.tol, opts.max_iter, opts.l, opts.m, 0, _dev_mode(mode))
            rep = _lib.CvkReport()
            _lib.check(op.L.cvk_solve(Device.default().handle, int(solver_id(solver)), op.hA, op.hM,
                                      C.byref(o), b.ctypes.data_as(P), x.ctypes.data_as(P), C.byref(rep)))
            table.rows.append(SweepRow(solver, float(f), omega, cav.n, int(rep.iterations), bool(rep.converged),
                                       rep.final_relres, rep.true_relres,
                                       op.L.cvk_breakdown_name(rep.breakdown).decode(), rep.device_time_s,
                                       time.perf_counter() - t0))
            if keep_solutions:
                table.solutions[float(f)] = x.copy()
    finally:
        op.close()
    return table
