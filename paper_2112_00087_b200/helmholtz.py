"""Matrix-assembly input of the solve path: the reference's 2-D cavity grid and
5-point Helmholtz assembly (helmholtz.hpp:18-83, helmholtz.cpp:14-168),
vectorised with numpy and rounded exactly as the reference (values are
bitwise identical -- tests/test_helmholtz.py checks against the golden
system.mtx).  Host-side setup: it runs once per system, the device assembles
per-frequency values for sweeps (sweep.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .cavac import CsrMatrix, InvalidArgument


def cdiv(a: complex, b: complex) -> complex:
    """libgcc __divdc3 rounding in Python floats (see csrc/cvk_complex.h)."""
    ar, ai, c, d = a.real, a.imag, b.real, b.imag
    if abs(c) < abs(d):
        ratio = c / d
        denom = (c * ratio) + d
        return complex(((ar * ratio) + ai) / denom, ((ai * ratio) - ar) / denom)
    ratio = d / c
    denom = (d * ratio) + c
    return complex(((ai * ratio) + ar) / denom, (ai - (ar * ratio)) / denom)


def cmul(a: complex, b: complex) -> complex:
    return complex(a.real * b.real - a.imag * b.imag, a.real * b.imag + a.imag * b.real)


def _round_half_away(v: float) -> float:
    return math.copysign(math.floor(abs(v) + 0.5), v)


@dataclass
class CavityGrid:
    """helmholtz.hpp:18-39: interior nodes only, node = iy * nx + ix."""
    width: float = 2.4
    height: float = 1.2
    h: float = 0.05
    nx: int = 0
    ny: int = 0
    roof_begin: int = 0
    roof_end: int = 0
    wall_admittance: complex = 0j

    def size(self) -> int:
        return self.nx * self.ny

    def node(self, ix: int, iy: int) -> int:
        return iy * self.nx + ix

    def x_of(self, ix):
        return (ix + 1) * self.h

    def y_of(self, iy):
        return (iy + 1) * self.h

    def roof_size(self) -> int:
        return self.roof_end - self.roof_begin


@dataclass
class HelmholtzProblem:
    grid: CavityGrid
    omega: float
    c: float
    dirichlet: np.ndarray
    A: CsrMatrix
    b: np.ndarray


def _interior_count(extent: float, h: float, what: str) -> int:
    rounded = _round_half_away(extent / h)
    if rounded < 4.0:
        raise InvalidArgument(f"build_grid: {what} too coarse, fewer than 3 interior nodes")
    return int(rounded) - 1


def build_grid(width: float, height: float, h: float, roof_fraction_start: float,
               roof_fraction_end: float, wall_admittance: complex = 0j) -> CavityGrid:
    """helmholtz.cpp:25-57."""
    if width <= 0 or height <= 0 or h <= 0:
        raise InvalidArgument("build_grid: nonpositive dimension")
    if not (0.0 <= roof_fraction_start < roof_fraction_end <= 1.0):
        raise InvalidArgument("build_grid: bad roof fractions")
    g = CavityGrid(width, height, h, _interior_count(width, h, "width"),
                   _interior_count(height, h, "height"), 0, 0, complex(wall_admittance))
    x0, x1 = roof_fraction_start * width, roof_fraction_end * width
    xs = (np.arange(g.nx, dtype=np.float64) + 1.0) * h
    inside = np.nonzero((xs >= x0 - 1e-9) & (xs <= x1 + 1e-9))[0]
    if len(inside) == 0:
        raise InvalidArgument("build_grid: empty roof span")
    g.roof_begin, g.roof_end = int(inside[0]), int(inside[-1]) + 1
    return g


def wall_weight(grid: CavityGrid, omega: float) -> complex:
    """1 for rigid walls, 1/(1 + i omega h beta) with admittance (helmholtz.cpp:68-73)."""
    if grid.wall_admittance == 0:
        return complex(1.0, 0.0)
    return cdiv(complex(1.0, 0.0), complex(1.0, 0.0) + cmul(complex(0.0, omega * grid.h), grid.wall_admittance))


def _nodes(grid: CavityGrid, rows):
    """(node, ix, iy) of the grid rows [r0, r1) (all rows when rows is None)."""
    r0, r1 = (0, grid.size()) if rows is None else (int(rows[0]), int(rows[1]))
    if not 0 <= r0 <= r1 <= grid.size():
        raise InvalidArgument("rows must satisfy 0 <= r0 <= r1 <= grid size")
    node = np.arange(r0, r1, dtype=np.int64)
    return node, node % grid.nx, node // grid.nx


def pattern(grid: CavityGrid, rows=None):
    """CSR pattern of the 5-point operator: per row below, left, diag, right,
    above (the stable (row, col) order csr_from_triplets produces).  Returns
    (row_offsets, col_indices, slot) with slot = 0..4 naming each entry.
    rows = (r0, r1): only those rows (row offsets from 0, global columns) --
    a rank's block of a distributed solve, assembled without the rest."""
    nx, ny = grid.nx, grid.ny
    node, ix, iy = _nodes(grid, rows)
    has = np.stack([iy > 0, ix > 0, np.ones_like(ix, bool), ix + 1 < nx, iy + 1 < ny], axis=1)
    off = np.array([-nx, -1, 0, 1, nx], dtype=np.int64)
    cols = node[:, None] + off[None, :]
    counts = has.sum(axis=1)
    rp = np.zeros(len(node) + 1, np.int64)
    rp[1:] = np.cumsum(counts)
    ci = cols[has]
    slot = np.broadcast_to(np.arange(5), has.shape)[has]
    return rp, ci, slot, has


def values(grid: CavityGrid, omega: float, c: float, pat=None, rows=None) -> np.ndarray:
    """helmholtz.cpp:78-113 values on the fixed pattern (diag 4k^2 - omega^2,
    minus k^2 w per missing wall neighbour in the order left, right, below,
    above; off-diagonals -k^2).  Each row's values depend only on its grid
    position, so rows=(r0, r1) gives bitwise those rows of the global values."""
    rp, ci, slot, has = pat if pat is not None else pattern(grid, rows)
    nx, ny = grid.nx, grid.ny
    k2 = c * c / (grid.h * grid.h)
    ww = wall_weight(grid, omega)
    kw_re, kw_im = k2 * ww.real, k2 * ww.imag
    _, ix, iy = _nodes(grid, rows)
    roof = (iy + 1 == ny) & (ix >= grid.roof_begin) & (ix < grid.roof_end)
    dre = np.full(len(ix), 4.0 * k2 - omega * omega)
    dim = np.zeros(len(ix))
    for cond in (ix == 0, ix + 1 == nx, iy == 0, (iy + 1 == ny) & ~roof):
        dre = np.where(cond, dre - kw_re, dre)
        dim = np.where(cond, dim - kw_im, dim)
    v = np.empty(len(ci), np.complex128)
    v.real = -k2
    v.imag = 0.0
    dpos = rp[:-1] + has[:, 0] + has[:, 1]  # diagonal entry index per row
    v.real[dpos] = dre
    v.imag[dpos] = dim
    return v


def rhs(grid: CavityGrid, c: float, dirichlet, rows=None) -> np.ndarray:
    """b: k^2 * dirichlet on the top row under the roof span (helmholtz.cpp:104-107)."""
    k2 = c * c / (grid.h * grid.h)
    d = np.asarray(dirichlet, np.complex128)
    r0, r1 = (0, grid.size()) if rows is None else (int(rows[0]), int(rows[1]))
    b = np.zeros(r1 - r0, np.complex128)
    nodes = (grid.ny - 1) * grid.nx + np.arange(grid.roof_begin, grid.roof_end)
    keep = (nodes >= r0) & (nodes < r1)
    b.real[nodes[keep] - r0] = 0.0 + k2 * d.real[keep]
    b.imag[nodes[keep] - r0] = 0.0 + k2 * d.imag[keep]
    return b


def assemble(grid: CavityGrid, omega: float, c: float, dirichlet) -> HelmholtzProblem:
    """helmholtz.cpp:59-115."""
    dirichlet = np.asarray(dirichlet, np.complex128)
    if len(dirichlet) != grid.roof_size():
        raise InvalidArgument("assemble: dirichlet length does not match roof span")
    pat = pattern(grid)
    v = values(grid, omega, c, pat)
    A = CsrMatrix(grid.size(), grid.size(), pat[0], pat[1], v)
    return HelmholtzProblem(grid, omega, c, dirichlet, A, rhs(grid, c, dirichlet))


def assemble_rows(grid: CavityGrid, omega: float, c: float, dirichlet, r0: int, r1: int):
    """Rows [r0, r1) of assemble(): (row_offsets from 0, global columns,
    values, rhs), bitwise the same rows of the global system, built without
    the other rows (a rank's share of a distributed solve)."""
    dirichlet = np.asarray(dirichlet, np.complex128)
    if len(dirichlet) != grid.roof_size():
        raise InvalidArgument("assemble: dirichlet length does not match roof span")
    pat = pattern(grid, (r0, r1))
    return pat[0], pat[1], values(grid, omega, c, pat, (r0, r1)), rhs(grid, c, dirichlet, (r0, r1))


@dataclass
class ManufacturedProblem:
    problem: HelmholtzProblem
    exact: np.ndarray = field(default=None)


def manufactured_problem(grid: CavityGrid, m: int, n: int, omega: float, c: float) -> ManufacturedProblem:
    """helmholtz.cpp:117-168: exact sin(m pi x/W) sin(n pi y/H), zero Dirichlet."""
    if m == 0 or n == 0:
        raise InvalidArgument("manufactured_problem: mode must be >= 1")
    W, H = grid.width, grid.height
    pi = math.pi
    lam = pi * pi * ((m * m) / (W * W) + (n * n) / (H * H))
    factor = -omega * omega + c * c * lam
    if abs(factor) < 1e-10 * c * c * lam:
        raise InvalidArgument(f"manufactured_problem: omega is resonant for mode ({m}, {n})")
    k2 = c * c / (grid.h * grid.h)
    nx, ny = grid.nx, grid.ny
    ix = np.tile(np.arange(nx), ny)
    iy = np.repeat(np.arange(ny), nx)
    x = (ix + 1) * grid.h
    y = (iy + 1) * grid.h
    psi = np.sin(m * pi * x / W) * np.sin(n * pi * y / H)
    rp, ci, slot, has = pattern(grid)
    v = np.empty(len(ci), np.complex128)
    v.real = -k2
    v.imag = 0.0
    dpos = rp[:-1] + has[:, 0] + has[:, 1]
    v.real[dpos] = 4.0 * k2 - omega * omega
    A = CsrMatrix(grid.size(), grid.size(), rp, ci, v)
    b = (factor * psi).astype(np.complex128)
    prob = HelmholtzProblem(grid, omega, c, np.zeros(0, np.complex128), A, b)
    return ManufacturedProblem(prob, psi.astype(np.complex128))
