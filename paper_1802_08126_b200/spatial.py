"""Geometric multigrid: hierarchy, Galerkin stencil tables, GPU V-cycle.

Mirrors spatial.py of the reference (MgHierarchy / build_mg_hierarchy,
spatial.py:87-113; MgVCycleSolver, spatial.py:116-169; make_solver,
spatial.py:172-183).  The host builds, once, the per-level 9-point Galerkin
stencils P^T A P of every operator in a batch ("operator sets"); the CUDA
V-cycle (csrc/mg.cu) then runs one launch per level over all planes.

Galerkin stencils are computed with the reference's own sparse product,
``(P.T @ A) @ P`` in scipy (spatial.py:140), on a small probe grid (16 cells
per side) holding the same stencil.  Every coarse coefficient is a sum over
a fixed local neighbourhood whose relative index order is the same on any
grid size, so the probe reproduces the full-size product bit for bit
(tests/test_host.py checks this against the oracle's full hierarchies) at a
cost independent of the mesh, for thousands of per-mode operators at once.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import InputError
from .linalg import STENCIL_2D, STENCIL_3D, grid_stencil, grid_stencil3

_PROBE_CELLS = 16
_CHUNK = 256


def _prolongation_1d(coarse_cells: int) -> sp.csr_matrix:
    """Linear interpolation from coarse_cells-1 to 2*coarse_cells-1 interior
    nodes (spatial.py:75-84)."""
    nc = coarse_cells - 1
    j = np.arange(nc)
    rows = np.concatenate([2 * j + 1, 2 * j, 2 * j + 2])
    cols = np.concatenate([j, j, j])
    vals = np.concatenate([np.ones(nc), np.full(2 * nc, 0.5)])
    return sp.coo_matrix((vals, (rows, cols)), shape=(2 * coarse_cells - 1, nc)).tocsr()


@dataclass
class MgHierarchy:
    """Grid transfers shared by all operators on one mesh (spatial.py:87-97)."""

    space: str
    cells: list
    prolongations: list

    @property
    def levels(self) -> int:
        return len(self.cells)

    @property
    def level_m(self) -> list:
        return [c - 1 for c in self.cells]


def build_mg_hierarchy(space: str, fine_cells: int) -> MgHierarchy:
    """Halve the cell count down to 2 or 3 per side (spatial.py:100-113)."""
    if fine_cells < 4 or fine_cells & (fine_cells - 1):
        raise InputError("fine cell count must be a power of two, at least 4")
    cells = [fine_cells]
    while cells[-1] // 2 >= 2 and cells[-1] > 3:
        cells.append(cells[-1] // 2)
    if space not in ("1d", "2d", "3d"):
        raise InputError(f"unknown space {space!r}")
    pro = []
    for c in cells[1:]:
        p1 = _prolongation_1d(c)
        if space == "1d":
            pro.append(p1)
        elif space == "2d":
            pro.append(sp.kron(p1, p1).tocsr())
        else:  # EXTENSION: trilinear transfers for the 3D configs
            pro.append(sp.kron(sp.kron(p1, p1), p1).tocsr())
    return MgHierarchy(space=space, cells=cells, prolongations=pro)


# damped-Jacobi weights: 1D 2/3 and 2D 4/5 (spatial.py:136); 3D 6/7 (EXTENSION)
DEFAULT_DAMPING = {"1d": 2.0 / 3.0, "2d": 4.0 / 5.0, "3d": 6.0 / 7.0}


def _batch_stencil_matrix(st: np.ndarray, m: int) -> sp.csr_matrix:
    """Block-diagonal CSR of B translation-invariant stencils on m x m grids."""
    B = st.shape[0]
    n = m * m
    j, i = np.divmod(np.arange(n), m)
    rows, cols, vals = [], [], []
    for k, (dy, dx) in enumerate(STENCIL_2D):
        ok = (j + dy >= 0) & (j + dy < m) & (i + dx >= 0) & (i + dx < m)
        r = (j * m + i)[ok]
        c = ((j + dy) * m + (i + dx))[ok]
        off = (np.arange(B) * n)[:, None]
        rows.append((off + r[None, :]).ravel())
        cols.append((off + c[None, :]).ravel())
        vals.append(np.repeat(st[:, k], r.size))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(B * n, B * n)).tocsr()


def _galerkin_step(st: np.ndarray, fine_cells: int) -> np.ndarray:
    """Coarse 9-point stencils of P^T A P for a batch of fine stencils."""
    cf = min(fine_cells, _PROBE_CELLS)
    mf, cc = cf - 1, cf // 2
    mc = cc - 1
    p1 = _prolongation_1d(cc)
    P = sp.kron(p1, p1).tocsr()
    out = np.zeros((st.shape[0], 9))
    centre = (mc // 2) * mc + mc // 2
    for s0 in range(0, st.shape[0], _CHUNK):
        blk = st[s0:s0 + _CHUNK]
        B = blk.shape[0]
        A = _batch_stencil_matrix(blk, mf)
        Pb = sp.block_diag([P] * B, format="csr")
        C = (Pb.T @ A @ Pb).tocsr()
        base = np.arange(B) * (mc * mc) + centre
        cy, cx = divmod(centre, mc)
        for k, (dy, dx) in enumerate(STENCIL_2D):
            if 0 <= cy + dy < mc and 0 <= cx + dx < mc:
                out[s0:s0 + B, k] = np.asarray(C[base, base + dy * mc + dx]).ravel()
    return out


def _batch_stencil_matrix3(st: np.ndarray, m: int) -> sp.csr_matrix:
    B, n = st.shape[0], m ** 3
    z, rem = np.divmod(np.arange(n), m * m)
    y, x = np.divmod(rem, m)
    rows, cols, vals = [], [], []
    for k, (dz, dy, dx) in enumerate(STENCIL_3D):
        ok = ((z + dz >= 0) & (z + dz < m) & (y + dy >= 0) & (y + dy < m)
              & (x + dx >= 0) & (x + dx < m))
        r = np.arange(n)[ok]
        c = ((z[ok] + dz) * m + (y[ok] + dy)) * m + (x[ok] + dx)
        off = (np.arange(B) * n)[:, None]
        rows.append((off + r[None, :]).ravel())
        cols.append((off + c[None, :]).ravel())
        vals.append(np.repeat(st[:, k], r.size))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(B * n, B * n)).tocsr()


def _galerkin_step3(st: np.ndarray, fine_cells: int) -> np.ndarray:
    """3D analogue of _galerkin_step (probe grid of 8 cells per side)."""
    cf = min(fine_cells, 8)
    mf, cc = cf - 1, cf // 2
    mc = cc - 1
    p1 = _prolongation_1d(cc)
    P = sp.kron(sp.kron(p1, p1), p1).tocsr()
    out = np.zeros((st.shape[0], 27))
    cz = cy = cx = mc // 2
    centre = (cz * mc + cy) * mc + cx
    chunk = 32
    for s0 in range(0, st.shape[0], chunk):
        blk = st[s0:s0 + chunk]
        B = blk.shape[0]
        A = _batch_stencil_matrix3(blk, mf)
        Pb = sp.block_diag([P] * B, format="csr")
        C = (Pb.T @ A @ Pb).tocsr()
        base = np.arange(B) * (mc ** 3) + centre
        for k, (dz, dy, dx) in enumerate(STENCIL_3D):
            if 0 <= cz + dz < mc and 0 <= cy + dy < mc and 0 <= cx + dx < mc:
                out[s0:s0 + B, k] = np.asarray(C[base, base + (dz * mc + dy) * mc + dx]).ravel()
    return out


def galerkin_tables(fine_stencils: np.ndarray, hierarchy: MgHierarchy,
                    damping: float) -> np.ndarray:
    """Per-(level, set) table of 9 stencil coefficients + dinv, shape (L, S, 10).

    dinv = damping / diag exactly as spatial.py:142; the coarsest level's
    centre coefficient is the 1x1 operator solved directly (spatial.py:143).
    """
    if hierarchy.space not in ("2d", "3d"):
        raise InputError("the GPU multigrid supports the 2d and 3d hierarchies")
    S, step = (9, _galerkin_step) if hierarchy.space == "2d" else (27, _galerkin_step3)
    st = np.atleast_2d(np.asarray(fine_stencils, dtype=np.float64))
    L = hierarchy.levels
    tab = np.zeros((L, st.shape[0], S + 1))
    cur = st
    for lev in range(L):
        tab[lev, :, :S] = cur
        tab[lev, :, S] = damping / cur[:, S // 2]
        if lev + 1 < L:
            cur = step(cur, hierarchy.cells[lev])
    return tab


class SpatialSolver:
    """Approximate inverse of an SPD spatial operator (spatial.py:26-39)."""

    def apply(self, b):
        raise NotImplementedError


def _check_mg_options(cycles: int, smooth_steps: int, damping):
    """cycles / smooth_steps as in spatial.py:116-169.  (1, 1) -- every
    BASELINE config -- runs the fused band kernels; other values run the
    general kernels of csrc/mg_generic.cu (pint_mg_set_options)."""
    for name, v in (("cycles", cycles), ("smooth_steps", smooth_steps)):
        if int(v) != v or v < 1:
            raise InputError(f"{name} must be a positive integer")


class MgVCycleSolver(SpatialSolver):
    """One symmetric V-cycle on the GPU (spatial.py:116-169) for a single
    operator; accepts one vector (n,) or a batch (B, n)."""

    def __init__(self, target, hierarchy: MgHierarchy, cycles: int = 1,
                 smooth_steps: int = 1, damping: float | None = None, device=None):
        _check_mg_options(cycles, smooth_steps, damping)
        if hierarchy.space != "2d":
            raise InputError("the standalone GPU V-cycle supports the 2d hierarchy")
        if damping is None:
            damping = DEFAULT_DAMPING["2d"]
        self.target = target
        self.hierarchy = hierarchy
        self.cycles = cycles
        self.smooth_steps = smooth_steps
        self.damping = damping
        m = hierarchy.cells[0] - 1
        self._m = m
        self._tables = galerkin_tables(grid_stencil(target, m)[None, :], hierarchy, damping)
        self._device = device
        self._ctx = None
        self._cap = 0

    def level_stencil(self, level: int) -> np.ndarray:
        return self._tables[level, 0, :9].copy()

    def _ensure(self, batch: int):
        from ._native import MG_ATILDE, Context

        if self._ctx is None:
            self._ctx = Context(self._device)
        if batch <= self._cap:
            return
        ctx, m = self._ctx, self._m
        steps = np.ones(batch)
        zero9 = np.zeros(9)
        one = np.ones(batch)
        sid = np.zeros(batch, dtype=np.int32)
        ctx.call("pint_problem_set", 2, m, batch, steps.ctypes.data, zero9.ctypes.data, 1,
                 zero9.ctypes.data, sid.ctypes.data, one.ctypes.data, zero9.ctypes.data, 1.0)
        lm = np.asarray(self.hierarchy.level_m, dtype=np.int32)
        tab = np.ascontiguousarray(self._tables)
        ctx.call("pint_mg_set", MG_ATILDE, len(lm), lm.ctypes.data, 1, tab.ctypes.data,
                 sid.ctypes.data)
        ctx.call("pint_mg_set_options", MG_ATILDE, int(self.cycles), int(self.smooth_steps))
        self._cap = batch

    def apply(self, b):
        from ._native import MG_ATILDE, as_buffer, empty_like_kind, ptr_of

        single = np.ndim(b) == 1
        shape = (1, self._m ** 2) if single else (np.shape(b)[0], self._m ** 2)
        self._ensure(shape[0])
        ptr, keep = as_buffer(b if not single else (b[None, :] if hasattr(b, "shape") else b),
                              shape)
        out = empty_like_kind(keep, shape)
        self._ctx.call("pint_vcycle", MG_ATILDE, shape[0], ptr, ptr_of(out))
        return out[0] if single else out


def make_solver(target, kind: str, hierarchy: MgHierarchy | None = None, **opts):
    """Solver factory (spatial.py:172-183); the GPU path provides 'mg'."""
    if kind == "mg":
        if hierarchy is None:
            raise InputError("mg solver needs a grid hierarchy")
        return MgVCycleSolver(target, hierarchy, **opts)
    if kind in ("direct", "jacobi"):
        raise InputError(f"solver kind {kind!r} is not on the GPU path; use kind='mg'")
    raise InputError(f"unknown solver kind {kind!r}")
