"""Per-problem device state shared by TimeGlobalSystem, BlockDiagSolver and
SchurPreconditioner.

The reference's three duck-typed objects each hold their own
numpy/scipy data; on the GPU they share one libpint context per ProblemSpec
so that ``uzawa_solve(system, atilde, htilde, cfg)`` runs with all state
resident in HBM.  The context is created on first use and cached on the
spec object.
"""

from __future__ import annotations

import math

import numpy as np

from ._native import MG_ATILDE, MG_HTILDE, Context
from .errors import InputError
from .linalg import grid_stencil, grid_stencil3
from .spatial import DEFAULT_DAMPING, MgHierarchy, galerkin_tables


def _grid_side(spec):
    """(dims, m) of the structured interior grid of a problem."""
    meta = getattr(spec, "meta", {}) or {}
    space = meta.get("space", "2d")
    if space not in ("2d", "3d"):
        raise InputError(f"the GPU path implements the 2d and 3d problems (got space={space!r})")
    dims = 2 if space == "2d" else 3
    mesh = meta.get("mesh")
    m = int(round(spec.dim ** (1.0 / dims)))
    if m ** dims != spec.dim or (mesh is not None and int(mesh) - 1 != m):
        raise InputError("spatial dimension is not a structured grid")
    return dims, m


def proportional_scales(spec):
    """c_n * tau_n when every A_n is a known multiple of A_1, else None
    (TimeGlobalSystem._proportional_scales, operators.py:41-49)."""
    base = spec.stiffness[0]
    s = np.empty(spec.N)
    for k, a in enumerate(spec.stiffness):
        r = a.proportionality(base)
        if r is None:
            return None
        s[k] = r
    return s * spec.grid.steps


class HostProblem:
    """Host-side arrays of one ProblemSpec that the C ABI consumes: stencils,
    step sizes, stiffness scales and the multigrid tables.  Pure numpy/scipy
    (setup); accepts the reference's ProblemSpec as well as ours."""

    def __init__(self, spec):
        self.spec = spec
        self.dims, self.m = _grid_side(spec)
        self.N = spec.N
        self.n = spec.dim
        m = self.m
        grid_stencil = self._stencil
        self.steps = np.ascontiguousarray(spec.grid.steps, dtype=np.float64)
        self.mass_st = grid_stencil(spec.mass, m)
        scales = proportional_scales(spec)
        if scales is not None:
            a_st = grid_stencil(spec.stiffness[0], m)[None, :]
            a_sid = np.zeros(self.N, dtype=np.int32)
            a_scale = scales
        else:
            ids: dict[int, int] = {}
            sets = []
            a_sid = np.empty(self.N, dtype=np.int32)
            for k, a in enumerate(spec.stiffness):
                if id(a) not in ids:
                    ids[id(a)] = len(sets)
                    sets.append(a)
                a_sid[k] = ids[id(a)]
            a_st = np.stack([grid_stencil(a, m) for a in sets])
            a_scale = self.steps.copy()
        self.scales = scales
        self.a_st = np.ascontiguousarray(a_st)
        self.a_sid = a_sid
        self.a_scale = np.ascontiguousarray(a_scale, dtype=np.float64)
        self.aref_st = grid_stencil(spec.a_ref, m)

    def _stencil(self, mat, m):
        return grid_stencil(mat, m) if self.dims == 2 else grid_stencil3(mat, m)

    def default_damping(self):
        return DEFAULT_DAMPING["2d" if self.dims == 2 else "3d"]

    def atilde_tables(self, hierarchy: MgHierarchy, damping: float):
        """Per-step hierarchies, one per distinct A_n object (solvers.py:134-140)."""
        ids: dict[int, int] = {}
        ops = []
        sid = np.empty(self.N, dtype=np.int32)
        for k, a in enumerate(self.spec.stiffness):
            if id(a) not in ids:
                ids[id(a)] = len(ops)
                ops.append(a)
            sid[k] = ids[id(a)]
        st = np.stack([self._stencil(a, self.m) for a in ops])
        return galerkin_tables(st, hierarchy, damping), sid

    def htilde_tables(self, hierarchy: MgHierarchy, damping: float, mu: np.ndarray):
        """H_k = mu_k M + tau_ref A_ref (schur.py:41-47): the coefficient of
        add_matrices(mu_k, M, 1.0, A_ref.scaled(tau_ref)) at every stencil
        position is fl(mu_k m) + fl(1.0 * fl(tau_ref a))."""
        ta = 1.0 * (float(self.spec.tau_ref) * self.aref_st)
        st = mu[:, None] * self.mass_st[None, :] + ta[None, :]
        return galerkin_tables(st, hierarchy, damping), np.arange(self.N, dtype=np.int32)


class GpuProblem(HostProblem):
    """Device copy of one ProblemSpec: stencils, steps, scales, MG sets."""

    def __init__(self, spec, device=None):
        super().__init__(spec)
        self.ctx = Context(device)
        self.ctx.call("pint_problem_set", self.dims, self.m, self.N, self.steps.ctypes.data,
                      self.mass_st.ctypes.data, self.a_st.shape[0], self.a_st.ctypes.data,
                      self.a_sid.ctypes.data, self.a_scale.ctypes.data,
                      self.aref_st.ctypes.data, float(spec.tau_ref))
        self.atilde_ready = False
        self.htilde_ready = False

    def set_atilde(self, hierarchy: MgHierarchy, damping: float):
        tab, sid = self.atilde_tables(hierarchy, damping)
        self._upload_set(MG_ATILDE, hierarchy, tab, sid)
        self.atilde_ready = True

    def set_htilde(self, hierarchy: MgHierarchy, damping: float, mu: np.ndarray):
        tab, sid = self.htilde_tables(hierarchy, damping, mu)
        self._upload_set(MG_HTILDE, hierarchy, tab, sid)
        self.htilde_ready = True

    def _upload_set(self, which, hierarchy, tables, sid):
        if hierarchy.cells[0] - 1 != self.m:
            raise InputError("hierarchy does not match the problem mesh")
        lm = np.asarray(hierarchy.level_m, dtype=np.int32)
        tab = np.ascontiguousarray(tables, dtype=np.float64)
        sid = np.ascontiguousarray(sid, dtype=np.int32)
        self.ctx.call("pint_mg_set", which, len(lm), lm.ctypes.data, tab.shape[1],
                      tab.ctypes.data, sid.ctypes.data)


def gpu_problem(spec, device=None) -> GpuProblem:
    gp = spec.__dict__.get("_pint_gpu")
    if gp is None:
        gp = GpuProblem(spec, device)
        spec.__dict__["_pint_gpu"] = gp
    return gp
