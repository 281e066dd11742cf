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

from ._native import MG_ATILDE, MG_EULER, MG_HTILDE, Context
from .errors import InputError
from .linalg import grid_fields, grid_stencil, grid_stencil3
from .problems import WeightedStiffness
from .spatial import DEFAULT_DAMPING, MgHierarchy, build_mg_hierarchy, galerkin_tables


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
    if isinstance(spec.stiffness, WeightedStiffness):
        return None
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
        self.field = self._field_mode(spec)
        scales = proportional_scales(spec)
        if self.field is not None:
            # per-point coefficients live in device fields; the stencil
            # arguments of pint_problem_set are placeholders
            a_st = np.zeros((1, self._st_size()))
            a_sid = np.zeros(self.N, dtype=np.int32)
            a_scale = self.steps.copy()
            scales = None
        elif scales is not None:
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
        self.aref_st = (np.zeros(self._st_size()) if self.field is not None
                        else grid_stencil(spec.a_ref, m))

    def _st_size(self):
        return 9 if self.dims == 2 else 27

    def _field_mode(self, spec):
        """None (translation-invariant stencils), "family" (WeightedStiffness,
        assembled on the GPU) or "explicit" (2D operators that are not
        translation invariant: compact per-point fields from the matrices)."""
        if isinstance(spec.stiffness, WeightedStiffness):
            if self.dims != 2:
                raise InputError("weighted stiffness families are 2D")
            return "family"
        if self.dims != 2:
            return None
        seen = set()
        for a in spec.stiffness:
            if id(a) in seen:
                continue
            seen.add(id(a))
            try:
                grid_stencil(a, self.m)
            except InputError as e:
                if "translation invariant" not in str(e):
                    raise
                return "explicit"
        try:
            grid_stencil(spec.a_ref, self.m)
        except InputError as e:
            if "translation invariant" not in str(e):
                raise
            return "explicit"
        return None

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


    def euler_tables(self, hierarchy: MgHierarchy, damping: float):
        """Operators M + tau_n A_n of the sequential implicit-Euler oracle
        (solvers.py:166-170), one set per distinct (A_n, tau_n); coefficient
        fl(1.0 m) + fl(tau_n a) as add_matrices(1.0, M, tau, A_n) forms it."""
        index: dict = {}
        sets = []
        sid = np.empty(self.N, dtype=np.int32)
        for k, (a, tau) in enumerate(zip(self.spec.stiffness, self.steps)):
            key = (id(a), float(tau))
            if key not in index:
                index[key] = len(sets)
                sets.append(1.0 * self.mass_st + float(tau) * self._stencil(a, self.m))
            sid[k] = index[key]
        return galerkin_tables(np.stack(sets), hierarchy, damping), sid


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
        if self.field is not None:
            self._upload_fields()

    _FIELD_CHUNK = 32

    def _upload_fields(self):
        """Per-point stiffness of every step and of A_ref into HBM."""
        spec, ctx = self.spec, self.ctx
        if self.field == "family" and spec.stiffness.terms is not None:
            a, c = spec.stiffness.terms
            ctx.call("pint_field_separable", int(a.shape[0]), a.ctypes.data, c.ctypes.data)
        elif self.field == "family":
            fam = spec.stiffness
            for n0 in range(0, self.N, self._FIELD_CHUNK):
                n1 = min(self.N, n0 + self._FIELD_CHUNK)
                w = np.ascontiguousarray(fam.cell_weights(n0, n1))
                ctx.call("pint_field_assemble", n0, n1 - n0, w.ctypes.data)
        else:
            cache: dict[int, np.ndarray] = {}
            for n, a in enumerate(spec.stiffness):
                f = cache.get(id(a))
                if f is None:
                    f = np.ascontiguousarray(grid_fields(a, self.m))
                    cache = {id(a): f}
                ctx.call("pint_field_set", n, 1, f.ctypes.data)
        step = getattr(spec.a_ref, "_family_step", None)
        if self.field == "family" and step is not None and spec.stiffness[step] is spec.a_ref:
            ctx.call("pint_field_aref", int(step), None)
        else:
            f = np.ascontiguousarray(grid_fields(spec.a_ref, self.m))
            ctx.call("pint_field_aref", 0, f.ctypes.data)

    def set_atilde(self, hierarchy: MgHierarchy, damping: float, cycles: int = 1,
                   smooth_steps: int = 1):
        if self.field is not None:
            self._set_field(MG_ATILDE, hierarchy, damping, None)
        else:
            tab, sid = self.atilde_tables(hierarchy, damping)
            self._upload_set(MG_ATILDE, hierarchy, tab, sid)
        self.ctx.call("pint_mg_set_options", MG_ATILDE, int(cycles), int(smooth_steps))
        self.atilde_ready = True

    def set_htilde(self, hierarchy: MgHierarchy, damping: float, mu: np.ndarray, cycles: int = 1,
                   smooth_steps: int = 1):
        if self.field is not None:
            self._set_field(MG_HTILDE, hierarchy, damping,
                            np.ascontiguousarray(mu, dtype=np.float64))
        else:
            tab, sid = self.htilde_tables(hierarchy, damping, mu)
            self._upload_set(MG_HTILDE, hierarchy, tab, sid)
        self.ctx.call("pint_mg_set_options", MG_HTILDE, int(cycles), int(smooth_steps))
        self.htilde_ready = True

    def ensure_exact(self):
        """Multigrid sets the device-side exact solves precondition with: the
        A~ set (operators A_n; configured with the default hierarchy unless a
        BlockDiagSolver already did) and the EULER set (M + tau_n A_n)."""
        if self.field is not None:
            raise InputError("exact solves are not built for per-point stiffness fields")
        if getattr(self, "exact_ready", False):
            return
        space = "2d" if self.dims == 2 else "3d"
        hier = build_mg_hierarchy(space, self.m + 1)
        damping = self.default_damping()
        if not self.atilde_ready:
            self.set_atilde(hier, damping)
        tab, sid = self.euler_tables(hier, damping)
        self._upload_set(MG_EULER, hier, tab, sid)
        self.exact_ready = True

    def _set_field(self, which, hierarchy, damping, mu):
        if hierarchy.cells[0] - 1 != self.m or hierarchy.space != "2d":
            raise InputError("hierarchy does not match the problem mesh")
        lm = np.asarray(hierarchy.level_m, dtype=np.int32)
        self.ctx.call("pint_mg_set_field", which, len(lm), lm.ctypes.data, float(damping),
                      None if mu is None else mu.ctypes.data)

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
