"""DST-diagonalised Schur-complement preconditioner on the GPU
(schur.py of the reference).

After the sine transform in time, mode k carries H_k = mu_k M + tau_ref A_ref
with mu_k = 2 sin((2k-1) pi / 4N) (schur.py:21-24, 41-47); one inverse
application is  DST^T, per-mode V-cycle / A_ref / V-cycle scaled by
2 tau_ref / N, DST  (schur.py:62-76).  On the GPU every mode's solves run in
the same batched V-cycle launches (csrc/mg.cu) and both transforms are the
batched FFT kernel (csrc/dst.cu).
"""

from __future__ import annotations

import numpy as np

from ._device import gpu_problem
from ._native import as_buffer, empty_like_kind, ptr_of
from .dst import DstPlan
from .errors import InputError
from .spatial import MgHierarchy, _check_mg_options, build_mg_hierarchy


def frequency_weights(N: int) -> np.ndarray:
    """mu_k = 2 sin((2k-1) pi / (4N)), k = 1..N (schur.py:21-24)."""
    k = np.arange(1, N + 1)
    return 2.0 * np.sin((2 * k - 1) * np.pi / (4 * N))


class SchurPreconditioner:
    """Approximate Schur-complement inverse H~^{-1} (schur.py:27-97)."""

    def __init__(self, spec, solver_kind: str = "mg", hierarchy: MgHierarchy | None = None,
                 cycles: int = 1, smooth_steps: int = 1, damping: float | None = None,
                 device=None):
        if solver_kind != "mg":
            raise InputError(f"solver kind {solver_kind!r} is not on the GPU path; use 'mg'")
        if hierarchy is None:
            raise InputError("mg solvers need a grid hierarchy")
        _check_mg_options(cycles, smooth_steps, damping)
        self.N = spec.N
        self.dim = spec.dim
        self.tau_ref = spec.tau_ref
        self.a_ref = spec.a_ref
        self.mu = frequency_weights(self.N)
        self.plan = DstPlan(self.N)
        self.solver_kind = solver_kind
        self.hierarchy = hierarchy
        self.cycles, self.smooth_steps = int(cycles), int(smooth_steps)
        self._gp = gpu_problem(spec, device)
        self._gp.set_htilde(hierarchy, self._gp.default_damping() if damping is None else damping,
                            self.mu, self.cycles, self.smooth_steps)

    def apply_inverse(self, r):
        """One preconditioner action (schur.py:62-76)."""
        shape = (self.N, self.dim)
        ptr, keep = as_buffer(r, shape)
        out = empty_like_kind(keep, shape)
        self._gp.ctx.call("pint_htilde_inv", ptr, ptr_of(out))
        return out

    def apply(self, u):
        raise InputError("forward application requires direct (exact) solvers")


def build_schur_preconditioner(spec, solver_kind: str = "mg", vcycles: int = 1,
                               smooth_steps: int = 1, jacobi_sweeps: int = 2,
                               device=None) -> SchurPreconditioner:
    """Builder tying the solver options to the problem mesh (schur.py:100-118)."""
    if solver_kind != "mg":
        raise InputError(f"solver kind {solver_kind!r} is not on the GPU path; use 'mg'")
    meta = getattr(spec, "meta", {}) or {}
    if "space" not in meta:
        raise InputError("mg solvers need mesh metadata on the problem")
    hierarchy = build_mg_hierarchy(meta["space"], meta["mesh"])
    return SchurPreconditioner(spec, "mg", hierarchy=hierarchy, cycles=vcycles,
                               smooth_steps=smooth_steps, device=device)
