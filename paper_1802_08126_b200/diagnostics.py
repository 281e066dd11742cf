"""Diagnostic mode of the reference, for the GPU solvers.

The reference measures convergence against the exact time-stepping solution
in its discrete parabolic norm when ``UzawaConfig(diagnostics=True)`` or
``stopping="s_norm_error"`` is requested (solvers.py:201-244): that is how its
``bench.run_table2`` reproduces the paper's Table 2 iteration counts
(bench.py:111-139; acceptance criterion 2, pkg/tests/test_acceptance.py:49-94).
These quantities need exact sparse factorisations of the spatial operators,
which the reference computes with SuperLU on the host (linalg.py:150-177);
they are evaluated here the same way, on the host, from the same matrices and
in the same operation order:

* :class:`SpdFactor`        -- linalg.py:150-177 (symmetric-mode LU, no pivoting)
* :func:`sequential_euler_solve` -- solvers.py:158-174
* :class:`ExactNorms`       -- the diagnostic operators of TimeGlobalSystem,
  operators.py:51-71 (exact A_bd^{-1}), 113-139 (P, S), 141-183 (a-norm,
  jump form, dual term, S bilinear form and norm)

This is reproduction tooling around the GPU iteration, never part of it: the
Uzawa step itself stays on the device; in diagnostic mode the iterate u is
copied to the host once per iteration (the reference's own cost model there).
"""

from __future__ import annotations

import numpy as np
import scipy.sparse.linalg as spla

from .errors import DimensionMismatchError, NotSpdError
from .linalg import add_matrices


class SpdFactor:
    """Cached factorisation of an SPD sparse operator (linalg.py:150-177):
    SuperLU in symmetric mode without off-diagonal pivoting, so a
    non-positive pivot flags a non-SPD operator."""

    def __init__(self, mat):
        self.dim = mat.dim
        csc = mat.tocsr().tocsc()
        try:
            self._lu = spla.splu(csc, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                                 options={"SymmetricMode": True})
        except RuntimeError as exc:
            raise NotSpdError(f"factorization failed: {exc}") from exc
        if np.any(self._lu.U.diagonal() <= 0.0):
            raise NotSpdError("non-positive pivot: operator is not SPD")

    def solve(self, b: np.ndarray) -> np.ndarray:
        b = np.asarray(b, dtype=np.float64)
        if b.shape[0] != self.dim and b.ndim == 2 and b.shape[1] == self.dim:
            return self._lu.solve(b.T).T
        return self._lu.solve(b)


def sequential_euler_solve(spec) -> np.ndarray:
    """Forward implicit-Euler sweep with exact per-step solves (solvers.py:158-174):
    (M + tau_n A_n) u_n = M u_{n-1} + tau_n load_n, one factorisation per
    distinct (A_n, tau_n)."""
    factors: dict = {}
    u = np.empty((spec.N, spec.dim))
    prev = spec.u_init
    for n in range(spec.N):
        tau = spec.grid.steps[n]
        a_n = spec.stiffness[n]
        key = (id(a_n), tau)
        if key not in factors:
            factors[key] = SpdFactor(add_matrices(1.0, spec.mass, tau, a_n))
        u[n] = factors[key].solve(spec.mass.dot(prev) + tau * spec.load[n])
        prev = u[n]
    return u


def _proportional_scales(spec):
    """c_n tau_n when every A_n is a scaled copy of A_0 (operators.py:41-49)."""
    base = spec.stiffness[0]
    scales = np.empty(spec.N)
    for n, a_n in enumerate(spec.stiffness):
        s = a_n.proportionality(base)
        if s is None:
            return None
        scales[n] = s
    return scales * spec.grid.steps


class ExactNorms:
    """Exact per-step inverses and the error norms of the reference's
    diagnostic mode (operators.py:51-71, 113-183), host side."""

    def __init__(self, spec):
        self.spec = spec
        self._scales = _proportional_scales(spec)
        self._base_factor = None
        self._block_factors = None
        if self._scales is not None:
            self._base_factor = SpdFactor(spec.stiffness[0])
        else:
            self._block_factors = [SpdFactor(a.scaled(t)) if t != 1.0 else SpdFactor(a)
                                   for a, t in zip(spec.stiffness, spec.grid.steps)]

    def _check(self, u) -> np.ndarray:
        u = np.asarray(u, dtype=np.float64)
        if u.shape != (self.spec.N, self.spec.dim):
            raise DimensionMismatchError(
                f"expected block vector of shape {(self.spec.N, self.spec.dim)}, got {u.shape}")
        return u

    def apply_Abd(self, u) -> np.ndarray:
        """tau_n A_n u_n with the host CSR products (operators.py:92-99)."""
        u = self._check(u)
        if self._scales is not None:
            return self._scales[:, None] * self.spec.stiffness[0].dot(u.T).T
        steps = self.spec.grid.steps
        return np.stack([t * a.dot(x) for a, t, x in zip(self.spec.stiffness, steps, u)])

    def apply_Abd_inv(self, b) -> np.ndarray:
        b = self._check(b)
        if self._base_factor is not None:
            return self._base_factor.solve(b.T).T / self._scales[:, None]
        return np.stack([f.solve(bn) for f, bn in zip(self._block_factors, b)])

    def a_norm(self, u) -> float:
        u = self._check(u)
        return float(np.sqrt(max(np.sum(u * self.apply_Abd(u)), 0.0)))

    def jump_form(self, u, v) -> float:
        """Final-value plus temporal-jump mass form, u_0 = v_0 = 0 (operators.py:146-153)."""
        u, v = self._check(u), self._check(v)
        du = np.diff(u, axis=0, prepend=0.0)
        dv = np.diff(v, axis=0, prepend=0.0)
        m = self.spec.mass
        return float(u[-1] @ m.dot(v[-1]) + np.sum(du * m.dot(dv.T).T))

    def dual_term(self, u, v) -> float:
        """sum_n tau_n (d_t u, d_t v) in the per-step dual inner product (operators.py:155-172)."""
        steps = self.spec.grid.steps
        mdu = self.spec.mass.dot(np.diff(u, axis=0, prepend=0.0).T).T / steps[:, None]
        mdv = self.spec.mass.dot(np.diff(v, axis=0, prepend=0.0).T).T / steps[:, None]
        if self._base_factor is not None:
            sol = self._base_factor.solve(mdv.T).T / (self._scales / steps)[:, None]
        else:
            sol = np.stack([f.solve(x) * t for f, x, t in zip(self._block_factors, mdv, steps)])
        return float(np.sum(steps[:, None] * mdu * sol))

    def s_bilinear(self, u, v) -> float:
        """Dual-derivative term + energy term + jump form (operators.py:174-178)."""
        u, v = self._check(u), self._check(v)
        energy = float(np.sum(u * self.apply_Abd(v)))
        return self.dual_term(u, v) + energy + self.jump_form(u, v)

    def s_norm(self, u) -> float:
        return float(np.sqrt(max(self.s_bilinear(u, u), 0.0)))
