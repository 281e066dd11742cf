"""Time-global operators on the GPU (operators.py:22-99 of the reference).

``TimeGlobalSystem`` keeps the reference's interface (``spec``, ``rhs``,
``apply_K``, ``apply_Kt``, ``apply_Abd``, ``apply_B``, ``apply_Bt``,
``apply_saddle``) with the arithmetic done by the sm_100a kernels of
csrc/stencil_ops.cu: block vectors of shape (N, dim), numpy (host) or CUDA
float64 torch tensors (device), results of the same kind.

Diagnostic mode (operators.py:51-214: exact A_bd^{-1}, P, S and the discrete
parabolic S-norm) runs on the device too (csrc/exact_solve.cu): the exact
per-step solves the reference does with SuperLU are multigrid-preconditioned
CG solves to the rounding floor (relative residual <= EXACT_TOL), batched
over all steps.  They measure errors; the Uzawa iteration never uses them.
"""

from __future__ import annotations

import ctypes

import numpy as np

from ._device import gpu_problem
from ._native import _is_tensor, as_buffer, empty_like_kind, ptr_of

# exact solves of diagnostic mode: relative residual target and CG iteration cap
EXACT_TOL = 1e-14
EXACT_MAX_ITER = 200
from .errors import DiagnosticModeRequiredError


def _host(x) -> np.ndarray:
    return x.detach().cpu().numpy() if _is_tensor(x) else np.asarray(x, dtype=np.float64)


def fold_rhs(spec) -> np.ndarray:
    """tau_n load_n, plus M u_init on block 1 (operators.py:22-26), on the GPU."""
    gp = gpu_problem(spec)
    load = np.ascontiguousarray(spec.load, dtype=np.float64)
    u0 = np.ascontiguousarray(spec.u_init, dtype=np.float64)
    out = np.empty((spec.N, spec.dim))
    gp.ctx.call("pint_fold_rhs", load.ctypes.data, u0.ctypes.data, out.ctypes.data)
    return out


class TimeGlobalSystem:
    """The time-global implicit-Euler system of one ProblemSpec, on the GPU."""

    def __init__(self, spec, diagnostic: bool = False, device=None):
        self.spec = spec
        self._gp = gpu_problem(spec, device)
        self.rhs = fold_rhs(spec)
        self._scales = self._gp.scales
        self._exact = None
        if diagnostic:
            self.build_exact_solvers()

    @property
    def diagnostic(self) -> bool:
        return self._exact is not None

    def build_exact_solvers(self) -> None:
        """Enable diagnostic mode (operators.py:51-61): configures the
        multigrid sets that precondition the device's exact solves."""
        self._gp.ensure_exact()
        self._exact = True

    def _need_exact(self):
        if self._exact is None:
            raise DiagnosticModeRequiredError(
                "exact per-step factorizations not built; pass diagnostic=True")

    # --- diagnostic-mode operators and norms (operators.py:113-183) --------
    def apply_Abd_inv(self, b):
        """diag(tau_n A_n)^{-1} b (operators.py:113-122)."""
        self._need_exact()
        shape = (self.spec.N, self.spec.dim)
        ptr, keep = as_buffer(b, shape)
        out = empty_like_kind(keep, shape)
        self._gp.ctx.call("pint_abd_inverse", ptr, ptr_of(out), EXACT_TOL, EXACT_MAX_ITER)
        return out

    def apply_P(self, u):
        """Optimal test functions A_bd^{-1} K u + u (operators.py:124-126)."""
        return self.apply_Abd_inv(self.apply_K(u)) + u

    def apply_Pt(self, u):
        return self.apply_Kt(self.apply_Abd_inv(u)) + u

    def apply_S(self, u):
        """Schur complement K^T A_bd^{-1} K u + K u + K^T u + A_bd u (operators.py:131-139)."""
        ku = self.apply_K(u)
        return self.apply_Kt(self.apply_Abd_inv(ku)) + ku + self.apply_Kt(u) + self.apply_Abd(u)

    def s_norm_diff(self, a, b=None) -> float:
        """|a - b|_S on the device (b = None: |a|_S)."""
        self._need_exact()
        shape = (self.spec.N, self.spec.dim)
        pa, ka = as_buffer(a, shape)
        pb, kb = as_buffer(b, shape) if b is not None else (None, None)
        if _is_tensor(ka) or _is_tensor(kb):
            import torch

            torch.cuda.synchronize(self._gp.ctx.device)
        out = ctypes.c_double()
        self._gp.ctx.call("pint_s_norm", pa, pb, EXACT_TOL, EXACT_MAX_ITER, ctypes.byref(out))
        return float(out.value)

    def s_norm(self, u) -> float:
        """Discrete parabolic norm (operators.py:182-183)."""
        return self.s_norm_diff(u)

    def s_bilinear(self, u, v) -> float:
        """s(u, v) by polarisation of the device S-norm (operators.py:174-178)."""
        return 0.25 * (self.s_norm_diff(u, -v) ** 2 - self.s_norm_diff(u, v) ** 2)

    def jump_form(self, u, v) -> float:
        """sum_n (u_n - u_{n-1}) . M (v_n - v_{n-1}) + u_N . M v_N, u_0 = v_0 = 0
        (operators.py:146-153), host sparse products."""
        u, v = _host(u), _host(v)
        m = self.spec.mass
        jumps_u = np.vstack([u[:1], u[1:] - u[:-1]])
        jumps_v = np.vstack([v[:1], v[1:] - v[:-1]])
        return float(np.einsum("ij,ij->", jumps_u, m.dot(jumps_v.T).T) + u[-1] @ m.dot(v[-1]))

    def _apply(self, name: str, u):
        shape = (self.spec.N, self.spec.dim)
        ptr, keep = as_buffer(u, shape)
        out = empty_like_kind(keep, shape)
        self._gp.ctx.call(name, ptr, ptr_of(out))
        return out

    def apply_K(self, u):
        """M u_n - M u_{n-1} (operators.py:78-83)."""
        return self._apply("pint_apply_K", u)

    def apply_Kt(self, u):
        """M u_n - M u_{n+1} (operators.py:85-90)."""
        return self._apply("pint_apply_Kt", u)

    def apply_Abd(self, u):
        """tau_n A_n u_n (operators.py:92-99)."""
        return self._apply("pint_apply_Abd", u)

    def apply_B(self, u):
        return self.apply_K(u) + self.apply_Abd(u)

    def apply_Bt(self, u):
        return self.apply_Kt(u) + self.apply_Abd(u)

    def apply_saddle(self, p, u):
        """Symmetric indefinite 2x2 block operator (operators.py:107-111):
        top = Abd p - K u, bottom = -Kt p - (K u + Kt u + Abd u), one
        pint_apply_saddle call (device kernels, the reference's operation
        order); numpy in -> numpy out, CUDA tensors in -> CUDA tensors out."""
        import torch

        shape = (self.spec.N, self.spec.dim)
        host = not (_is_tensor(p) and _is_tensor(u))
        dev = torch.device("cuda", self._gp.ctx.device)

        def dev_of(x):
            if _is_tensor(x):
                _, t = as_buffer(x, shape)
                return t
            a = np.ascontiguousarray(x, dtype=np.float64)
            if a.shape != shape:
                from .errors import DimensionMismatchError

                raise DimensionMismatchError(f"expected block vector of shape {shape}, got {a.shape}")
            return torch.from_numpy(a).to(dev)

        pd, ud = dev_of(p), dev_of(u)
        top = torch.empty(shape, dtype=torch.float64, device=dev)
        bottom = torch.empty(shape, dtype=torch.float64, device=dev)
        torch.cuda.synchronize(dev)  # uploads (torch stream) before the library stream reads
        self._gp.ctx.call("pint_apply_saddle", pd.data_ptr(), ud.data_ptr(), top.data_ptr(),
                          bottom.data_ptr())
        self._gp.ctx.call("pint_sync")
        if host:
            return top.cpu().numpy(), bottom.cpu().numpy()
        return top, bottom

    def a_norm(self, u) -> float:
        return float(np.sqrt(max(float((u * self.apply_Abd(u)).sum()), 0.0)))
