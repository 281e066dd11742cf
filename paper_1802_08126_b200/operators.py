"""Time-global operators on the GPU (operators.py:22-99 of the reference).

``TimeGlobalSystem`` keeps the reference's interface (``spec``, ``rhs``,
``apply_K``, ``apply_Kt``, ``apply_Abd``, ``apply_B``, ``apply_Bt``,
``apply_saddle``) with the arithmetic done by the sm_100a kernels of
csrc/stencil_ops.cu: block vectors of shape (N, dim), numpy (host) or CUDA
float64 torch tensors (device), results of the same kind.  Diagnostic-mode
operators (exact per-step inverses, S-norm, P, S; operators.py:51-214) are
the reference's host-side SuperLU computations (diagnostics.py); they serve
error measurement, never the iteration.
"""

from __future__ import annotations

import numpy as np

from ._device import gpu_problem
from ._native import _is_tensor, as_buffer, empty_like_kind, ptr_of
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
        """Exact per-step factorisations on the host (operators.py:51-61)."""
        if self._exact is None:
            from .diagnostics import ExactNorms

            self._exact = ExactNorms(self.spec)

    def _need_exact(self):
        if self._exact is None:
            raise DiagnosticModeRequiredError(
                "exact per-step factorizations not built; pass diagnostic=True")
        return self._exact

    # --- diagnostic-mode operators and norms (operators.py:113-183) --------
    def apply_Abd_inv(self, b):
        return self._need_exact().apply_Abd_inv(_host(b))

    def apply_P(self, u):
        """Optimal-test-function map (operators.py:124-126)."""
        return self.apply_Abd_inv(self.apply_K(_host(u))) + _host(u)

    def apply_Pt(self, u):
        return self.apply_Kt(self.apply_Abd_inv(_host(u))) + _host(u)

    def apply_S(self, u):
        """Schur complement operator (operators.py:131-139)."""
        u = _host(u)
        ku = self.apply_K(u)
        return self.apply_Kt(self.apply_Abd_inv(ku)) + ku + self.apply_Kt(u) + self.apply_Abd(u)

    def a_norm(self, u) -> float:
        return self._need_exact().a_norm(_host(u))

    def jump_form(self, u, v) -> float:
        return self._need_exact().jump_form(_host(u), _host(v))

    def s_bilinear(self, u, v) -> float:
        return self._need_exact().s_bilinear(_host(u), _host(v))

    def s_norm(self, u) -> float:
        return self._need_exact().s_norm(_host(u))

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
