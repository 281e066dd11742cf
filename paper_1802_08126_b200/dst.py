"""Sine transforms over the time index on the GPU (dst.py of the reference).

forward   uhat_k = (2/N) sum_n (1 + delta_nN)^-1 u_n sin((2k-1) n pi / 2N)  (dst.py:57-65)
inverse   u_n    = sum_k uhat_k sin((2k-1) n pi / 2N)                      (dst.py:67-73)
and their transposes (dst.py:75-93), along axis 0 of an (N, dim) array.
Power-of-two N runs the FFT kernel of csrc/dst.cu; other N a dense kernel
(the reference's own split, dst.py:60-93).
"""

from __future__ import annotations

import numpy as np

from ._native import Context, as_buffer, empty_like_kind, ptr_of
from .errors import DimensionMismatchError

_KIND = {"inverse": 0, "inverse_transpose": 1, "forward": 2, "forward_transpose": 3}
_shared_ctx = None


def _ctx() -> Context:
    global _shared_ctx
    if _shared_ctx is None:
        _shared_ctx = Context()
    return _shared_ctx


class DstPlan:
    """Reusable transform plan for a fixed number of time blocks (dst.py:31-55)."""

    def __init__(self, N: int):
        if N < 1:
            raise DimensionMismatchError("transform length must be >= 1")
        self.N = int(N)
        self.fast = (N & (N - 1)) == 0

    def kernel(self) -> np.ndarray:
        k = np.arange(1, self.N + 1)[:, None]
        n = np.arange(1, self.N + 1)[None, :]
        return np.sin((2 * k - 1) * n * np.pi / (2 * self.N))

    def _run(self, kind: str, u):
        shape = tuple(np.shape(u)) if not hasattr(u, "shape") else tuple(u.shape)
        if len(shape) == 0 or shape[0] != self.N:
            raise DimensionMismatchError(
                f"block count {shape[0] if shape else 0} does not match plan length {self.N}")
        ptr, keep = as_buffer(u, shape)
        out = empty_like_kind(keep, shape)
        ncols = int(np.prod(shape[1:])) if len(shape) > 1 else 1
        _ctx().call("pint_dst_raw", _KIND[kind], self.N, ncols, ptr, ptr_of(out))
        return out

    def forward(self, u):
        return self._run("forward", u)

    def inverse(self, uhat):
        return self._run("inverse", uhat)

    def forward_transpose(self, v):
        return self._run("forward_transpose", v)

    def inverse_transpose(self, u):
        return self._run("inverse_transpose", u)

    def forward_matrix(self) -> np.ndarray:
        w = np.ones(self.N)
        w[-1] = 0.5
        return (2.0 / self.N) * self.kernel() * w[None, :]

    def inverse_matrix(self) -> np.ndarray:
        return self.kernel().T


def dst_forward(plan: DstPlan, u):
    return plan.forward(u)


def dst_inverse(plan: DstPlan, uhat):
    return plan.inverse(uhat)


def dst_forward_transpose(plan: DstPlan, v):
    return plan.forward_transpose(v)


def dst_inverse_transpose(plan: DstPlan, u):
    return plan.inverse_transpose(u)
