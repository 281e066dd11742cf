"""Inexact Uzawa iteration on the GPU (solvers.py of the reference).

``uzawa_solve(system, atilde, htilde, cfg, initial=None, u_oracle=None)``
keeps the reference signature and semantics (solvers.py:177-264):

* ref = sqrt(max(f.A~^-1 f + f.H~^-1 f, 0)); ref == 0 -> converged, 0 iterations;
* per iteration  r1 = K u - A p - f;  p += A~^-1 r1;
  z = f - K^T p - (K u + K^T u + A u);  u += omega H~^-1 z;
  res = sqrt(max(sum r1.dp + sum z.y, 0)) / ref, recorded before the tests;
* divergence when res > 1e6 * first_res (SolverDivergenceError);
* stop when res < tol (the converging iteration is counted).

The iteration itself is one call per iteration into libpint
(pint_uzawa_step); the state (f, p, u and all work slabs) stays in HBM and
only the two partial sums come back.  ``fft_seconds`` / ``spatial_seconds``
are cumulative device time of the DST and multigrid phases (CUDA events).
Diagnostic mode (exact S-norm error per iteration, stopping='s_norm_error',
solvers.py:201-244) stays on the device end to end: the sequential
implicit-Euler solution and every S-norm come from the device's exact solves
(csrc/exact_solve.cu, ``sequential_euler_solve`` below), and the error of
the iterate held in HBM is measured in place (pint_uzawa_s_error).
The reference's rate theory (solvers.py:77-124) is analysis tooling, out of
scope for the GPU path.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from ._device import gpu_problem
from ._native import as_buffer, empty_like_kind, ptr_of
from .errors import InputError
from .operators import EXACT_MAX_ITER, EXACT_TOL
from .spatial import MgHierarchy, _check_mg_options


@dataclass
class UzawaConfig:
    """solvers.py:21-36."""

    omega: float = 0.9
    max_iter: int = 200
    tol: float = 1e-8
    stopping: str = "preconditioned_residual"
    record_history: bool = True
    diagnostics: bool = False

    def __post_init__(self):
        if self.omega <= 0.0:
            raise InputError("damping parameter must be positive")
        if self.tol <= 0.0:
            raise InputError("tolerance must be positive")
        if self.stopping not in ("preconditioned_residual", "s_norm_error"):
            raise InputError(f"unknown stopping rule {self.stopping!r}")


@dataclass
class ConvergenceHistory:
    """Per-iteration record (solvers.py:39-74); same CSV format."""

    residual: list = field(default_factory=list)
    s_norm_error: list = field(default_factory=list)
    d_norm_error: list = field(default_factory=list)
    wall_seconds: list = field(default_factory=list)
    fft_seconds: list = field(default_factory=list)
    spatial_seconds: list = field(default_factory=list)
    converged: bool = False

    @property
    def iterations(self) -> int:
        return len(self.residual)

    def append(self, residual, s_err, d_err, wall, fft, spatial) -> None:
        self.residual.append(residual)
        self.s_norm_error.append(s_err)
        self.d_norm_error.append(d_err)
        self.wall_seconds.append(wall)
        self.fft_seconds.append(fft)
        self.spatial_seconds.append(spatial)

    def to_csv(self) -> str:
        head = "iter,residual,s_norm_error,d_norm_error,wall_seconds,fft_seconds,spatial_seconds"
        out = [head]
        for i in range(self.iterations):
            s = "" if self.s_norm_error[i] is None else f"{self.s_norm_error[i]:.17g}"
            d = "" if self.d_norm_error[i] is None else f"{self.d_norm_error[i]:.17g}"
            out.append(f"{i + 1},{self.residual[i]:.17g},{s},{d},{self.wall_seconds[i]:.17g},"
                       f"{self.fft_seconds[i]:.17g},{self.spatial_seconds[i]:.17g}")
        return "\n".join(out) + "\n"


class BlockDiagSolver:
    """A~^{-1}: one V-cycle per step on A_n, divided by tau_n (solvers.py:127-155),
    all steps in one batched launch per level."""

    def __init__(self, spec, kind: str = "mg", hierarchy: MgHierarchy | None = None,
                 cycles: int = 1, smooth_steps: int = 1, damping: float | None = None,
                 device=None):
        if kind != "mg":
            raise InputError(f"solver kind {kind!r} is not on the GPU path; use kind='mg'")
        if hierarchy is None:
            raise InputError("mg solver needs a grid hierarchy")
        _check_mg_options(cycles, smooth_steps, damping)
        self.spec = spec
        self.kind = kind
        self.steps = spec.grid.steps
        self.hierarchy = hierarchy
        self.cycles, self.smooth_steps = int(cycles), int(smooth_steps)
        self._gp = gpu_problem(spec, device)
        self._gp.set_atilde(hierarchy, self._gp.default_damping() if damping is None else damping,
                            self.cycles, self.smooth_steps)

    def apply_inverse(self, b):
        shape = (self.spec.N, self.spec.dim)
        ptr, keep = as_buffer(b, shape)
        out = empty_like_kind(keep, shape)
        self._gp.ctx.call("pint_atilde_inv", ptr, ptr_of(out))
        return out

    def forward(self, x):
        raise InputError("forward application requires direct (exact) solvers")


def _sequential_euler_device(gp):
    """u_n = (M + tau_n A_n)^{-1} (M u_{n-1} + tau_n load_n) on the device as a
    CUDA tensor (the oracle of solvers.py:158-174, exact_solve.cu)."""
    import torch

    gp.ensure_exact()
    spec = gp.spec
    dev = torch.device("cuda", gp.ctx.device)
    load = torch.from_numpy(np.ascontiguousarray(spec.load, dtype=np.float64)).to(dev)
    u0 = torch.from_numpy(np.ascontiguousarray(spec.u_init, dtype=np.float64)).to(dev)
    out = torch.empty((spec.N, spec.dim), dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    it = ctypes.c_int()
    rel = ctypes.c_double()
    gp.ctx.call("pint_sequential_euler", load.data_ptr(), u0.data_ptr(), out.data_ptr(),
                EXACT_TOL, EXACT_MAX_ITER, ctypes.byref(it), ctypes.byref(rel))
    return out


def sequential_euler_solve(spec, device=None) -> np.ndarray:
    """Forward implicit-Euler sweep with exact per-step solves (the oracle of
    solvers.py:158-174), on the GPU: one multigrid-preconditioned CG solve of
    (M + tau_n A_n) u_n = M u_{n-1} + tau_n load_n per step, to the rounding
    floor.  Returns a numpy array (N, dim)."""
    return _sequential_euler_device(gpu_problem(spec, device)).cpu().numpy()


def _is_cuda(x) -> bool:
    return x is not None and type(x).__module__.startswith("torch") and x.is_cuda


def _shared_problem(system, atilde, htilde):
    gp = system._gp
    if getattr(atilde, "_gp", None) is not gp or getattr(htilde, "_gp", None) is not gp:
        raise InputError("system, atilde and htilde must be built from the same ProblemSpec")
    if not (gp.atilde_ready and gp.htilde_ready):
        raise InputError("multigrid sets not configured")
    return gp


def uzawa_solve(system, atilde, htilde, cfg: UzawaConfig, initial=None, u_oracle=None):
    """Damped two-stage inexact Uzawa iteration (solvers.py:177-264) on the GPU.

    Returns ((p, u), ConvergenceHistory) with p, u numpy arrays (or CUDA
    tensors when ``initial`` holds CUDA tensors).
    """
    diagnostics = cfg.diagnostics or cfg.stopping == "s_norm_error"
    gp = _shared_problem(system, atilde, htilde)
    ctx = gp.ctx
    shape = (system.spec.N, system.spec.dim)
    f_ptr, f_keep = as_buffer(system.rhs, shape)
    if initial is not None:
        p_ptr, p_keep = as_buffer(initial[0], shape)
        u_ptr, u_keep = as_buffer(initial[1], shape)
        like = p_keep
    else:
        p_ptr = u_ptr = None
        like = f_keep
    hist = ConvergenceHistory()
    # diagnostic mode (solvers.py:201-210): the exact solution and its S-norm
    # on the device; the error of the device-resident iterate is measured in
    # place each iteration
    u_star = s_norm_ref = None
    if diagnostics:
        system.build_exact_solvers()
        if u_oracle is not None:
            u_star = u_oracle
        else:
            u_star = _sequential_euler_device(gp)
        s_norm_ref = system.s_norm(u_star)
        us_ptr, us_keep = as_buffer(u_star, shape)
    if any(_is_cuda(x) for x in (f_keep, p_ptr and p_keep, u_ptr and u_keep)):
        # the library reads device inputs on its own stream: order it after
        # torch's pending writes (.contiguous(), .cuda(), the caller's kernels)
        import torch

        torch.cuda.synchronize(gp.ctx.device)
    ref = ctypes.c_double(0.0)
    ctx.call("pint_uzawa_begin", f_ptr, p_ptr, u_ptr, ctypes.byref(ref))
    p_out = empty_like_kind(like, shape)
    u_out = empty_like_kind(like, shape)
    if ref.value == 0.0:
        hist.converged = True
        ctx.call("pint_uzawa_end", ptr_of(p_out), ptr_of(u_out))
        return (p_out, u_out), hist
    for arr in (p_out, u_out):
        if isinstance(arr, np.ndarray):
            # fault the host output pages in while the device iterates
            ctx.call("pint_host_prefault", arr.ctypes.data, arr.nbytes)
    ctx.call("pint_set_timing", 1)
    ms = np.zeros(3)
    num = ctypes.c_double(0.0)
    first = None
    t0 = time.perf_counter()
    try:
        for _ in range(cfg.max_iter):
            ctx.call("pint_uzawa_step", float(cfg.omega), ctypes.byref(num))
            res = float(num.value) / ref.value
            if first is None:
                first = max(res, 1e-300)
            ctx.call("pint_phase_ms", ms.ctypes.data)
            s_err = None
            if diagnostics:
                err = ctypes.c_double()
                ctx.call("pint_uzawa_s_error", us_ptr, EXACT_TOL, EXACT_MAX_ITER,
                         ctypes.byref(err))
                s_err = err.value / s_norm_ref
            hist.append(res, s_err, None, time.perf_counter() - t0, ms[0] / 1e3, ms[1] / 1e3)
            if res > 1e6 * first:
                from .errors import SolverDivergenceError

                raise SolverDivergenceError(f"residual grew to {res:.3e} from {first:.3e}")
            if cfg.stopping == "preconditioned_residual" and res < cfg.tol:
                hist.converged = True
                break
            if cfg.stopping == "s_norm_error" and s_err < cfg.tol:
                hist.converged = True
                break
    finally:
        ctx.call("pint_set_timing", 0)
        # background first-touch threads write into p_out / u_out: they must
        # finish before an exception can release those arrays
        ctx.call("pint_host_prefault_join")
    ctx.call("pint_uzawa_end", ptr_of(p_out), ptr_of(u_out))
    return (p_out, u_out), hist


def minres_solve(system, atilde, htilde, tol: float = 1e-8, max_iter: int = 500):
    """Block-diagonally preconditioned MINRES on the saddle-point system
    (solvers.py:267-327) with every vector resident on the GPU.

    The Krylov recurrence is scipy.sparse.linalg.minres (the reference's own
    solver, Paige-Saunders; restated step for step: same scalar updates, same
    stopping tests test1 = |r|/(|A||x|) <= rtol, test2 = |Ar|/(|A||r|) <= rtol,
    Acond >= 0.1/eps, ...), with the operator ``apply_saddle``
    (operators.py:107-111) and the preconditioner diag(A~^-1, H~^-1) as the
    library's kernels and the vector updates as pint_lincomb in numpy's
    operation order.  As in the reference, the callback evaluates the true
    preconditioned residual sqrt(max(r.M r, 0))/ref of every iterate,
    r = g - A x, g = (-f, -f).  Inner products are deterministic device
    reductions (a different summation order than numpy's BLAS dot).
    Returns ((p, u), ConvergenceHistory); p, u are numpy arrays.
    """
    import torch

    gp = _shared_problem(system, atilde, htilde)
    ctx = gp.ctx
    spec = system.spec
    N, n = spec.N, spec.dim
    nd = N * n
    dev = torch.device("cuda", ctx.device)
    eps = float(np.finfo(np.float64).eps)

    def new():
        return torch.empty(2 * nd, dtype=torch.float64, device=dev)

    def halves(t):
        return t.data_ptr(), t.data_ptr() + nd * 8

    def matvec(w, out):
        wp, wu = halves(w)
        op, ou = halves(out)
        ctx.call("pint_apply_saddle", wp, wu, op, ou)

    def precond(w, out):
        wp, wu = halves(w)
        op, ou = halves(out)
        ctx.call("pint_atilde_inv", wp, op)
        ctx.call("pint_htilde_inv", wu, ou)

    def lincomb(out, x0, a1=0.0, x1=None, a2=0.0, x2=None, scale=None):
        ctx.call("pint_lincomb", out.data_ptr(), 2 * nd, x0.data_ptr(), float(a1),
                 None if x1 is None else x1.data_ptr(), float(a2),
                 None if x2 is None else x2.data_ptr(),
                 1.0 if scale is None else float(scale), 0 if scale is None else 1)

    def dot(a, b):
        v = ctypes.c_double()
        ctx.call("pint_dot", a.data_ptr(), b.data_ptr(), 2 * nd, ctypes.byref(v))
        return v.value

    def upload(arr):
        t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64).ravel()).to(dev)
        torch.cuda.synchronize(dev)  # torch-stream copy before the library stream reads it
        return t

    # g = (-f, -f) formed on the device from one upload of f (the host
    # concatenation and the second half's transfer cost more than 20 iterations)
    f_dev = upload(system.rhs)
    g = new()
    g[:nd].copy_(f_dev).neg_()
    g[nd:].copy_(g[:nd])
    del f_dev
    torch.cuda.synchronize(dev)
    tmp, tmp2 = new(), new()

    # cheap positivity probe of the preconditioner (solvers.py:297-302)
    # (three seeded N(0,1) probes as in the reference; drawn on the device --
    # the host generator costs seconds per probe at config-2 size)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234)
    for _ in range(3):
        w = torch.randn(2 * nd, dtype=torch.float64, device=dev, generator=gen)
        torch.cuda.synchronize(dev)
        precond(w, tmp)
        if dot(w, tmp) <= 0.0:
            from .errors import NotSpdError

            raise NotSpdError("block preconditioner is not positive definite")
        del w

    hist = ConvergenceHistory()
    t0 = time.perf_counter()
    precond(g, tmp)
    ref = float(np.sqrt(dot(g, tmp)))
    if ref == 0.0:
        hist.converged = True
        z = np.zeros((N, n))
        return (z, z.copy()), hist

    def callback(xk):
        matvec(xk, tmp)
        lincomb(tmp, g, -1.0, tmp)           # r = g - A x
        precond(tmp, tmp2)
        res = float(np.sqrt(max(dot(tmp, tmp2), 0.0))) / ref
        hist.append(res, None, None, time.perf_counter() - t0, 0.0, 0.0)

    # ---- scipy.sparse.linalg.minres (x0 = None, shift = 0) ----
    x = torch.zeros(2 * nd, dtype=torch.float64, device=dev)
    torch.cuda.synchronize(dev)
    r1 = new()
    lincomb(r1, g)                           # r1 = b.copy()
    y = new()
    precond(r1, y)
    beta1 = dot(r1, y)
    if beta1 < 0:
        raise InputError("indefinite preconditioner")
    info = 0
    if beta1 == 0 or float(np.sqrt(max(dot(g, g), 0.0))) == 0.0:
        hist.converged = True
    else:
        beta1 = float(np.sqrt(beta1))
        oldb, beta, dbar, epsln = 0.0, beta1, 0.0, 0.0
        phibar = beta1
        rhs1, rhs2, tnorm2 = beta1, 0.0, 0.0
        gmax, gmin = 0.0, float(np.finfo(np.float64).max)
        cs, sn = -1.0, 0.0
        w = torch.zeros(2 * nd, dtype=torch.float64, device=dev)
        w2 = torch.zeros(2 * nd, dtype=torch.float64, device=dev)
        torch.cuda.synchronize(dev)
        w1 = new()
        v = new()
        r2 = new()
        lincomb(r2, r1)                      # r2 = r1
        istop, itn = 0, 0
        while itn < max_iter:
            itn += 1
            s = 1.0 / beta
            lincomb(v, y, scale=s)           # v = s*y
            matvec(v, y)                     # y = A v  (shift = 0: y - 0*v == y)
            if itn >= 2:
                lincomb(y, y, -(beta / oldb), r1)
            alfa = dot(v, y)
            lincomb(y, y, -(alfa / beta), r2)
            r1, r2 = r2, r1
            lincomb(r2, y)                   # r2 = y
            precond(r2, y)
            oldb = beta
            beta = dot(r2, y)
            if beta < 0:
                raise InputError("non-symmetric matrix")
            beta = float(np.sqrt(beta))
            tnorm2 += alfa ** 2 + oldb ** 2 + beta ** 2
            if itn == 1 and beta / beta1 <= 10 * eps:
                istop = -1
            oldeps = epsln
            delta = cs * dbar + sn * alfa
            gbar = sn * dbar - cs * alfa
            epsln = sn * beta
            dbar = -cs * beta
            root = float(np.linalg.norm([gbar, dbar]))
            gamma = float(np.linalg.norm([gbar, beta]))
            gamma = max(gamma, eps)
            cs = gbar / gamma
            sn = beta / gamma
            phi = cs * phibar
            phibar = sn * phibar
            denom = 1.0 / gamma
            w1, w2, w = w2, w, w1
            lincomb(w, v, -oldeps, w1, -delta, w2, scale=denom)
            lincomb(x, x, phi, w)
            gmax = max(gmax, gamma)
            gmin = min(gmin, gamma)
            z = rhs1 / gamma
            rhs1 = rhs2 - delta * z
            rhs2 = -epsln * z
            Anorm = float(np.sqrt(tnorm2))
            ynorm = float(np.sqrt(max(dot(x, x), 0.0)))
            epsx = Anorm * ynorm * eps
            rnorm = phibar
            test1 = np.inf if (ynorm == 0 or Anorm == 0) else rnorm / (Anorm * ynorm)
            test2 = np.inf if Anorm == 0 else root / Anorm
            Acond = gmax / gmin
            if istop == 0:
                if 1 + test2 <= 1:
                    istop = 2
                if 1 + test1 <= 1:
                    istop = 1
                if itn >= max_iter:
                    istop = 6
                if Acond >= 0.1 / eps:
                    istop = 4
                if epsx >= beta1:
                    istop = 3
                if test2 <= tol:
                    istop = 2
                if test1 <= tol:
                    istop = 1
            callback(x)
            if istop != 0:
                break
        info = max_iter if istop == 6 else 0
        hist.converged = info == 0
    ctx.call("pint_sync")
    # each half straight into its own numpy array (no host-side re-copy)
    p_out, u_out = np.empty((N, n)), np.empty((N, n))
    torch.from_numpy(p_out).copy_(x[:nd].view(N, n))
    torch.from_numpy(u_out).copy_(x[nd:].view(N, n))
    return (p_out, u_out), hist
