"""Time-partitioned Uzawa iteration over several ranks.

The time axis is split into contiguous blocks of steps, one per rank.  The
arithmetic stays in the rank-local building blocks (``GpuLocalOps`` calls the
C ABI of libpint; the CPU tests plug in numpy ops); this module moves data:

* ghost planes: u's boundary planes to both neighbours, p's first plane to the
  left neighbour (K u, K^T u, K^T p couple adjacent steps, operators.py:78-90);
* H~^{-1} (schur.py:62-76) needs the whole time column: the z slab is
  transposed time-sharded -> column-sharded, sine-transformed along the full
  time axis, transposed to mode-sharded planes for the per-mode V-cycles, and
  back the same way; the transposes are grouped point-to-point exchanges
  (NCCL groups them into one all-to-all; gloo has no all-to-all);
* the two residual partial sums are one all-reduce per iteration.

The residual, stopping rule and divergence guard are the reference's
(solvers.py:212-263), evaluated identically on every rank.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from .errors import InputError, SolverDivergenceError
from .solvers import ConvergenceHistory, UzawaConfig


@dataclass(frozen=True)
class Partition:
    """Balanced contiguous split of `total` items into `parts` blocks."""

    total: int
    parts: int

    def count(self, r: int) -> int:
        return self.total // self.parts + (1 if r < self.total % self.parts else 0)

    def start(self, r: int) -> int:
        return r * (self.total // self.parts) + min(r, self.total % self.parts)

    def slice(self, r: int) -> slice:
        s = self.start(r)
        return slice(s, s + self.count(r))


class Comm:
    """The few collectives the time-partitioned iteration needs."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # P2POp takes GLOBAL peer ranks; rank/world above are group-local
        self._global = [q if group is None else dist.get_global_rank(group, q)
                        for q in range(self.world)]

    def peer(self, q: int) -> int:
        return self._global[q]

    def _run(self, ops):
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def halo(self, ext: torch.Tensor, nl: int, prev: bool, nxt: bool) -> None:
        """ext = [ghost_prev, local_0 .. local_{nl-1}, ghost_next] along dim 0.
        prev: fill ghost_prev with the left rank's last plane;
        nxt:  fill ghost_next with the right rank's first plane."""
        r, w = self.rank, self.world
        ops = []
        if prev:
            if r + 1 < w:
                ops.append(dist.P2POp(dist.isend, ext[nl].contiguous(), self.peer(r + 1), self.group))
            if r > 0:
                ops.append(dist.P2POp(dist.irecv, ext[0], self.peer(r - 1), self.group))
        if nxt:
            if r > 0:
                ops.append(dist.P2POp(dist.isend, ext[1].contiguous(), self.peer(r - 1), self.group))
            if r + 1 < w:
                ops.append(dist.P2POp(dist.irecv, ext[nl + 1], self.peer(r + 1), self.group))
        self._run(ops)

    def exchange(self, send: list, recv: list) -> None:
        """send[q] -> rank q, recv[q] <- rank q (own block copied locally)."""
        ops = []
        for q in range(self.world):
            if q == self.rank:
                recv[q].copy_(send[q])
                continue
            ops.append(dist.P2POp(dist.isend, send[q], self.peer(q), self.group))
            ops.append(dist.P2POp(dist.irecv, recv[q], self.peer(q), self.group))
        self._run(ops)

    def allreduce(self, vals, device) -> list:
        t = torch.tensor(list(vals), dtype=torch.float64, device=device)
        dist.all_reduce(t, group=self.group)
        return [float(x) for x in t.cpu()]


class Transposer:
    """Layout changes between time-sharded [N_r][n], column-sharded [N][n_c]
    and mode-sharded [N_r][n] slabs (modes split like steps)."""

    def __init__(self, comm: Comm, N: int, n: int, device):
        self.comm = comm
        self.tp = Partition(N, comm.world)
        self.cp = Partition(n, comm.world)
        self.N, self.n, self.device = N, n, device
        r = comm.rank
        self.nl = self.tp.count(r)
        self.nc = self.cp.count(r)

    def rows_to_cols(self, x: torch.Tensor) -> torch.Tensor:
        """[N_r][n] sharded by rows (steps or modes) -> [N][n_c] sharded by columns."""
        c, w, r = self.comm, self.comm.world, self.comm.rank
        send = [x[:, self.cp.slice(q)].contiguous() for q in range(w)]
        out = torch.empty((self.N, self.nc), dtype=x.dtype, device=x.device)
        recv = [out[self.tp.slice(q)] for q in range(w)]  # contiguous row blocks
        c.exchange(send, recv)
        del r
        return out

    def cols_to_rows(self, y: torch.Tensor) -> torch.Tensor:
        """[N][n_c] sharded by columns -> [N_r][n] sharded by rows."""
        c, w = self.comm, self.comm.world
        send = [y[self.tp.slice(q)].contiguous() for q in range(w)]
        recv = [torch.empty((self.nl, self.cp.count(q)), dtype=y.dtype, device=y.device)
                for q in range(w)]
        c.exchange(send, recv)
        out = torch.empty((self.nl, self.n), dtype=y.dtype, device=y.device)
        for q in range(w):
            out[:, self.cp.slice(q)] = recv[q]
        return out


class LocalOps:
    """Rank-local arithmetic of one Uzawa iteration (interface).

    Slabs are torch tensors; ``u_ext``/``p_ext`` carry one ghost plane before
    and after the local steps."""

    def r1(self, u_ext, p_ext, f):  # -> r1 [N_r][n]
        raise NotImplementedError

    def z(self, u_ext, p_ext, f):  # -> z [N_r][n]
        raise NotImplementedError

    def atilde_update(self, r1, p_ext):  # p_local += A~^-1 r1 ; -> sum r1.dp  (p_ext None: dot only)
        raise NotImplementedError

    def dst_cols(self, kind, x):  # kind 1: S x ; kind 0: S^T x  along dim 0 of [N][n_c]
        raise NotImplementedError

    def htilde_modes(self, zh, want_w=True):  # -> (w or None, sum zh.w)
        raise NotImplementedError

    def axpy(self, u_local, y, omega):  # u_local += omega * y
        raise NotImplementedError


class DistUzawa:
    """Time-partitioned damped two-stage inexact Uzawa (solvers.py:177-264).

    ``begin()`` computes the reference norm (solvers.py:212-217); each
    ``step()`` is one iteration (solvers.py:224-233) and returns the residual
    numerator sqrt(max(sum r1.dp + sum z.y, 0)), identical on every rank."""

    def __init__(self, ops: LocalOps, comm: Comm, N: int, n: int, f_local: torch.Tensor,
                 initial=None):
        self.ops, self.comm = ops, comm
        self.dev = f_local.device
        self.tr = tr = Transposer(comm, N, n, self.dev)
        nl = self.nl = tr.nl
        if f_local.shape != (nl, n):
            raise InputError(f"local rhs has shape {tuple(f_local.shape)}, expected {(nl, n)}")
        self.f = f_local
        self.u_ext = torch.zeros((nl + 2, n), dtype=torch.float64, device=self.dev)
        self.p_ext = torch.zeros((nl + 2, n), dtype=torch.float64, device=self.dev)
        if initial is not None:
            self.p_ext[1:nl + 1].copy_(initial[0])
            self.u_ext[1:nl + 1].copy_(initial[1])
        self.u, self.p = self.u_ext[1:nl + 1], self.p_ext[1:nl + 1]

    def begin(self) -> float:
        ops, tr = self.ops, self.tr
        a = ops.atilde_update(self.f, None)
        fh = tr.cols_to_rows(ops.dst_cols(1, tr.rows_to_cols(self.f)))
        h = ops.htilde_modes(fh, want_w=False)[1]
        tot = self.comm.allreduce([a, h], self.dev)
        return float(np.sqrt(max(tot[0] + tot[1], 0.0)))

    def step(self, omega: float) -> float:
        ops, tr, comm, nl = self.ops, self.tr, self.comm, self.nl
        comm.halo(self.u_ext, nl, prev=True, nxt=True)
        r1 = ops.r1(self.u_ext, self.p_ext, self.f)
        d1 = ops.atilde_update(r1, self.p_ext)
        comm.halo(self.p_ext, nl, prev=False, nxt=True)
        z = ops.z(self.u_ext, self.p_ext, self.f)
        zh = tr.cols_to_rows(ops.dst_cols(1, tr.rows_to_cols(z)))  # mode-sharded S z
        w, d2 = ops.htilde_modes(zh, want_w=True)
        y = tr.cols_to_rows(ops.dst_cols(0, tr.rows_to_cols(w)))  # time-sharded S^T w
        ops.axpy(self.u, y, omega)
        s = comm.allreduce([d1, d2], self.dev)
        return float(np.sqrt(max(s[0] + s[1], 0.0)))


def dist_uzawa_solve(ops: LocalOps, comm: Comm, N: int, n: int, f_local: torch.Tensor,
                     cfg: UzawaConfig, initial=None):
    """uzawa_solve (solvers.py:177-264) on a time-partitioned problem.
    Returns (p_local, u_local, ConvergenceHistory) on every rank."""
    if cfg.diagnostics or cfg.stopping == "s_norm_error":
        raise InputError("diagnostic stopping is not available on the partitioned path")
    it = DistUzawa(ops, comm, N, n, f_local, initial)
    ref = it.begin()
    hist = ConvergenceHistory()
    if ref == 0.0:
        hist.converged = True
        return it.p.clone(), it.u.clone(), hist
    first = None
    t0 = time.perf_counter()
    for _ in range(cfg.max_iter):
        res = it.step(cfg.omega) / ref
        if first is None:
            first = max(res, 1e-300)
        hist.append(res, None, None, time.perf_counter() - t0, 0.0, 0.0)
        if res > 1e6 * first:
            raise SolverDivergenceError(f"residual grew to {res:.3e} from {first:.3e}")
        if res < cfg.tol:
            hist.converged = True
            break
    return it.p.clone(), it.u.clone(), hist


class GpuLocalOps(LocalOps):
    """libpint building blocks for this rank's steps / modes (CUDA tensors)."""

    def __init__(self, spec, hierarchy, part: Partition, rank: int, device=None,
                 damping: float | None = None):
        from ._device import HostProblem
        from ._native import MG_ATILDE, MG_HTILDE, Context
        from .schur import frequency_weights

        hp = HostProblem(spec)
        if damping is None:
            damping = hp.default_damping()
        sl = part.slice(rank)
        self.N, self.n, self.nl = hp.N, hp.n, part.count(rank)
        self.n0 = part.start(rank)
        self.ctx = ctx = Context(device)
        self.dev = torch.device("cuda", ctx.device)
        # launch on the torch stream so the transposes (torch copies, NCCL)
        # and the kernels are ordered without host synchronisation
        with torch.cuda.device(self.dev):
            ctx.call("pint_set_stream", torch.cuda.current_stream().cuda_stream, 0)
        steps = np.ascontiguousarray(hp.steps[sl])
        a_sid = np.ascontiguousarray(hp.a_sid[sl])
        used = np.unique(a_sid)
        remap = {int(s): i for i, s in enumerate(used)}
        a_st = np.ascontiguousarray(hp.a_st[used])
        a_sid = np.array([remap[int(s)] for s in a_sid], dtype=np.int32)
        a_scale = np.ascontiguousarray(hp.a_scale[sl])
        ctx.call("pint_problem_set", hp.dims, hp.m, self.nl, steps.ctypes.data,
                 hp.mass_st.ctypes.data, a_st.shape[0], a_st.ctypes.data, a_sid.ctypes.data,
                 a_scale.ctypes.data, hp.aref_st.ctypes.data, float(spec.tau_ref))
        ctx.call("pint_set_partition", self.n0, self.N, int(self.n0 > 0),
                 int(self.n0 + self.nl < self.N))
        lm = np.asarray(hierarchy.level_m, dtype=np.int32)
        tab_a, sid_a = hp.atilde_tables(hierarchy, damping)
        tab_a = np.ascontiguousarray(tab_a)
        sid_a = np.ascontiguousarray(sid_a[sl])
        ctx.call("pint_mg_set", MG_ATILDE, len(lm), lm.ctypes.data, tab_a.shape[1],
                 tab_a.ctypes.data, sid_a.ctypes.data)
        mu = frequency_weights(self.N)[sl]
        tab_h, _ = hp.htilde_tables(hierarchy, damping, mu)
        tab_h = np.ascontiguousarray(tab_h)
        sid_h = np.arange(self.nl, dtype=np.int32)
        ctx.call("pint_mg_set", MG_HTILDE, len(lm), lm.ctypes.data, self.nl,
                 tab_h.ctypes.data, sid_h.ctypes.data)

    @staticmethod
    def _ptr(t):
        return t.data_ptr()

    def r1(self, u_ext, p_ext, f):
        out = torch.empty_like(f)
        self.ctx.call("pint_residual_r1", u_ext[1].data_ptr(), p_ext[1].data_ptr(),
                      f.data_ptr(), out.data_ptr())
        return out

    def z(self, u_ext, p_ext, f):
        out = torch.empty_like(f)
        self.ctx.call("pint_residual_z", u_ext[1].data_ptr(), p_ext[1].data_ptr(),
                      f.data_ptr(), out.data_ptr())
        return out

    def atilde_update(self, r1, p_ext):
        import ctypes

        d = ctypes.c_double()
        self.ctx.call("pint_atilde_update", r1.data_ptr(),
                      None if p_ext is None else p_ext[1].data_ptr(), ctypes.byref(d))
        return d.value

    def dst_cols(self, kind, x):
        x = x.contiguous()
        out = torch.empty_like(x)
        self.ctx.call("pint_dst_raw", int(kind), int(x.shape[0]), int(x.shape[1]),
                      x.data_ptr(), out.data_ptr())
        return out

    def htilde_modes(self, zh, want_w=True):
        import ctypes

        d = ctypes.c_double()
        w = torch.empty_like(zh) if want_w else None
        self.ctx.call("pint_htilde_modes", zh.data_ptr(), None if w is None else w.data_ptr(),
                      ctypes.byref(d))
        return w, d.value

    def axpy(self, u_local, y, omega):
        self.ctx.call("pint_axpy", u_local.data_ptr(), y.contiguous().data_ptr(), float(omega),
                      int(u_local.numel()))
