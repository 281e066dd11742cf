"""Time-partitioned Uzawa iteration over several GPUs.

One process per GPU (torchrun); the time axis is split into contiguous blocks
of steps, one per rank, as the north_star prescribes.  The arithmetic stays in
the rank-local building blocks (``GpuLocalOps``: the partition-aware C ABI of
libpint; the CPU tests plug in numpy ops); this module moves data:

* ghost planes: u's boundary planes to both neighbours, p's first plane to the
  left neighbour (K u, K^T u, K^T p couple adjacent steps, operators.py:78-90);
* H~^{-1} (schur.py:62-76) needs whole time columns: z is transposed
  time-sharded -> column-sharded, sine-transformed along the full time axis,
  and transposed back mode-sharded for the per-mode V-cycles; w goes the same
  way back and lands as the u update.  The transposes are split into column
  chunks and pipelined: with NCCL every chunk is an asynchronous
  all_to_all_single on NCCL's stream, so chunk j+1 moves over NVLink while the
  transform of chunk j runs (gloo, used by the CPU tests, exchanges
  point-to-point and synchronously);
* the two residual partial sums stay on the device and are one all-reduce per
  iteration; the host reads the residual once per iteration (the reference's
  stopping and divergence rules, solvers.py:234-263).

Every libpint call is stream-ordered on torch's current stream
(pint_set_stream), so the kernels, the NCCL exchanges and the packing copies
are ordered without host synchronisation.  With one rank there is nothing to
transpose and the u update is fused into the final transform
(pint_dst_raw_axpy).
"""

from __future__ import annotations

import argparse
import ctypes
import os
import sys
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
    """The collectives the time-partitioned iteration needs, on a process
    group (default: the world)."""

    def __init__(self, group=None, pipelined=None):
        """pipelined: run the transposes as chunked asynchronous all-to-alls
        (default: on NCCL; the CPU tests force it on gloo to cover that path)."""
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        # P2POp takes GLOBAL peer ranks; rank/world above are group-local
        self._global = [q if group is None else dist.get_global_rank(group, q)
                        for q in range(self.world)]
        self.nccl = (dist.get_backend(group) == "nccl") if pipelined is None else bool(pipelined)

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
                ops.append(dist.P2POp(dist.isend, ext[nl], self.peer(r + 1), self.group))
            if r > 0:
                ops.append(dist.P2POp(dist.irecv, ext[0], self.peer(r - 1), self.group))
        if nxt:
            if r > 0:
                ops.append(dist.P2POp(dist.isend, ext[1], self.peer(r - 1), self.group))
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

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits):
        """Asynchronous all-to-all of contiguous split blocks (NCCL); returns
        the work handle, whose wait() orders the current stream after it."""
        return dist.all_to_all_single(out, inp, list(out_splits), list(in_splits),
                                      group=self.group, async_op=True)

    def allreduce_(self, t: torch.Tensor) -> None:
        dist.all_reduce(t, group=self.group)


class Transposer:
    """Row-sharded [N_r][n] (steps or modes; modes split like steps) <->
    column-sharded [N][n_c] around a transform of whole time columns,
    pipelined over column chunks."""

    def __init__(self, comm, N: int, n: int, chunks: int = 4):
        self.comm = comm
        w = comm.world
        self.tp = Partition(N, w)
        self.cp = Partition(n, w)
        self.N, self.n = N, n
        self.nl = self.tp.count(comm.rank)
        # chunk j of rank q's columns: cols[q][j] (a slice of the global columns)
        self.chunks = max(1, chunks)
        self.cols = []
        for q in range(w):
            s = self.cp.slice(q)
            sub = Partition(s.stop - s.start, self.chunks)
            self.cols.append([slice(s.start + sub.start(j), s.start + sub.start(j) + sub.count(j))
                              for j in range(self.chunks)])

    def _width(self, q: int, j: int) -> int:
        s = self.cols[q][j]
        return s.stop - s.start

    def apply(self, x: torch.Tensor, transform, out: torch.Tensor, omega=None) -> None:
        """out[:, :] (row-sharded) = rows of transform(column-sharded x);
        with omega: out += omega * (...) (the fused u update).
        transform(cols_in [N][w], cols_out [N][w]) acts along dim 0."""
        comm, w, me = self.comm, self.comm.world, self.comm.rank
        nl, N = self.nl, self.N
        rows = [self.tp.count(q) for q in range(w)]
        if getattr(comm, "nccl", False):
            # pack every chunk for every destination (contiguous blocks), then
            # stream the chunks: a2a in (async) -> transform -> a2a out (async)
            packs, handles, recvs = [], [], []
            for j in range(self.chunks):
                blocks = [x[:, self.cols[q][j]] for q in range(w)]
                packs.append(torch.cat([b.reshape(-1) for b in blocks]))
            for j in range(self.chunks):
                wj = self._width(me, j)
                recv = torch.empty((N, wj), dtype=x.dtype, device=x.device)
                handles.append(comm.all_to_all(
                    recv.view(-1), packs[j], [r * wj for r in rows],
                    [nl * self._width(q, j) for q in range(w)]))
                recvs.append(recv)
            backs, outs = [], []
            for j in range(self.chunks):
                handles[j].wait()
                res = torch.empty_like(recvs[j])
                transform(recvs[j], res)
                back = torch.empty(sum(nl * self._width(q, j) for q in range(w)),
                                   dtype=x.dtype, device=x.device)
                backs.append((back, comm.all_to_all(
                    back, res.view(-1), [nl * self._width(q, j) for q in range(w)],
                    [r * self._width(me, j) for r in rows])))
            for j in range(self.chunks):
                back, h = backs[j]
                h.wait()
                off = 0
                for q in range(w):
                    wq = self._width(q, j)
                    blk = back[off:off + nl * wq].view(nl, wq)
                    off += nl * wq
                    if omega is None:
                        out[:, self.cols[q][j]] = blk
                    else:
                        out[:, self.cols[q][j]].add_(blk, alpha=omega)
            return
        # synchronous point-to-point path (gloo / loopback): whole columns
        mine = self.cp.slice(me)
        send = [x[:, self.cp.slice(q)].contiguous() for q in range(w)]
        cols_in = torch.empty((N, mine.stop - mine.start), dtype=x.dtype, device=x.device)
        comm.exchange(send, [cols_in[self.tp.slice(q)] for q in range(w)])
        cols_out = torch.empty_like(cols_in)
        transform(cols_in, cols_out)
        send = [cols_out[self.tp.slice(q)].contiguous() for q in range(w)]
        recv = [torch.empty((nl, self.cp.count(q)), dtype=x.dtype, device=x.device)
                for q in range(w)]
        comm.exchange(send, recv)
        for q in range(w):
            if omega is None:
                out[:, self.cp.slice(q)] = recv[q]
            else:
                out[:, self.cp.slice(q)].add_(recv[q], alpha=omega)


class LocalOps:
    """Rank-local arithmetic of one Uzawa iteration (interface).

    Slabs are torch tensors; ``u_ext``/``p_ext`` carry one ghost plane before
    and after the local steps.  Partial sums are written into 1-element
    tensors on the slab's device (``dot``), never returned to the host."""

    def r1(self, u_ext, p_ext, f, out):  # out = r1 [N_r][n]
        raise NotImplementedError

    def z(self, u_ext, p_ext, f, out):  # out = z [N_r][n]
        raise NotImplementedError

    def atilde_update(self, r1, p_ext, dot):  # p_local += A~^-1 r1; dot = sum r1.dp (p_ext None: dot only)
        raise NotImplementedError

    def dst_cols(self, kind, x, out, base=None, alpha=1.0):  # out = [base + alpha*] T x along dim 0
        raise NotImplementedError

    def htilde_modes(self, zh, w, dot):  # w = modes of H~^-1 (None: dot only); dot = sum zh.w
        raise NotImplementedError


class DistUzawa:
    """Time-partitioned damped two-stage inexact Uzawa (solvers.py:177-264).

    ``begin()`` computes the reference norm (solvers.py:212-217); each
    ``step()`` is one iteration (solvers.py:224-233) and returns the residual
    numerator sqrt(max(sum r1.dp + sum z.y, 0)), identical on every rank."""

    def __init__(self, ops: LocalOps, comm, N: int, n: int, f_local: torch.Tensor,
                 initial=None, chunks: int = 4):
        self.ops, self.comm = ops, comm
        self.dev = f_local.device
        self.tr = tr = Transposer(comm, N, n, chunks)
        nl = self.nl = tr.nl
        if f_local.shape != (nl, n):
            raise InputError(f"local rhs has shape {tuple(f_local.shape)}, expected {(nl, n)}")
        self.N, self.n = N, n
        self.f = f_local
        kw = dict(dtype=torch.float64, device=self.dev)
        self.u_ext = torch.zeros((nl + 2, n), **kw)
        self.p_ext = torch.zeros((nl + 2, n), **kw)
        if initial is not None:
            self.p_ext[1:nl + 1].copy_(initial[0])
            self.u_ext[1:nl + 1].copy_(initial[1])
        self.u, self.p = self.u_ext[1:nl + 1], self.p_ext[1:nl + 1]
        self.r1 = torch.empty((nl, n), **kw)
        self.z = torch.empty((nl, n), **kw)
        self.zh = torch.empty((nl, n), **kw)
        self.w = torch.empty((nl, n), **kw)
        self.dots = torch.zeros(2, **kw)
        self.single = comm.world == 1

    def _transform(self, kind):
        ops = self.ops

        def run(x, out):
            ops.dst_cols(kind, x, out)

        return run

    def _modes(self, x, out):
        """out = S x (mode-sharded rows) for the time-sharded slab x."""
        if self.single:
            self.ops.dst_cols(1, x, out)
        else:
            self.tr.apply(x, self._transform(1), out)

    def begin(self) -> float:
        self.ops.atilde_update(self.f, None, self.dots[0:1])
        self._modes(self.f, self.zh)
        self.ops.htilde_modes(self.zh, None, self.dots[1:2])
        self.comm.allreduce_(self.dots)
        a, h = (float(v) for v in self.dots.cpu())
        return float(np.sqrt(max(a + h, 0.0)))

    def step(self, omega: float) -> float:
        ops, comm, nl = self.ops, self.comm, self.nl
        comm.halo(self.u_ext, nl, prev=True, nxt=True)
        ops.r1(self.u_ext, self.p_ext, self.f, self.r1)
        ops.atilde_update(self.r1, self.p_ext, self.dots[0:1])
        comm.halo(self.p_ext, nl, prev=False, nxt=True)
        ops.z(self.u_ext, self.p_ext, self.f, self.z)
        self._modes(self.z, self.zh)
        ops.htilde_modes(self.zh, self.w, self.dots[1:2])
        # u += omega S^T w   (y = H~^{-1} z never materialised time-sharded)
        if self.single:
            ops.dst_cols(0, self.w, self.u, base=self.u, alpha=omega)
        else:
            self.tr.apply(self.w, self._transform(0), self.u, omega=omega)
        comm.allreduce_(self.dots)
        s = self.dots.cpu()  # the one host read per iteration (stopping rule)
        return float(np.sqrt(max(float(s[0]) + float(s[1]), 0.0)))


def dist_uzawa_solve(ops: LocalOps, comm, N: int, n: int, f_local: torch.Tensor,
                     cfg: UzawaConfig, initial=None, chunks: int = 4):
    """uzawa_solve (solvers.py:177-264) on a time-partitioned problem.
    Returns (p_local, u_local, ConvergenceHistory) on every rank."""
    if cfg.diagnostics or cfg.stopping == "s_norm_error":
        raise InputError("diagnostic stopping is not available on the partitioned path")
    it = DistUzawa(ops, comm, N, n, f_local, initial, chunks)
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
    """libpint building blocks for this rank's steps / modes (CUDA tensors):
    2D and 3D problems with stencil operators, and 2D per-point stiffness
    fields (BASELINE config 4: every rank holds the coefficient fields of
    its own steps, or the term tables of a separable family, the A_ref field
    and the H~ hierarchies of its own modes)."""

    def __init__(self, spec, hierarchy, part: Partition, rank: int, device=None,
                 damping: float | None = None):
        from ._device import HostProblem
        from ._native import MG_ATILDE, MG_HTILDE, Context
        from .schur import frequency_weights

        from .linalg import grid_fields

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
        mu = frequency_weights(self.N)[sl]
        if hp.field is not None:
            self._upload_fields(hp, spec, sl, grid_fields)
            ctx.call("pint_mg_set_field", MG_ATILDE, len(lm), lm.ctypes.data, float(damping), None)
            mu = np.ascontiguousarray(mu, dtype=np.float64)
            ctx.call("pint_mg_set_field", MG_HTILDE, len(lm), lm.ctypes.data, float(damping),
                     mu.ctypes.data)
            return
        tab_a, sid_a = hp.atilde_tables(hierarchy, damping)
        tab_a = np.ascontiguousarray(tab_a)
        sid_a = np.ascontiguousarray(sid_a[sl])
        ctx.call("pint_mg_set", MG_ATILDE, len(lm), lm.ctypes.data, tab_a.shape[1],
                 tab_a.ctypes.data, sid_a.ctypes.data)
        tab_h, _ = hp.htilde_tables(hierarchy, damping, mu)
        tab_h = np.ascontiguousarray(tab_h)
        sid_h = np.arange(self.nl, dtype=np.int32)
        ctx.call("pint_mg_set", MG_HTILDE, len(lm), lm.ctypes.data, self.nl,
                 tab_h.ctypes.data, sid_h.ctypes.data)

    _FIELD_CHUNK = 32

    def _upload_fields(self, hp, spec, sl, grid_fields):
        """Coefficient fields of the local steps (GpuProblem._upload_fields on
        the slice) and the A_ref field, which every rank needs in full."""
        ctx, fam = self.ctx, spec.stiffness
        if hp.field == "family" and fam.terms is not None:
            a, c = fam.terms
            c = np.ascontiguousarray(c[sl])
            ctx.call("pint_field_separable", int(a.shape[0]), a.ctypes.data, c.ctypes.data)
        elif hp.field == "family":
            for k0 in range(0, self.nl, self._FIELD_CHUNK):
                k1 = min(self.nl, k0 + self._FIELD_CHUNK)
                w = np.ascontiguousarray(fam.cell_weights(self.n0 + k0, self.n0 + k1))
                ctx.call("pint_field_assemble", k0, k1 - k0, w.ctypes.data)
        else:
            for k in range(self.nl):
                f = np.ascontiguousarray(grid_fields(spec.stiffness[self.n0 + k], hp.m))
                ctx.call("pint_field_set", k, 1, f.ctypes.data)
        f = np.ascontiguousarray(grid_fields(spec.a_ref, hp.m))
        ctx.call("pint_field_aref", 0, f.ctypes.data)

    def r1(self, u_ext, p_ext, f, out):
        self.ctx.call("pint_residual_r1", u_ext[1].data_ptr(), p_ext[1].data_ptr(),
                      f.data_ptr(), out.data_ptr())

    def z(self, u_ext, p_ext, f, out):
        self.ctx.call("pint_residual_z", u_ext[1].data_ptr(), p_ext[1].data_ptr(),
                      f.data_ptr(), out.data_ptr())

    def atilde_update(self, r1, p_ext, dot):
        self.ctx.call("pint_atilde_update", r1.data_ptr(),
                      None if p_ext is None else p_ext[1].data_ptr(),
                      ctypes.cast(dot.data_ptr(), ctypes.POINTER(ctypes.c_double)))

    def dst_cols(self, kind, x, out, base=None, alpha=1.0):
        x = x.contiguous()
        if base is None:
            self.ctx.call("pint_dst_raw", int(kind), int(x.shape[0]), int(x.shape[1]),
                          x.data_ptr(), out.data_ptr())
        else:
            self.ctx.call("pint_dst_raw_axpy", int(kind), int(x.shape[0]), int(x.shape[1]),
                          x.data_ptr(), out.data_ptr(), base.data_ptr(), float(alpha))

    def htilde_modes(self, zh, w, dot):
        self.ctx.call("pint_htilde_modes", zh.data_ptr(), None if w is None else w.data_ptr(),
                      ctypes.cast(dot.data_ptr(), ctypes.POINTER(ctypes.c_double)))


# ----------------------------------------------------------------------------
# torchrun worker: python -m torch.distributed.run --nproc-per-node G
#     -m paper_1802_08126_b200.distributed --space 3d --h 64 --N 512 ...
# prints "scaling,<s/iter>,<total s>,<fft share>,<spatial share>" on rank 0
# (cli.py scaling; the shares are not split per phase on this path: 0)
# ----------------------------------------------------------------------------

def _worker_main(argv=None) -> int:
    from . import build_mg_hierarchy, build_time_grid, make_heat_problem

    ap = argparse.ArgumentParser()
    ap.add_argument("--space", default="2d")
    ap.add_argument("--h", type=int, default=32)
    ap.add_argument("--N", type=int, default=256)
    ap.add_argument("--T", type=float, default=1.0)
    ap.add_argument("--omega", type=float, default=0.9)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--repeats", type=int, default=5)
    ap.add_argument("--chunks", type=int, default=4)
    args = ap.parse_args(argv)
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        comm = Comm()
        spec = make_heat_problem(args.space, args.h, build_time_grid("uniform", args.N, args.T),
                                 data="sine")
        part = Partition(args.N, comm.world)
        ops = GpuLocalOps(spec, build_mg_hierarchy(args.space, args.h), part, comm.rank,
                          device=local)
        f_all = spec.grid.steps[:, None] * spec.load
        f_all[0] += spec.mass.dot(spec.u_init)      # fold_rhs (operators.py:22-26)
        f = torch.from_numpy(np.ascontiguousarray(f_all[part.slice(comm.rank)])).to(ops.dev)
        times = []
        for _ in range(args.repeats + 1):
            it = DistUzawa(ops, comm, args.N, spec.dim, f, chunks=args.chunks)
            it.begin()
            dist.barrier()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.iters):
                it.step(args.omega)
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / 1e3], device=ops.dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            times.append(float(t.item()))
        total = float(np.median(times[1:]))
        if comm.rank == 0:
            print(f"scaling,{total / args.iters!r},{total!r},0.0,0.0", flush=True)
    finally:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(_worker_main())
