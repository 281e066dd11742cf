"""TEST INFRASTRUCTURE ONLY -- CPU restatement of the reference Uzawa path.

Restates, in plain numpy/scipy, the algorithm of the reference package
``pintsolve`` for the hot path named by BASELINE.json ``north_star``:
the damped inexact-Uzawa iteration on the time-global implicit-Euler saddle
system with a DST-diagonalised Schur preconditioner and geometric-multigrid
spatial solves.  Each function cites the reference ``file:line`` (paths
relative to ``/root/reference/pkg/src/pintsolve/``) whose arithmetic it
follows.  It reuses the reference's own third-party kernels (scipy CSR
SpMV/SpGEMM, SuperLU, ``scipy.fft.dst``) and the same association order so
that it is bit-identical to the reference on the same inputs
(pinned by ``tests/test_oracle.py`` against ``tests/golden``).

Import rule: only tests/, __graft_entry__.smoke() and bench.py's CPU legs may
use this module.  The product never does.

Extensions beyond the reference (marked EXTENSION) cover what BASELINE.json's
configs need and the reference lacks: a 3D P1 (Kuhn split) discretisation with
trilinear multigrid, and a variable coefficient a(x, t) stiffness.  They are
written in the same style as the 1D/2D code they extend; their parity is
pinned only against this oracle itself (there is no reference output).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np
import scipy.fft
import scipy.sparse as sp
import scipy.sparse.linalg as spla

__all__ = [
    "OracleInputError", "OracleDivergence", "OracleNotSpd",
    "SymOp", "sym_add", "LUFactor",
    "time_nodes", "p1_1d", "p1_2d", "p1_3d", "stiffness_2d_weighted",
    "Problem", "heat_problem",
    "fold_rhs", "stiffness_scales", "op_K", "op_Kt", "op_Abd",
    "MgLevels", "mg_levels", "VCycle",
    "dst_kernel", "dst_forward", "dst_inverse", "dst_forward_T", "dst_inverse_T",
    "frequency_weights", "SchurInv", "BlockInv",
    "UzawaResult", "uzawa", "sequential_euler", "ExactNorms",
    "MinresResult", "op_saddle", "minres",
    "set_num_threads", "get_num_threads",
]


class OracleInputError(ValueError):
    """errors.py:4-5 (InputError) restated."""


class OracleDivergence(RuntimeError):
    """errors.py:20-21 (SolverDivergenceError) restated."""


class OracleNotSpd(ValueError):
    """errors.py:12-13 (NotSpdError) restated."""


# ----------------------------------------------------------------------------
# symmetric sparse operators  (linalg.py:24-127, 150-177)
# ----------------------------------------------------------------------------

class SymOp:
    """Symmetric sparse operator, canonical upper triangle + full CSR.

    Restates ``SpatialMatrix`` (linalg.py:24-115): triplets are folded into
    the upper triangle and duplicates summed (linalg.py:37-44), then the full
    matrix is materialised once as CSR (linalg.py:49-59).  ``scaled`` keeps a
    proportionality root (linalg.py:99-112).
    """

    def __init__(self, dim: int, rows, cols, vals):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        swap = rows > cols
        ur = np.where(swap, cols, rows)
        uc = np.where(swap, rows, cols)
        up = sp.coo_matrix((vals, (ur, uc)), shape=(dim, dim)).tocsr()
        up.sum_duplicates()
        up = up.tocoo()
        self.dim = int(dim)
        self.rows, self.cols, self.vals = up.row, up.col, up.data
        off = self.rows < self.cols
        self.csr = sp.coo_matrix(
            (np.concatenate([self.vals, self.vals[off]]),
             (np.concatenate([self.rows, self.cols[off]]),
              np.concatenate([self.cols, self.rows[off]]))),
            shape=(dim, dim)).tocsr()
        self.root = self
        self.scale = 1.0

    @classmethod
    def from_upper_of(cls, m) -> "SymOp":
        """linalg.py:66-69 (``from_sparse``)."""
        coo = sp.coo_matrix(m)
        keep = coo.row <= coo.col
        return cls(coo.shape[0], coo.row[keep], coo.col[keep], coo.data[keep])

    def scaled(self, c: float) -> "SymOp":
        out = SymOp(self.dim, self.rows, self.cols, c * self.vals)
        out.root = self.root
        out.scale = c * self.scale
        return out

    def ratio_to(self, other: "SymOp"):
        if self.root is other.root:
            return self.scale / other.scale
        return None

    def diagonal(self) -> np.ndarray:
        return self.csr.diagonal()

    def dot(self, x):
        return self.csr.dot(x)

    def dense(self) -> np.ndarray:
        return self.csr.toarray()


def sym_add(a: float, x: SymOp, b: float, y: SymOp) -> SymOp:
    """a*X + b*Y via triplet concatenation (linalg.py:118-127)."""
    return SymOp(x.dim, np.concatenate([x.rows, y.rows]),
                 np.concatenate([x.cols, y.cols]),
                 np.concatenate([a * x.vals, b * y.vals]))


class LUFactor:
    """SuperLU factor with no off-diagonal pivoting (linalg.py:150-177)."""

    def __init__(self, op):
        m = op.csr if isinstance(op, SymOp) else sp.csr_matrix(op)
        self.dim = m.shape[0]
        try:
            self.lu = spla.splu(m.tocsc(), permc_spec="MMD_AT_PLUS_A",
                                diag_pivot_thresh=0.0,
                                options={"SymmetricMode": True})
        except RuntimeError as exc:
            raise OracleNotSpd(str(exc)) from exc
        if np.any(self.lu.U.diagonal() <= 0.0):
            raise OracleNotSpd("non-positive pivot")

    def solve(self, b):
        b = np.asarray(b, dtype=np.float64)
        if b.ndim == 2 and b.shape[0] != self.dim and b.shape[1] == self.dim:
            return self.lu.solve(b.T).T
        return self.lu.solve(b)


# ----------------------------------------------------------------------------
# discretisation  (problems.py:53-138)
# ----------------------------------------------------------------------------

def time_nodes(kind: str, N: int, T: float, perturbation: float = 0.0,
               seed: int = 0) -> np.ndarray:
    """Uniform or seeded quasi-uniform grid nodes (problems.py:53-75)."""
    if N < 1 or T <= 0.0:
        raise OracleInputError("bad time grid")
    if kind == "uniform":
        w = np.ones(N)
    elif kind == "perturbed":
        w = 1.0 + perturbation * np.random.default_rng(seed).uniform(-1.0, 1.0, N)
    else:
        raise OracleInputError(kind)
    tau = T * w / w.sum()
    return np.concatenate([[0.0], np.cumsum(tau)])


def p1_1d(cells: int):
    """P1 mass/stiffness on (0,1), Dirichlet (problems.py:78-90)."""
    h = 1.0 / cells
    n = cells - 1
    d = np.arange(n)
    o = np.arange(n - 1)
    r = np.concatenate([d, o])
    c = np.concatenate([d, o + 1])
    m = np.concatenate([np.full(n, 4 * h / 6), np.full(n - 1, h / 6)])
    a = np.concatenate([np.full(n, 2.0 / h), np.full(n - 1, -1.0 / h)])
    return SymOp(n, r, c, m), SymOp(n, r, c, a)


_K2 = 0.5 * np.array([[2.0, -1.0, -1.0], [-1.0, 1.0, 0.0], [-1.0, 0.0, 1.0]])
_M2 = np.array([[2.0, 1.0, 1.0], [1.0, 2.0, 1.0], [1.0, 1.0, 2.0]]) / 12.0


def _tri_triplets(cells: int):
    """Element node lists of the structured diagonal split, in the
    reference's element order (problems.py:114-121): cell (i, j) with i
    fastest, triangles (lr, ur, ll) then (ul, ll, ur)."""
    c = cells
    j, i = np.meshgrid(np.arange(c), np.arange(c), indexing="ij")
    i = i.ravel()
    j = j.ravel()
    ll = j * (c + 1) + i
    lr = ll + 1
    ul = ll + (c + 1)
    ur = ul + 1
    t1 = np.stack([lr, ur, ll], axis=1)
    t2 = np.stack([ul, ll, ur], axis=1)
    return np.stack([t1, t2], axis=1).reshape(-1, 3)


def _assemble_p1_2d(cells: int, elem_stiff_weight=None):
    c = cells
    h = 1.0 / c
    tris = _tri_triplets(c)
    rows = np.repeat(tris, 3, axis=1).ravel()          # a outer, b inner
    cols = np.tile(tris, (1, 3)).ravel()
    area = 0.5 * h * h
    mvals = np.tile((area * _M2).ravel(), len(tris))
    if elem_stiff_weight is None:
        avals = np.tile(_K2.ravel(), len(tris))
    else:  # EXTENSION: per-triangle weights w_e * K_el (order as above)
        avals = (elem_stiff_weight[:, None] * _K2.ravel()[None, :]).ravel()
    nn = (c + 1) * (c + 1)
    mfull = sp.coo_matrix((mvals, (rows, cols)), shape=(nn, nn)).tocsr()
    afull = sp.coo_matrix((avals, (rows, cols)), shape=(nn, nn)).tocsr()
    jj, ii = np.meshgrid(np.arange(1, c), np.arange(1, c), indexing="ij")
    interior = (jj * (c + 1) + ii).ravel().astype(np.int64)
    return (SymOp.from_upper_of(mfull[np.ix_(interior, interior)]),
            SymOp.from_upper_of(afull[np.ix_(interior, interior)]))


def p1_2d(cells: int):
    """P1 on the unit square, lower-left/upper-right diagonal split,
    interior nodes j*(c-1)+i (problems.py:99-138)."""
    if cells < 2:
        raise OracleInputError("need at least 2 cells per side")
    return _assemble_p1_2d(cells)


def stiffness_2d_weighted(cells: int, weight: np.ndarray) -> SymOp:
    """EXTENSION (config 4): stiffness of -div(a grad u) with a piecewise
    constant per cell, ``weight[j, i]`` for cell (i, j); both triangles of a
    cell carry the cell weight.  Same assembly path as problems.py:99-138."""
    w = np.repeat(np.asarray(weight, dtype=np.float64).reshape(-1), 2)
    return _assemble_p1_2d(cells, elem_stiff_weight=w)[1]


# EXTENSION (configs 3 and 5): P1 on the Kuhn 6-tetrahedron split of each
# cube, the 3D analogue of the 2D diagonal split.  Vertex bit k of a cube
# corner is the offset along axis k (x = bit 0).  Each tetrahedron follows
# one monotone path 0 -> e_a -> e_a+e_b -> (1,1,1).
_KUHN = [(0, 1, 3, 7), (0, 1, 5, 7), (0, 2, 3, 7), (0, 2, 6, 7), (0, 4, 5, 7), (0, 4, 6, 7)]


def _tet_element(h: float, corners):
    pts = np.array([[(v >> 0) & 1, (v >> 1) & 1, (v >> 2) & 1] for v in corners],
                   dtype=np.float64) * h
    jac = (pts[1:] - pts[0]).T / h                         # 0/1 matrix, det +-1
    vol = h * h * h / 6.0
    ginv = np.round(np.linalg.inv(jac))                     # exact integer inverse
    grads = np.vstack([-ginv.sum(axis=0), ginv])           # rows: h * grad of basis
    kel = (vol / (h * h)) * (grads @ grads.T)
    mel = vol / 20.0 * (np.ones((4, 4)) + np.eye(4))
    return mel, kel


def p1_3d(cells: int):
    """EXTENSION: P1 mass/stiffness on the unit cube (Kuhn split), interior
    nodes ordered (k*(c-1) + j)*(c-1) + i, x fastest."""
    if cells < 2:
        raise OracleInputError("need at least 2 cells per side")
    c = cells
    h = 1.0 / c
    c1 = c + 1
    rows, cols, mv, av = [], [], [], []
    k, j, i = np.meshgrid(np.arange(c), np.arange(c), np.arange(c), indexing="ij")
    base = ((k * c1 + j) * c1 + i).ravel()
    for tet in _KUHN:
        mel, kel = _tet_element(h, tet)
        nodes = [base + ((v >> 2) & 1) * c1 * c1 + ((v >> 1) & 1) * c1 + (v & 1) for v in tet]
        for a in range(4):
            for b in range(4):
                rows.append(nodes[a])
                cols.append(nodes[b])
                mv.append(np.full(base.size, mel[a, b]))
                av.append(np.full(base.size, kel[a, b]))
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    nn = c1 ** 3
    mfull = sp.coo_matrix((np.concatenate(mv), (rows, cols)), shape=(nn, nn)).tocsr()
    afull = sp.coo_matrix((np.concatenate(av), (rows, cols)), shape=(nn, nn)).tocsr()
    kk, jj, ii = np.meshgrid(np.arange(1, c), np.arange(1, c), np.arange(1, c), indexing="ij")
    interior = ((kk * c1 + jj) * c1 + ii).ravel().astype(np.int64)
    return (SymOp.from_upper_of(mfull[np.ix_(interior, interior)]),
            SymOp.from_upper_of(afull[np.ix_(interior, interior)]))


@dataclass
class Problem:
    """Restates ``ProblemSpec`` (problems.py:153-182)."""

    mass: SymOp
    stiffness: list
    nodes: np.ndarray
    load: np.ndarray
    u_init: np.ndarray
    tau_ref: float
    a_ref: SymOp
    space: str
    cells: int
    meta: dict = field(default_factory=dict)

    @property
    def steps(self) -> np.ndarray:
        return np.diff(self.nodes)

    @property
    def N(self) -> int:
        return len(self.nodes) - 1

    @property
    def dim(self) -> int:
        return self.mass.dim


def heat_problem(space: str, cells: int, nodes: np.ndarray,
                 coeff: Callable[[float], float] | None = None,
                 load: np.ndarray | None = None, u_init: np.ndarray | None = None,
                 data: str | None = None, seed: int = 0,
                 stiffness: Sequence[SymOp] | None = None,
                 tau_ref: float | None = None, a_ref: SymOp | None = None) -> Problem:
    """Heat problem (problems.py:228-297) with explicit data or one of the
    reference data descriptors (problems.py:263-280)."""
    mass, a0 = {"1d": p1_1d, "2d": p1_2d, "3d": p1_3d}[space](cells)
    N = len(nodes) - 1
    n = mass.dim
    if stiffness is None:
        cf = coeff if coeff is not None else (lambda t: 1.0)
        cv = np.array([cf(t) for t in nodes[1:]], dtype=np.float64)
        if np.any(cv <= 0.0):
            raise OracleInputError("diffusion coefficient must be positive")
        stiffness = [a0 if s == 1.0 else a0.scaled(float(s)) for s in cv]
    stiffness = list(stiffness)
    if data is not None:
        if data == "zero":
            u_init, load = np.zeros(n), np.zeros((N, n))
        elif data == "random":
            rng = np.random.default_rng(seed)
            u_init = rng.standard_normal(n)
            load = rng.standard_normal((N, n))
        elif data == "sine":
            u_init = _sine(space, cells)
            load = np.zeros((N, n))
        else:
            raise OracleInputError(data)
    if load is None:
        load = np.zeros((N, n))
    if u_init is None:
        u_init = np.zeros(n)
    steps = np.diff(nodes)
    if tau_ref is None:
        tau_ref = float(np.exp(np.mean(np.log(steps))))
    if a_ref is None:
        a_ref = stiffness[math.ceil(N / 2) - 1]
    return Problem(mass, stiffness, np.asarray(nodes, dtype=np.float64),
                   np.asarray(load, dtype=np.float64), np.asarray(u_init, dtype=np.float64),
                   float(tau_ref), a_ref, space, cells)


def _sine(space: str, cells: int) -> np.ndarray:
    """problems.py:219-225."""
    g = np.arange(1, cells) / cells
    if space == "1d":
        return np.sin(np.pi * g)
    if space == "2d":
        x, y = np.meshgrid(g, g)
        return np.sin(np.pi * x.ravel()) * np.sin(np.pi * y.ravel())
    z, y, x = np.meshgrid(g, g, g, indexing="ij")
    return (np.sin(np.pi * x) * np.sin(np.pi * y) * np.sin(np.pi * z)).ravel()


# ----------------------------------------------------------------------------
# time-global operators  (operators.py:22-99)
# ----------------------------------------------------------------------------

def fold_rhs(pb: Problem) -> np.ndarray:
    """f_n = tau_n load_n, plus M u_I on block 1 (operators.py:22-26)."""
    f = pb.steps[:, None] * pb.load
    f[0] += pb.mass.dot(pb.u_init)
    return f


def stiffness_scales(pb: Problem):
    """c_n tau_n when every A_n is a known multiple of A_1, else None
    (operators.py:41-49)."""
    first = pb.stiffness[0]
    s = np.empty(pb.N)
    for k, a in enumerate(pb.stiffness):
        r = a.ratio_to(first)
        if r is None:
            return None
        s[k] = r
    return s * pb.steps


def op_K(pb: Problem, u: np.ndarray) -> np.ndarray:
    """M u_n - M u_{n-1} (operators.py:78-83)."""
    mu = pb.mass.dot(u.T).T
    out = mu.copy()
    out[1:] -= mu[:-1]
    return out


def op_Kt(pb: Problem, u: np.ndarray) -> np.ndarray:
    """M u_n - M u_{n+1} (operators.py:85-90)."""
    mu = pb.mass.dot(u.T).T
    out = mu.copy()
    out[:-1] -= mu[1:]
    return out


def op_Abd(pb: Problem, u: np.ndarray, scales=None) -> np.ndarray:
    """tau_n A_n u_n (operators.py:92-99)."""
    if scales is None:
        scales = stiffness_scales(pb)
    if scales is not None:
        return scales[:, None] * pb.stiffness[0].dot(u.T).T
    return np.stack([t * a.dot(v) for t, a, v in zip(pb.steps, pb.stiffness, u)])


# ----------------------------------------------------------------------------
# geometric multigrid  (spatial.py:75-169)
# ----------------------------------------------------------------------------

def _interp_1d(coarse_cells: int) -> sp.csr_matrix:
    """Linear interpolation (spatial.py:75-84)."""
    nf, nc = 2 * coarse_cells - 1, coarse_cells - 1
    j = np.arange(nc)
    r = np.concatenate([2 * j + 1, 2 * j, 2 * j + 2])
    c = np.concatenate([j, j, j])
    v = np.concatenate([np.ones(nc), np.full(nc, 0.5), np.full(nc, 0.5)])
    return sp.coo_matrix((v, (r, c)), shape=(nf, nc)).tocsr()


@dataclass
class MgLevels:
    space: str
    cells: list
    prolong: list


def mg_levels(space: str, fine_cells: int) -> MgLevels:
    """Halve cells down to 2 or 3 (spatial.py:100-113); 2D/3D transfers are
    Kronecker products of the 1D interpolation (3D: EXTENSION)."""
    if fine_cells < 4 or fine_cells & (fine_cells - 1):
        raise OracleInputError("fine cell count must be a power of two >= 4")
    cells = [fine_cells]
    while cells[-1] // 2 >= 2 and cells[-1] > 3:
        cells.append(cells[-1] // 2)
    pro = []
    for c in cells[1:]:
        p1 = _interp_1d(c)
        if space == "1d":
            pro.append(p1)
        elif space == "2d":
            pro.append(sp.kron(p1, p1).tocsr())
        elif space == "3d":
            pro.append(sp.kron(sp.kron(p1, p1), p1).tocsr())
        else:
            raise OracleInputError(space)
    return MgLevels(space, cells, pro)


_DAMPING = {"1d": 2.0 / 3.0, "2d": 4.0 / 5.0, "3d": 6.0 / 7.0}   # 3d: EXTENSION


class VCycle:
    """Symmetric V-cycle, damped Jacobi, Galerkin coarse operators, direct
    coarsest solve (spatial.py:116-169)."""

    def __init__(self, op: SymOp, levels: MgLevels, cycles: int = 1,
                 smooth_steps: int = 1, damping: float | None = None):
        self.levels = levels
        self.cycles = cycles
        self.smooth = smooth_steps
        self.damping = _DAMPING[levels.space] if damping is None else damping
        mats = [op.csr]
        for p in levels.prolong:
            mats.append((p.T @ mats[-1] @ p).tocsr())
        self.mats = mats
        self.dinv = [self.damping / np.asarray(m.diagonal()) for m in mats]
        self.coarse = LUFactor(SymOp.from_upper_of(mats[-1]))

    def _cycle(self, lev: int, b: np.ndarray) -> np.ndarray:
        if lev == len(self.mats) - 1:
            return self.coarse.solve(b)
        a, d = self.mats[lev], self.dinv[lev]
        x = d * b
        for _ in range(self.smooth - 1):
            x += d * (b - a.dot(x))
        p = self.levels.prolong[lev]
        x = x + p.dot(self._cycle(lev + 1, p.T.dot(b - a.dot(x))))
        for _ in range(self.smooth):
            x += d * (b - a.dot(x))
        return x

    def apply(self, b: np.ndarray) -> np.ndarray:
        x = self._cycle(0, b)
        for _ in range(self.cycles - 1):
            x += self._cycle(0, b - self.mats[0].dot(x))
        return x


# ----------------------------------------------------------------------------
# sine transforms in time  (dst.py:31-102)
# ----------------------------------------------------------------------------

def _pow2(n: int) -> bool:
    return n >= 1 and n & (n - 1) == 0


def dst_kernel(N: int) -> np.ndarray:
    """sin((2k-1) n pi / 2N), k rows, n columns (dst.py:40-47)."""
    k = np.arange(1, N + 1)[:, None]
    n = np.arange(1, N + 1)[None, :]
    return np.sin((2 * k - 1) * n * np.pi / (2 * N))


def dst_forward(u: np.ndarray) -> np.ndarray:
    """Weighted type-III analysis map (dst.py:57-65)."""
    N = u.shape[0]
    if _pow2(N):
        return scipy.fft.dst(u, type=3, axis=0) / N
    w = u.copy()
    w[-1] *= 0.5
    return (2.0 / N) * np.tensordot(dst_kernel(N), w, axes=(1, 0))


def dst_inverse(uh: np.ndarray) -> np.ndarray:
    """u_n = sum_k uh_k sin(...) (dst.py:67-73)."""
    N = uh.shape[0]
    if _pow2(N):
        return scipy.fft.dst(uh, type=2, axis=0) / 2.0
    return np.tensordot(dst_kernel(N).T, uh, axes=(1, 0))


def dst_forward_T(v: np.ndarray) -> np.ndarray:
    """dst.py:75-84."""
    N = v.shape[0]
    if _pow2(N):
        out = scipy.fft.dst(v, type=2, axis=0) / N
    else:
        out = (2.0 / N) * np.tensordot(dst_kernel(N).T, v, axes=(1, 0))
    out[-1] *= 0.5
    return out


def dst_inverse_T(u: np.ndarray) -> np.ndarray:
    """r_k = sum_n u_n sin(...) (dst.py:86-93)."""
    N = u.shape[0]
    if _pow2(N):
        w = u.copy()
        w[-1] *= 2.0
        return scipy.fft.dst(w, type=3, axis=0) / 2.0
    return np.tensordot(dst_kernel(N), u, axes=(1, 0))


# ----------------------------------------------------------------------------
# preconditioners  (schur.py:21-76, solvers.py:127-150)
# ----------------------------------------------------------------------------

def frequency_weights(N: int) -> np.ndarray:
    """mu_k = 2 sin((2k-1) pi / 4N) (schur.py:21-24)."""
    k = np.arange(1, N + 1)
    return 2.0 * np.sin((2 * k - 1) * np.pi / (4 * N))


# ----------------------------------------------------------------------------
# thread pool of the block loops  (parallel.py:19-43)
# ----------------------------------------------------------------------------

_POOL = None
_THREADS = 1


def set_num_threads(n: int) -> None:
    """Process-wide pool for the per-step / per-mode loops of BlockInv and
    SchurInv (parallel.py:19-29); 1 = serial.  Slots are disjoint, so results
    do not depend on the thread count (parallel.py:1-6)."""
    global _POOL, _THREADS
    if n < 1:
        raise OracleInputError("thread count must be >= 1")
    if _POOL is not None:
        _POOL.shutdown(wait=True)
        _POOL = None
    _THREADS = n
    if n > 1:
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(max_workers=n)


def get_num_threads() -> int:
    return _THREADS


def _block_map(fn, count: int) -> None:
    """fn(k) for k < count, on the pool when there is one (parallel.py:36-43)."""
    if _POOL is None or count < 2:
        for k in range(count):
            fn(k)
    else:
        list(_POOL.map(fn, range(count)))


class SchurInv:
    """H~^{-1} = Phi^{-1} diag(scale * H_k^{-1} A_ref H_k^{-1}) Phi^{-T}
    with one MG V-cycle per H_k^{-1} (schur.py:30-52, 62-76)."""

    def __init__(self, pb: Problem, levels: MgLevels, cycles: int = 1,
                 smooth_steps: int = 1, dense_dst: bool = False):
        # dense_dst: evaluate both transforms with the dense sine kernel, the
        # reference's own non-power-of-two path (dst.py:64,73,81,93); used to
        # measure the reference's intrinsic reassociation noise
        self.dense = dst_kernel(pb.N) if dense_dst else None
        self.N = pb.N
        self.tau_ref = pb.tau_ref
        self.a_ref = pb.a_ref
        self.mu = frequency_weights(self.N)
        ta = pb.a_ref.scaled(pb.tau_ref)
        self.blocks = [sym_add(m, pb.mass, 1.0, ta) for m in self.mu]
        self.solvers = [VCycle(h, levels, cycles, smooth_steps) for h in self.blocks]

    def apply(self, r: np.ndarray) -> np.ndarray:
        rh = dst_inverse_T(r) if self.dense is None else self.dense @ r
        out = np.empty_like(rh)
        s = 2.0 * self.tau_ref / self.N

        def mode(k):  # schur.py:69-75
            sol = self.solvers[k]
            y = sol.apply(rh[k])
            y = self.a_ref.dot(y)
            out[k] = s * sol.apply(y)

        _block_map(mode, len(self.solvers))
        return dst_inverse(out) if self.dense is None else self.dense.T @ out


class BlockInv:
    """A~^{-1}: one V-cycle per step on A_n, divided by tau_n; solvers are
    shared between steps that share the operator object (solvers.py:127-150)."""

    def __init__(self, pb: Problem, levels: MgLevels, cycles: int = 1,
                 smooth_steps: int = 1):
        cache = {}
        self.solvers = []
        for a in pb.stiffness:
            if id(a) not in cache:
                cache[id(a)] = VCycle(a, levels, cycles, smooth_steps)
            self.solvers.append(cache[id(a)])
        self.steps = pb.steps

    def apply(self, b: np.ndarray) -> np.ndarray:
        out = np.empty_like(b)

        def step(k):  # solvers.py:145-149
            out[k] = self.solvers[k].apply(b[k]) / self.steps[k]

        _block_map(step, len(self.solvers))
        return out


# ----------------------------------------------------------------------------
# Uzawa  (solvers.py:177-264)
# ----------------------------------------------------------------------------

@dataclass
class UzawaResult:
    p: np.ndarray
    u: np.ndarray
    residual: list
    converged: bool
    wall: list


def uzawa(pb: Problem, atilde: BlockInv, htilde: SchurInv, omega: float = 0.9,
          tol: float = 1e-8, max_iter: int = 200, initial=None,
          on_iter: Callable | None = None) -> UzawaResult:
    """Damped two-stage inexact Uzawa with the preconditioned-residual stop
    (solvers.py:177-264; diagnostics branch omitted)."""
    f = fold_rhs(pb)
    scales = stiffness_scales(pb)
    if initial is not None:
        p, u = initial[0].copy(), initial[1].copy()
    else:
        p = np.zeros((pb.N, pb.dim))
        u = np.zeros((pb.N, pb.dim))
    ref = np.sqrt(max(np.sum(f * atilde.apply(f)) + np.sum(f * htilde.apply(f)), 0.0))
    res_hist, wall = [], []
    if ref == 0.0:
        return UzawaResult(p, u, res_hist, True, wall)
    first = None
    t0 = time.perf_counter()
    converged = False
    for _ in range(max_iter):
        r1 = op_K(pb, u) - op_Abd(pb, p, scales) - f
        dp = atilde.apply(r1)
        p = p + dp
        z = f - op_Kt(pb, p) - (op_K(pb, u) + op_Kt(pb, u) + op_Abd(pb, u, scales))
        y = htilde.apply(z)
        u = u + omega * y
        res = float(np.sqrt(max(np.sum(r1 * dp) + np.sum(z * y), 0.0))) / ref
        if first is None:
            first = max(res, 1e-300)
        res_hist.append(res)
        wall.append(time.perf_counter() - t0)
        if on_iter is not None:
            on_iter(len(res_hist), res)
        if res > 1e6 * first:
            raise OracleDivergence(f"residual grew to {res:.3e} from {first:.3e}")
        if res < tol:
            converged = True
            break
    return UzawaResult(p, u, res_hist, converged, wall)


@dataclass
class MinresResult:
    p: np.ndarray
    u: np.ndarray
    residual: list
    converged: bool


def op_saddle(pb: Problem, p: np.ndarray, u: np.ndarray, scales=None):
    """Symmetric indefinite 2x2 block operator (operators.py:107-111)."""
    top = op_Abd(pb, p, scales) - op_K(pb, u)
    bottom = -op_Kt(pb, p) - (op_K(pb, u) + op_Kt(pb, u) + op_Abd(pb, u, scales))
    return top, bottom


def minres(pb: Problem, atilde: BlockInv, htilde: SchurInv, tol: float = 1e-8,
           max_iter: int = 500) -> MinresResult:
    """Block-diagonally preconditioned MINRES on the saddle-point system
    (solvers.py:267-327): scipy.sparse.linalg.minres (the reference's own
    dependency, Paige-Saunders) with the reference's callback, which records
    the true preconditioned residual of every iterate."""
    import scipy.sparse.linalg as spla

    f = fold_rhs(pb)
    scales = stiffness_scales(pb)
    N, n = pb.N, pb.dim
    nd = N * n
    g = np.concatenate([-f.ravel(), -f.ravel()])

    def matvec(w):
        top, bottom = op_saddle(pb, w[:nd].reshape(N, n), w[nd:].reshape(N, n), scales)
        return np.concatenate([top.ravel(), bottom.ravel()])

    def precond(w):
        return np.concatenate([atilde.apply(w[:nd].reshape(N, n)).ravel(),
                               htilde.apply(w[nd:].reshape(N, n)).ravel()])

    rng = np.random.default_rng(1234)
    for _ in range(3):
        w = rng.standard_normal(2 * nd)
        if w @ precond(w) <= 0.0:
            raise OracleNotSpd("block preconditioner is not positive definite")
    op = spla.LinearOperator((2 * nd, 2 * nd), matvec=matvec)
    mop = spla.LinearOperator((2 * nd, 2 * nd), matvec=precond)
    res = []
    ref = float(np.sqrt(g @ precond(g)))
    if ref == 0.0:
        z = np.zeros((N, n))
        return MinresResult(z, z.copy(), res, True)

    def callback(xk):
        r = g - matvec(xk)
        res.append(float(np.sqrt(max(r @ precond(r), 0.0))) / ref)

    w, info = spla.minres(op, g, M=mop, rtol=tol, maxiter=max_iter, callback=callback)
    return MinresResult(w[:nd].reshape(N, n), w[nd:].reshape(N, n), res, info == 0)


def sequential_euler(pb: Problem) -> np.ndarray:
    """Implicit Euler sweep with exact solves (solvers.py:158-174)."""
    fac = {}
    u = np.empty((pb.N, pb.dim))
    prev = pb.u_init
    for n in range(pb.N):
        t = pb.steps[n]
        key = (id(pb.stiffness[n]), t)
        if key not in fac:
            fac[key] = LUFactor(sym_add(1.0, pb.mass, t, pb.stiffness[n]))
        u[n] = fac[key].solve(pb.mass.dot(prev) + t * pb.load[n])
        prev = u[n]
    return u


class ExactNorms:
    """Discrete parabolic S-norm (operators.py:40-49, 127-135, 176-214)."""

    def __init__(self, pb: Problem):
        self.pb = pb
        self.scales = stiffness_scales(pb)
        if self.scales is not None:
            self.base = LUFactor(pb.stiffness[0])
            self.blocks = None
        else:
            self.base = None
            self.blocks = [LUFactor(a.scaled(t)) if t != 1.0 else LUFactor(a)
                           for a, t in zip(pb.stiffness, pb.steps)]

    def _dual(self, u, v) -> float:
        pb = self.pb
        st = pb.steps
        mdu = pb.mass.dot(np.diff(u, axis=0, prepend=0.0).T).T / st[:, None]
        mdv = pb.mass.dot(np.diff(v, axis=0, prepend=0.0).T).T / st[:, None]
        if self.base is not None:
            sol = self.base.solve(mdv.T).T / (self.scales / st)[:, None]
        else:
            sol = np.stack([f.solve(x) * t for f, x, t in zip(self.blocks, mdv, st)])
        return float(np.sum(st[:, None] * mdu * sol))

    def _jump(self, u, v) -> float:
        du = np.diff(u, axis=0, prepend=0.0)
        dv = np.diff(v, axis=0, prepend=0.0)
        m = self.pb.mass
        return float(u[-1] @ m.dot(v[-1]) + np.sum(du * m.dot(dv.T).T))

    def s_bilinear(self, u, v) -> float:
        energy = float(np.sum(u * op_Abd(self.pb, v, self.scales)))
        return self._dual(u, v) + energy + self._jump(u, v)

    def s_norm(self, u) -> float:
        return float(np.sqrt(max(self.s_bilinear(u, u), 0.0)))
