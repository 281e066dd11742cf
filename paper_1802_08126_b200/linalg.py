"""Host-side spatial operators and their translation to GPU stencils.

``SpatialMatrix`` mirrors the reference type (linalg.py:24-115): a symmetric
sparse operator stored as its canonical upper triangle, materialised once as
full CSR, with the proportionality provenance that ``scaled`` records
(linalg.py:99-112).  It is setup-time data: the GPU path never multiplies
with it; :func:`grid_stencil` converts it to the 9 stencil coefficients the
CUDA kernels consume, after checking that the matrix really is a
translation-invariant stencil on the structured grid (the only operators the
reference's assembly produces, problems.py:99-138).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from .errors import DimensionMismatchError, InputError, NotSpdError

DEFAULT_DENSE_EIG_LIMIT = 20_000

# CSR column order of an interior row of a 2D 9-point operator: (dy, dx)
STENCIL_2D = ((-1, -1), (-1, 0), (-1, 1), (0, -1), (0, 0), (0, 1), (1, -1), (1, 0), (1, 1))
# ... and of a 3D 27-point operator: (dz, dy, dx), z slowest (EXTENSION, configs 3/5)
STENCIL_3D = tuple((dz, dy, dx) for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1))


class SpatialMatrix:
    """Symmetric sparse operator with canonical upper-triangle storage."""

    def __init__(self, dim: int, rows, cols, vals):
        if dim <= 0:
            raise InputError("matrix dimension must be positive")
        r = np.asarray(rows, dtype=np.int64)
        c = np.asarray(cols, dtype=np.int64)
        v = np.asarray(vals, dtype=np.float64)
        lo = np.minimum(r, c)
        hi = np.maximum(r, c)
        upper = sp.coo_matrix((v, (lo, hi)), shape=(dim, dim)).tocsr()
        upper.sum_duplicates()
        upper = upper.tocoo()
        self.dim = int(dim)
        self.rows, self.cols, self.vals = upper.row, upper.col, upper.data
        off = self.rows != self.cols
        self._csr = sp.coo_matrix(
            (np.concatenate([self.vals, self.vals[off]]),
             (np.concatenate([self.rows, self.cols[off]]),
              np.concatenate([self.cols, self.rows[off]]))),
            shape=(dim, dim)).tocsr()
        self._base = None
        self._scale = 1.0
        self._stencil = None  # cached (m, coefficients) once verified

    @classmethod
    def from_sparse(cls, m) -> "SpatialMatrix":
        coo = sp.coo_matrix(m)
        keep = coo.row <= coo.col
        return cls(coo.shape[0], coo.row[keep], coo.col[keep], coo.data[keep])

    @classmethod
    def from_dense(cls, m) -> "SpatialMatrix":
        m = np.asarray(m, dtype=np.float64)
        if m.ndim != 2 or m.shape[0] != m.shape[1]:
            raise InputError("matrix must be square")
        if not np.allclose(m, m.T, rtol=1e-12, atol=1e-14 * max(1.0, np.abs(m).max())):
            raise InputError("matrix must be symmetric")
        r, c = np.nonzero(np.triu(m))
        return cls(m.shape[0], r, c, m[r, c])

    @classmethod
    def identity(cls, dim: int) -> "SpatialMatrix":
        i = np.arange(dim)
        return cls(dim, i, i, np.ones(dim))

    def tocsr(self) -> sp.csr_matrix:
        return self._csr

    def todense(self) -> np.ndarray:
        return self._csr.toarray()

    def diagonal(self) -> np.ndarray:
        return self._csr.diagonal()

    def dot(self, x):
        return self._csr.dot(x)

    def __matmul__(self, x):
        return self.dot(x)

    def scaled(self, c: float) -> "SpatialMatrix":
        out = SpatialMatrix(self.dim, self.rows, self.cols, c * self.vals)
        out._base = self._base if self._base is not None else self
        out._scale = c * self._scale
        if self._stencil is not None:
            m, st = self._stencil
            out._stencil = (m, c * st)  # same triplets, same products: still a stencil
        return out

    def proportionality(self, other) -> float | None:
        a = self._base if self._base is not None else self
        b = getattr(other, "_base", None) or other
        if a is b:
            return self._scale / getattr(other, "_scale", 1.0)
        return None


def add_matrices(a: float, x, b: float, y) -> SpatialMatrix:
    """a X + b Y by triplet concatenation (linalg.py:118-127)."""
    if x.dim != y.dim:
        raise DimensionMismatchError("operator dimensions differ")
    return SpatialMatrix(x.dim, np.concatenate([x.rows, y.rows]),
                         np.concatenate([x.cols, y.cols]),
                         np.concatenate([a * x.vals, b * y.vals]))


def spmv(mat, x):
    x = np.asarray(x, dtype=np.float64)
    if x.shape[-1] != mat.dim:
        raise DimensionMismatchError(f"operator dim {mat.dim} does not match vector dim {x.shape[-1]}")
    return mat.dot(x)


def weighted_norm(mat, x) -> float:
    x = np.asarray(x, dtype=np.float64)
    q = float(x @ spmv(mat, x))
    if q < 0.0:
        if q < -1e-14 * float(x @ x):
            raise NotSpdError("negative quadratic form: operator is not SPD")
        q = 0.0
    return float(np.sqrt(q))


def dense_generalized_eig_extremal(a, b, dense_limit: int = DEFAULT_DENSE_EIG_LIMIT):
    """Extremal eigenvalues of A x = lambda B x (linalg.py:188-208); setup only."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    n = a.shape[0]
    if n > dense_limit:
        raise InputError(f"dimension {n} exceeds dense limit {dense_limit}; use the Lanczos path")
    if a.shape != b.shape or a.shape != (n, n):
        raise DimensionMismatchError("pencil matrices must be square of equal size")
    try:
        w = scipy.linalg.eigh(a, b, eigvals_only=True)
    except scipy.linalg.LinAlgError as exc:
        raise NotSpdError(f"B factorization failed: {exc}") from exc
    return float(w[0]), float(w[-1])


def _csr_of(mat) -> sp.csr_matrix:
    if hasattr(mat, "tocsr"):
        return sp.csr_matrix(mat.tocsr())
    return sp.csr_matrix(mat)


def stencil_matrix_2d(st: np.ndarray, m: int) -> sp.csr_matrix:
    """The m^2 x m^2 CSR matrix of a translation-invariant 9-point stencil."""
    st = np.asarray(st, dtype=np.float64)
    j, i = np.divmod(np.arange(m * m), m)
    rows, cols, vals = [], [], []
    for k, (dy, dx) in enumerate(STENCIL_2D):
        if st[k] == 0.0:
            continue
        ok = (j + dy >= 0) & (j + dy < m) & (i + dx >= 0) & (i + dx < m)
        rows.append((j * m + i)[ok])
        cols.append(((j + dy) * m + (i + dx))[ok])
        vals.append(np.full(int(ok.sum()), st[k]))
    if not rows:
        return sp.csr_matrix((m * m, m * m))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(m * m, m * m)).tocsr()


def stencil_matrix_3d(st: np.ndarray, m: int) -> sp.csr_matrix:
    """The m^3 x m^3 CSR matrix of a translation-invariant 27-point stencil."""
    st = np.asarray(st, dtype=np.float64)
    z, rem = np.divmod(np.arange(m ** 3), m * m)
    y, x = np.divmod(rem, m)
    rows, cols, vals = [], [], []
    for k, (dz, dy, dx) in enumerate(STENCIL_3D):
        if st[k] == 0.0:
            continue
        ok = ((z + dz >= 0) & (z + dz < m) & (y + dy >= 0) & (y + dy < m)
              & (x + dx >= 0) & (x + dx < m))
        idx = np.arange(m ** 3)[ok]
        rows.append(idx)
        cols.append(((z[ok] + dz) * m + (y[ok] + dy)) * m + (x[ok] + dx))
        vals.append(np.full(idx.size, st[k]))
    if not rows:
        return sp.csr_matrix((m ** 3, m ** 3))
    return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(m ** 3, m ** 3)).tocsr()


def grid_stencil3(mat, m: int) -> np.ndarray:
    """27-point stencil of a structured-grid operator on an m^3 interior grid
    (EXTENSION): exact translation-invariance check as in grid_stencil."""
    cached = getattr(mat, "_stencil", None)
    if cached is not None and cached[0] == ("3d", m):
        return cached[1].copy()
    csr = _csr_of(mat)
    if csr.shape != (m ** 3, m ** 3):
        raise DimensionMismatchError(f"operator of shape {csr.shape} is not on a {m}^3 grid")
    coo = csr.tocoo()
    zr, rr = np.divmod(coo.row, m * m)
    yr, xr = np.divmod(rr, m)
    zc, rc = np.divmod(coo.col, m * m)
    yc, xc = np.divmod(rc, m)
    dz, dy, dx = zc - zr, yc - yr, xc - xr
    if coo.nnz and max(np.abs(dz).max(), np.abs(dy).max(), np.abs(dx).max()) > 1:
        raise InputError("operator is not a 27-point stencil on the structured grid")
    code = ((dz + 1) * 3 + (dy + 1)) * 3 + (dx + 1)
    st = np.zeros(27)
    for k in range(27):
        sel = coo.data[code == k]
        nz = sel[sel != 0.0]
        if nz.size:
            st[k] = nz[0]
    diff = (csr - stencil_matrix_3d(st, m)).tocoo()
    if np.any(diff.data != 0.0):
        raise InputError("operator is not translation invariant")
    if hasattr(mat, "_stencil"):
        try:
            mat._stencil = (("3d", m), st.copy())
        except AttributeError:
            pass
    return st


def grid_stencil(mat, m: int) -> np.ndarray:
    """9-point stencil of a structured-grid operator on an m x m interior grid.

    Raises InputError when the operator is not exactly a translation-invariant
    9-point stencil (the GPU kernels evaluate the operator from the stencil).
    The check is exact (value by value), so the GPU product is bit-identical
    to the CSR product.
    """
    cached = getattr(mat, "_stencil", None)
    if cached is not None and cached[0] == m:
        return cached[1].copy()
    csr = _csr_of(mat)
    if csr.shape != (m * m, m * m):
        raise DimensionMismatchError(f"operator of shape {csr.shape} is not on a {m}x{m} grid")
    coo = csr.tocoo()
    jr, ir = np.divmod(coo.row, m)
    jc, ic = np.divmod(coo.col, m)
    dy, dx = jc - jr, ic - ir
    if coo.nnz and (np.abs(dy).max() > 1 or np.abs(dx).max() > 1):
        raise InputError("operator is not a 9-point stencil on the structured grid")
    code = (dy + 1) * 3 + (dx + 1)
    st = np.zeros(9)
    for k in range(9):
        sel = coo.data[code == k]
        nz = sel[sel != 0.0]
        if nz.size:
            st[k] = nz[0]
    ref = stencil_matrix_2d(st, m)
    diff = (csr - ref).tocoo()
    if np.any(diff.data != 0.0):
        raise InputError("operator is not translation invariant; the GPU path needs "
                         "structured-grid stencils")
    if hasattr(mat, "_stencil"):
        try:
            mat._stencil = (m, st.copy())
        except AttributeError:
            pass
    return st


def grid_fields(mat, m: int) -> np.ndarray:
    """Compact per-point form (3, m*m) = centre, east (i, i+1), north (i, i+m)
    coefficients of a symmetric operator on an m x m grid whose only
    non-zeros are the S, W, C, E, N positions (the P1 diagonal-split pattern;
    SW / NE may hold stored zeros).  EXTENSION for the GPU field mode
    (csrc/field2d.cu): operators that are not translation invariant.
    Exact: raises InputError unless the lower triangle mirrors the upper
    one bit for bit and nothing else is non-zero."""
    csr = _csr_of(mat)
    n = m * m
    if csr.shape != (n, n):
        raise DimensionMismatchError(f"operator of shape {csr.shape} is not on a {m}x{m} grid")
    coo = csr.tocoo()
    jr, ir = np.divmod(coo.row, m)
    jc, ic = np.divmod(coo.col, m)
    dy, dx = jc - jr, ic - ir
    allowed = (np.abs(dy) + np.abs(dx)) <= 1
    if np.any(coo.data[~allowed] != 0.0):
        raise InputError("operator is not a 5-point-pattern P1 stiffness on the structured grid")
    idx = np.arange(n)
    y, x = np.divmod(idx, m)
    out = np.zeros((3, n))
    out[0] = csr.diagonal()
    e_ok = x < m - 1
    n_ok = y < m - 1
    out[1, e_ok] = np.asarray(csr[idx[e_ok], idx[e_ok] + 1]).ravel()
    out[2, n_ok] = np.asarray(csr[idx[n_ok], idx[n_ok] + m]).ravel()
    west = np.asarray(csr[idx[e_ok] + 1, idx[e_ok]]).ravel()
    south = np.asarray(csr[idx[n_ok] + m, idx[n_ok]]).ravel()
    if np.any(west != out[1, e_ok]) or np.any(south != out[2, n_ok]):
        raise InputError("operator is not exactly symmetric")
    return out
