"""Field mode (per-point 2D stiffness, BASELINE config 4): host-side pins.

The GPU kernels of csrc/field2d.cu evaluate the weighted P1 assembly and the
Galerkin products in fixed summation orders.  These CPU tests restate those
orders in numpy and check them bit for bit against the oracle's scipy
assembly (oracle.stiffness_2d_weighted, problems.py:99-138 with w_e K_e) and
its (P^T A) P hierarchy (spatial.py:140), so the orders the kernels hard-code
are pinned before any GPU run.
"""

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as orc
import paper_1802_08126_b200 as pg
from paper_1802_08126_b200.linalg import grid_fields

WT = np.array([0.5, 1.0, 0.5])


def _weights(cells, seed):
    return np.random.default_rng(seed).uniform(0.05, 2.0, (cells, cells))


def _assemble_fields_np(W):
    """numpy restatement of k_f_assemble: centre in scipy's duplicate order."""
    c = W.shape[0]
    j, i = np.meshgrid(np.arange(1, c), np.arange(1, c), indexing="ij")

    def cw(ci, cj):
        return W[cj, ci]

    s = cw(i - 1, j - 1) * 0.5
    s = s + cw(i, j) * 0.5
    s = s + cw(i, j) * 0.5
    s = s + cw(i - 1, j) * 1.0
    s = s + cw(i, j - 1) * 1.0
    s = s + cw(i - 1, j - 1) * 0.5
    e = np.where(i < c - 1, cw(i, j) * -0.5 + cw(i, j - 1) * -0.5, 0.0)
    n = np.where(j < c - 1, cw(i, j) * -0.5 + cw(i - 1, j) * -0.5, 0.0)
    return np.stack([s.ravel(), e.ravel(), n.ravel()])


def _row_coefs(csr, m):
    """(9, m, m): coefficient of every row at each CSR stencil position."""
    out = np.zeros((9, m, m))
    y, x = np.divmod(np.arange(m * m), m)
    for k, (dy, dx) in enumerate(pg.linalg.STENCIL_2D):
        ok = (y + dy >= 0) & (y + dy < m) & (x + dx >= 0) & (x + dx < m)
        r = np.arange(m * m)[ok]
        out[k].reshape(-1)[r] = np.asarray(csr[r, r + dy * m + dx]).ravel()
    return out


def _galerkin_np(A, m):
    """numpy restatement of k_f_galerkin (scipy SpGEMM order)."""
    mc = (m - 1) // 2
    Y, X = np.meshgrid(np.arange(mc), np.arange(mc), indexing="ij")
    B = np.zeros((5, 5, mc, mc))
    for a in range(3):
        for q in range(3):
            ly, lx = 2 * Y + a, 2 * X + q
            pl = WT[a] * WT[q]
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    k = (dy + 1) * 3 + (dx + 1)
                    ky, kx = ly + dy, lx + dx
                    ok = (ky >= 0) & (ky < m) & (kx >= 0) & (kx < m)
                    alk = np.where(ok, A[k][ly, lx], 0.0)
                    B[a + dy + 1, q + dx + 1] = np.where(ok, B[a + dy + 1, q + dx + 1] + alk * pl,
                                                         B[a + dy + 1, q + dx + 1])
    C = np.zeros((9, mc, mc))
    for jy in (-1, 0, 1):
        for jx in (-1, 0, 1):
            J = (jy + 1) * 3 + (jx + 1)
            cv = np.zeros((mc, mc))
            for ry in range(3):
                for rx in range(3):
                    by, bx = 2 * jy + ry + 1, 2 * jx + rx + 1
                    if 0 <= by <= 4 and 0 <= bx <= 4:
                        cv = cv + (WT[ry] * WT[rx]) * B[by, bx]
            ok = (Y + jy >= 0) & (Y + jy < mc) & (X + jx >= 0) & (X + jx < mc)
            C[J] = np.where(ok, cv, 0.0)
    return C


@pytest.mark.parametrize("cells", [4, 8, 32])
def test_weighted_assembly_order(cells):
    W = _weights(cells, cells)
    a = orc.stiffness_2d_weighted(cells, W)
    np.testing.assert_array_equal(_assemble_fields_np(W), grid_fields(a.csr, cells - 1))
    # the package's own scipy assembly (the reference element loop) agrees too
    _, ap = pg.assemble_mass_stiffness_2d(cells, cell_weights=W)
    np.testing.assert_array_equal(ap.tocsr().toarray(), a.csr.toarray())


@pytest.mark.parametrize("cells", [8, 16, 32])
def test_field_galerkin_order_matches_oracle_hierarchy(cells):
    """(P^T A) P of a variable-coefficient operator, every level, bitwise."""
    W = _weights(cells, 7 * cells)
    om, _ = orc.p1_2d(cells)
    ops = [orc.stiffness_2d_weighted(cells, W)]
    ops.append(orc.sym_add(0.37, om, 1.0, ops[0].scaled(0.0123)))   # an H_k-type operator
    lev = orc.mg_levels("2d", cells)
    for op in ops:
        vc = orc.VCycle(op, lev)
        for l in range(len(vc.mats) - 1):
            m = lev.cells[l] - 1
            mc = lev.cells[l + 1] - 1
            C = _galerkin_np(_row_coefs(vc.mats[l], m), m)
            got = _row_coefs(vc.mats[l + 1], mc) if mc > 1 else None
            if mc > 1:
                np.testing.assert_array_equal(C, got)
            else:
                assert C[4, 0, 0] == vc.mats[l + 1].toarray()[0, 0]


def test_weighted_family_items_match_oracle():
    cells, N = 8, 5
    grid = pg.build_time_grid("uniform", N, 2.0)
    w = pg.c4_cell_weights(cells, grid, seed=3)
    fam = pg.WeightedStiffness(cells, N, w)
    assert len(fam) == N and fam.dim == 49
    for n in range(N):
        ref = orc.stiffness_2d_weighted(cells, w(n))
        np.testing.assert_array_equal(fam[n].tocsr().toarray(), ref.csr.toarray())
    spec = pg.make_weighted_problem(cells, grid, w, np.zeros((N, 49)), np.zeros(49), alpha=1.0)
    assert spec.a_ref is spec.stiffness[2] and spec.a_ref._family_step == 2


def test_grid_fields_rejects():
    m = 5
    a = pg.assemble_mass_stiffness_2d(m + 1)[1]
    f = grid_fields(a.tocsr(), m)
    assert f.shape == (3, m * m)
    nine = sp.csr_matrix(pg.linalg.stencil_matrix_2d(np.arange(1.0, 10.0), m))
    with pytest.raises(pg.InputError):
        grid_fields(nine, m)
    asym = a.tocsr().tolil()
    asym[0, 1] = asym[0, 1] * 2.0
    with pytest.raises(pg.InputError):
        grid_fields(asym.tocsr(), m)
