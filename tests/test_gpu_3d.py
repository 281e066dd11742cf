"""GPU parity for the 3D discretisation (BASELINE configs 3 and 5): 27-point
stencils on the unit cube (Kuhn-split P1, oracle.p1_3d), trilinear multigrid.

Same bars as the 2D path (tests/test_gpu_parity.py): stencil operators,
fold_rhs, V-cycles and A~^{-1} bit-identical to the oracle; H~^{-1} within
1e-12 relative; Uzawa residual histories within 1e-10 relative.
"""

import numpy as np
import pytest

import oracle as orc
import paper_1802_08126_b200 as pg
import ulp_floor

pytestmark = pytest.mark.gpu


def _case(cells, N, seed, coeff=None, T=0.5):
    n = (cells - 1) ** 3
    rng = np.random.default_rng(seed)
    load = rng.standard_normal((N, n))
    u0 = rng.uniform(0.0, 1.0, n)
    nodes = orc.time_nodes("uniform", N, T)
    opb = orc.heat_problem("3d", cells, nodes, coeff=coeff, load=load, u_init=u0)
    spec = pg.problem_from_arrays("3d", cells, pg.TimeGrid(nodes), load, u0, coeff=coeff)
    return rng, opb, spec


@pytest.mark.parametrize("cells,N", [(4, 5), (8, 7), (16, 4), (32, 3)])
def test_operators_and_preconditioners_3d(cells, N):
    rng, opb, spec = _case(cells, N, cells + N, coeff=lambda t: 1.0 + 0.5 * t)
    system = pg.TimeGlobalSystem(spec)
    hier = pg.build_mg_hierarchy("3d", cells)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=hier)
    ht = pg.build_schur_preconditioner(spec, "mg")
    lev = orc.mg_levels("3d", cells)
    x = rng.standard_normal((N, spec.dim))
    np.testing.assert_array_equal(system.rhs, orc.fold_rhs(opb))
    np.testing.assert_array_equal(system.apply_K(x), orc.op_K(opb, x))
    np.testing.assert_array_equal(system.apply_Kt(x), orc.op_Kt(opb, x))
    np.testing.assert_array_equal(system.apply_Abd(x), orc.op_Abd(opb, x))
    np.testing.assert_array_equal(at.apply_inverse(x), orc.BlockInv(opb, lev).apply(x))
    href = orc.SchurInv(opb, lev).apply(x)
    assert np.max(np.abs(ht.apply_inverse(x) - href)) <= 1e-12 * np.max(np.abs(href))


def test_uzawa_3d_matches_oracle():
    cells, N = 16, 16
    rng, opb, spec = _case(cells, N, 3, T=1.0)
    lev = orc.mg_levels("3d", cells)
    ref = orc.uzawa(opb, orc.BlockInv(opb, lev), orc.SchurInv(opb, lev), 0.9, 1e-8, 200)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("3d", cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    (p, u), hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-8))
    assert hist.converged and abs(hist.iterations - len(ref.residual)) <= 1
    k = min(hist.iterations, len(ref.residual))
    rel = np.abs(np.array(hist.residual[:k]) - ref.residual[:k]) / np.array(ref.residual[:k])
    print(f"3d uzawa: {hist.iterations} iterations, max rel residual drift {rel.max():.3e}")
    ref_res = np.array(ref.residual[:k])
    # 1e-10 while res > 1e-7; on the tail, the oracle's own drift under a
    # 1-ulp perturbation of its transforms (tests/ulp_floor.py)
    assert rel[ref_res > 1e-7].max() <= 1e-10, rel
    bar = ulp_floor.bar("uzawa3d_c16_N16", k)
    print(f"oracle 1-ulp floor {bar.max():.3e}")
    assert np.all(rel <= bar), (rel.max(), bar.max())
    nrm = orc.ExactNorms(opb)
    assert nrm.s_norm(u - ref.u) / nrm.s_norm(ref.u) <= 1e-8


def test_c3_full_mesh_short_history():
    """BASELINE config 3's full spatial mesh (cells = 64, 63^3 = 250,047 nodes
    per step, the 6-level hierarchy of the benchmarked run) with N = 8 steps:
    6 Uzawa iterations against the oracle, u0 ~ U[0,1] as in c3."""
    cells, N = 64, 8
    rng, opb, spec = _case(cells, N, 0, T=N / 512.0)
    lev = orc.mg_levels("3d", cells)
    ref = orc.uzawa(opb, orc.BlockInv(opb, lev), orc.SchurInv(opb, lev), 0.9, 1e-300, 6)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("3d", cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    x = rng.standard_normal((N, spec.dim))
    np.testing.assert_array_equal(at.apply_inverse(x), orc.BlockInv(opb, lev).apply(x))
    (p, u), hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(tol=1e-300, max_iter=6))
    rel = np.abs(np.array(hist.residual) - ref.residual) / np.array(ref.residual)
    print(f"c3 mesh, N=8: max rel residual drift over 6 iterations {rel.max():.3e}")
    assert rel.max() <= 1e-12, rel
    assert np.max(np.abs(u - ref.u)) <= 1e-12 * np.max(np.abs(ref.u))
    assert np.max(np.abs(p - ref.p)) <= 1e-12 * np.max(np.abs(ref.p))
