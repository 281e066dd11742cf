"""V-cycle options cycles > 1 / smooth_steps > 1 (spatial.py:116-169) on the
GPU (csrc/mg_generic.cu) against the oracle's VCycle, which restates the same
lines: A~^{-1} and the standalone V-cycle bit-identical, H~^{-1} within the
transform bar, a short Uzawa history within 1e-12."""

import numpy as np
import pytest

import oracle as orc
import paper_1802_08126_b200 as pg

pytestmark = pytest.mark.gpu


def _case(space, cells, N, seed):
    n = (cells - 1) ** (3 if space == "3d" else 2)
    rng = np.random.default_rng(seed)
    load = rng.standard_normal((N, n))
    u0 = rng.uniform(0.0, 1.0, n)
    nodes = orc.time_nodes("uniform", N, 0.5)
    coeff = lambda t: 1.0 + 0.5 * t  # noqa: E731
    opb = orc.heat_problem(space, cells, nodes, coeff=coeff, load=load, u_init=u0)
    spec = pg.problem_from_arrays(space, cells, pg.TimeGrid(nodes), load, u0, coeff=coeff)
    return rng, opb, spec


@pytest.mark.parametrize("space,cells,N,cycles,smooth",
                         [("2d", 16, 6, 2, 1), ("2d", 32, 5, 1, 2), ("2d", 128, 4, 2, 2),
                          ("3d", 8, 5, 2, 2), ("3d", 16, 4, 3, 1), ("3d", 16, 3, 1, 3)])
def test_preconditioners_with_options(space, cells, N, cycles, smooth):
    rng, opb, spec = _case(space, cells, N, cells + cycles + 7 * smooth)
    hier = pg.build_mg_hierarchy(space, cells)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=hier, cycles=cycles, smooth_steps=smooth)
    ht = pg.build_schur_preconditioner(spec, "mg", vcycles=cycles, smooth_steps=smooth)
    lev = orc.mg_levels(space, cells)
    x = rng.standard_normal((N, spec.dim))
    np.testing.assert_array_equal(at.apply_inverse(x),
                                  orc.BlockInv(opb, lev, cycles, smooth).apply(x))
    href = orc.SchurInv(opb, lev, cycles, smooth).apply(x)
    assert np.max(np.abs(ht.apply_inverse(x) - href)) <= 1e-12 * np.max(np.abs(href))


def test_standalone_vcycle_with_options():
    cells = 32
    mass, stiff = pg.assemble_mass_stiffness_2d(cells)
    hier = pg.build_mg_hierarchy("2d", cells)
    sol = pg.MgVCycleSolver(stiff, hier, cycles=2, smooth_steps=3)
    b = np.random.default_rng(3).standard_normal((4, (cells - 1) ** 2))
    _, ostiff = orc.p1_2d(cells)
    ref = orc.VCycle(ostiff, orc.mg_levels("2d", cells), cycles=2, smooth_steps=3)
    np.testing.assert_array_equal(sol.apply(b), np.stack([ref.apply(v) for v in b]))


def test_uzawa_with_options_matches_oracle():
    rng, opb, spec = _case("2d", 32, 8, 11)
    lev = orc.mg_levels("2d", 32)
    ref = orc.uzawa(opb, orc.BlockInv(opb, lev, 2, 2), orc.SchurInv(opb, lev, 2, 2), 0.9, 1e-300, 6)
    system = pg.TimeGlobalSystem(spec)
    hier = pg.build_mg_hierarchy("2d", 32)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=hier, cycles=2, smooth_steps=2)
    ht = pg.build_schur_preconditioner(spec, "mg", vcycles=2, smooth_steps=2)
    (p, u), hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(tol=1e-300, max_iter=6))
    rel = np.abs(np.array(hist.residual) - ref.residual) / np.array(ref.residual)
    assert rel.max() <= 1e-12, rel
    assert np.max(np.abs(u - ref.u)) <= 1e-12 * np.max(np.abs(ref.u))
    # back to the fused kernels on the same problem: options are per solver object
    # (this context runs the default FMA-contracted build of the fused 2D kernels:
    # within 1e-13 of the largest entry, tests/test_gpu_parity.py FAST_RTOL)
    at1 = pg.BlockDiagSolver(spec, "mg", hierarchy=hier)
    x = rng.standard_normal((8, spec.dim))
    want = orc.BlockInv(opb, lev).apply(x)
    assert np.max(np.abs(at1.apply_inverse(x) - want)) <= 1e-13 * np.max(np.abs(want))


def test_field_mode_rejects_options():
    cells, N = 16, 4
    n = (cells - 1) ** 2
    grid = pg.build_time_grid("uniform", N, 2.0)
    spec = pg.make_weighted_problem(cells, grid, pg.c4_cell_weights(cells, grid, seed=0),
                                    np.zeros((N, n)), np.zeros(n), alpha=1.0)
    with pytest.raises(pg.InputError):
        pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("2d", cells), cycles=2)
