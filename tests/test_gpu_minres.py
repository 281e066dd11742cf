"""minres_solve on the GPU (solvers.py:267-327) against the reference's
MINRES runs (tests/golden/make_golden_minres.py), through the C ABI."""

import os

import numpy as np
import pytest

import oracle as orc
import ulp_floor
import paper_1802_08126_b200 as pg
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

CASES = ["minres_c16_N16", "minres_sine_c8_N32"]


def _build(d):
    cells = int(d["cells"])
    spec = pg.problem_from_arrays(str(d["space"]), cells, pg.TimeGrid(d["nodes"]), d["load"],
                                  d["u_init"])
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy(str(d["space"]), cells))
    ht = pg.build_schur_preconditioner(spec, "mg", vcycles=1)
    return spec, system, at, ht


@pytest.mark.parametrize("name", CASES)
def test_minres_matches_reference(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    spec, system, at, ht = _build(d)
    (p, u), hist = pg.minres_solve(system, at, ht, tol=float(d["mr_tol"]),
                                   max_iter=int(d["mr_max_iter"]))
    ref = d["mr_res"]
    # iteration count within 1 of the reference (north_star), residual history
    # within 1e-10 relative where the reference residual is above 1e-7 of the
    # start (deeper, the Krylov recurrence amplifies rounding of the inner
    # products exactly as it does between BLAS builds)
    assert abs(hist.iterations - len(ref)) <= 1, (hist.iterations, len(ref))
    assert hist.converged == bool(d["mr_converged"])
    k = min(hist.iterations, len(ref))
    res = np.array(hist.residual[:k])
    rel = np.abs(res - ref[:k]) / ref[:k]
    head = ref[:k] > 1e-7 * ref[0]
    pb = orc.heat_problem(str(d["space"]), int(d["cells"]), d["nodes"], load=d["load"],
                          u_init=d["u_init"])
    # bar: 1e-10, or the reference arithmetic's own drift under a 1-ulp
    # perturbation of its transforms (tests/ulp_floor.py)
    bar = ulp_floor.bar(name, k, pg.get_arithmetic())
    print(f"{name}: {hist.iterations} vs {len(ref)} iterations, max rel drift {rel.max():.2e}, "
          f"head {rel[head].max():.2e}, reference 1-ulp floor {bar[head].max():.2e}")
    assert np.all(rel[head] <= bar[head]), (rel[head].max(), bar[head].max())
    nrm = orc.ExactNorms(pb)
    ref_u = d["mr_u"]
    assert nrm.s_norm(u - ref_u) <= 1e-8 * nrm.s_norm(ref_u)


def test_apply_saddle_bitwise():
    d = np.load(os.path.join(GOLDEN, "minres_c16_N16.npz"))
    spec, system, at, ht = _build(d)
    rng = np.random.default_rng(3)
    p = rng.standard_normal((spec.N, spec.dim))
    u = rng.standard_normal((spec.N, spec.dim))
    top, bottom = system.apply_saddle(p, u)
    pb = orc.heat_problem("2d", int(d["cells"]), d["nodes"], load=d["load"], u_init=d["u_init"])
    t0, b0 = orc.op_saddle(pb, p, u, orc.stiffness_scales(pb))
    np.testing.assert_array_equal(top, t0)
    np.testing.assert_array_equal(bottom, b0)


@pytest.mark.parametrize("arith", ["fast", "exact"])
@pytest.mark.parametrize("space,cells,N", [("2d", 128, 6), ("2d", 64, 5), ("3d", 16, 5), ("3d", 64, 3)])
def test_apply_saddle_band_sizes(space, cells, N, arith):
    """apply_saddle on the grids the fused residual kernels serve (2D band
    kernels, 3D z-marching / TMA kernels, c(t) coefficient): bit-identical to
    the oracle in exact arithmetic, within 1e-13 of the largest entry in the
    FMA-contracted one (pint_apply_saddle = the two Uzawa residuals at f = 0)."""
    n = (cells - 1) ** (3 if space == "3d" else 2)
    rng = np.random.default_rng(cells + N)
    load = rng.standard_normal((N, n))
    u0 = rng.standard_normal(n)
    nodes = orc.time_nodes("perturbed", N, 0.5, 0.2, 7)
    pb = orc.heat_problem(space, cells, nodes, coeff=lambda t: 1.0 + t, load=load, u_init=u0)
    spec = pg.problem_from_arrays(space, cells, pg.TimeGrid(nodes), load, u0,
                                  coeff=lambda t: 1.0 + t)
    prev = pg.set_arithmetic(arith)
    try:
        system = pg.TimeGlobalSystem(spec)
        p = rng.standard_normal((N, n))
        u = rng.standard_normal((N, n))
        top, bottom = system.apply_saddle(p, u)
    finally:
        pg.set_arithmetic(prev)
    t0, b0 = orc.op_saddle(pb, p, u, orc.stiffness_scales(pb))
    if arith == "exact" or space == "3d":
        np.testing.assert_array_equal(top, t0)
        np.testing.assert_array_equal(bottom, b0)
    else:
        assert np.max(np.abs(top - t0)) <= 1e-13 * np.max(np.abs(t0))
        assert np.max(np.abs(bottom - b0)) <= 1e-13 * np.max(np.abs(b0))
