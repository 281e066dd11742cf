"""Diagnostic mode on the device (csrc/exact_solve.cu) against the reference.

The reference computes the sequential implicit-Euler oracle and the discrete
parabolic S-norm with SuperLU (solvers.py:158-174, operators.py:113-183);
the GPU path solves the same SPD systems by multigrid-preconditioned CG to
the rounding floor.  Bars: 1e-12 relative against the reference's golden
outputs (tests/golden/c1_uzawa.npz, written by the unmodified pintsolve)
and against the oracle's restatement on a perturbed grid with a c(t)
coefficient and in 3D.
"""

import os

import numpy as np
import pytest

import oracle as orc
import paper_1802_08126_b200 as pg
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _c1():
    load = np.random.default_rng(0).standard_normal((64, 961))
    spec = pg.problem_from_arrays("2d", 32, pg.build_time_grid("uniform", 64, 1.0), load,
                                  np.zeros(961))
    return spec, np.load(os.path.join(GOLDEN, "c1_uzawa.npz"))


def test_sequential_euler_matches_reference():
    spec, g = _c1()
    u = pg.sequential_euler_solve(spec)
    assert np.max(np.abs(u - g["u_seq"])) <= 1e-12 * np.max(np.abs(g["u_seq"]))


def test_s_norms_match_reference():
    spec, g = _c1()
    system = pg.TimeGlobalSystem(spec, diagnostic=True)
    assert abs(system.s_norm(g["u_seq"]) / float(g["s_norm_seq"]) - 1.0) <= 1e-12
    err = system.s_norm_diff(g["u"], g["u_seq"]) / float(g["s_norm_seq"])
    # the reference's own error of its Uzawa iterate (6.2e-9): a difference
    # of two nearby vectors, so the exact-solve floor enters relative to it
    assert abs(err / float(g["s_norm_err"]) - 1.0) <= 1e-6
    with pytest.raises(pg.DiagnosticModeRequiredError):
        pg.TimeGlobalSystem(spec).s_norm(g["u"])


@pytest.mark.parametrize("space,cells,N", [("2d", 8, 6), ("2d", 64, 5), ("3d", 8, 4)])
def test_exact_solves_match_oracle(space, cells, N):
    """c(t) coefficient on a perturbed time grid: sequential Euler, S-norm,
    s_bilinear and A_bd^{-1} against the oracle's SuperLU restatement."""
    rng = np.random.default_rng(3 + cells)
    n = (cells - 1) ** (2 if space == "2d" else 3)
    nodes = orc.time_nodes("perturbed", N, 0.5, perturbation=0.3, seed=4)
    load = rng.standard_normal((N, n))
    u0 = rng.standard_normal(n)
    cf = lambda t: 1.0 + 2.0 * t  # noqa: E731
    opb = orc.heat_problem(space, cells, nodes, coeff=cf, load=load, u_init=u0)
    spec = pg.problem_from_arrays(space, cells, pg.TimeGrid(nodes), load, u0, coeff=cf)
    system = pg.TimeGlobalSystem(spec, diagnostic=True)
    nrm = orc.ExactNorms(opb)
    x = rng.standard_normal((N, n))
    y = rng.standard_normal((N, n))
    assert abs(system.s_norm(x) / nrm.s_norm(x) - 1.0) <= 1e-12
    sb = nrm.s_bilinear(x, y)
    assert abs(system.s_bilinear(x, y) - sb) <= 1e-11 * nrm.s_norm(x) * nrm.s_norm(y)
    useq = pg.sequential_euler_solve(spec)
    ref = orc.sequential_euler(opb)
    assert np.max(np.abs(useq - ref)) <= 1e-12 * np.max(np.abs(ref))
    # A_bd^{-1}: A_bd (A_bd^{-1} x) = x
    back = system.apply_Abd(system.apply_Abd_inv(x))
    assert np.max(np.abs(back - x)) <= 1e-11 * np.max(np.abs(x))


def test_diagnostic_uzawa_history_matches_reference_error():
    """uzawa_solve(diagnostics=True) records the exact S-norm error of every
    iterate on the device; the last one equals the reference's s_norm_err."""
    spec, g = _c1()
    system = pg.TimeGlobalSystem(spec, diagnostic=True)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("2d", 32))
    ht = pg.build_schur_preconditioner(spec, "mg", vcycles=1)
    cfg = pg.UzawaConfig(omega=0.9, tol=1e-8, max_iter=200, diagnostics=True)
    (_, u), hist = pg.uzawa_solve(system, at, ht, cfg)
    assert hist.iterations == 66
    errs = np.array(hist.s_norm_error)
    assert np.all(np.isfinite(errs)) and errs[-1] < errs[0]
    assert abs(errs[-1] / float(g["s_norm_err"]) - 1.0) <= 1e-3
