"""Diagnostic mode on the host (paper_1802_08126_b200/diagnostics.py) against
the reference's own outputs (tests/golden/c1_uzawa.npz, written by the
unmodified pintsolve: sequential_euler_solve and s_norm, solvers.py:158-174,
operators.py:174-183) and against the CPU oracle.  No GPU needed."""

import os

import numpy as np

import oracle as orc
from conftest import GOLDEN
from paper_1802_08126_b200 import build_time_grid, problem_from_arrays
from paper_1802_08126_b200.diagnostics import ExactNorms, sequential_euler_solve


def _c1_spec():
    load = np.random.default_rng(0).standard_normal((64, 961))
    return problem_from_arrays("2d", 32, build_time_grid("uniform", 64, 1.0), load,
                               np.zeros(961)), load


def test_sequential_euler_matches_reference():
    g = np.load(os.path.join(GOLDEN, "c1_uzawa.npz"))
    spec, _ = _c1_spec()
    u = sequential_euler_solve(spec)
    # same matrices, same SuperLU options and operation order as the reference
    assert np.max(np.abs(u - g["u_seq"])) <= 1e-14 * np.max(np.abs(g["u_seq"]))


def test_s_norms_match_reference():
    g = np.load(os.path.join(GOLDEN, "c1_uzawa.npz"))
    spec, _ = _c1_spec()
    nrm = ExactNorms(spec)
    assert abs(nrm.s_norm(g["u_seq"]) / float(g["s_norm_seq"]) - 1.0) <= 1e-13
    err = nrm.s_norm(g["u"] - g["u_seq"]) / nrm.s_norm(g["u_seq"])
    assert abs(err / float(g["s_norm_err"]) - 1.0) <= 1e-9


def test_exact_norms_match_oracle_perturbed_grid():
    """c(t) coefficient on a perturbed time grid against the oracle's
    restatement of operators.py:141-183 and solvers.py:158-174."""
    rng = np.random.default_rng(3)
    cells, N = 8, 6
    n = (cells - 1) ** 2
    nodes = orc.time_nodes("perturbed", N, 0.5, perturbation=0.3, seed=4)
    load = rng.standard_normal((N, n))
    opb = orc.heat_problem("2d", cells, nodes, coeff=lambda t: 1.0 + 2.0 * t, load=load,
                           u_init=rng.standard_normal(n))
    from paper_1802_08126_b200 import TimeGrid

    spec = problem_from_arrays("2d", cells, TimeGrid(nodes), load, opb.u_init,
                               coeff=lambda t: 1.0 + 2.0 * t)
    ours, ref = ExactNorms(spec), orc.ExactNorms(opb)
    x = rng.standard_normal((N, n))
    assert abs(ours.s_norm(x) / ref.s_norm(x) - 1.0) <= 1e-13
    useq = sequential_euler_solve(spec)
    assert np.max(np.abs(useq - orc.sequential_euler(opb))) <= 1e-12 * np.max(np.abs(useq))
