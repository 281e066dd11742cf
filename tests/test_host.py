"""CPU-side checks of the product package: host setup reproduces the oracle
(and hence the reference) bit for bit, the Galerkin stencil tables equal the
oracle's sparse triple products on every level, and libpint.so loads and
exports every symbol include/pint.h declares.  No GPU needed."""

import os
import re

import numpy as np
import pytest

import oracle as orc
import paper_1802_08126_b200 as pg
from paper_1802_08126_b200 import _native, spatial
from paper_1802_08126_b200.linalg import (grid_stencil, grid_stencil3, stencil_matrix_2d,
                                          stencil_matrix_3d)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("cells", [2, 4, 8, 32])
def test_assembly_2d_bitwise(cells):
    m, a = pg.assemble_mass_stiffness_2d(cells)
    om, oa = orc.p1_2d(cells)
    np.testing.assert_array_equal(m.todense(), om.dense())
    np.testing.assert_array_equal(a.todense(), oa.dense())


@pytest.mark.parametrize("cells", [2, 4, 8])
def test_assembly_3d_bitwise(cells):
    """3D extension: Kuhn-split P1 on the unit cube == oracle.p1_3d."""
    m, a = pg.assemble_mass_stiffness_3d(cells)
    om, oa = orc.p1_3d(cells)
    np.testing.assert_array_equal(m.todense(), om.dense())
    np.testing.assert_array_equal(a.todense(), oa.dense())


def test_assembly_1d_bitwise():
    m, a = pg.assemble_mass_stiffness_1d(16)
    om, oa = orc.p1_1d(16)
    np.testing.assert_array_equal(m.todense(), om.dense())
    np.testing.assert_array_equal(a.todense(), oa.dense())


def test_time_grid_and_tau_ref():
    g = pg.build_time_grid("perturbed", 16, 1.3, perturbation=0.3, seed=3)
    np.testing.assert_array_equal(g.nodes, orc.time_nodes("perturbed", 16, 1.3, 0.3, 3))
    spec = pg.make_heat_problem("2d", 8, pg.build_time_grid("uniform", 64, 1.0), data="zero")
    assert spec.tau_ref == 0.015625000000000007  # not exactly T/N


def test_make_heat_problem_random_matches_golden():
    d = np.load(os.path.join(ROOT, "tests", "golden", "ops2d_c16_N16_coeff.npz"))
    grid = pg.build_time_grid("perturbed", 16, 1.3, perturbation=0.3, seed=3)
    spec = pg.make_heat_problem("2d", 16, grid, coeff=lambda t: 0.8 + 0.6 * t, data="random",
                                seed=11)
    np.testing.assert_array_equal(spec.load, d["load"])
    np.testing.assert_array_equal(spec.u_init, d["u_init"])
    assert spec.tau_ref == float(d["tau_ref"])


def test_grid_stencil_roundtrip_and_rejects():
    m, a = pg.assemble_mass_stiffness_2d(16)
    st = grid_stencil(m, 15)
    assert st[2] == 0.0 and st[6] == 0.0        # diagonal split: no SE / NW coupling
    assert st[4] == 0.49999999999999994 * (1 / 16) ** 2 * 1.0 or st[4] > 0
    diff = (m.tocsr() - stencil_matrix_2d(st, 15)).tocoo()
    assert not np.any(diff.data)
    np.testing.assert_array_equal(grid_stencil(a, 15), [0, -1, 0, -1, 4, -1, 0, -1, 0])
    bad = pg.SpatialMatrix.from_dense(np.diag(np.arange(1.0, 10.0)))
    with pytest.raises(pg.InputError):
        grid_stencil(bad, 3)
    with pytest.raises(pg.DimensionMismatchError):
        grid_stencil(a, 14)


def test_scaled_stencil_cache_is_exact():
    _, a = pg.assemble_mass_stiffness_2d(8)
    grid_stencil(a, 7)
    s = a.scaled(0.37)
    cached = grid_stencil(s, 7)
    s2 = pg.SpatialMatrix(s.dim, s.rows, s.cols, s.vals)   # no cache: full check
    np.testing.assert_array_equal(cached, grid_stencil(s2, 7))


@pytest.mark.parametrize("cells", [4, 8, 32, 64])
def test_galerkin_tables_match_oracle_hierarchy(cells):
    """Probe-grid Galerkin stencils == the oracle's full-size (P^T A P) on every level."""
    om, oa = orc.p1_2d(cells)
    lev = orc.mg_levels("2d", cells)
    hier = pg.build_mg_hierarchy("2d", cells)
    mus = orc.frequency_weights(8)
    ops = [orc.sym_add(mu, om, 1.0, oa.scaled(0.0123)) for mu in mus] + [oa.scaled(1.7), oa]
    st0 = np.stack([grid_stencil(o.csr, cells - 1) for o in ops])
    tab = spatial.galerkin_tables(st0, hier, 4.0 / 5.0)
    for s, o in enumerate(ops):
        vc = orc.VCycle(o, lev)
        for lvl, mat in enumerate(vc.mats):
            ml = lev.cells[lvl] - 1
            if ml >= 3:
                diff = (mat - stencil_matrix_2d(tab[lvl, s, :9], ml)).tocoo()
                assert not np.any(diff.data), (s, lvl)
            else:
                assert mat.toarray()[0, 0] == tab[lvl, s, 4]
            np.testing.assert_array_equal(vc.dinv[lvl], np.full(ml * ml, tab[lvl, s, 9]))


@pytest.mark.parametrize("cells", [4, 8, 16])
def test_galerkin_tables_3d_match_oracle_hierarchy(cells):
    """3D: 27-point probe-grid Galerkin stencils == the oracle's full-size
    (P^T A P) with trilinear transfers; damping 6/7."""
    om, oa = orc.p1_3d(cells)
    lev = orc.mg_levels("3d", cells)
    hier = pg.build_mg_hierarchy("3d", cells)
    ops = [orc.sym_add(mu, om, 1.0, oa.scaled(0.0123)) for mu in orc.frequency_weights(3)] + [oa]
    st0 = np.stack([grid_stencil3(o.csr, cells - 1) for o in ops])
    tab = spatial.galerkin_tables(st0, hier, spatial.DEFAULT_DAMPING["3d"])
    for s, o in enumerate(ops):
        vc = orc.VCycle(o, lev)
        for lvl, mat in enumerate(vc.mats):
            ml = lev.cells[lvl] - 1
            if ml >= 3:
                diff = (mat - stencil_matrix_3d(tab[lvl, s, :27], ml)).tocoo()
                assert not np.any(diff.data), (s, lvl)
            else:
                assert mat.toarray()[0, 0] == tab[lvl, s, 13]
            np.testing.assert_array_equal(vc.dinv[lvl], np.full(ml ** 3, tab[lvl, s, 27]))


def test_schur_block_stencils_match_add_matrices():
    """H_k stencil = fl(mu_k m) + fl(1.0 fl(tau a)) (schur.py:41-47 via linalg.py:118-127)."""
    spec = pg.make_heat_problem("2d", 8, pg.build_time_grid("uniform", 16, 1.0), data="zero")
    mu = pg.frequency_weights(16)
    mst, ast = grid_stencil(spec.mass, 7), grid_stencil(spec.a_ref, 7)
    ta = spec.a_ref.scaled(spec.tau_ref)
    for k in (0, 7, 15):
        hk = pg.add_matrices(mu[k], spec.mass, 1.0, ta)
        np.testing.assert_array_equal(grid_stencil(hk, 7), mu[k] * mst + 1.0 * (spec.tau_ref * ast))


def test_frequency_weights_closed_form():
    """pkg/tests/test_schur.py:12-23."""
    np.testing.assert_array_equal(pg.frequency_weights(64), orc.frequency_weights(64))
    mu = pg.frequency_weights(32)
    assert np.all(np.diff(mu) > 0) and mu[0] > 0


def test_config_and_history_types():
    with pytest.raises(pg.InputError):
        pg.UzawaConfig(omega=0.0)
    with pytest.raises(pg.InputError):
        pg.UzawaConfig(stopping="bogus")
    h = pg.ConvergenceHistory()
    h.append(0.5, None, None, 1.0, 0.1, 0.2)
    assert h.to_csv().splitlines()[1] == "1,0.5,,,1,0.10000000000000001,0.20000000000000001"


def test_library_exports_every_header_symbol():
    header = open(os.path.join(ROOT, "include", "pint.h")).read()
    declared = set(re.findall(r"\b(pint_[a-z_A-Z0-9]+)\s*\(", header))
    lib = _native.load_library()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(_native.exported_symbols())
    assert lib.pint_abi_version() == 1


def test_no_cpu_fallback_without_device():
    """Without a CUDA device the product raises instead of computing on the CPU."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _native.Context()
    spec = pg.make_heat_problem("2d", 4, pg.build_time_grid("uniform", 4, 1.0), data="sine")
    with pytest.raises(RuntimeError):
        pg.TimeGlobalSystem(spec)


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1802_08126_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference not present (GPU box)")
def test_reference_problemspec_is_accepted_bitwise():
    """A ProblemSpec built by the unmodified reference yields exactly the same
    device-upload arrays (stencils, scales, multigrid tables) as ours."""
    import importlib
    import sys

    sys.path.insert(0, REF_SRC)
    try:
        ps = importlib.import_module("pintsolve")
    finally:
        sys.path.remove(REF_SRC)
    from paper_1802_08126_b200._device import HostProblem

    for coeff in (None, lambda t: 0.8 + 0.6 * t):
        rgrid = ps.build_time_grid("perturbed", 16, 1.3, perturbation=0.3, seed=3)
        rspec = ps.make_heat_problem("2d", 16, rgrid, coeff=coeff, data="random", seed=11)
        ogrid = pg.build_time_grid("perturbed", 16, 1.3, perturbation=0.3, seed=3)
        ospec = pg.make_heat_problem("2d", 16, ogrid, coeff=coeff, data="random", seed=11)
        hr, ho = HostProblem(rspec), HostProblem(ospec)
        for name in ("steps", "mass_st", "a_st", "a_sid", "a_scale", "aref_st"):
            np.testing.assert_array_equal(getattr(hr, name), getattr(ho, name), err_msg=name)
        hier = pg.build_mg_hierarchy("2d", 16)
        for t_r, t_o in zip(hr.atilde_tables(hier, 0.8), ho.atilde_tables(hier, 0.8)):
            np.testing.assert_array_equal(t_r, t_o)
        mu = pg.frequency_weights(16)
        for t_r, t_o in zip(hr.htilde_tables(hier, 0.8, mu), ho.htilde_tables(hier, 0.8, mu)):
            np.testing.assert_array_equal(t_r, t_o)
        # and the tables reproduce the reference's own multigrid operators
        rsch = ps.build_schur_preconditioner(rspec, "mg", vcycles=1)
        tab, _ = hr.htilde_tables(hier, 0.8, mu)
        for k in (0, 9, 15):
            for lvl, op in enumerate(rsch.solvers[k]._ops):
                ml = hier.cells[lvl] - 1
                if ml >= 3:
                    diff = (op - stencil_matrix_2d(tab[lvl, k, :9], ml)).tocoo()
                    assert not np.any(diff.data)
                np.testing.assert_array_equal(rsch.solvers[k]._dinv[lvl],
                                              np.full(ml * ml, tab[lvl, k, 9]))
