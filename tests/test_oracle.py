"""Pin the CPU oracle (oracle/) against golden vectors from the unmodified
reference (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

import oracle as orc
from conftest import GOLDEN

CASES = ["ops2d_c16_N16_coeff", "ops1d_c16_N12", "sine2d_c8_N16"]


def load_case(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    c0, c1 = (float(v) for v in d["coeff"])
    coeff = None if (c0, c1) == (1.0, 0.0) else (lambda t: c0 + c1 * t)
    pb = orc.heat_problem(str(d["space"]), int(d["cells"]), d["nodes"], coeff=coeff,
                          load=d["load"], u_init=d["u_init"])
    return d, pb


@pytest.fixture(scope="module", params=CASES)
def case(request):
    d, pb = load_case(request.param)
    lev = orc.mg_levels(pb.space, pb.cells)
    return d, pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev)


def test_problem_setup_bitwise(case):
    d, pb, _, _ = case
    assert pb.tau_ref == float(d["tau_ref"])
    np.testing.assert_array_equal(orc.fold_rhs(pb), d["rhs"])
    np.testing.assert_array_equal(orc.frequency_weights(pb.N), d["mu"])
    if d["mass_dense"].size:
        np.testing.assert_array_equal(pb.mass.dense(), d["mass_dense"])
        np.testing.assert_array_equal(pb.stiffness[0].dense(), d["a0_dense"])


def test_time_operators_bitwise(case):
    d, pb, _, _ = case
    x = d["x"]
    np.testing.assert_array_equal(orc.op_K(pb, x), d["K_x"])
    np.testing.assert_array_equal(orc.op_Kt(pb, x), d["Kt_x"])
    np.testing.assert_array_equal(orc.op_Abd(pb, x), d["Abd_x"])


def test_dst_bitwise(case):
    d, _, _, _ = case
    x = d["x"]
    np.testing.assert_array_equal(orc.dst_forward(x), d["dst_fwd_x"])
    np.testing.assert_array_equal(orc.dst_inverse(x), d["dst_inv_x"])
    np.testing.assert_array_equal(orc.dst_forward_T(x), d["dst_fwdT_x"])
    np.testing.assert_array_equal(orc.dst_inverse_T(x), d["dst_invT_x"])


def test_preconditioners_bitwise(case):
    d, pb, at, ht = case
    np.testing.assert_array_equal(at.apply(d["x"]), d["atilde_x"])
    np.testing.assert_array_equal(ht.apply(d["x"]), d["htilde_x"])
    np.testing.assert_array_equal(at.solvers[0].apply(d["y"][0]), d["vcyc_a0_y"])
    np.testing.assert_array_equal(ht.solvers[-1].apply(d["y"][-1]), d["vcyc_h_last_y"])


def test_uzawa_bitwise(case):
    d, pb, at, ht = case
    res = orc.uzawa(pb, at, ht, omega=float(d["uz_omega"]), tol=float(d["uz_tol"]),
                    max_iter=int(d["uz_max_iter"]))
    np.testing.assert_array_equal(np.array(res.residual), d["uz_res"])
    np.testing.assert_array_equal(res.u, d["uz_u"])
    np.testing.assert_array_equal(res.p, d["uz_p"])
    assert res.converged == bool(d["uz_converged"])
    np.testing.assert_array_equal(orc.sequential_euler(pb), d["u_seq"])
    nrm = orc.ExactNorms(pb)
    err = nrm.s_norm(res.u - d["u_seq"]) / nrm.s_norm(d["u_seq"])
    assert err == pytest.approx(float(d["s_norm_err"]), rel=1e-12)


def test_config1_bitwise():
    """BASELINE config 1 end to end: 66 iterations, bit-identical history."""
    d = np.load(os.path.join(GOLDEN, "c1_uzawa.npz"))
    nodes = orc.time_nodes("uniform", 64, 1.0)
    load = np.random.default_rng(0).standard_normal((64, 961))
    pb = orc.heat_problem("2d", 32, nodes, load=load, u_init=np.zeros(961))
    lev = orc.mg_levels("2d", 32)
    res = orc.uzawa(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), 0.9, 1e-8, 200)
    assert len(res.residual) == 66
    np.testing.assert_array_equal(np.array(res.residual), d["residual"])
    np.testing.assert_array_equal(res.u, d["u"])
    np.testing.assert_array_equal(res.p, d["p"])


def test_zero_data_zero_iterations():
    """solvers.py:212-217 / test_solvers.py:108-115."""
    nodes = orc.time_nodes("uniform", 4, 1.0)
    pb = orc.heat_problem("2d", 4, nodes, data="zero")
    lev = orc.mg_levels("2d", 4)
    res = orc.uzawa(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev))
    assert res.converged and res.residual == []


def test_divergence_raises():
    """solvers.py:254-257 / test_solvers.py:117-123."""
    nodes = orc.time_nodes("uniform", 8, 1.0)
    pb = orc.heat_problem("2d", 8, nodes, data="sine")
    lev = orc.mg_levels("2d", 8)
    with pytest.raises(orc.OracleDivergence):
        orc.uzawa(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), omega=40.0,
                  tol=1e-12, max_iter=500)


def test_3d_extension_stencils():
    """EXTENSION pin: the Kuhn-split P1 stiffness is the 7-point h(6,-1x6)
    stencil and the mass has 15 points with centre 2h^3/5."""
    c = 4
    m, a = orc.p1_3d(c)
    h = 1.0 / c
    n = c - 1
    mid = (1 * n + 1) * n + 1
    arow = a.dense()[mid]
    nz = np.nonzero(arow)[0]
    assert len(nz) == 7
    assert arow[mid] == pytest.approx(6 * h)
    assert sorted(arow[nz])[:6] == pytest.approx([-h] * 6)
    mrow = m.dense()[mid]
    assert np.count_nonzero(mrow) == 15
    assert mrow[mid] == pytest.approx(2 * h ** 3 / 5)
    assert mrow.sum() == pytest.approx(h ** 3)      # interior row sums to |supp| * ... = h^3


MINRES_CASES = ["minres_c16_N16", "minres_sine_c8_N32"]


def load_minres(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    pb = orc.heat_problem(str(d["space"]), int(d["cells"]), d["nodes"], load=d["load"],
                          u_init=d["u_init"])
    return d, pb


@pytest.mark.parametrize("name", MINRES_CASES)
def test_minres_bitwise(name):
    """minres_solve (solvers.py:267-327): the oracle reproduces the
    reference's residual history and iterate bit for bit
    (tests/golden/make_golden_minres.py)."""
    d, pb = load_minres(name)
    lev = orc.mg_levels(pb.space, pb.cells)
    r = orc.minres(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), tol=float(d["mr_tol"]),
                   max_iter=int(d["mr_max_iter"]))
    np.testing.assert_array_equal(np.array(r.residual), d["mr_res"])
    assert r.converged == bool(d["mr_converged"])
    np.testing.assert_array_equal(r.p, d["mr_p"])
    np.testing.assert_array_equal(r.u, d["mr_u"])


@pytest.mark.parametrize("name", MINRES_CASES)
def test_sequential_euler_and_s_norm(name):
    """sequential_euler_solve (solvers.py:158-174) and s_norm
    (operators.py:176-183) against the reference."""
    d, pb = load_minres(name)
    u = orc.sequential_euler(pb)
    np.testing.assert_allclose(u, d["u_seq"], rtol=0, atol=1e-13 * np.abs(d["u_seq"]).max())
    nrm = orc.ExactNorms(pb)
    assert nrm.s_norm(d["x"]) == pytest.approx(float(d["s_norm_x"]), rel=1e-13)
    assert nrm.s_norm(d["u_seq"]) == pytest.approx(float(d["s_norm_seq"]), rel=1e-13)
