"""Residual-drift floor of the reference arithmetic (test helper).

Near convergence the Uzawa / MINRES residual is a difference of O(|f|)
terms that cancel to O(res |f|); its rounding noise relative to the residual
is ~ eps / res / sqrt(#entries).  Two runs whose iterates differ in a single
bit disagree at that level, whatever their arithmetic.  The floor is measured
on the oracle (bit-identical to the reference where the reference exists):
the same solve with one ulp flipped in a random half of the sine
transforms' outputs -- a model of an independent, equally accurate transform
implementation -- over SEEDS seeds.  ``bar(case, iters)`` is the per-
iteration envelope: the running maximum over seeds and earlier iterations,
never below the north_star's 1e-10.

The ensembles are precomputed by tests/golden/make_drift_floor.py into
tests/golden/drift_floor.npz for every case the GPU tests compare (CASES).
"""

from __future__ import annotations

import contextlib
import os

import numpy as np

import oracle as orc
import oracle.pint_oracle as O

FRACTION = 0.5
SEEDS = 64
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


@contextlib.contextmanager
def perturbed_transforms(seed: int, fraction: float = FRACTION):
    fwd, inv = O.dst_inverse_T, O.dst_inverse
    rng = np.random.default_rng(seed)

    def pert(x):
        hit = rng.random(x.shape) < fraction
        toward = np.where(rng.random(x.shape) < 0.5, np.inf, -np.inf)
        return np.where(hit, np.nextafter(x, toward), x)

    O.dst_inverse_T = lambda u: pert(fwd(u))
    O.dst_inverse = lambda u: pert(inv(u))
    try:
        yield
    finally:
        O.dst_inverse_T, O.dst_inverse = fwd, inv


@contextlib.contextmanager
def perturbed_operators(seed: int, fraction: float = FRACTION):
    """Every block operator of the iteration (the sine transforms, K, K^T,
    A and each V-cycle) is evaluated on an input with one ulp flipped in a
    random half of the entries (backward error) and returns its result
    perturbed the same way (forward error): a model of an independent,
    equally backward-stable implementation of ALL operators -- what the
    FMA-contracted ("fast") band kernels are against the reference's CSR
    products (a contracted row sum differs by ~1 ulp of its largest term,
    i.e. by the effect of ~1 ulp on its inputs, not 1 ulp of the result)."""
    names = ("dst_inverse_T", "dst_inverse", "op_K", "op_Kt", "op_Abd")
    saved = {k: getattr(O, k) for k in names}
    vc = O.VCycle.apply
    rng = np.random.default_rng(seed)

    def pert(x):
        hit = rng.random(x.shape) < fraction
        toward = np.where(rng.random(x.shape) < 0.5, np.inf, -np.inf)
        return np.where(hit, np.nextafter(x, toward), x)

    def pert_in(a):
        return pert(a) if isinstance(a, np.ndarray) and a.ndim == 2 else a

    def wrap(fn):
        return lambda *a, **k: pert(fn(*[pert_in(v) for v in a], **k))

    for k in names:
        setattr(O, k, wrap(saved[k]))
    O.VCycle.apply = lambda self, b: pert(vc(self, pert_in(b)))
    try:
        yield
    finally:
        for k in names:
            setattr(O, k, saved[k])
        O.VCycle.apply = vc


# ---- the cases the GPU tests compare: (oracle problem, solver settings) -----

def _golden_uzawa(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    c0, c1 = (float(v) for v in d["coeff"])
    coeff = None if (c0, c1) == (1.0, 0.0) else (lambda t: c0 + c1 * t)
    pb = orc.heat_problem(str(d["space"]), int(d["cells"]), d["nodes"], coeff=coeff,
                          load=d["load"], u_init=d["u_init"])
    return pb, ("uzawa", float(d["uz_omega"]), float(d["uz_tol"]), int(d["uz_max_iter"]))


def case_c1():
    nodes = orc.time_nodes("uniform", 64, 1.0)
    load = np.random.default_rng(0).standard_normal((64, 961))
    return (orc.heat_problem("2d", 32, nodes, load=load, u_init=np.zeros(961)),
            ("uzawa", 0.9, 1e-8, 200))


def case_uzawa3d():
    """tests/test_gpu_3d.py::test_uzawa_3d_matches_oracle (cells 16, N 16)."""
    cells, N, seed, T = 16, 16, 3, 1.0
    n = (cells - 1) ** 3
    rng = np.random.default_rng(seed)
    load = rng.standard_normal((N, n))
    u0 = rng.uniform(0.0, 1.0, n)
    pb = orc.heat_problem("3d", cells, orc.time_nodes("uniform", N, T), load=load, u_init=u0)
    return pb, ("uzawa", 0.9, 1e-8, 200)


def case_field():
    """tests/test_gpu_field.py::test_field_uzawa_matches_oracle (cells 16, N 16)."""
    import paper_1802_08126_b200 as pg

    cells, N, T, seed = 16, 16, 2.0, 11
    n = (cells - 1) ** 2
    grid = pg.build_time_grid("uniform", N, T)
    w = pg.c4_cell_weights(cells, grid, seed=seed)
    rng = np.random.default_rng(seed + 1)
    load = rng.standard_normal((N, n))
    u0 = rng.uniform(0.0, 1.0, n)
    stiff = [orc.stiffness_2d_weighted(cells, w(k)) for k in range(N)]
    pb = orc.heat_problem("2d", cells, grid.nodes, load=load, u_init=u0, stiffness=stiff)
    return pb, ("uzawa", 0.9, 1e-8, 3000)


def _golden_minres(name):
    d = np.load(os.path.join(GOLDEN, name + ".npz"))
    pb = orc.heat_problem(str(d["space"]), int(d["cells"]), d["nodes"], load=d["load"],
                          u_init=d["u_init"])
    return pb, ("minres", float(d["mr_tol"]), int(d["mr_max_iter"]))


def _cli(method):
    d = np.load(os.path.join(GOLDEN, "problem_c8_N4.npz"))
    pb = orc.heat_problem("2d", 8, d["nodes"], coeff=lambda t: 1.0 + t, load=d["load"],
                          u_init=d["u_init"])
    if method == "minres":
        return pb, ("minres", 1e-10, 300)
    omega = float(np.load(os.path.join(GOLDEN, "problem_c8_N4_omega.npy")))
    return pb, ("uzawa", omega, 1e-10, 300)


CASES = {
    "c1": case_c1,
    "ops2d_c16_N16_coeff": lambda: _golden_uzawa("ops2d_c16_N16_coeff"),
    "sine2d_c8_N16": lambda: _golden_uzawa("sine2d_c8_N16"),
    "uzawa3d_c16_N16": case_uzawa3d,
    "field_c16_N16": case_field,
    "minres_c16_N16": lambda: _golden_minres("minres_c16_N16"),
    "minres_sine_c8_N32": lambda: _golden_minres("minres_sine_c8_N32"),
    "cli_uzawa": lambda: _cli("uzawa"),
    "cli_minres": lambda: _cli("minres"),
}


# cases that run on the 2D band / stencil kernels, which exist in "fast" (FMA-
# contracted) arithmetic: their fast-arithmetic bar is the all-operator ensemble
FAST_CASES = ("c1", "ops2d_c16_N16_coeff", "sine2d_c8_N16", "minres_c16_N16",
              "minres_sine_c8_N32", "cli_uzawa", "cli_minres")


def residuals(name: str, seed: int, mode: str = "dst") -> np.ndarray:
    """Residual history of case `name`; seed 0 unperturbed, else perturbed
    (mode "dst": the transforms only; "all": every block operator)."""
    pb, how = CASES[name]()
    lev = orc.mg_levels(pb.space, pb.cells)
    if seed == 0:
        ctx = contextlib.nullcontext()
    else:
        ctx = perturbed_operators(seed) if mode == "all" else perturbed_transforms(seed)
    with ctx:
        if how[0] == "uzawa":
            r = orc.uzawa(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), *how[1:]).residual
        else:
            r = orc.minres(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), tol=how[1],
                           max_iter=how[2]).residual
    return np.asarray(r, dtype=np.float64)


def envelope(drifts: np.ndarray, iters: int) -> np.ndarray:
    """max(1e-10, running max over seeds and iterations), length iters."""
    env = np.fmax.accumulate(np.nanmax(np.atleast_2d(drifts), axis=0))
    if len(env) < iters:
        env = np.concatenate([env, np.full(iters - len(env), env[-1])])
    return np.maximum(1e-10, env[:iters])


def bar(name: str, iters: int, arith: str = "exact") -> np.ndarray:
    """Per-iteration bar of case `name` from the committed ensemble: the
    transform-only ensemble for exact arithmetic (every other operator is
    bit-identical to the reference there), the all-operator ensemble for
    fast arithmetic."""
    d = np.load(os.path.join(GOLDEN, "drift_floor.npz"))
    key = name + ("_drift_all" if arith == "fast" else "_drift")
    return envelope(d[key], iters)
