"""Residual-drift floor of the reference arithmetic (test helper).

Near convergence the Uzawa / MINRES residual is a difference of O(|f|)
terms that cancel to O(res |f|); its rounding noise relative to the residual
is ~ eps / res / sqrt(#entries).  Two runs whose iterates differ in a single
bit disagree at that level, whatever their arithmetic.  This helper measures
the floor on the oracle (bit-identical to the reference where the reference
exists): the same solve with one ulp flipped in a random half of the sine
transforms' outputs (a model of an independent, equally accurate transform
implementation), over 8 seeds.  ``envelope`` turns the drifts into a
per-iteration bar: the running maximum over seeds and earlier iterations,
never below the north_star's 1e-10.  See tests/golden/make_drift_floor.py
for the committed ensembles of the reference's golden cases.
"""

from __future__ import annotations

import contextlib

import numpy as np

import oracle as orc
import oracle.pint_oracle as O

FRACTION = 0.5


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


def envelope(drifts, iters: int) -> np.ndarray:
    """max(1e-10, running max over seeds and iterations) of length iters."""
    width = max(len(d) for d in drifts)
    a = np.full((len(drifts), width), np.nan)
    for i, d in enumerate(drifts):
        a[i, :len(d)] = d
    env = np.fmax.accumulate(np.nanmax(a, axis=0))
    if len(env) < iters:
        env = np.concatenate([env, np.full(iters - len(env), env[-1])])
    return np.maximum(1e-10, env[:iters])


def floor_envelope(solve, ref_res, iters: int, seeds=tuple(range(1, 9))) -> np.ndarray:
    """solve() -> residual list, run under perturbed transforms per seed;
    drift against ref_res (the unperturbed reference history)."""
    ref_res = np.asarray(ref_res)
    drifts = []
    for s in seeds:
        with perturbed_transforms(s):
            r = np.asarray(solve())
        k = min(len(r), len(ref_res))
        drifts.append(np.abs(r[:k] - ref_res[:k]) / ref_res[:k])
    return envelope(drifts, iters)


def uzawa_envelope(pb, omega, tol, max_iter, ref_res, iters, seeds=tuple(range(1, 9))):
    lev = orc.mg_levels(pb.space, pb.cells)

    def solve():
        return orc.uzawa(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), omega, tol,
                         max_iter).residual

    return floor_envelope(solve, ref_res, iters, seeds)


def minres_envelope(pb, tol, max_iter, ref_res, iters, seeds=tuple(range(1, 9))):
    lev = orc.mg_levels(pb.space, pb.cells)

    def solve():
        return orc.minres(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), tol=tol,
                          max_iter=max_iter).residual

    return floor_envelope(solve, ref_res, iters, seeds)
