"""Residual-drift floor of the reference algorithm itself (build host only).

    python tests/golden/make_drift_floor.py [--seeds 64] [--jobs 6] [--cases a,b]

The north_star asks for per-iteration Uzawa residuals within 1e-10 relative
of the reference.  Near convergence (res ~ tol) the residual
sqrt(sum r1.dp + sum z.y) is evaluated from r1 = (K u - A p) - f and
z = ..., each a difference of O(|f|) terms that cancel to O(res |f|); its
rounding noise, relative to the residual, is ~ eps / res / sqrt(#entries).
Two runs whose iterates differ in even a single bit therefore disagree at
that level on the last iterations, whatever the arithmetic.

This script measures that floor on the reference's own arithmetic: it runs
the oracle (bit-identical to ``pintsolve``, tests/test_oracle.py) on every
case the GPU tests compare (tests/ulp_floor.py CASES) with the sine
transforms' outputs perturbed by one ulp in a random half of their entries
-- a model of an independent, equally accurate implementation of the
transforms -- for SEEDS seeds, and records the relative drift of every
iteration's residual against the unperturbed run.  The GPU tests hold the
device to max(1e-10, the ensemble's running maximum) per iteration.

Fixture: tests/golden/drift_floor.npz, one array per case:
    <case>_drift      [seeds, iterations]  relative residual drift per seed, transforms perturbed
    <case>_drift_all  the same with every block operator perturbed (--mode all): the bar of
                      the FMA-contracted "fast" band kernels
"""

from __future__ import annotations

import argparse
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]


def _run(args):
    import ulp_floor

    name, seed, mode = args
    return name, seed, ulp_floor.residuals(name, seed, mode)


def main():
    import ulp_floor

    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=ulp_floor.SEEDS)
    ap.add_argument("--jobs", type=int, default=6)
    ap.add_argument("--cases", default=None)
    ap.add_argument("--mode", default="dst", choices=["dst", "all"],
                    help="dst: perturb the sine transforms (-> <case>_drift); all: perturb "
                         "every block operator (-> <case>_drift_all, the fast-arithmetic bar)")
    args = ap.parse_args()
    default = ulp_floor.FAST_CASES if args.mode == "all" else ulp_floor.CASES
    cases = [c for c in (args.cases.split(",") if args.cases else default) if c]
    suffix = "_drift_all" if args.mode == "all" else "_drift"
    work = [(c, s, args.mode) for c in cases for s in range(args.seeds + 1)]
    with ProcessPoolExecutor(args.jobs) as ex:
        runs = list(ex.map(_run, work, chunksize=4))
    path = os.path.join(HERE, "drift_floor.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
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
        out[c + suffix] = np.array(rows)
        m = np.nanmax(out[c + suffix], axis=1)
        print(f"{c}: {len(base)} iterations; per-seed max drift median {np.median(m):.1e}, "
              f"max {m.max():.1e}; seeds over 1e-10: {int(np.sum(m > 1e-10))}/{len(m)}")
    out["fraction"] = np.array(ulp_floor.FRACTION)
    np.savez_compressed(path, **out)


if __name__ == "__main__":
    main()
