"""c2 residual history under the selected arithmetic (PINT_ARITH) and fusion
knobs: iteration count and the last residuals, for comparison with the
reference run (60 iterations, final 7.941816e-09)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    load = bench.c2_load()
    pg, spec, system, at, ht = bench.build_solver(load, 0)
    (p, u), hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-8, max_iter=200))
    r = np.array(hist.residual)
    env = {k: v for k, v in os.environ.items() if k.startswith("PINT_")}
    print(json.dumps({"env": env, "arith": pg.get_arithmetic(), "iters": hist.iterations,
                      "res": [float(x) for x in r]}))


if __name__ == "__main__":
    main()
