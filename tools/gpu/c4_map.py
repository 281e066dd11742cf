"""Where does Uzawa (omega = 0.9) on the c4 coefficient stop converging?  Map over
(cells, N) at T = 2 (GPU box)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1802_08126_b200 as pg  # noqa: E402

for cells, N in [(64, 64), (128, 64), (256, 64), (512, 64), (128, 256), (256, 256), (512, 256),
                 (256, 1024), (512, 1024)]:
    n = (cells - 1) ** 2
    grid = pg.build_time_grid("uniform", N, 2.0)
    load = np.random.default_rng(1).standard_normal((N, n))
    spec = pg.make_weighted_problem(cells, grid, pg.c4_cell_weights(cells, grid, seed=0), load,
                                    np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("2d", cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    t0 = time.perf_counter()
    try:
        _, hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-8, max_iter=3000))
        print(f"cells {cells} N {N}: {hist.iterations} iterations, converged {hist.converged}, "
              f"final {hist.residual[-1]:.3e}, {time.perf_counter() - t0:.1f}s", flush=True)
    except pg.SolverDivergenceError as e:
        print(f"cells {cells} N {N}: DIVERGED ({e}), {time.perf_counter() - t0:.1f}s", flush=True)
    del system, at, ht, spec
