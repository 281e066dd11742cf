"""First residuals of the c4 problem (cells = 512, T = 2) for growing N (GPU box)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1802_08126_b200 as pg  # noqa: E402

cells = int(os.environ.get("CELLS", "512"))
for N in [int(a) for a in sys.argv[1:]] or [1024, 2048, 3072, 4096]:
    n = (cells - 1) ** 2
    grid = pg.build_time_grid("uniform", N, 2.0)
    load = np.random.default_rng(1).standard_normal((N, n))
    spec = pg.make_weighted_problem(cells, grid, pg.c4_cell_weights(cells, grid, seed=0), load,
                                    np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("2d", cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    try:
        _, hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-30, max_iter=40))
        r = hist.residual
    except pg.SolverDivergenceError as e:
        r = [str(e)]
    print(f"N {N}:", " ".join(f"{v:.4e}" if isinstance(v, float) else v for v in r[:12]), "...",
          " ".join(f"{v:.3e}" for v in r[-3:] if isinstance(v, float)), flush=True)
    del system, at, ht, spec
