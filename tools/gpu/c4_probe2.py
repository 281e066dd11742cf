"""c4-coefficient Uzawa at small cells, large N: first residuals on the GPU and
(CELLS <= 32) from the CPU oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as orc  # noqa: E402
import paper_1802_08126_b200 as pg  # noqa: E402

for cells, N, with_oracle in [(64, 2048, False), (32, 2048, False), (16, 2048, True), (16, 1024, True)]:
    n = (cells - 1) ** 2
    grid = pg.build_time_grid("uniform", N, 2.0)
    w = pg.c4_cell_weights(cells, grid, seed=0)
    load = np.random.default_rng(1).standard_normal((N, n))
    spec = pg.make_weighted_problem(cells, grid, w, load, np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("2d", cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    try:
        _, hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-30, max_iter=12))
        r = hist.residual
    except pg.SolverDivergenceError as e:
        r = [str(e)]
    print(f"GPU cells {cells} N {N}:", " ".join(f"{v:.6e}" if isinstance(v, float) else v for v in r), flush=True)
    if with_oracle:
        stiff = [orc.stiffness_2d_weighted(cells, w(k)) for k in range(N)]
        opb = orc.heat_problem("2d", cells, grid.nodes, load=load, u_init=np.zeros(n), stiffness=stiff)
        lev = orc.mg_levels("2d", cells)
        ref = orc.uzawa(opb, orc.BlockInv(opb, lev), orc.SchurInv(opb, lev), 0.9, 1e-30, 12)
        print(f"ORC cells {cells} N {N}:", " ".join(f"{v:.6e}" for v in ref.residual), flush=True)
    del system, at, ht, spec
