"""Per-iteration residual drift of a golden Uzawa case in both arithmetics
against the reference history and the committed drift bars (GPU box)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle as orc  # noqa: E402
import paper_1802_08126_b200 as pg  # noqa: E402
import ulp_floor  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "ops2d_c16_N16_coeff"
d = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
c0, c1 = (float(v) for v in d["coeff"])
coeff = None if (c0, c1) == (1.0, 0.0) else (lambda t: c0 + c1 * t)
ref = d["uz_res"]
for arith in ("exact", "fast"):
    pg.set_arithmetic(arith)
    spec = pg.problem_from_arrays(str(d["space"]), int(d["cells"]), pg.TimeGrid(d["nodes"]),
                                  d["load"], d["u_init"], coeff=coeff)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy(str(d["space"]), int(d["cells"])))
    ht = pg.build_schur_preconditioner(spec, "mg")
    cfg = pg.UzawaConfig(omega=float(d["uz_omega"]), tol=float(d["uz_tol"]),
                         max_iter=int(d["uz_max_iter"]))
    (p, u), hist = pg.uzawa_solve(system, at, ht, cfg)
    k = min(hist.iterations, len(ref))
    rel = np.abs(np.array(hist.residual[:k]) - ref[:k]) / ref[:k]
    bar = ulp_floor.bar(name, k, arith)
    print(arith, hist.iterations, len(ref), "worst ratio", float(np.max(rel / bar)),
          "at", int(np.argmax(rel / bar)))
    for i in range(0, k, 1):
        if rel[i] > 0.25 * bar[i] or i % 20 == 0:
            print(f"  {i:4d} res {ref[i]:.3e} rel {rel[i]:.3e} bar {bar[i]:.3e}")
