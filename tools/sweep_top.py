"""Diagnostic: time the fused residual kernels (r1, z) and DSTs under env overrides."""
import ctypes, os, subprocess, sys, json
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

def run_one():
    import paper_1802_08126_b200 as pg
    cells, N = 256, 1024
    n = (cells - 1) ** 2
    grid = pg.build_time_grid("uniform", N, 1.0)
    load = np.random.default_rng(0).standard_normal((N, n))
    spec = pg.problem_from_arrays("2d", cells, grid, load, np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("2d", cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    ctx = system._gp.ctx
    f = np.ascontiguousarray(system.rhs)
    ref = ctypes.c_double()
    ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
    nums = np.zeros(4); ms = ctypes.c_double()
    ctx.call("pint_uzawa_run", 0.9, 2, nums.ctypes.data, ctypes.byref(ms))
    ctx.call("pint_profile", 1)
    ctx.call("pint_uzawa_run", 0.9, 2, nums.ctypes.data, ctypes.byref(ms))
    st = ctx.kernel_stats()
    out = {k: round(v[0] / v[1], 4) for k, v in st.items() if v[1] and (k.startswith("timeop") or k.startswith("dst"))}
    print(json.dumps({"env": {k: os.environ.get(k) for k in ("PINT_STAGES", "PINT_CTAS")}, "ms": out}), flush=True)

if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "one":
        run_one(); sys.exit(0)
    for stages in (2, 3, 4):
        for ctas in (1, 2):
            env = dict(os.environ, PINT_STAGES=str(stages), PINT_CTAS=str(ctas))
            subprocess.run([sys.executable, __file__, "one"], env=env)
