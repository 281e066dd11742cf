"""Per-iteration timing and kernel shares for the non-headline BASELINE
configs (c3: 3D 63^3, N=512; c5 at G=1: 3D 63^3, N=1024).  Development tool;
bench.py remains the contract for the headline c2 line."""

import argparse
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

CFG = {
    "c3": dict(space="3d", cells=64, N=512, T=1.0),
    "c5": dict(space="3d", cells=64, N=1024, T=1.0),
    "c2": dict(space="2d", cells=256, N=1024, T=1.0),
    "c4": dict(space="2d", cells=512, N=4096, T=2.0),
    "c4s": dict(space="2d", cells=512, N=1024, T=2.0),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(CFG))
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--N", type=int, default=0)
    ap.add_argument("--separable", action="store_true", help="c4: separable family (pint_field_separable)")
    args = ap.parse_args()
    import paper_1802_08126_b200 as pg

    c = CFG[args.config]
    cells, N, space = c["cells"], args.N or c["N"], c["space"]
    n = (cells - 1) ** (3 if space == "3d" else 2)
    import time
    t0 = time.perf_counter()
    grid = pg.build_time_grid("uniform", N, c["T"])
    if args.config.startswith("c4"):
        load = np.random.default_rng(1).standard_normal((N, n))
        spec = pg.make_weighted_problem(cells, grid, pg.c4_cell_weights(cells, grid, seed=0),
                                        load, np.zeros(n), alpha=1.0, separable=args.separable)
    else:
        rng = np.random.default_rng(0)
        load = rng.standard_normal((N, n))
        u0 = rng.uniform(0.0, 1.0, n) if args.config == "c3" else np.zeros(n)
        spec = pg.problem_from_arrays(space, cells, grid, load, u0, alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy(space, cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    ctx = system._gp.ctx
    setup_s = time.perf_counter() - t0
    f = np.ascontiguousarray(system.rhs)
    ref = ctypes.c_double()
    ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
    nums = np.zeros(64)
    ms = ctypes.c_double()
    ctx.call("pint_uzawa_run", 0.9, 3, nums.ctypes.data, ctypes.byref(ms))
    ctx.call("pint_uzawa_run", 0.9, args.steps, nums.ctypes.data, ctypes.byref(ms))
    ms_it = ms.value / args.steps
    ctx.call("pint_profile", 1)
    ctx.call("pint_uzawa_run", 0.9, 2, nums.ctypes.data, ctypes.byref(ms))
    stats = ctx.kernel_stats()
    ctx.call("pint_profile", 0)
    tot = sum(v[0] for v in stats.values())
    import torch
    out = {"config": args.config, "n": n, "N": N, "ms_per_iter": ms_it, "setup_s": setup_s,
           "gpu_mem_GB": torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9,
           "DoF_per_s": N * n / (ms_it / 1e3),
           "iteration_alg_GBps": 224.0 * N * n / (ms_it / 1e3) / 1e9,
           "kernels": {k: {"ms": v[0] / v[1], "share": round(v[0] / tot, 4),
                           "GBps": round(v[2] / v[0] / 1e6, 1), "launches": v[1]}
                       for k, v in sorted(stats.items(), key=lambda kv: -kv[1][0]) if v[1]}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
