"""End-to-end breakdown of uzawa_solve on c2 from host numpy arrays:
H2D + reference norm (pint_uzawa_begin), iterations, D2H (pint_uzawa_end)."""
import ctypes
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    load = bench.c2_load()
    pg, spec, system, at, ht = bench.build_solver(load, 0)
    ctx = system._gp.ctx
    f = np.ascontiguousarray(system.rhs)
    out = {"cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0))}
    ref = ctypes.c_double()
    nums = np.zeros(8)
    ms = ctypes.c_double()
    for rep in range(2):
        p = np.empty_like(f)
        u = np.empty_like(f)
        t0 = time.perf_counter()
        ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
        t1 = time.perf_counter()
        ctx.call("pint_uzawa_run", 0.9, 5, nums.ctypes.data, ctypes.byref(ms))
        t2 = time.perf_counter()
        ctx.call("pint_uzawa_end", p.ctypes.data, u.ctypes.data)
        t3 = time.perf_counter()
        out[f"rep{rep}"] = {"begin_s": t1 - t0, "iter5_s": t2 - t1, "end_s": t3 - t2,
                            "h2d_GBps": f.nbytes / (t1 - t0) / 1e9,
                            "d2h_GBps": 2 * f.nbytes / (t3 - t2) / 1e9}
    for rep in range(2):
        t0 = time.perf_counter()
        (p_h, u_h), hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-8))
        out[f"solve{rep}"] = {"wall_s": time.perf_counter() - t0, "iters": hist.iterations,
                              "loop_s": hist.wall_seconds[-1]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
