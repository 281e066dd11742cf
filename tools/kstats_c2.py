"""Per-kernel device times of the c2 Uzawa step (profiling mode), for A/B
runs of the diagnostic environment knobs (PINT_*)."""
import ctypes
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    load = bench.c2_load()
    pg, spec, system, at, ht = bench.build_solver(load, 0)
    ctx = system._gp.ctx
    f = np.ascontiguousarray(system.rhs)
    ref = ctypes.c_double()
    ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
    nums = np.zeros(8)
    ms = ctypes.c_double()
    ctx.call("pint_uzawa_run", 0.9, 3, nums.ctypes.data, ctypes.byref(ms))
    ctx.call("pint_uzawa_run", 0.9, 5, nums.ctypes.data, ctypes.byref(ms))
    step = ms.value / 5
    ctx.call("pint_profile", 1)
    ctx.call("pint_uzawa_run", 0.9, 2, nums.ctypes.data, ctypes.byref(ms))
    st = ctx.kernel_stats()
    env = {k: v for k, v in os.environ.items() if k.startswith("PINT_")}
    print(json.dumps({"env": env, "ms_per_step": round(step, 4),
                      "ms": {k: round(v[0] / v[1], 4) for k, v in st.items() if v[1]}}))


if __name__ == "__main__":
    main()
