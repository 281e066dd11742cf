"""Minimal c2 driver for ncu captures: setup, pint_uzawa_begin, K iterations."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    iters = int(sys.argv[1]) if len(sys.argv) > 1 else 2
    load = bench.c2_load()
    pg, spec, system, at, ht = bench.build_solver(load, 0)
    ctx = system._gp.ctx
    f = np.ascontiguousarray(system.rhs)
    ref = ctypes.c_double()
    ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
    nums = np.zeros(max(iters, 1))
    ms = ctypes.c_double()
    ctx.call("pint_uzawa_run", 0.9, iters, nums.ctypes.data, ctypes.byref(ms))
    print("ms/iter", ms.value / max(iters, 1), "res", nums[:iters] / ref.value)


if __name__ == "__main__":
    main()
