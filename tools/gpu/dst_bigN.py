"""DST throughput at large N (the c4 time axis): S^T and S on an (N, n) slab,
for the column-pair counts PINT_DST_P allows.  usage: dst_bigN.py N cells"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1802_08126_b200 as pg  # noqa: E402

N, cells = int(sys.argv[1]), int(sys.argv[2])
n = (cells - 1) ** 2
plan = pg.DstPlan(N)
x = torch.randn(N, n, dtype=torch.float64, device="cuda")
for name, fn in (("S^T", plan.inverse_transpose), ("S", plan.inverse)):
    y = fn(x)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        y = fn(x)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 5
    print(f"PINT_DST_P={os.environ.get('PINT_DST_P', 'default')} N={N} n={n} {name}: {dt * 1e3:.3f} ms, "
          f"{16.0 * N * n / dt / 1e9:.0f} GB/s")
