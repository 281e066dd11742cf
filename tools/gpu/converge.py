"""Run one BASELINE config to convergence through the public API (GPU box):
iterations, time-to-1e-8, final residual.  usage: converge.py c3|c5|c4 [max_iter]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

name = sys.argv[1]
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 200
t0 = time.perf_counter()
out = bench.converge_config(name, max_iter=max_iter)
out["total_s"] = time.perf_counter() - t0
print(json.dumps(out))
