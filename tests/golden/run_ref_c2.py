"""Full BASELINE config-2 run of the UNMODIFIED reference (build host only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/run_ref_c2.py /tmp/refruns

Writes the Uzawa history, final (p, u), the sequential implicit-Euler
solution and the reference's own S-norm errors into DIR; ``make_golden.py
--c2 DIR`` condenses them into the committed ``c2_summary.npz``.  Needs
~25 GB of RAM and ~35 minutes on one core.
"""
import json
import math
import os
import sys
import time

import numpy as np
import pintsolve as ps
from pintsolve.problems import ProblemSpec, compute_alpha

out_dir = sys.argv[1] if len(sys.argv) > 1 else "/tmp/refruns"
os.makedirs(out_dir, exist_ok=True)
ps.parallel.set_num_threads(int(os.environ.get("REF_THREADS", "1")))
cells, N, T = 256, 1024, 1.0
t0 = time.time()
grid = ps.build_time_grid("uniform", N, T)
mass, a0 = ps.assemble_mass_stiffness_2d(cells)
n = mass.dim
g = np.random.default_rng(0).standard_normal((N, n))
dinv = (4.0 / 5.0) / a0.diagonal()
load = g - dinv[None, :] * a0.dot(g.T).T
stiff = [a0] * N
tau_ref = float(np.exp(np.mean(np.log(grid.steps))))
a_ref = stiff[math.ceil(N / 2) - 1]
alpha = compute_alpha(mass, stiff, grid, tau_ref, a_ref)
spec = ProblemSpec(mass=mass, stiffness=stiff, grid=grid, load=load, u_init=np.zeros(n),
                   tau_ref=tau_ref, a_ref=a_ref, alpha=alpha, meta={"space": "2d", "mesh": cells})
system = ps.TimeGlobalSystem(spec)
hier = ps.build_mg_hierarchy("2d", cells)
at = ps.BlockDiagSolver(spec, "mg", hierarchy=hier)
ht = ps.build_schur_preconditioner(spec, "mg", vcycles=1)
t1 = time.time()
print("setup", t1 - t0, flush=True)
cfg = ps.UzawaConfig(omega=0.9, tol=1e-8, max_iter=200)
(p, u), hist = ps.uzawa_solve(system, at, ht, cfg)
t2 = time.time()
print("solve", t2 - t1, hist.iterations, hist.residual[0], hist.residual[-1], flush=True)
np.save(os.path.join(out_dir, "c2_u.npy"), u)
np.save(os.path.join(out_dir, "c2_p.npy"), p)
del at, ht
u_seq = ps.sequential_euler_solve(spec)
np.save(os.path.join(out_dir, "c2_useq.npy"), u_seq)
system.build_exact_solvers()
s_seq = system.s_norm(u_seq)
s_err = system.s_norm(u - u_seq)
s_u = system.s_norm(u)
t3 = time.time()
print("s-norm", s_err / s_seq, "seq+norm s", t3 - t2, flush=True)
json.dump({"residual": hist.residual, "wall": hist.wall_seconds, "fft": hist.fft_seconds,
           "spatial": hist.spatial_seconds, "iterations": hist.iterations,
           "converged": hist.converged, "setup_s": t1 - t0, "solve_s": t2 - t1,
           "tau_ref": tau_ref, "s_norm_seq": s_seq, "s_norm_u": s_u, "s_norm_err": s_err},
          open(os.path.join(out_dir, "c2_hist.json"), "w"))
