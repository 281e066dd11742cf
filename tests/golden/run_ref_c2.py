import sys, time, math, json, numpy as np
import pintsolve as ps
from pintsolve.problems import ProblemSpec, compute_alpha
cells, N, T = 256, 1024, 1.0
t0=time.time()
grid = ps.build_time_grid("uniform", N, T)
mass, a0 = ps.assemble_mass_stiffness_2d(cells)
n = mass.dim
g = np.random.default_rng(0).standard_normal((N, n))
dinv = (4.0/5.0) / a0.diagonal()
load = g - dinv[None, :] * a0.dot(g.T).T
stiff = [a0] * N
tau_ref = float(np.exp(np.mean(np.log(grid.steps))))
a_ref = stiff[math.ceil(N/2)-1]
alpha = compute_alpha(mass, stiff, grid, tau_ref, a_ref)
spec = ProblemSpec(mass=mass, stiffness=stiff, grid=grid, load=load, u_init=np.zeros(n),
                   tau_ref=tau_ref, a_ref=a_ref, alpha=alpha, meta={"space":"2d","mesh":cells})
system = ps.TimeGlobalSystem(spec)
hier = ps.build_mg_hierarchy("2d", cells)
at = ps.BlockDiagSolver(spec, "mg", hierarchy=hier)
ht = ps.build_schur_preconditioner(spec, "mg", vcycles=1)
t1=time.time(); print("setup", t1-t0, flush=True)
cfg = ps.UzawaConfig(omega=0.9, tol=1e-8, max_iter=200)
(p,u), hist = ps.uzawa_solve(system, at, ht, cfg)
t2=time.time()
print("solve", t2-t1, hist.iterations, hist.residual[0], hist.residual[-1], flush=True)
np.save("/tmp/refruns/c2_u.npy", u); np.save("/tmp/refruns/c2_p.npy", p)
json.dump({"residual": hist.residual, "wall": hist.wall_seconds, "fft": hist.fft_seconds,
           "spatial": hist.spatial_seconds, "iterations": hist.iterations, "converged": hist.converged,
           "setup_s": t1-t0, "solve_s": t2-t1, "tau_ref": tau_ref},
          open("/tmp/refruns/c2_hist.json","w"))
