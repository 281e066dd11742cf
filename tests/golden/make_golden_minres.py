"""Golden vectors for the second solver entry point and the diagnostic
oracle pieces, from the UNMODIFIED reference package:

  * minres_solve (solvers.py:267-327) on two small 2D cases,
  * sequential_euler_solve (solvers.py:158-174) and TimeGlobalSystem.s_norm
    (operators.py:176-183) on the same cases.

Run in the build container (the GPU box never runs it):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_minres.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, os.environ.get("PINTSOLVE_REF", "/root/reference/pkg/src"))
import pintsolve as ps  # noqa: E402
from make_golden import spec_from_arrays  # noqa: E402


def case(name, spec, tol, max_iter, seed):
    system = ps.TimeGlobalSystem(spec)
    hier = ps.build_mg_hierarchy(spec.meta["space"], spec.meta["mesh"])
    at = ps.BlockDiagSolver(spec, "mg", hierarchy=hier)
    ht = ps.build_schur_preconditioner(spec, "mg", vcycles=1)
    (p, u), hist = ps.minres_solve(system, at, ht, tol=tol, max_iter=max_iter)
    u_seq = ps.sequential_euler_solve(spec)
    system.build_exact_solvers()
    x = np.random.default_rng(seed).standard_normal((spec.N, spec.dim))
    np.savez_compressed(
        os.path.join(HERE, name), nodes=spec.grid.nodes, load=spec.load, u_init=spec.u_init,
        cells=np.array(spec.meta["mesh"]), space=spec.meta["space"],
        mr_res=np.array(hist.residual), mr_converged=np.array(hist.converged),
        mr_tol=np.array(tol), mr_max_iter=np.array(max_iter), mr_p=p, mr_u=u,
        u_seq=u_seq, s_norm_seq=np.array(system.s_norm(u_seq)),
        x=x, s_norm_x=np.array(system.s_norm(x)), s_norm_err=np.array(system.s_norm(u - u_seq)))


def main():
    # BASELINE-style data on a small grid: f ~ N(0,1) seed 0, u0 = 0
    grid = ps.build_time_grid("uniform", 16, 1.0)
    load = np.random.default_rng(0).standard_normal((16, 15 * 15))
    case("minres_c16_N16.npz", spec_from_arrays("2d", 16, grid, load, np.zeros(15 * 15)),
         tol=1e-8, max_iter=300, seed=21)
    # the reference's sine problem (test_solvers.py:134-143 style), N = 32
    grid = ps.build_time_grid("uniform", 32, 1.0)
    spec = ps.make_heat_problem("2d", 8, grid, data="sine")
    case("minres_sine_c8_N32.npz", spec, tol=1e-10, max_iter=300, seed=22)
    print("minres golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
