"""Problem files written by the UNMODIFIED reference (problems.py:300-345)
for the problem-file I/O parity tests.  Build container only:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_problem_io.py
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("PINTSOLVE_REF", "/root/reference/pkg/src"))
import pintsolve as ps  # noqa: E402


def main():
    grid = ps.build_time_grid("perturbed", 4, 1.0, perturbation=0.2, seed=5)
    spec = ps.make_heat_problem("2d", 8, grid, coeff=lambda t: 1.0 + t, data="random", seed=3)
    path = os.path.join(HERE, "problem_c8_N4.txt")
    ps.save_problem(spec, path)
    back = ps.load_problem(path)
    np.savez_compressed(os.path.join(HERE, "problem_c8_N4.npz"), nodes=back.grid.nodes,
                        load=back.load, u_init=back.u_init, tau_ref=np.array(back.tau_ref),
                        alpha=np.array(back.alpha), mass=back.mass.todense(),
                        a_ref=back.a_ref.todense(),
                        stiff=np.stack([a.todense() for a in back.stiffness]))
    # Solver histories on the loaded problem.  The reference CLI cannot run
    # --solver mg on a problem file (load_problem leaves meta empty and
    # cli.py:145 reads meta["space"]), so the runs use the API with the mesh
    # metadata restored, as paper_1802_08126_b200.load_problem does.
    back.meta.update({"space": "2d", "mesh": 8})
    system = ps.TimeGlobalSystem(back)
    hier = ps.build_mg_hierarchy("2d", 8)
    at = ps.BlockDiagSolver(back, "mg", hierarchy=hier)
    ht = ps.build_schur_preconditioner(back, "mg", vcycles=1)
    omega = ps.safe_damping(back.alpha)
    _, h1 = ps.uzawa_solve(system, at, ht, ps.UzawaConfig(omega=omega, tol=1e-10, max_iter=300))
    np.save(os.path.join(HERE, "problem_c8_N4_omega.npy"), np.array(omega))
    open(os.path.join(HERE, "problem_c8_N4_uzawa.csv"), "w").write(h1.to_csv())
    _, h2 = ps.minres_solve(system, at, ht, tol=1e-10, max_iter=300)
    open(os.path.join(HERE, "problem_c8_N4_minres.csv"), "w").write(h2.to_csv())
    print("written", path)


if __name__ == "__main__":
    main()

