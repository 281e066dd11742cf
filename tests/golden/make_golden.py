"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container, where the reference is importable:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [--c2 /tmp/refruns]

It imports ``pintsolve`` from $PINTSOLVE_REF (default
/root/reference/pkg/src), builds small seeded cases through the reference's
public API (make_heat_problem / ProblemSpec, TimeGlobalSystem,
BlockDiagSolver, build_schur_preconditioner, DstPlan, uzawa_solve) and writes
their inputs and outputs as .npz fixtures next to this script.  The GPU box
never runs this script; tests read only the committed .npz files.

``--c2 DIR`` additionally summarises a full config-2 reference run produced by
``tests/golden/run_ref_c2.py`` (1871 s, 23 GB RAM on the build host).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.environ.get("PINTSOLVE_REF", "/root/reference/pkg/src"))
import pintsolve as ps  # noqa: E402
from pintsolve.problems import ProblemSpec, compute_alpha  # noqa: E402


def spec_from_arrays(space, cells, grid, load, u_init, coeff=None):
    mass, a0 = (ps.assemble_mass_stiffness_2d if space == "2d"
                else ps.assemble_mass_stiffness_1d)(cells)
    cf = coeff or (lambda t: 1.0)
    cv = [cf(t) for t in grid.nodes[1:]]
    stiff = [a0 if c == 1.0 else a0.scaled(float(c)) for c in cv]
    tau_ref = float(np.exp(np.mean(np.log(grid.steps))))
    a_ref = stiff[math.ceil(grid.N / 2) - 1]
    alpha = compute_alpha(mass, stiff, grid, tau_ref, a_ref)
    return ProblemSpec(mass=mass, stiffness=stiff, grid=grid, load=load, u_init=u_init,
                       tau_ref=tau_ref, a_ref=a_ref, alpha=alpha,
                       meta={"space": space, "mesh": cells})


def operator_case(spec, seed, uzawa_tol, max_iter=300, omega=0.9):
    rng = np.random.default_rng(seed)
    N, n = spec.N, spec.dim
    x = rng.standard_normal((N, n))
    y = rng.standard_normal((N, n))
    system = ps.TimeGlobalSystem(spec)
    hier = ps.build_mg_hierarchy(spec.meta["space"], spec.meta["mesh"])
    at = ps.BlockDiagSolver(spec, "mg", hierarchy=hier)
    ht = ps.build_schur_preconditioner(spec, "mg", vcycles=1)
    plan = ps.DstPlan(N)
    out = dict(
        nodes=spec.grid.nodes, load=spec.load, u_init=spec.u_init, tau_ref=spec.tau_ref,
        x=x, y=y, rhs=system.rhs,
        K_x=system.apply_K(x), Kt_x=system.apply_Kt(x), Abd_x=system.apply_Abd(x),
        atilde_x=at.apply_inverse(x), htilde_x=ht.apply_inverse(x),
        dst_fwd_x=plan.forward(x), dst_inv_x=plan.inverse(x),
        dst_fwdT_x=plan.forward_transpose(x), dst_invT_x=plan.inverse_transpose(x),
        vcyc_a0_y=at.solvers[0].apply(y[0]),
        vcyc_h_last_y=ht.solvers[-1].apply(y[-1]),
        mu=ps.frequency_weights(N),
        mass_dense=spec.mass.todense() if n <= 400 else np.zeros(0),
        a0_dense=spec.stiffness[0].todense() if n <= 400 else np.zeros(0),
    )
    cfg = ps.UzawaConfig(omega=omega, tol=uzawa_tol, max_iter=max_iter)
    (p, u), hist = ps.uzawa_solve(system, at, ht, cfg)
    out.update(uz_p=p, uz_u=u, uz_res=np.array(hist.residual),
               uz_converged=np.array(hist.converged), uz_tol=np.array(uzawa_tol),
               uz_omega=np.array(omega), uz_max_iter=np.array(max_iter))
    u_star = ps.sequential_euler_solve(spec)
    system.build_exact_solvers()
    out.update(u_seq=u_star, s_norm_err=np.array(system.s_norm(u - u_star) / system.s_norm(u_star)))
    return out


def write_c2_summary(run_dir):
    """c2_summary.npz from a full config-2 reference run (run_ref_c2.py):
    17-digit residual history, reference S-norms, seeded samples of the final
    p, u and of the sequential-Euler solution, and per-plane 2-norms."""
    h = json.load(open(os.path.join(run_dir, "c2_hist.json")))
    u = np.load(os.path.join(run_dir, "c2_u.npy"))
    p = np.load(os.path.join(run_dir, "c2_p.npy"))
    useq = np.load(os.path.join(run_dir, "c2_useq.npy"))
    idx = np.sort(np.random.default_rng(123).choice(u.size, 4096, replace=False))
    np.savez_compressed(os.path.join(HERE, "c2_summary.npz"),
                        residual=np.array(h["residual"]), converged=np.array(h["converged"]),
                        sample_idx=idx, u_sample=u.ravel()[idx], p_sample=p.ravel()[idx],
                        useq_sample=useq.ravel()[idx],
                        u_plane_norms=np.linalg.norm(u, axis=1),
                        p_plane_norms=np.linalg.norm(p, axis=1),
                        useq_plane_norms=np.linalg.norm(useq, axis=1),
                        s_norm_seq=np.array(h["s_norm_seq"]), s_norm_u=np.array(h["s_norm_u"]),
                        s_norm_err=np.array(h["s_norm_err"]),
                        solve_s=np.array(h["solve_s"]), setup_s=np.array(h["setup_s"]),
                        wall=np.array(h["wall"]), fft=np.array(h["fft"]),
                        spatial=np.array(h["spatial"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c2", default=None, help="directory with the c2 reference run")
    ap.add_argument("--only-c2", action="store_true", help="write c2_summary.npz only")
    args = ap.parse_args()
    if args.only_c2:
        write_c2_summary(args.c2)
        return

    # A: 2D, perturbed grid, c(t) coefficient, random data (test-suite style)
    grid = ps.build_time_grid("perturbed", 16, 1.3, perturbation=0.3, seed=3)
    spec = ps.make_heat_problem("2d", 16, grid, coeff=lambda t: 0.8 + 0.6 * t,
                                data="random", seed=11)
    np.savez_compressed(os.path.join(HERE, "ops2d_c16_N16_coeff.npz"),
                        space="2d", cells=16, coeff=np.array([0.8, 0.6]),
                        **operator_case(spec, seed=5, uzawa_tol=1e-10,
                                       omega=ps.safe_damping(spec.alpha)))

    # B: 1D, uniform grid, non-power-of-two N (dense DST path)
    grid = ps.build_time_grid("uniform", 12, 1.0)
    spec = ps.make_heat_problem("1d", 16, grid, data="random", seed=7)
    np.savez_compressed(os.path.join(HERE, "ops1d_c16_N12.npz"), space="1d", cells=16,
                        coeff=np.array([1.0, 0.0]),
                        **operator_case(spec, seed=6, uzawa_tol=1e-10))

    # C: the reference's own 2D multigrid Uzawa test problem (test_solvers.py:134-143)
    grid = ps.build_time_grid("uniform", 16, 1.0)
    spec = ps.make_heat_problem("2d", 8, grid, data="sine")
    np.savez_compressed(os.path.join(HERE, "sine2d_c8_N16.npz"), space="2d", cells=8,
                        coeff=np.array([1.0, 0.0]),
                        **operator_case(spec, seed=8, uzawa_tol=1e-9))

    # D: BASELINE config 1 (cells=32 -> 31x31 interior, N=64, T=1, f~N(0,1) seed 0, u0=0)
    grid = ps.build_time_grid("uniform", 64, 1.0)
    load = np.random.default_rng(0).standard_normal((64, 31 * 31))
    spec = spec_from_arrays("2d", 32, grid, load, np.zeros(31 * 31))
    system = ps.TimeGlobalSystem(spec)
    hier = ps.build_mg_hierarchy("2d", 32)
    at = ps.BlockDiagSolver(spec, "mg", hierarchy=hier)
    ht = ps.build_schur_preconditioner(spec, "mg", vcycles=1)
    (p, u), hist = ps.uzawa_solve(system, at, ht, ps.UzawaConfig(omega=0.9, tol=1e-8, max_iter=200))
    u_star = ps.sequential_euler_solve(spec)
    system.build_exact_solvers()
    np.savez_compressed(os.path.join(HERE, "c1_uzawa.npz"),
                        residual=np.array(hist.residual), converged=np.array(hist.converged),
                        p=p, u=u, u_seq=u_star,
                        s_norm_err=np.array(system.s_norm(u - u_star) / system.s_norm(u_star)),
                        s_norm_seq=np.array(system.s_norm(u_star)))

    if args.c2:
        write_c2_summary(args.c2)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
