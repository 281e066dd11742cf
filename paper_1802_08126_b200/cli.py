"""Command-line entry point: ``python -m paper_1802_08126_b200 solve ...``.

Mirrors the reference's ``pintsolve solve`` (cli.py:60-76, 131-155): build a
heat problem (or load one with --problem-file, problems.py:348-395), run the
Uzawa or MINRES solver on the GPU and write the ConvergenceHistory CSV
(solvers.py:64-74) to --out or stdout.  Exit codes as the reference: 0
success, 1 bad input, 3 solver divergence.  The GPU path implements the
multigrid spatial solver only; --solver direct/jacobi and
--method sequential are rejected with exit code 1.
"""

from __future__ import annotations

import argparse
import sys

from .errors import InputError, SolverDivergenceError


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_1802_08126_b200",
        description="Time-parallel solvers for implicit-Euler parabolic problems (B200 path)")
    sub = parser.add_subparsers(dest="command", required=True)
    p = sub.add_parser("solve", help="solve one heat problem and report convergence")
    p.add_argument("--out", help="output CSV path (default: stdout)")
    p.add_argument("--seed", type=int, default=7)
    p.add_argument("--T", type=float, default=1.0, help="final time")
    p.add_argument("--space", choices=["2d", "3d"], default="2d")
    p.add_argument("--h", type=int, default=64, help="mesh cells per side (h=1/cells)")
    p.add_argument("--N", type=int, default=64, help="number of time steps")
    p.add_argument("--data", default="sine", help="sine | random | zero")
    p.add_argument("--problem-file", help="load the problem from a file instead")
    p.add_argument("--method", choices=["uzawa", "minres", "sequential"], default="uzawa")
    p.add_argument("--solver", choices=["direct", "mg", "jacobi"], default="mg")
    p.add_argument("--vcycles", type=int, default=1)
    p.add_argument("--omega", type=float, default=0.9)
    p.add_argument("--tol", type=float, default=1e-8)
    p.add_argument("--max-iter", type=int, default=200)
    return parser


def _cmd_solve(args) -> str:
    from . import (BlockDiagSolver, TimeGlobalSystem, UzawaConfig, build_mg_hierarchy,
                   build_schur_preconditioner, build_time_grid, load_problem,
                   make_heat_problem, minres_solve, uzawa_solve)

    if args.method == "sequential":
        raise InputError("--method sequential (exact per-step factorisations) is not on the GPU path")
    if args.solver != "mg":
        raise InputError("the GPU path implements the multigrid spatial solver (--solver mg)")
    if args.problem_file:
        spec = load_problem(args.problem_file)
        if not spec.meta:
            raise InputError("problem file is not on a structured 2^k-cell grid")
    else:
        grid = build_time_grid("uniform", args.N, args.T)
        spec = make_heat_problem(args.space, args.h, grid, data=args.data, seed=args.seed)
    system = TimeGlobalSystem(spec)
    hier = build_mg_hierarchy(spec.meta["space"], spec.meta["mesh"])
    at = BlockDiagSolver(spec, "mg", hierarchy=hier, cycles=args.vcycles)
    ht = build_schur_preconditioner(spec, "mg", vcycles=args.vcycles)
    if args.method == "minres":
        _, hist = minres_solve(system, at, ht, tol=args.tol, max_iter=args.max_iter)
    else:
        cfg = UzawaConfig(omega=args.omega, tol=args.tol, max_iter=args.max_iter)
        _, hist = uzawa_solve(system, at, ht, cfg)
    return hist.to_csv()


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    try:
        text = _cmd_solve(args)
    except SolverDivergenceError as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 3
    except (InputError, ValueError, OSError) as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 1
    if args.out:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(text)
    else:
        sys.stdout.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
