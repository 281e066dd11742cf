"""Command-line entry point: ``python -m paper_1802_08126_b200 solve ...``.

Mirrors the reference's ``pintsolve solve`` (cli.py:60-76, 131-155): build a
heat problem (or load one with --problem-file, problems.py:348-395), run the
Uzawa or MINRES solver on the GPU and write the ConvergenceHistory CSV
(solvers.py:64-74) to --out or stdout; ``--diagnostics`` adds the exact
S-norm error column, ``--method sequential`` writes the time-stepping
oracle's first node (both host-side SuperLU, diagnostics.py).  ``table2``
mirrors ``pintsolve table2`` (cli.py:86-92, bench.py:111-139): the paper's
iteration-count table, Uzawa on the GPU stopped on the S-norm error.  Exit
codes as the reference: 0 success, 1 bad input, 3 solver divergence.  The
GPU path implements the multigrid spatial solver only;
--solver direct/jacobi is rejected with exit code 1.
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
    p.add_argument("--diagnostics", action="store_true",
                   help="record exact error norms against the sequential sweep")
    p = sub.add_parser("table2", help="iteration-count table (2d, multigrid)")
    p.add_argument("--out", help="output CSV path (default: stdout)")
    p.add_argument("--T", type=float, default=1.0, help="final time")
    p.add_argument("--h", type=_int_list, default=[8, 16, 32, 64])
    p.add_argument("--N", type=_int_list, default=[128, 256, 512, 1024])
    p.add_argument("--omega", type=float, default=0.9)
    p.add_argument("--tol", type=float, default=1e-6)
    p.add_argument("--vcycles", type=int, default=1)
    return parser


def _int_list(text: str) -> list[int]:
    try:
        return [int(v) for v in text.split(",") if v.strip()]
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers: {text!r}") from exc


def run_table2(h_list=None, n_list=None, T: float = 1.0, omega: float = 0.9, tol: float = 1e-6,
               vcycles: int = 1) -> list[dict]:
    """Iteration counts of the two-stage iteration on the 2d heat problem with
    one-V-cycle multigrid, stopped on the relative S-norm error against the
    time-stepping oracle (bench.py:111-139 of the reference), Uzawa on the GPU."""
    from . import (BlockDiagSolver, TimeGlobalSystem, UzawaConfig, build_mg_hierarchy,
                   build_schur_preconditioner, build_time_grid, make_heat_problem,
                   sequential_euler_solve, uzawa_solve)

    rows = []
    for cells in h_list or [8, 16, 32, 64]:
        hier = build_mg_hierarchy("2d", cells)
        for N in n_list or [128, 256, 512, 1024]:
            spec = make_heat_problem("2d", cells, build_time_grid("uniform", N, T), data="sine")
            system = TimeGlobalSystem(spec, diagnostic=True)
            u_star = sequential_euler_solve(spec)
            at = BlockDiagSolver(spec, "mg", hierarchy=hier, cycles=vcycles)
            ht = build_schur_preconditioner(spec, "mg", vcycles=vcycles)
            cfg = UzawaConfig(omega=omega, tol=tol, stopping="s_norm_error", max_iter=200)
            _, hist = uzawa_solve(system, at, ht, cfg, u_oracle=u_star)
            rows.append({"h": f"1/{cells}", "N": N, "iterations": hist.iterations})
    return rows


def _rows_to_csv(header: str, rows: list[dict]) -> str:
    cols = header.split(",")
    return "\n".join([header] + [",".join(str(r[c]) for c in cols) for r in rows]) + "\n"


def _cmd_solve(args) -> str:
    from . import (BlockDiagSolver, TimeGlobalSystem, UzawaConfig, build_mg_hierarchy,
                   build_schur_preconditioner, build_time_grid, load_problem,
                   make_heat_problem, minres_solve, uzawa_solve)

    if args.problem_file:
        spec = load_problem(args.problem_file)
    else:
        grid = build_time_grid("uniform", args.N, args.T)
        spec = make_heat_problem(args.space, args.h, grid, data=args.data, seed=args.seed)
    if args.method == "sequential":
        from .diagnostics import sequential_euler_solve

        u = sequential_euler_solve(spec)
        lines = ["step,node"] + [f"{n + 1},{u[n, 0]:.17g}" for n in range(spec.N)]
        return "\n".join(lines) + "\n"
    if args.solver != "mg":
        raise InputError("the GPU path implements the multigrid spatial solver (--solver mg)")
    if not spec.meta:
        raise InputError("problem file is not on a structured 2^k-cell grid")
    system = TimeGlobalSystem(spec, diagnostic=args.diagnostics)
    hier = build_mg_hierarchy(spec.meta["space"], spec.meta["mesh"])
    at = BlockDiagSolver(spec, "mg", hierarchy=hier, cycles=args.vcycles)
    ht = build_schur_preconditioner(spec, "mg", vcycles=args.vcycles)
    if args.method == "minres":
        _, hist = minres_solve(system, at, ht, tol=args.tol, max_iter=args.max_iter)
    else:
        cfg = UzawaConfig(omega=args.omega, tol=args.tol, max_iter=args.max_iter,
                          diagnostics=args.diagnostics)
        _, hist = uzawa_solve(system, at, ht, cfg)
    return hist.to_csv()


def main(argv=None) -> int:
    parser = build_parser()
    try:
        args = parser.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 1
    try:
        if args.command == "table2":
            rows = run_table2(args.h, args.N, T=args.T, omega=args.omega, tol=args.tol,
                              vcycles=args.vcycles)
            text = _rows_to_csv("h,N,iterations", rows)
        else:
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
