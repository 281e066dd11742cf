"""Command line: ``python -m paper_1802_08126_b200 <command> [options]``.

The reference's ``pintsolve`` CLI (cli.py:46-228) for the commands that run
on the GPU path:

  solve    one heat problem (or ``--problem-file``), Uzawa / MINRES / the
           sequential oracle; writes the ConvergenceHistory CSV
  table2   the paper's iteration-count table (bench.py:111-139)
  history  S-norm error decay of the multigrid Uzawa iteration (bench.py:142-183,
           the "mg1" variant: the GPU path runs one V-cycle per block)
  scaling  device time per Uzawa iteration and its DST / multigrid shares
           versus the number of GPUs (bench.py:264-310 times threads; the
           GPU analogue partitions the time axis over 1..G GPUs)

``--config FILE`` supplies ``key=value`` defaults (``#`` comments; a key is
an option name without the leading dashes); options given on the command
line win (cli.py:32-43, 161-181).  Exit codes: 0 success, 1 bad input,
3 solver divergence.  Only the multigrid spatial solver exists on the GPU:
``--solver direct|jacobi`` is rejected with exit code 1.
"""

from __future__ import annotations

import argparse
import os
import subprocess
import sys

from .errors import InputError, SolverDivergenceError


def _int_list(text: str) -> list[int]:
    try:
        return [int(v) for v in text.split(",") if v.strip()]
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers: {text!r}") from exc


# (flags, keyword arguments) per option; grouped so commands share them
_COMMON = [
    (("--out",), dict(help="output CSV path (default: stdout)")),
    (("--seed",), dict(type=int, default=7)),
    (("--T",), dict(type=float, default=1.0, help="final time")),
]
_PROBLEM = [
    (("--space",), dict(choices=["2d", "3d"], default="2d")),
    (("--h",), dict(type=int, default=64, help="mesh cells per side (h = 1/cells)")),
    (("--N",), dict(type=int, default=64, help="number of time steps")),
]
_ITERATION = [
    (("--omega",), dict(type=float, default=0.9)),
    (("--tol",), dict(type=float, default=1e-8)),
    (("--max-iter",), dict(type=int, default=200)),
]
_COMMANDS = {
    "solve": ("solve one heat problem and report convergence", _COMMON + _PROBLEM + _ITERATION + [
        (("--data",), dict(default="sine", choices=["sine", "zero", "manufactured", "random"])),
        (("--problem-file",), dict(help="load the problem from a file instead")),
        (("--method",), dict(choices=["uzawa", "minres", "sequential"], default="uzawa")),
        (("--solver",), dict(choices=["direct", "mg", "jacobi"], default="mg")),
        (("--vcycles",), dict(type=int, default=1)),
        (("--diagnostics",), dict(action="store_true",
                                  help="record exact S-norm errors against the sequential sweep")),
    ]),
    "table2": ("iteration-count table (2d, multigrid)", _COMMON + [
        (("--h",), dict(type=_int_list, default=[8, 16, 32, 64])),
        (("--N",), dict(type=_int_list, default=[128, 256, 512, 1024])),
        (("--omega",), dict(type=float, default=0.9)),
        (("--tol",), dict(type=float, default=1e-6)),
        (("--vcycles",), dict(type=int, default=1)),
    ]),
    "history": ("S-norm error decay of the multigrid iteration", _COMMON + [
        (("--space",), dict(choices=["2d", "3d"], default="2d")),
        (("--h",), dict(type=int, default=64)),
        (("--N",), dict(type=int, default=512)),
        (("--omega",), dict(type=float, default=0.9)),
        (("--tol",), dict(type=float, default=1e-10)),
        (("--max-iter",), dict(type=int, default=200)),
    ]),
    "scaling": ("device time per iteration versus GPUs", _COMMON + [
        (("--space",), dict(choices=["2d", "3d"], default="2d")),
        (("--h",), dict(type=int, default=32)),
        (("--N",), dict(type=int, default=256)),
        (("--omega",), dict(type=float, default=0.9)),
        (("--iters",), dict(type=int, default=10)),
        (("--repeats",), dict(type=int, default=5)),
        (("--gpu-list",), dict(type=_int_list, default=[1])),
    ]),
}

HEADERS = {
    "table2": "h,N,iterations",
    "history": "iter,solver,s_norm_error,residual",
    "scaling": "gpus,time_per_iter,total_time,fft_share,spatial_share",
}


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(
        prog="paper_1802_08126_b200",
        description="Time-parallel solvers for implicit-Euler parabolic problems (B200 path)")
    parser.add_argument("--config", help="key=value file; the command line overrides it")
    sub = parser.add_subparsers(dest="command", required=True)
    for name, (text, options) in _COMMANDS.items():
        p = sub.add_parser(name, help=text)
        for flags, kw in options:
            p.add_argument(*flags, **kw)
    return parser


def read_config(path: str) -> dict[str, str]:
    """``key = value`` lines; ``#`` starts a comment; blank lines ignored."""
    entries: dict[str, str] = {}
    with open(path, encoding="utf-8") as fh:
        for number, raw in enumerate(fh, start=1):
            text = raw.partition("#")[0].strip()
            if not text:
                continue
            key, eq, value = text.partition("=")
            if not eq or not key.strip():
                raise InputError(f"bad config line {number}: {raw.strip()!r}")
            entries[key.strip()] = value.strip()
    return entries


def merge_config(argv: list[str], entries: dict[str, str]) -> list[str]:
    """Insert ``--key value`` for every config key not given on the command
    line, right after the subcommand so the subparser sees them."""
    given = {a.split("=", 1)[0] for a in argv if a.startswith("--")}
    extra: list[str] = []
    for key, value in entries.items():
        flag = "--" + key
        if flag in given:
            continue
        extra.append(flag)
        if value.lower() not in ("true", ""):
            extra.append(value)
    cmd = next((i for i, a in enumerate(argv) if a in _COMMANDS), len(argv))
    return argv[:cmd + 1] + extra + argv[cmd + 1:]


# ---------------------------------------------------------------------------
# commands
# ---------------------------------------------------------------------------


def _fmt(x) -> str:
    return f"{x:.17g}" if isinstance(x, float) else str(x)


def rows_to_csv(header: str, rows: list[dict]) -> str:
    cols = header.split(",")
    body = [",".join(_fmt(row[c]) if row[c] is not None else "" for c in cols) for row in rows]
    return "\n".join([header, *body]) + "\n"


def _solvers(spec, vcycles: int = 1, diagnostic: bool = False):
    from . import (BlockDiagSolver, TimeGlobalSystem, build_mg_hierarchy,
                   build_schur_preconditioner)

    if not spec.meta:
        raise InputError("problem is not on a structured 2^k-cell grid")
    hier = build_mg_hierarchy(spec.meta["space"], spec.meta["mesh"])
    system = TimeGlobalSystem(spec, diagnostic=diagnostic)
    return (system, BlockDiagSolver(spec, "mg", hierarchy=hier, cycles=vcycles),
            build_schur_preconditioner(spec, "mg", vcycles=vcycles))


def cmd_solve(args) -> str:
    from . import (UzawaConfig, build_time_grid, load_problem, make_heat_problem, minres_solve,
                   sequential_euler_solve, uzawa_solve)

    if args.problem_file:
        spec = load_problem(args.problem_file)
    else:
        spec = make_heat_problem(args.space, args.h, build_time_grid("uniform", args.N, args.T),
                                 data=args.data, seed=args.seed)
    if args.method == "sequential":
        u = sequential_euler_solve(spec)
        return rows_to_csv("step,node", [{"step": k + 1, "node": float(u[k, 0])}
                                         for k in range(spec.N)])
    if args.solver != "mg":
        raise InputError("the GPU path implements the multigrid spatial solver (--solver mg)")
    system, at, ht = _solvers(spec, args.vcycles, args.diagnostics)
    if args.method == "minres":
        _, hist = minres_solve(system, at, ht, tol=args.tol, max_iter=args.max_iter)
    else:
        cfg = UzawaConfig(omega=args.omega, tol=args.tol, max_iter=args.max_iter,
                          diagnostics=args.diagnostics)
        _, hist = uzawa_solve(system, at, ht, cfg)
    return hist.to_csv()


def run_table2(h_list=None, n_list=None, T: float = 1.0, omega: float = 0.9, tol: float = 1e-6,
               vcycles: int = 1) -> list[dict]:
    """Iteration counts of the multigrid Uzawa iteration on the 2d sine
    problem, stopped on the relative S-norm error against the sequential
    oracle (bench.py:111-139); oracle and norms on the device."""
    from . import UzawaConfig, build_time_grid, make_heat_problem, uzawa_solve

    rows = []
    for cells in h_list or [8, 16, 32, 64]:
        for N in n_list or [128, 256, 512, 1024]:
            spec = make_heat_problem("2d", cells, build_time_grid("uniform", N, T), data="sine")
            system, at, ht = _solvers(spec, vcycles, diagnostic=True)
            cfg = UzawaConfig(omega=omega, tol=tol, stopping="s_norm_error", max_iter=200)
            _, hist = uzawa_solve(system, at, ht, cfg)
            rows.append({"h": f"1/{cells}", "N": N, "iterations": hist.iterations})
    return rows


def run_history(N=512, cells=64, space="2d", T=1.0, omega=0.9, tol=1e-10,
                max_iter=200) -> list[dict]:
    """Per-iteration S-norm error and residual of the one-V-cycle multigrid
    Uzawa iteration on the sine problem (the "mg1" rows of bench.py:142-183)."""
    from . import UzawaConfig, build_time_grid, make_heat_problem, uzawa_solve

    spec = make_heat_problem(space, cells, build_time_grid("uniform", N, T), data="sine")
    system, at, ht = _solvers(spec, 1, diagnostic=True)
    cfg = UzawaConfig(omega=omega, tol=tol, stopping="s_norm_error", max_iter=max_iter,
                      diagnostics=True)
    _, hist = uzawa_solve(system, at, ht, cfg)
    return [{"iter": i + 1, "solver": "mg1", "s_norm_error": hist.s_norm_error[i],
             "residual": hist.residual[i]} for i in range(hist.iterations)]


def time_iterations(spec, omega: float, iters: int, repeats: int) -> dict:
    """Median device time of `iters` Uzawa iterations and the DST / multigrid
    shares of it (CUDA events around the phases, as timing.py's counters)."""
    import ctypes
    import statistics

    import numpy as np

    system, at, ht = _solvers(spec)
    ctx = system._gp.ctx
    f = np.ascontiguousarray(system.rhs)
    ref = ctypes.c_double()
    ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
    nums = np.zeros(max(iters, 2))
    ms = ctypes.c_double()
    ctx.call("pint_uzawa_run", float(omega), 2, nums.ctypes.data, ctypes.byref(ms))  # warm-up
    totals, shares = [], (0.0, 0.0)
    phase = np.zeros(3)
    for _ in range(repeats):
        ctx.call("pint_set_timing", 1)
        ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
        ctx.call("pint_uzawa_run", float(omega), iters, nums.ctypes.data, ctypes.byref(ms))
        ctx.call("pint_phase_ms", phase.ctypes.data)
        ctx.call("pint_set_timing", 0)
        totals.append(ms.value / 1e3)
        shares = (phase[0] / ms.value, phase[1] / ms.value)
    total = statistics.median(totals)
    return {"time_per_iter": total / iters, "total_time": total, "fft_share": float(shares[0]),
            "spatial_share": float(shares[1])}


def run_scaling(gpu_list=None, N=256, cells=32, space="2d", T=1.0, omega=0.9, iters=10,
                repeats=5) -> list[dict]:
    """Device time per iteration with the time axis partitioned over G GPUs
    (G = 1 in this process; G > 1 through torchrun, one process per GPU,
    paper_1802_08126_b200.distributed)."""
    from . import build_time_grid, make_heat_problem

    rows = []
    for G in gpu_list or [1]:
        if G == 1:
            spec = make_heat_problem(space, cells, build_time_grid("uniform", N, T), data="sine")
            row = time_iterations(spec, omega, iters, repeats)
        else:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone",
                   "--nproc-per-node", str(G), "-m", "paper_1802_08126_b200.distributed",
                   "--space", space, "--h", str(cells), "--N", str(N), "--T", repr(T),
                   "--omega", repr(omega), "--iters", str(iters), "--repeats", str(repeats)]
            env = dict(os.environ, MASTER_ADDR="127.0.0.1")
            out = subprocess.run(cmd, capture_output=True, text=True, env=env, check=False)
            if out.returncode != 0:
                raise InputError(f"{G}-GPU run failed: {out.stderr.strip()[-300:]}")
            vals = [ln for ln in out.stdout.splitlines() if ln.startswith("scaling,")][-1]
            t, tot, fs, ss = (float(v) for v in vals.split(",")[1:5])
            row = {"time_per_iter": t, "total_time": tot, "fft_share": fs, "spatial_share": ss}
        rows.append({"gpus": G, **row})
    return rows


def _run(args) -> str:
    if args.command == "solve":
        return cmd_solve(args)
    if args.command == "table2":
        return rows_to_csv(HEADERS["table2"], run_table2(args.h, args.N, T=args.T, omega=args.omega,
                                                         tol=args.tol, vcycles=args.vcycles))
    if args.command == "history":
        return rows_to_csv(HEADERS["history"], run_history(
            N=args.N, cells=args.h, space=args.space, T=args.T, omega=args.omega, tol=args.tol,
            max_iter=args.max_iter))
    return rows_to_csv(HEADERS["scaling"], run_scaling(
        args.gpu_list, N=args.N, cells=args.h, space=args.space, T=args.T, omega=args.omega,
        iters=args.iters, repeats=args.repeats))


def main(argv=None) -> int:
    argv = list(sys.argv[1:] if argv is None else argv)
    parser = build_parser()
    try:
        probe, _ = parser.parse_known_args(argv)
        if probe.config:
            argv = merge_config(argv, read_config(probe.config))
        args = parser.parse_args(argv)
    except SystemExit as exc:
        return 0 if exc.code == 0 else 1
    except (InputError, OSError) as exc:
        sys.stderr.write(f"error: {exc}\n")
        return 1
    try:
        text = _run(args)
    except SolverDivergenceError as exc:
        sys.stderr.write(f"divergence: {exc}\n")
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
