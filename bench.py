"""Benchmark: space-time DoF/s per Uzawa iteration on BASELINE config 2.

Workload (BASELINE.json configs[1]): 2D heat equation on the
unit square, cells=256 (255x255 = 65,025 interior nodes, the MG-compatible
mesh for "256x256"), implicit Euler N=1024, T=1, fp64, u(0)=0, load
f = g - (4/5) D_A^-1 (A g) with g ~ N(0,1) seeded 0 (one damped-Jacobi
smoothing sweep), MG V-cycles (1 pre + 1 post sweep), omega=0.9, tol=1e-8.

One bench "step" = one Uzawa iteration over the whole space-time slab
(r1, A~^-1, z, H~^-1, updates, residual), state resident in HBM (each slab
is 533 MB > 126 MB L2, so no L2 flush is needed between steps).
``value``  = N*n / device time per iteration (CUDA events on the library stream).
``e2e``    = the same metric through the public API (uzawa_solve) from host
             numpy arrays to host numpy arrays, to convergence, wall clock
             including H2D of f and D2H of p, u (time-to-1e-8 also reported).
``roofline`` = dominant kernel's algorithmic bytes / its event-timed duration.
``cpu_baseline`` = the CPU oracle port (oracle/, the reference algorithm in
             numpy/scipy) on an N=64 slice of the same grid, per iteration.

--impl reference runs that CPU oracle arm alone (the reference is pure
Python and is not installable on the GPU box; oracle/ restates it and is
pinned bit-for-bit to it, tests/test_oracle.py).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CELLS, NSTEPS, T_END = 256, 1024, 1.0
WORKLOAD = ("c2: 2D heat u_t - Lap u = f, unit square, cells=256 (255^2=65025 interior), "
            "implicit Euler N=1024, T=1, f=Jacobi-smoothed N(0,1) seed 0, u0=0, "
            "MG V(1,1), omega=0.9, tol=1e-8")


def c2_load(cells=CELLS, N=NSTEPS, seed=0):
    """g ~ N(0,1) (seed) smoothed by one damped Jacobi sweep: g - (4/5) D^-1 A g."""
    import scipy.sparse as sp  # noqa: F401

    from paper_1802_08126_b200 import assemble_mass_stiffness_2d

    _, a = assemble_mass_stiffness_2d(cells)
    g = np.random.default_rng(seed).standard_normal((N, a.dim))
    dinv = (4.0 / 5.0) / a.diagonal()
    return g - dinv[None, :] * a.dot(g.T).T


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the newest committed ncu launch
    summary (profiles/*_c2_traffic.json, tools/traffic_summary.py), or None."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_c2_traffic.json")))
    if not files:
        return None, None
    try:
        with open(files[-1]) as fh:
            d = json.load(fh)
        return float(d["kernels"][kernel]["dram_bytes_per_launch"]), os.path.relpath(files[-1], ROOT)
    except Exception:
        return None, None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """SM clock and throttle reasons during the timed region: NVML in process
    (a few ms per sample, so even the 35 ms headline region gets several),
    nvidia-smi every 0.2 s when pynvml is not importable."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index=0):
        self.index = index
        self.sm, self.mx, self.reasons = [], [], set()
        self.source = None
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run_nvml(self):
        import pynvml as nv

        nv.nvmlInit()
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        idx = self.index
        if vis and all(v.strip().isdigit() for v in vis.split(",")):
            ids = [int(v) for v in vis.split(",")]
            idx = ids[self.index] if self.index < len(ids) else self.index
        h = nv.nvmlDeviceGetHandleByIndex(idx)
        bits = [(nv.nvmlClocksEventReasonHwSlowdown, "hw_slowdown"),
                (nv.nvmlClocksEventReasonHwThermalSlowdown, "hw_thermal_slowdown"),
                (nv.nvmlClocksEventReasonSwThermalSlowdown, "sw_thermal_slowdown"),
                (nv.nvmlClocksEventReasonSwPowerCap, "sw_power_cap")]
        try:
            get_reasons = nv.nvmlDeviceGetCurrentClocksEventReasons
        except AttributeError:
            get_reasons = nv.nvmlDeviceGetCurrentClocksThrottleReasons
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        self.source = "nvml"
        while not self._stop.is_set():
            self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
            self.mx.append(mx)
            r = get_reasons(h)
            for bit, name in bits:
                if r & bit:
                    self.reasons.add(name)
            self._stop.wait(0.004)

    def _run_smi(self):
        self.source = "nvidia-smi"
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    r = [x.strip() for x in out.stdout.strip().split(",")]
                    if r[0].replace(".", "").isdigit():
                        self.sm.append(float(r[0]))
                    if r[1].replace(".", "").isdigit():
                        self.mx.append(float(r[1]))
                    for i, name in enumerate(self.NAMES):
                        if len(r) > 3 + i and r[3 + i].lower().startswith("active"):
                            self.reasons.add(name)
            except Exception:
                return
            self._stop.wait(0.2)

    def _run(self):
        try:
            self._run_nvml()
        except Exception:
            if not self.sm:
                self._run_smi()

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.sm:
            return None
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


# ----------------------------------------------------------------------------
# CPU oracle arm (reference algorithm restated in numpy/scipy)
# ----------------------------------------------------------------------------

def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


_ORACLE_CASE = {}


def cpu_oracle_rate(cells=CELLS, n_slice=64, iters=4, repeats=1, threads=1):
    """Marginal per-iteration time of the oracle Uzawa on an N-slice of the
    c2 grid ((t(k=iters) - t(k=iters/2)) / (iters/2)), with
    `threads` workers on the per-step / per-mode loops (parallel.py:19-43)."""
    import oracle as orc

    orc.set_num_threads(threads)
    n = (cells - 1) ** 2
    key = (cells, n_slice)
    if key not in _ORACLE_CASE:  # problem and preconditioners are built once per process
        load = c2_load(cells, n_slice)
        nodes = orc.time_nodes("uniform", n_slice, T_END * n_slice / NSTEPS)
        pb = orc.heat_problem("2d", cells, nodes, load=load, u_init=np.zeros(n))
        lev = orc.mg_levels("2d", cells)
        _ORACLE_CASE[key] = (pb, orc.BlockInv(pb, lev), orc.SchurInv(pb, lev))
    pb, at, ht = _ORACLE_CASE[key]
    best = None
    for _ in range(repeats):
        times = []
        res = orc.uzawa(pb, at, ht, 0.9, 1e-300, iters,
                        on_iter=lambda j, r: times.append(time.perf_counter()))
        half = iters // 2
        dt = (times[-1] - times[half - 1]) / (iters - half)
        best = dt if best is None else min(best, dt)
        del res
    orc.set_num_threads(1)
    return n_slice * n / best, best


def run_reference(args):
    """The reference algorithm on the host cores (the CPU oracle, pinned
    bit-for-bit to the pure-Python reference, which cannot travel to the GPU
    box): each step times the marginal Uzawa iteration on an N = 64 slice of
    the c2 grid with every host thread the reference's pool can use; the
    first three timed steps also run it with one thread; `value` is the better
    of the two medians."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    steps, warm = max(1, args.steps), max(0, args.warmup)
    iters = 2 * max(1, min(steps, 3))
    cores = host_cores()
    rates = {1: [], cores: []}
    t0 = time.perf_counter()
    for k in range(warm + steps):
        for th in sorted(rates, reverse=True):
            if th == 1 and cores > 1 and not warm <= k < warm + 3:
                continue  # the one-thread leg on three timed steps only (wall budget)
            rate, dt = cpu_oracle_rate(iters=iters, threads=th)
            if k >= warm:
                rates[th].append((rate, dt))
    wall = time.perf_counter() - t0
    med = {th: (float(np.median([r for r, _ in v])), float(np.median([d for _, d in v])))
           for th, v in rates.items()}
    best = max(med, key=lambda th: med[th][0])
    val, dt = med[best]
    line = {
        "metric": "space-time DoF/s per Uzawa iteration", "value": val,
        "unit": "DoF/s", "n_gpus": args.gpus, "steps": steps, "warmup": warm,
        "ms_per_step": dt * 1e3 * (NSTEPS / 64),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "same_config": False,
                   "sample": "N=64 slice (1/16 of the time steps) of the c2 grid, marginal "
                             "per-iteration time of the CPU oracle; ms_per_step is that time "
                             "EXTRAPOLATED linearly to N=1024 (the full-size reference run "
                             "took 31 s per iteration, SURVEY 8(d), so the extrapolation "
                             "favours the CPU)"},
        "cpu_baseline": {"value": val, "unit": "DoF/s", "cores": best, "kind": "port",
                         "host_cores": cores,
                         "by_threads": {str(th): {"DoF_per_s": med[th][0], "s_per_iter": med[th][1]}
                                        for th in med},
                         "sample": f"oracle uzawa, cells=256, N=64 slice, {iters} iterations "
                                   f"per step, marginal; wall {wall:.1f}s"},
        "e2e": {"value": val, "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def build_solver(load, device):
    import paper_1802_08126_b200 as pg

    grid = pg.build_time_grid("uniform", NSTEPS, T_END)
    n = (CELLS - 1) ** 2
    spec = pg.problem_from_arrays("2d", CELLS, grid, load, np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec, device=device)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("2d", CELLS))
    ht = pg.build_schur_preconditioner(spec, "mg", vcycles=1)
    return pg, spec, system, at, ht


OTHER_CONFIGS = {
    # BASELINE configs[2]/[4] (G=1)/[3]: MG-compatible meshes
    "c3": dict(space="3d", cells=64, N=512, T=1.0,
               workload="c3: 3D heat, unit cube, cells=64 (63^3=250047 interior), N=512, T=1, "
                        "f~N(0,1) seed 0, u0~U[0,1] seed 0 (drawn after f)"),
    "c5": dict(space="3d", cells=64, N=1024, T=1.0,
               workload="c5 (G=1 slice of the weak-scaling series): 3D heat, cells=64, N=1024, "
                        "T=1, f~N(0,1) seed 0, u0=0"),
    "c4": dict(space="2d", cells=512, N=4096, T=2.0,
               workload="c4: 2D -div(a(x,t) grad u), a=1+0.5 sin(2 pi t)(x1^2+x2^2)+0.1 U_cell "
                        "(seed 0), cells=512 (511^2=261121 interior), N=4096, T=2, "
                        "f~N(0,1) seed 1, u0=0"),
}


def build_config(name):
    """(pg, spec, system, at, ht, setup seconds) of OTHER_CONFIGS[name]."""
    import paper_1802_08126_b200 as pg

    c = OTHER_CONFIGS[name]
    cells, N, space = c["cells"], c["N"], c["space"]
    n = (cells - 1) ** (3 if space == "3d" else 2)
    t0 = time.perf_counter()
    grid = pg.build_time_grid("uniform", N, c["T"])
    if name == "c4":
        load = np.random.default_rng(1).standard_normal((N, n))
        spec = pg.make_weighted_problem(cells, grid, pg.c4_cell_weights(cells, grid, seed=0),
                                        load, np.zeros(n), alpha=1.0)
    else:
        rng = np.random.default_rng(0)
        load = rng.standard_normal((N, n))
        u0 = rng.uniform(0.0, 1.0, n) if name == "c3" else np.zeros(n)
        spec = pg.problem_from_arrays(space, cells, grid, load, u0, alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy(space, cells))
    ht = pg.build_schur_preconditioner(spec, "mg")
    return pg, spec, system, at, ht, time.perf_counter() - t0


# iteration caps of the convergence runs: the reference default 200 (solvers.py:24)
# except c4, whose count grows with the mesh (~10^3 at cells=512)
MAX_ITER = {"c3": 200, "c5": 200, "c4": 4000}


def converge_config(name, max_iter=None):
    """One uzawa_solve of a BASELINE config to tol 1e-8 through the public API
    (host numpy in / out): iterations, time-to-tol (BASELINE's second metric),
    clocks during the solve."""
    import gc

    max_iter = max_iter or MAX_ITER[name]
    pg, spec, system, at, ht, setup = build_config(name)
    N, n = spec.N, spec.dim
    with ClockSampler(0) as clk:
        t0 = time.perf_counter()
        (p, u), hist = pg.uzawa_solve(system, at, ht,
                                      pg.UzawaConfig(omega=0.9, tol=1e-8, max_iter=max_iter))
        wall = time.perf_counter() - t0
    out = {"iterations": hist.iterations, "converged": bool(hist.converged),
           "max_iter": max_iter, "time_to_tol_s": wall, "setup_s": setup,
           "first_residual": hist.residual[0] if hist.residual else None,
           "final_residual": hist.residual[-1] if hist.residual else None,
           "e2e_DoF_per_s": N * n * hist.iterations / wall if wall > 0 else None,
           "h2d_bytes": int(8 * N * n), "d2h_bytes": int(16 * N * n),
           "clocks": clk.summary()}
    del p, u, system, at, ht, spec
    gc.collect()
    return out


def measure_config(name, steps=3, warm=2, converge=True, budget_s=None):
    """Per-iteration device time of one more BASELINE config on this GPU
    (CUDA events on the library stream, state resident in HBM), with the
    iteration roofline fraction and the per-kernel shares; then the solve to
    tol 1e-8 through the public API (iterations, time-to-tol, clocks).  A
    config whose projected solve exceeds `budget_s` is run with the iteration
    cap that fits the budget and reported as not converged."""
    import ctypes
    import gc

    c = OTHER_CONFIGS[name]
    pg, spec, system, at, ht, setup = build_config(name)
    N, n = spec.N, spec.dim
    ctx = system._gp.ctx
    f = np.ascontiguousarray(system.rhs)
    ref = ctypes.c_double()
    ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
    nums = np.zeros(max(steps, warm, 2))
    ms = ctypes.c_double()
    ctx.call("pint_uzawa_run", 0.9, warm, nums.ctypes.data, ctypes.byref(ms))
    with ClockSampler(0) as clk:
        ctx.call("pint_uzawa_run", 0.9, steps, nums.ctypes.data, ctypes.byref(ms))
    ms_it = ms.value / steps
    ctx.call("pint_profile", 1)
    ctx.call("pint_uzawa_run", 0.9, 1, nums.ctypes.data, ctypes.byref(ms))
    stats = ctx.kernel_stats()
    ctx.call("pint_profile", 0)
    hbm, _ = peaks()
    tot = sum(v[0] for v in stats.values()) or 1.0
    dom = max(stats.items(), key=lambda kv: kv[1][0])
    iter_bytes = 224.0 * N * n
    out = {"workload": c["workload"], "n": n, "N": N, "ms_per_iter": ms_it,
           "value": N * n / (ms_it / 1e3), "unit": "DoF/s", "setup_s": setup,
           "iteration_frac": iter_bytes / (ms_it / 1e3) / 1e9 / hbm,
           "clocks": clk.summary(),
           "dominant_kernel": {"name": dom[0], "share": dom[1][0] / tot,
                               "GBps": dom[1][2] / dom[1][0] / 1e6 if dom[1][0] else None},
           "kernel_shares": {k: round(v[0] / tot, 4) for k, v in
                             sorted(stats.items(), key=lambda kv: -kv[1][0]) if v[1]}}
    del f
    if converge:
        max_iter = MAX_ITER[name]
        if budget_s is not None:
            max_iter = max(10, min(max_iter, int(budget_s / (ms_it / 1e3))))
        with ClockSampler(0) as clk2:
            t0 = time.perf_counter()
            try:
                (p, u), hist = pg.uzawa_solve(
                    system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-8, max_iter=max_iter))
                wall = time.perf_counter() - t0
                out["solve"] = {
                    "iterations": hist.iterations, "converged": bool(hist.converged),
                    "max_iter": max_iter, "reference_default_max_iter": 200,
                    "time_to_tol_s": wall if hist.converged else None, "wall_s": wall,
                    "first_residual": hist.residual[0] if hist.residual else None,
                    "final_residual": hist.residual[-1] if hist.residual else None,
                    "e2e_DoF_per_s": N * n * hist.iterations / wall,
                    "h2d_bytes": int(8 * N * n), "d2h_bytes": int(16 * N * n)}
                del p, u
            except pg.SolverDivergenceError as e:
                # the reference's own divergence rule (solvers.py:236-237)
                out["solve"] = {"converged": False, "diverged": True, "omega": 0.9,
                                "max_iter": max_iter, "error": str(e),
                                "wall_s": time.perf_counter() - t0}
        out["solve"]["clocks"] = clk2.summary()
    del system, spec, ctx, at, ht
    gc.collect()
    return out


PART_CONFIGS = {
    # the headline grid, time axis split over the ranks (strong scaling)
    "c2": dict(space="2d", cells=CELLS, N=NSTEPS, T=T_END, weak=False),
    # BASELINE configs[2] (strong scaling 1/2/4/8) and configs[4] (weak: N = 1024 G)
    "c3": dict(space="3d", cells=64, N=512, T=1.0, weak=False),
    "c5": dict(space="3d", cells=64, N=1024, T=1.0, weak=True),
    # BASELINE config 4 ("time-sharded across 8 B200"): per-step coefficient
    # fields, every rank assembles those of its own steps
    "c4": dict(space="2d", cells=512, N=4096, T=2.0, weak=False),
}


def _part_problem(name, world, rank):
    """(spec, f_local, part) of a partitioned config; the load of c3/c5 is
    generated per plane with default_rng((seed, step)) so every rank builds
    only its own slab."""
    import paper_1802_08126_b200 as pg
    from paper_1802_08126_b200.distributed import Partition

    c = PART_CONFIGS[name]
    N = c["N"] * (world if c["weak"] else 1)
    if name == "c4" and os.environ.get("PINT_BENCH_C4_N"):
        N = int(os.environ["PINT_BENCH_C4_N"])  # one-GPU validation of this path (163 GB at N = 4096)
    T = c["T"] * N / c["N"] if c["weak"] else c["T"]
    grid = pg.build_time_grid("uniform", N, T)
    n = (c["cells"] - 1) ** (3 if c["space"] == "3d" else 2)
    part = Partition(N, world)
    sl = part.slice(rank)
    if name == "c2":
        load = c2_load()
        mine = load[sl]
    else:
        # only this rank's slab exists on the host (c5 at G = 8 is 16 GB in all)
        mine = np.stack([np.random.default_rng((1 if name == "c4" else 0, t)).standard_normal(n)
                         for t in range(sl.start, sl.stop)])
        load = np.broadcast_to(np.zeros(1), (N, n))
    if name == "c4":
        spec = pg.make_weighted_problem(c["cells"], grid,
                                        pg.c4_cell_weights(c["cells"], grid, seed=0), load,
                                        np.zeros(n), alpha=1.0)
    else:
        spec = pg.problem_from_arrays(c["space"], c["cells"], grid, load, np.zeros(n), alpha=1.0)
    f_loc = np.ascontiguousarray(spec.grid.steps[sl, None] * mine)  # fold_rhs, u0 = 0
    return spec, f_loc, part


def measure_partitioned(name, world, rank, local, steps, warm, e2e=False):
    """Per-iteration device time (max over ranks) of the time-partitioned
    Uzawa step on config `name`; optionally the end-to-end solve."""
    import torch
    import torch.distributed as dist

    import paper_1802_08126_b200 as pg
    from paper_1802_08126_b200.distributed import Comm, DistUzawa, GpuLocalOps, dist_uzawa_solve

    spec, f_loc_h, part = _part_problem(name, world, rank)
    c = PART_CONFIGS[name]
    hier = pg.build_mg_hierarchy(c["space"], c["cells"])
    ops = GpuLocalOps(spec, hier, part, rank, device=local)
    comm = Comm()
    f_host = torch.from_numpy(f_loc_h).pin_memory()
    f_loc = f_host.to(ops.dev)
    N, n = spec.N, spec.dim
    it = DistUzawa(ops, comm, N, n, f_loc)
    it.begin()
    for _ in range(warm):
        it.step(0.9)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = ops.ctx.launches()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record()
        for _ in range(steps):
            it.step(0.9)
        ev1.record()
        torch.cuda.synchronize()
    launches = ops.ctx.launches() - l0
    t = torch.tensor([ev0.elapsed_time(ev1) / steps], device=ops.dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    hbm, _ = peaks()
    out = {"config": name, "N": N, "n": n, "ms_per_iter": ms, "value": N * n / (ms / 1e3),
           "unit": "DoF/s", "scaling": "weak" if c["weak"] else "strong",
           "iteration_frac_per_gpu": 224.0 * N * n / world / (ms / 1e3) / 1e9 / hbm,
           "launches": launches, "clocks": clk.summary()}
    if e2e:
        dist.barrier()
        t0 = time.perf_counter()
        f2 = f_host.to(ops.dev)
        _, u_l, hist = dist_uzawa_solve(ops, comm, N, n, f2,
                                        pg.UzawaConfig(omega=0.9, tol=1e-8, max_iter=200))
        u_host = u_l.cpu()
        wall = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=ops.dev)
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
        del u_host
        out["e2e"] = {"iterations": hist.iterations, "time_to_tol_s": float(wall.item()),
                      "converged": hist.converged,
                      "final_residual": hist.residual[-1] if hist.residual else None,
                      "h2d_bytes_per_step": int(f_loc_h.nbytes),
                      "d2h_bytes_per_step": int(f_loc_h.nbytes)}
    del it, ops, f_loc
    torch.cuda.empty_cache()
    return out


def run_gpu_partitioned(args, world, rank, local):
    """N > 1 GPUs (or --partitioned): the headline c2 time axis split across
    ranks (strong scaling, the same workload as the N = 1 line so the driver's
    scaling efficiency compares like with like), plus BASELINE's own
    multi-GPU configs c3 (strong), c5 (weak, N = 1024 G) and c4 (strong, field
    mode; per-iteration time only: it diverges at omega = 0.9 in the reference
    algorithm too) as other_configs."""
    import torch
    import torch.distributed as dist

    # NCCL_DEBUG=VERSION makes NCCL print its version on stdout, in front of the
    # one JSON line this script owes the driver
    if os.environ.get("NCCL_DEBUG", "").upper() == "VERSION":
        os.environ["NCCL_DEBUG"] = "WARN"
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    steps, warm = args.steps, max(3, args.warmup)
    head = measure_partitioned("c2", world, rank, local, steps, warm, e2e=True)
    others = {}
    if not args.no_other:
        for name in ("c3", "c5", "c4"):
            if name == "c4" and world == 1 and not os.environ.get("PINT_BENCH_C4_N"):
                continue  # does not fit one GPU next to the driver's own slabs
            try:
                others[name] = measure_partitioned(name, world, rank, local, max(2, steps // 3),
                                                   3)
            except Exception as e:  # report, do not lose the headline line
                others[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
    hbm, peak_kind = peaks()
    N, n, ms_step = head["N"], head["n"], head["ms_per_iter"]
    iter_bytes = 224.0 * N * n
    if rank == 0:
        e = head["e2e"]
        line = {
            "metric": "space-time DoF/s per Uzawa iteration", "value": head["value"],
            "unit": "DoF/s", "n_gpus": world, "steps": steps, "warmup": warm,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": n, "N": N,
                       "parallelism": f"time-sharded x{world} (ghost planes, chunked async "
                                      "all-to-all transposes around the DSTs, device "
                                      "all-reduce of the 2 partial sums)",
                       "l2": "inputs larger than L2, no flush"},
            "e2e": {"value": N * n * e["iterations"] / e["time_to_tol_s"], "unit": "DoF/s",
                    **e, "step": "one partitioned solve from host arrays to convergence"},
            "roofline": {"bound": "hbm", "kernel": "iteration", "achieved":
                         iter_bytes / world / (ms_step / 1e3) / 1e9, "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": iter_bytes / world / (ms_step / 1e3) / 1e9 / hbm,
                         "traffic": None},
            "cpu_baseline": None,
            "clocks": head["clocks"],
            "gpu_launches": head["launches"],
            "other_configs": others or None,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_gpu(args):
    import ctypes

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1 or args.partitioned:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        return run_gpu_partitioned(args, world, rank, local)
    dist = None
    load = c2_load()
    pg, spec, system, at, ht = build_solver(load, local)
    gp = system._gp
    ctx = gp.ctx
    f = np.ascontiguousarray(system.rhs)
    N, n = spec.N, spec.dim
    steps, warm = args.steps, max(3, args.warmup)

    # ---- device-resident timed region -------------------------------------
    ref = ctypes.c_double()
    ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
    nums = np.zeros(max(warm, steps))
    ms = ctypes.c_double()
    ctx.call("pint_uzawa_run", 0.9, warm, nums.ctypes.data, ctypes.byref(ms))
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches()
    with ClockSampler(local) as clk:
        ctx.call("pint_uzawa_run", 0.9, steps, nums.ctypes.data, ctypes.byref(ms))
    launches = (ctx.launches() - l0)
    torch.cuda.synchronize()
    ms_step = ms.value / steps
    if dist:
        t = torch.tensor([ms_step], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = world * N * n / (ms_step / 1e3)

    # ---- per-kernel roofline (profiling pass, outside the timed region) ----
    ctx.call("pint_profile", 1)
    ctx.call("pint_uzawa_run", 0.9, 2, nums.ctypes.data, ctypes.byref(ms))
    stats = ctx.kernel_stats()
    ctx.call("pint_profile", 0)
    hbm, peak_kind = peaks()
    tot = sum(v[0] for v in stats.values())
    dom = max(stats.items(), key=lambda kv: kv[1][0])
    dname, (dms, dcnt, dbytes) = dom
    achieved = (dbytes / dcnt) / (dms / dcnt / 1e3) / 1e9
    kernels = {k: {"ms_per_launch": v[0] / v[1], "share": v[0] / tot,
                   "GBps": (v[2] / v[0] / 1e6) if v[0] > 0 else None, "launches": v[1]}
               for k, v in stats.items() if v[1] > 0}
    iter_bytes = 224.0 * N * n  # 28 fp64 block-vector passes per iteration
    traffic, traffic_src = ncu_traffic(dname)
    # ---- end to end through the public API (host numpy in / out) ----------
    t0 = time.perf_counter()
    (p_h, u_h), hist = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(omega=0.9, tol=1e-8,
                                                                        max_iter=200))
    wall = time.perf_counter() - t0
    e2e_val = world * N * n * hist.iterations / wall

    others = {}
    if rank == 0 and world == 1 and not args.no_other:
        # second solver entry point on the headline config (solvers.py:267-327)
        try:
            t0 = time.perf_counter()
            _, mh = pg.minres_solve(system, at, ht, tol=1e-8, max_iter=500)
            mw = time.perf_counter() - t0
            others["c2_minres"] = {
                "workload": WORKLOAD + "; minres_solve (block-diagonally preconditioned MINRES)",
                "iterations": mh.iterations, "converged": bool(mh.converged),
                "time_to_tol_s": mw,
                "ms_per_iter": (mh.wall_seconds[-1] / max(1, mh.iterations) * 1e3
                                if mh.wall_seconds else None),
                "final_residual": mh.residual[-1] if mh.residual else None,
                "note": "wall clock from host numpy f to host numpy (p, u); each iteration "
                        "applies the saddle operator, A~^-1 and H~^-1 once"}
        except Exception as e:
            others["c2_minres"] = {"error": f"{type(e).__name__}: {e}"[:300]}
        del system, at, ht, spec, gp, ctx
        import gc

        gc.collect()
        torch.cuda.empty_cache()
        for name in ("c3", "c5", "c4"):
            try:
                # c4 needs ~10^3 iterations: its solve gets a wall budget
                others[name] = measure_config(name, converge=not args.no_converge,
                                              budget_s=args.c4_budget if name == "c4" else None)
            except Exception as e:  # report, do not lose the headline line
                others[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
            gc.collect()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = host_cores()
        rate1, dt1 = cpu_oracle_rate(iters=4, threads=1)
        ratec, dtc = cpu_oracle_rate(iters=4, threads=cores) if cores > 1 else (rate1, dt1)
        best = cores if ratec > rate1 else 1
        cpu = {"value": max(rate1, ratec), "unit": "DoF/s", "cores": best, "kind": "port",
               "host_cores": cores,
               "by_threads": {"1": {"DoF_per_s": rate1, "s_per_iter": dt1},
                              str(cores): {"DoF_per_s": ratec, "s_per_iter": dtc}},
               "sample": "CPU oracle uzawa (numpy/scipy restatement of the reference, its "
                         "thread pool on the per-step / per-mode loops), cells=256, N=64 "
                         f"slice, marginal s/iter: {dt1:.3f} (1 thread), {dtc:.3f} "
                         f"({cores} threads)"}
    if rank == 0:
        line = {
            "metric": "space-time DoF/s per Uzawa iteration", "value": value, "unit": "DoF/s",
            "n_gpus": world, "steps": steps, "warmup": warm, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": WORKLOAD, "n": n, "N": N,
                       "parallelism": "single",
                       "l2": "inputs larger than L2 (533 MB per slab), no flush"},
            "e2e": {"value": e2e_val, "unit": "DoF/s", "iterations": hist.iterations,
                    "time_to_tol_s": wall, "converged": hist.converged,
                    "final_residual": hist.residual[-1] if hist.residual else None,
                    "h2d_bytes_per_step": int(f.nbytes), "d2h_bytes_per_step": int(2 * f.nbytes),
                    "step": "one uzawa_solve call from host arrays to convergence"},
            "roofline": {"bound": "hbm", "kernel": dname, "achieved": achieved, "peak": hbm,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "traffic_source": traffic_src,
                         "algorithmic_bytes_per_launch": dbytes / dcnt,
                         "iteration_alg_GBps": iter_bytes / (ms_step / 1e3) / 1e9,
                         "iteration_frac": iter_bytes / (ms_step / 1e3) / 1e9 / hbm},
            "kernels": kernels,
            "cpu_baseline": cpu,
            "clocks": clk.summary(),
            "gpu_launches": launches,
            "other_configs": others or None,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-other", action="store_true",
                    help="skip the per-iteration measurements of configs c3, c5 (G=1), c4")
    ap.add_argument("--no-converge", action="store_true",
                    help="other configs: per-iteration timing only, no solve to tol")
    ap.add_argument("--c4-budget", type=float, default=240.0,
                    help="wall budget (s) of the c4 solve; its iteration cap is "
                         "min(4000, budget / measured iteration time)")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the time-partitioned driver even on one GPU (validation)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
