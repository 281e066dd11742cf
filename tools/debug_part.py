"""Debug: time-partitioned driver (1 rank, NCCL) vs the fused single-GPU path."""
import os, sys, ctypes
import numpy as np
import torch, torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_08126_b200 as pg
from paper_1802_08126_b200.distributed import Comm, DistUzawa, GpuLocalOps, Partition

os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0"); os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
for cells, N in [(32, 64), (128, 64), (256, 128), (256, 1024)]:
    n = (cells - 1) ** 2
    load = np.random.default_rng(0).standard_normal((N, n))
    grid = pg.build_time_grid("uniform", N, 1.0)
    spec = pg.problem_from_arrays("2d", cells, grid, load, np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    hier = pg.build_mg_hierarchy("2d", cells)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=hier)
    ht = pg.build_schur_preconditioner(spec, "mg")
    (p, u), h = pg.uzawa_solve(system, at, ht, pg.UzawaConfig(tol=1e-300, max_iter=4))
    ops = GpuLocalOps(spec, hier, Partition(N, 1), 0)
    f = torch.from_numpy(np.ascontiguousarray(system.rhs)).cuda()
    it = DistUzawa(ops, Comm(), N, n, f)
    ref = it.begin()
    res = [it.step(0.9) / ref for _ in range(4)]
    print(cells, N, "single", h.residual, "\n      part  ", res, flush=True)
    # operator-level comparisons
    x = torch.from_numpy(np.random.default_rng(1).standard_normal((N, n))).cuda()
    xc = x.clone()
    d1 = ops.dst_cols(1, xc).cpu().numpy(); d1s = pg.DstPlan(N).inverse_transpose(x.cpu().numpy())
    print("   dst1 maxdiff", np.abs(d1 - d1s).max())
    w, dot = ops.htilde_modes(x, True)
    print("   htilde_modes finite", bool(torch.isfinite(w).all()), dot)
dist.destroy_process_group()
