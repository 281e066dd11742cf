import os, sys
import numpy as np
import torch, torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_08126_b200 as pg
from paper_1802_08126_b200.distributed import GpuLocalOps, Partition
torch.cuda.set_device(0)
for cells, N in [(128, 16), (256, 16)]:
    n = (cells - 1) ** 2
    rng = np.random.default_rng(0)
    load = rng.standard_normal((N, n))
    grid = pg.build_time_grid("uniform", N, 1.0)
    spec = pg.problem_from_arrays("2d", cells, grid, load, np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    hier = pg.build_mg_hierarchy("2d", cells)
    at = pg.BlockDiagSolver(spec, "mg", hierarchy=hier)
    ops = GpuLocalOps(spec, hier, Partition(N, 1), 0)
    f = system.rhs
    u = rng.standard_normal((N, n)); p = rng.standard_normal((N, n))
    u_ext = torch.zeros((N + 2, n), dtype=torch.float64, device="cuda"); u_ext[1:N+1] = torch.from_numpy(u)
    p_ext = torch.zeros((N + 2, n), dtype=torch.float64, device="cuda"); p_ext[1:N+1] = torch.from_numpy(p)
    ft = torch.from_numpy(np.ascontiguousarray(f)).cuda()
    r1 = ops.r1(u_ext, p_ext, ft).cpu().numpy()
    r1_ref = (system.apply_K(u) - system.apply_Abd(p)) - f
    z = ops.z(u_ext, p_ext, ft).cpu().numpy()
    z_ref = (f - system.apply_Kt(p)) - ((system.apply_K(u) + system.apply_Kt(u)) + system.apply_Abd(u))
    print(cells, "r1 diff", np.abs(r1 - r1_ref).max(), "z diff", np.abs(z - z_ref).max())
    r1t = torch.from_numpy(r1_ref).cuda()
    d = ops.atilde_update(r1t, p_ext)
    dp = at.apply_inverse(r1_ref)
    print(cells, "p update diff", np.abs(p_ext[1:N+1].cpu().numpy() - (p + dp)).max(), "dot", d, np.sum(r1_ref * dp))
    # same with aligned (fresh) p
    p2 = torch.from_numpy(p).cuda().contiguous()
    pe2 = torch.zeros((N + 2, n), dtype=torch.float64, device="cuda")
