import os, sys
import numpy as np
import torch, torch.distributed as dist
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1802_08126_b200 as pg
from paper_1802_08126_b200.distributed import GpuLocalOps, Partition
torch.cuda.set_device(0)
for cells, N in [(128, 16), (256, 16), (256, 64)]:
    n = (cells - 1) ** 2
    rng = np.random.default_rng(0)
    load = rng.standard_normal((N, n))
    grid = pg.build_time_grid("uniform", N, 1.0)
    spec = pg.problem_from_arrays("2d", cells, grid, load, np.zeros(n), alpha=1.0)
    system = pg.TimeGlobalSystem(spec)
    hier = pg.build_mg_hierarchy("2d", cells)
    ht = pg.build_schur_preconditioner(spec, "mg")
    ops = GpuLocalOps(spec, hier, Partition(N, 1), 0)
    z = rng.standard_normal((N, n))
    zt = torch.from_numpy(z).cuda()
    zh = ops.dst_cols(1, zt)
    w, d = ops.htilde_modes(zh, True)
    y = ops.dst_cols(0, w).cpu().numpy()
    yref = ht.apply_inverse(z)
    print(cells, N, "htilde diff", np.abs(y - yref).max() / np.abs(yref).max(), flush=True)
    w2, d2 = ops.htilde_modes(zh, False)
    print("   dot", d, d2, np.sum(z * yref))
