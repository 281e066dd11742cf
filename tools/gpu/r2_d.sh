# ncu of the fused 3D band kernels (c3 shapes, short N)
python - <<'PY' > /dev/null 2>&1
PY
cat > /tmp/c3small.py <<'PY'
import sys, ctypes, numpy as np
sys.path.insert(0, '.')
import paper_1802_08126_b200 as pg
cells, N = 64, 64
n = 63**3
grid = pg.build_time_grid("uniform", N, 1.0)
rng = np.random.default_rng(0)
spec = pg.problem_from_arrays("3d", cells, grid, rng.standard_normal((N, n)), np.zeros(n), alpha=1.0)
system = pg.TimeGlobalSystem(spec)
pg.BlockDiagSolver(spec, "mg", hierarchy=pg.build_mg_hierarchy("3d", cells))
pg.build_schur_preconditioner(spec, "mg")
ctx = system._gp.ctx
f = np.ascontiguousarray(system.rhs)
ref = ctypes.c_double()
ctx.call("pint_uzawa_begin", f.ctypes.data, None, None, ctypes.byref(ref))
nums = np.zeros(8); ms = ctypes.c_double()
ctx.call("pint_uzawa_run", 0.9, 2, nums.ctypes.data, ctypes.byref(ms))
print("ok", ms.value)
PY
timeout 600 ncu -f --set full --import-source on --clock-control none -k regex:"kb3_p" -c 4 -o /tmp/kb3 python /tmp/c3small.py > gpurun_out/ncu_kb3.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/kb3.ncu-rep --page details --csv > gpurun_out/kb3_details.csv 2>&1
ncu -i /tmp/kb3.ncu-rep --page raw --csv > gpurun_out/kb3_raw.csv 2>&1
