import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2208_09899_b200 as L
import bench
wl = bench.build_workload(2, 0, 1)
ctx = L.Context(wl["n_global"], wl["s"], wl["m"], *wl["A"])
B = torch.from_numpy(wl["B"]).cuda(); X = torch.zeros_like(B)
m, tol = wl["m"], wl["tol"]
L.lsba_bgmres_solve(ctx.ctx, B, X, m, tol, 2)
torch.cuda.synchronize()
for r in range(3):
    t0 = time.perf_counter(); i = L.lsba_bgmres_solve(ctx.ctx, B, X, m, tol, 0); torch.cuda.synchronize(); print('device solve 1 cycle', (time.perf_counter()-t0)*1e3, 'ms', i.iterations, i.cycles)
Bh = torch.from_numpy(wl["B"]).pin_memory().numpy()
Xh = torch.zeros(B.shape, dtype=torch.float64).pin_memory().numpy()
for r in range(4):
    t0 = time.perf_counter(); i = L.lsba_solve_host(ctx.ctx, Bh, Xh, m, tol, 0); print('host solve 1 cycle', (time.perf_counter()-t0)*1e3, 'ms', i.seconds*1e3, i.iterations, i.cycles)
Xd = torch.empty_like(B)
for r in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter(); Xd.copy_(torch.from_numpy(Bh), non_blocking=True); torch.cuda.synchronize(); print('h2d 32MB', (time.perf_counter()-t0)*1e3)
