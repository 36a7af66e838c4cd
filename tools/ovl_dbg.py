import sys, time, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2208_09899_b200 as L
from lsba_inputs import make_twin
p = make_twin(2)
print('n', p.n, 's', p.s, flush=True)
ctx = L.Context(p.n, p.s, 6, p.row_ptr, p.col_idx, p.vals)
B = torch.from_numpy(p.B).cuda()
print('begin', ctx.begin(B), flush=True)
for k in range(4):
    t = time.time(); i = ctx.step(); torch.cuda.synchronize(); print('step', k + 1, i.chol_flag, time.time() - t, flush=True)
X = torch.zeros_like(B)
t = time.time(); info = ctx.solve(B, X, 6, p.tol, 3); torch.cuda.synchronize(); print('solve', info.cycles, info.iterations, time.time() - t, flush=True)
