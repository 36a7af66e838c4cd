"""P = 2 real NCCL ranks (one process per GPU, torchrun) against P = 1 — runs only where at
least two GPUs are visible (skipped on the one-GPU boxes of this build; the loopback tests of
tests/test_gpu_multirank.py cover the same library path on one GPU)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import os, sys, json
sys.path.insert(0, os.environ["LSBA_ROOT"])
import numpy as np, torch, torch.distributed as dist
import paper_2208_09899_b200 as L
from lsba_inputs import make_twin
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
p = make_twin(5)                                   # 3D Laplacian 24^3, s = 8, m = 40
plane = 24 * 24
q, r = divmod(24, world)
u0 = rank * q + min(rank, r); u1 = u0 + q + (1 if rank < r else 0)
r0, r1 = u0 * plane, u1 * plane
idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
if rank == 0:
    idt.copy_(torch.frombuffer(bytearray(L.lsba_get_unique_id()), dtype=torch.uint8))
dist.broadcast(idt, 0)
rp = p.row_ptr[r0:r1 + 1] - p.row_ptr[r0]
ci, va = p.col_idx[p.row_ptr[r0]:p.row_ptr[r1]], p.vals[p.row_ptr[r0]:p.row_ptr[r1]]
with L.Context(p.n, p.s, p.m, rp, ci, va, row_begin=r0, row_end=r1, rank=rank, nranks=world,
               nccl_id=bytes(idt.cpu().numpy().tobytes()), device=rank) as ctx:
    B = torch.from_numpy(np.ascontiguousarray(p.B[r0:r1])).cuda()
    X = torch.zeros_like(B)
    assert ctx.begin(B, "cl") == 0
    for _ in range(5):
        assert ctx.step().chol_flag == 0
    H = ctx.hessenberg(5, p.s)
    info = ctx.solve(B, X, p.m, p.tol, 2000, cond_threshold=1e8)
    Xl = X.cpu().numpy()
out = [None] * world
dist.all_gather_object(out, (H.tolist(), info.as_dict(), Xl.tolist()))
if rank == 0:
    json.dump(out, open(os.environ["LSBA_OUT"], "w"))
dist.destroy_process_group()
'''


@pytest.mark.parametrize("devar", ["0", "1"])
def test_two_nccl_ranks_match_one(devar, tmp_path):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    import json
    import paper_2208_09899_b200 as L
    from lsba_inputs import make_twin
    script = tmp_path / "worker.py"
    script.write_text(WORKER)
    out = tmp_path / "out.json"
    env = dict(os.environ, LSBA_ROOT=ROOT, LSBA_OUT=str(out), LSBA_DEVAR=devar)
    subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                    "--master-addr", "127.0.0.1", "--master-port", "29533", str(script)],
                   check=True, env=env, timeout=600)
    res = json.load(open(out))
    p = make_twin(5)
    with L.Context(p.n, p.s, p.m, p.row_ptr, p.col_idx, p.vals) as ctx:
        B = torch.from_numpy(p.B).cuda()
        X = torch.zeros_like(B)
        assert ctx.begin(B, "cl") == 0
        for _ in range(5):
            ctx.step()
        H1 = ctx.hessenberg(5, p.s)
        i1 = ctx.solve(B, X, p.m, p.tol, 2000, cond_threshold=1e8)
        X1 = X.cpu().numpy()
    H = np.array(res[0][0])
    assert np.array_equal(H, np.array(res[1][0]))           # replicated on both ranks
    assert np.linalg.norm(H - H1) <= 1e-12 * np.linalg.norm(H1)
    i2 = res[0][1]
    assert i2["outcome"] == L.LSBA_CONVERGED and abs(i2["cycles"] - i1.cycles) <= 1
    X2 = np.concatenate([np.array(r[2]) for r in res])
    if (i2["cycles"], i2["iterations"]) == (i1.cycles, i1.iterations):
        assert np.linalg.norm(X2 - X1) <= 1e-8 * np.linalg.norm(X1)
