"""The diagnostic environment switches of DESIGN.md 6.5 change only how the step is scheduled or
cached, never what it computes: with each non-default setting a restarted solve still matches
the oracle (true residual <= tol checked with the oracle's SpMM, cycles within one), and the
first Arnoldi steps match the default run to rounding.  The switches are read at lsba_create."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SWITCHES = [
    {"LSBA_PDL": "0"},
    {"LSBA_PDL_PROJ": "0"},
    {"LSBA_L2PERSIST": "0"},
    {"LSBA_L2PERSIST": "1"},
    {"LSBA_NO_FUSE": "1"},
    {"LSBA_UPD_MAIN": "1"},
    {"LSBA_G7": "2"},
    {"LSBA_SPEC_END": "0"},
    {"LSBA_DEVJOIN": "0"},
    {"LSBA_DEVJOIN": "2"},
]


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2208_09899_b200 as L
    return L


def _run(L, env, p, skel="pip"):
    import torch
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        with L.Context(p.n, p.s, p.m, p.row_ptr, p.col_idx, p.vals) as ctx:
            B = torch.from_numpy(p.B).cuda()
            X = torch.zeros_like(B)
            info = ctx.solve(B, X, p.m, p.tol, 2000, skel=skel)
            L.lsba_set_skeleton(ctx.ctx, skel)
            assert ctx.begin(B, "cl") == 0
            for _ in range(4):
                ctx.step()
            H = ctx.hessenberg(4, p.s)
            return X.cpu().numpy(), info, H
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("env", SWITCHES, ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_switch_keeps_results(L, env):
    from lsba_inputs import make_twin
    from oracle import lsba_oracle as O
    p = make_twin(2)                                   # 2D Laplacian 64^2, s = 4
    X0, i0, H0 = _run(L, {}, p)
    X1, i1, H1 = _run(L, env, p)
    A = (p.row_ptr, p.col_idx, p.vals)
    for X, info in ((X0, i0), (X1, i1)):
        assert info.outcome == L.LSBA_CONVERGED
        rel = np.linalg.norm(p.B - O.spmm(*A, X)) / np.linalg.norm(p.B)
        assert rel <= p.tol * (1 + 1e-6)
    assert abs(i1.cycles - i0.cycles) <= 1
    assert np.linalg.norm(H1 - H0) <= 1e-12 * np.linalg.norm(H0)


def _run_forced(L, env, p, max_restarts, sing_cycle):
    import torch
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        with L.Context(p.n, p.s, p.m, p.row_ptr, p.col_idx, p.vals) as ctx:
            L.lsba_set_force_singular(ctx.ctx, sing_cycle)
            B = torch.from_numpy(p.B).cuda()
            X = torch.zeros_like(B)
            info = ctx.solve(B, X, p.m, p.tol, max_restarts)
            return X.cpu().numpy(), info
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("spec", ["0", "1"])
@pytest.mark.parametrize("sing_cycle,max_restarts", [(2, 50), (2, 1), (3, 50)])
def test_singular_cycle_end_keeps_last_good_x(L, spec, sing_cycle, max_restarts):
    """A singular cycle-end projected solve (forced) ends the solve DEAD with the X of the
    cycle before it, whether or not the next cycle's end was enqueued speculatively
    (LSBA_SPEC_END): the speculative end checks the pending guard and no-ops."""
    from lsba_inputs import make_twin
    p = make_twin(2)                          # 2D Laplacian 64^2, s = 4, m = 20: ~33 cycles to m
    Xref, iref = _run_forced(L, {"LSBA_SPEC_END": spec}, p, sing_cycle - 2, 0)   # cycles 1..c-1
    assert iref.outcome == L.LSBA_MAX_RESTARTS and iref.cycles == sing_cycle - 1
    X, info = _run_forced(L, {"LSBA_SPEC_END": spec}, p, max_restarts, sing_cycle)
    assert info.outcome == L.LSBA_DEAD
    assert info.cycles == sing_cycle          # the cycle whose end was singular is counted
    assert np.all(np.isfinite(X))
    assert np.array_equal(X, Xref)            # bitwise: the same deterministic kernels
    assert info.true_relres == pytest.approx(iref.true_relres, rel=1e-12)


def test_caller_allocator_owns_workspace(L):
    """lsba_create_with_allocator (SURVEY.md 8(b)'s caller-owned workspace): with PyTorch's
    caching allocator the context's device buffers are torch's (memory_allocated grows by the
    workspace and falls back after destroy), and the solve is bitwise the default one."""
    import torch
    from lsba_inputs import make_twin
    p = make_twin(5)
    with L.Context(p.n, p.s, p.m, p.row_ptr, p.col_idx, p.vals) as ctx:
        B = torch.from_numpy(p.B).cuda()
        X0 = torch.zeros_like(B)
        i0 = ctx.solve(B, X0, p.m, p.tol, 2000, cond_threshold=1e8)
    torch.cuda.synchronize()
    before = torch.cuda.memory_allocated()
    ctx = L.Context(p.n, p.s, p.m, p.row_ptr, p.col_idx, p.vals, allocator="torch")
    try:
        ws = L.lsba_workspace_bytes(ctx.ctx)
        grown = torch.cuda.memory_allocated() - before
        assert grown >= 0.9 * ws and ws > 8 * p.n * p.s * (p.m + 1)
        X1 = torch.zeros_like(B)
        i1 = ctx.solve(B, X1, p.m, p.tol, 2000, cond_threshold=1e8)
        assert (i1.cycles, i1.iterations) == (i0.cycles, i0.iterations)
        assert torch.equal(X0, X1)
    finally:
        ctx.close()
    torch.cuda.synchronize()
    assert torch.cuda.memory_allocated() - before < 0.1 * ws
