"""Device-side join of the update kernel ("a3/a5 small step"): on one rank the
Gram's tail acquires the previous step's update kernel (sequence word released at its exit)
instead of the main stream waiting on its event.  It only reorders WHEN the Gram starts, so
every solve must be BITWISE identical to the event join (LSBA_DEVJOIN=0 vs 2 = at any size) — including the
endings where the update ends the cycle while the next speculative Gram already streams
(convergence mid-cycle, the kappa trigger, NaN-flags, forced flags, happy breakdown)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2208_09899_b200 as L
    return L


def _problem(name):
    from lsba_inputs import identity, make_twin, rhs, tridiag, tridiag_rhs
    if name == "tridiag100":
        A = tridiag(100)
        return A, tridiag_rhs(100), 50, 1e-10
    if name == "identity300":
        return identity(300), rhs(300, 4, seed=5), 5, 1e-10
    p = make_twin({"tiny": 1, "lapl2d": 2, "cd3d": 3, "rand": 4, "lapl3d": 5}[name])
    return (p.row_ptr, p.col_idx, p.vals), p.B, p.m, p.tol


def _solve(L, env, name, ip, mod, tau, force, max_restarts=2000):
    import torch
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        A, B, m, tol = _problem(name)
        n, s = B.shape
        with L.Context(n, s, m, *A) as ctx:
            if force:
                L.lsba_set_force_flag(ctx.ctx, force)
            X = torch.zeros(n, s, dtype=torch.float64, device="cuda")
            info = ctx.solve(torch.from_numpy(np.ascontiguousarray(B)).cuda(), X, m, tol, max_restarts,
                             ip=ip, mod=mod, cond_threshold=tau)
            torch.cuda.synchronize()
            return X.cpu().numpy(), info
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


CASES = [
    ("tiny", "cl", "gmres", float("inf"), 0, 2000),
    ("tiny", "cl", "fom", float("inf"), 6, 2000),       # forced NaN-flag at step 6
    ("lapl2d", "cl", "gmres", float("inf"), 0, 2000),   # converges mid-cycle
    ("lapl2d", "cl", "fom", float("inf"), 0, 2000),
    ("cd3d", "cl", "gmres", 1e8, 0, 2000),
    ("rand", "cl", "gmres", float("inf"), 0, 2000),
    ("lapl3d", "cl", "gmres", 1e8, 0, 2000),
    ("tridiag100", "cl", "fom", 1e8, 0, 50),           # kappa trigger at k = 15
    ("tridiag100", "cl", "fom", float("inf"), 0, 50),  # NaN-flags
    ("identity300", "cl", "gmres", float("inf"), 0, 5),  # happy breakdown
]


@pytest.mark.parametrize("name,ip,mod,tau,force,maxr", CASES,
                         ids=[f"{c[0]}-{c[2]}-tau{c[3]:g}-f{c[4]}" for c in CASES])
def test_device_join_bitwise(L, name, ip, mod, tau, force, maxr):
    X0, i0 = _solve(L, {"LSBA_DEVJOIN": "0"}, name, ip, mod, tau, force, maxr)
    X1, i1 = _solve(L, {"LSBA_DEVJOIN": "2"}, name, ip, mod, tau, force, maxr)
    assert i1.outcome == i0.outcome
    for f in ("cycles", "iterations", "nan_flags", "cond_restarts", "m_final", "happy"):
        assert getattr(i1, f) == getattr(i0, f), f
    assert np.array_equal(X1, X0)
    assert i1.true_relres == i0.true_relres
