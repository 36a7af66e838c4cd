"""The library's OWN multi-rank path (PAPER.md:57 row-partitioned block vectors,
PAPER.md:209 replicated small computations) run on one GPU.

P contexts, one per host thread, each holding a contiguous row range (whole z-planes of the
stencils), are joined by a loopback group (lsba_create_loopback): the library executes exactly
its P > 1 code -- create-time partition check and ghost-plan exchange, the halo pack and
grouped send/recv overlapped with the interior-row SpMM, ONE allreduce of the partial Gram per
block step, the unfused small step, replicated device-side decisions and the P > 1 enqueue rule
(every rank enqueues the same steps) -- with the collectives carried out by host rendezvous and
stream-ordered device copies instead of NCCL (no kernel waits on another rank's kernel).

Checked against the single-rank run of the same library (and the oracle's SpMM for the final
residual): Hessenberg and basis after 5 steps within 1e-12 (only the Gram's summation order
changes with P), full solves with equal cycle counts (+-1, reading R20), X within 1e-8 when the
trajectories agree, true residual <= tol.  A one-rank NCCL communicator (LSBA_FORCE_COMM=1)
runs the same distributed path through real ncclAllReduce calls.
"""
import os
import threading

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


def z_partition(p, P):
    """Row ranges of P ranks: whole planes of the slowest stencil dimension (or even row
    blocks for the random matrix)."""
    n = p.n
    meta = p.meta
    unit = meta["N"] ** (meta["dims"] - 1) if meta["kind"] == "stencil" else 1
    units = n // unit
    q, r = divmod(units, P)
    out = []
    for k in range(P):
        u0 = k * q + min(k, r)
        u1 = u0 + q + (1 if k < r else 0)
        out.append((u0 * unit, u1 * unit))
    return out


def run_ranks(L, p, P, fn, env=None, timeout=600):
    """fn(ctx, B_dev, X_dev, rank, (r0, r1)) on P threads with a loopback group; returns the
    per-rank results in rank order."""
    import torch
    parts = z_partition(p, P)
    group = L.lsba_loopback_create(P)
    res, errs = [None] * P, [None] * P
    old = {k: os.environ.get(k) for k in (env or {})}
    os.environ.update(env or {})

    def work(rank):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            r0, r1 = parts[rank]
            rp = p.row_ptr[r0:r1 + 1] - p.row_ptr[r0]
            ci = p.col_idx[p.row_ptr[r0]:p.row_ptr[r1]]
            va = p.vals[p.row_ptr[r0]:p.row_ptr[r1]]
            with torch.cuda.stream(st):
                ctx = L.Context(p.n, p.s, p.m, rp, ci, va, row_begin=r0, row_end=r1, rank=rank, nranks=P,
                                device=0, stream=st.cuda_stream, loopback=group)
                try:
                    B = torch.from_numpy(np.ascontiguousarray(p.B[r0:r1])).cuda()
                    X = torch.zeros_like(B)
                    st.synchronize()
                    res[rank] = fn(ctx, B, X, rank, (r0, r1))
                    st.synchronize()
                finally:
                    ctx.close()
        except BaseException as e:       # surfaced below
            errs[rank] = e

    try:
        th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout)
        assert not any(t.is_alive() for t in th), "loopback ranks hung"
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    for e in errs:
        if e is not None:
            raise e
    L.lsba_loopback_destroy(group)
    return res


def steps_fn(ip, K):
    def fn(ctx, B, X, rank, rows):
        b = ctx.s if ip == "cl" else 1
        assert ctx.begin(B, ip) == 0
        for _ in range(K):
            assert ctx.step().chol_flag == 0
        H = ctx.hessenberg(K, b)
        Vs = [ctx.basis_block(j).cpu().numpy() for j in range(1, K + 2)]
        return H, Vs
    return fn


def solve_fn(ip, tau):
    def fn(ctx, B, X, rank, rows):
        info = ctx.solve(B, X, ctx.m_max, 1e-8, 2000, ip=ip, cond_threshold=tau)
        return info.as_dict(), X.cpu().numpy()
    return fn


def single(L, p, fn):
    import torch
    with L.Context(p.n, p.s, p.m, p.row_ptr, p.col_idx, p.vals) as ctx:
        B = torch.from_numpy(p.B).cuda()
        X = torch.zeros_like(B)
        return fn(ctx, B, X, 0, (0, p.n))


CASES = [(5, "cl", 2), (5, "cl", 3), (5, "cl", 4), (2, "cl", 2), (2, "cl", 4), (4, "cl", 2), (4, "gl", 3),
         (3, "cl", 3)]


@pytest.mark.parametrize("ovl", ["1", "0"])
@pytest.mark.parametrize("twin,ip,P", CASES)
def test_loopback_steps_match_single_rank(L, twin, ip, P, ovl):
    from lsba_inputs import make_twin
    p = make_twin(twin)
    K = 5
    H1, V1 = single(L, p, steps_fn(ip, K))
    out = run_ranks(L, p, P, steps_fn(ip, K), env={"LSBA_HALO_OVERLAP": ovl})
    b = p.s if ip == "cl" else 1
    for r in range(1, P):                 # replicated small state: identical on every rank
        assert np.array_equal(out[r][0], out[0][0])
    # stencils: 1e-12; the random s = 16 twin amplifies the Gram's rounding ~10x per step
    # through Omega - H^T H (SURVEY.md 8(c) parity note), so the north star's 1e-10 applies
    tol = 1e-10 if p.meta["kind"] == "random" else 1e-12
    H = out[0][0]
    for k in range(K):
        col, col1 = H[:, k * b:(k + 1) * b], H1[:, k * b:(k + 1) * b]
        assert np.linalg.norm(col - col1) <= tol * np.linalg.norm(col1), k
    for j in range(K + 1):
        Vj = np.concatenate([o[1][j] for o in out])
        assert np.linalg.norm(Vj - V1[j]) <= tol * np.linalg.norm(V1[j]), j


# (the random twin has no interior block: with the overlap on it runs the local/ghost split)
SOLVES = [(5, "cl", 2, 1e8), (5, "cl", 3, 1e8), (2, "cl", 4, float("inf")), (4, "gl", 2, float("inf")),
          (4, "cl", 3, float("inf")), (3, "cl", 2, 1e8)]


@pytest.mark.parametrize("twin,ip,P,tau", SOLVES)
@pytest.mark.parametrize("ovl", ["1", "0"])
def test_loopback_solve_matches_single_rank(L, twin, ip, P, tau, ovl):
    from lsba_inputs import make_twin
    from oracle import lsba_oracle as O
    p = make_twin(twin)
    i1, X1 = single(L, p, solve_fn(ip, tau))
    out = run_ranks(L, p, P, solve_fn(ip, tau), env={"LSBA_HALO_OVERLAP": ovl})
    infos = [o[0] for o in out]
    for r in range(1, P):                 # every rank takes the same decisions
        for key in ("outcome", "cycles", "iterations", "nan_flags", "cond_restarts", "true_relres"):
            assert infos[r][key] == infos[0][key], key
    ip_ = infos[0]
    X = np.concatenate([o[1] for o in out])
    assert ip_["outcome"] == L.LSBA_CONVERGED and ip_["true_relres"] <= p.tol
    rel = np.linalg.norm(p.B - O.spmm(p.row_ptr, p.col_idx, p.vals, X)) / np.linalg.norm(p.B)
    assert rel <= p.tol * (1 + 1e-6)
    assert abs(ip_["cycles"] - i1["cycles"]) <= 1
    if (ip_["cycles"], ip_["iterations"]) == (i1["cycles"], i1["iterations"]):
        assert np.linalg.norm(X - X1) <= 1e-8 * np.linalg.norm(X1)
    assert ip_["syncs"] == ip_["iterations"] + ip_["cycles"]


@pytest.mark.parametrize("devar", ["0", "1"])
@pytest.mark.parametrize("twin,ip", [(2, "cl"), (5, "cl"), (4, "gl"), (4, "cl")])
def test_force_comm_one_rank_nccl(L, twin, ip, devar):
    """LSBA_FORCE_COMM=1: one rank through the distributed path with a real NCCL communicator;
    LSBA_DEVAR=1 adds f2: the Gram allreduce in the Gram kernel's tail through the NCCL device
    API (symmetric window + LSA barrier) with the small step fused again."""
    import torch
    from lsba_inputs import make_twin
    p = make_twin(twin)
    tau = p.cond_threshold
    i1, X1 = single(L, p, solve_fn(ip, tau))
    H1, V1 = single(L, p, steps_fn(ip, 5))
    os.environ["LSBA_FORCE_COMM"] = "1"
    os.environ["LSBA_DEVAR"] = devar
    try:
        i2, X2 = single(L, p, solve_fn(ip, tau))
        H2, V2 = single(L, p, steps_fn(ip, 5))
    finally:
        os.environ.pop("LSBA_FORCE_COMM", None)
        os.environ.pop("LSBA_DEVAR", None)
    assert i2["outcome"] == L.LSBA_CONVERGED and i2["true_relres"] <= p.tol
    assert abs(i2["cycles"] - i1["cycles"]) <= 1
    if (i2["cycles"], i2["iterations"]) == (i1["cycles"], i1["iterations"]):
        assert np.linalg.norm(X2 - X1) <= 1e-8 * np.linalg.norm(X1)
    # one rank: the allreduce is the identity, the fused and unfused small steps agree bitwise
    assert np.linalg.norm(H2 - H1) <= 1e-13 * np.linalg.norm(H1)
    torch.cuda.synchronize()


@pytest.mark.parametrize("skel", ["cwy", "icwy", "irols", "bmgs", "pio"])
@pytest.mark.parametrize("ip", ["cl", "gl"])
def test_loopback_other_skeletons(L, skel, ip):
    """The comparison / lagged skeletons (Alg 2, 4, 6, 7) through the P > 1 path: the same
    decisions on every rank, converged, cycles within one of the one-rank run, X within 1e-8
    when the counts agree."""
    from lsba_inputs import make_twin
    p = make_twin(5)

    def fn(ctx, B, X, rank, rows):
        info = ctx.solve(B, X, ctx.m_max, 1e-8, 2000, ip=ip, cond_threshold=1e8, skel=skel)
        return info.as_dict(), X.cpu().numpy()

    i1, X1 = single(L, p, fn)
    out = run_ranks(L, p, 3, fn)
    infos = [o[0] for o in out]
    for r in range(1, 3):
        for key in ("outcome", "cycles", "iterations", "nan_flags", "true_relres", "syncs"):
            assert infos[r][key] == infos[0][key], key
    i2 = infos[0]
    X = np.concatenate([o[1] for o in out])
    assert i2["outcome"] == L.LSBA_CONVERGED and i2["true_relres"] <= p.tol
    assert abs(i2["cycles"] - i1["cycles"]) <= 1
    if (i2["cycles"], i2["iterations"]) == (i1["cycles"], i1["iterations"]):
        assert np.linalg.norm(X - X1) <= 1e-8 * np.linalg.norm(X1)
        assert i2["syncs"] == i1["syncs"]          # the paper's counters do not depend on P


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_ilu0_block_jacobi(L, P):
    """Left ILU(0) at P > 1 is block-Jacobi ILU(0) of the local diagonal blocks (R28): every rank
    takes the same decisions and the solve converges in the preconditioned norm; the plain
    residual of X is checked with the oracle's SpMM."""
    from lsba_inputs import make_twin
    from oracle import lsba_oracle as O
    p = make_twin(5)

    def fn(ctx, B, X, rank, rows):
        info = ctx.solve(B, X, ctx.m_max, 1e-8, 2000, ip="cl", cond_threshold=1e8, prec="ilu0")
        return info.as_dict(), X.cpu().numpy()

    out = run_ranks(L, p, P, fn)
    infos = [o[0] for o in out]
    for r in range(1, P):
        for key in ("outcome", "cycles", "iterations", "true_relres"):
            assert infos[r][key] == infos[0][key], key
    assert infos[0]["outcome"] == L.LSBA_CONVERGED
    X = np.concatenate([o[1] for o in out])
    rel = np.linalg.norm(p.B - O.spmm(p.row_ptr, p.col_idx, p.vals, X)) / np.linalg.norm(p.B)
    assert rel <= 1e-6            # (tol 1e-8 holds in the block-Jacobi-preconditioned norm)
