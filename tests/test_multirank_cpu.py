"""Multi-rank (N > 1) host logic on CPU with the gloo backend, world size 2 and 3.

The CUDA library's N > 1 path is: contiguous row
partition; a ghost plan from ``lsba_ghost_plan`` (exported host code of liblsba.so, exercised
here without a GPU); per step one halo exchange of the ghost rows and exactly ONE allreduce of
the partial Gram (the step's single sync); replicated small state.  This test
runs that decomposition with gloo point-to-point and allreduce around the oracle's arithmetic
and checks it against the single-rank oracle:
  * the halo-extended local SpMM equals the global SpMM rows bitwise (same CSR order);
  * the allreduced partial Gram equals the global Gram to rounding;
  * K distributed BCGS-PIP steps (one halo + one allreduce each) reproduce the single-rank
    H and basis, with exactly K + 1 Gram allreduces (IO + K steps);
  * the same for K BMGS-CWY steps (Alg 6): loop iteration 1 + K steps, K + 1 allreduces;
  * and for K BCGS-IRO-LS steps (Alg 7): K + 1 allreduces, H and basis equal to the oracle's.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(kind):
    from lsba_inputs import random_sparse, rhs, stencil
    if kind == "stencil":
        A = stencil(2, 24, (10.0, 5.0), shape=[24, 40])
    else:
        A = random_sparse(3000)
    n = A[0].size - 1
    return A, rhs(n, 4)


def _partition(n, world):
    return np.array([n * r // world for r in range(world + 1)], dtype=np.int64)


def _worker(rank, world, port, kind, K, out):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from oracle import lsba_oracle as O
    import paper_2208_09899_b200 as L

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B = _problem(kind)
        rp, ci, va = A
        n, s = B.shape
        part = _partition(n, world)
        r0, r1 = int(part[rank]), int(part[rank + 1])
        rp_loc = rp[r0:r1 + 1] - rp[r0]
        ci_loc, va_loc = ci[rp[r0]:rp[r1]], va[rp[r0]:rp[r1]]

        # ghost plan (the library's host code) and the send lists it implies
        col_local, ghosts, recv_counts = L.lsba_ghost_plan(r0, r1, ci_loc, part)
        assert recv_counts[rank] == 0 and recv_counts.sum() == ghosts.size
        everyone = [None] * world
        dist.all_gather_object(everyone, ghosts.tolist())
        send_rows = {r: np.array([g for g in everyone[r] if r0 <= g < r1], dtype=np.int64) - r0
                     for r in range(world) if r != rank}
        recv_off = np.concatenate([[0], np.cumsum(recv_counts)])
        A_loc = (rp_loc, col_local, va_loc)
        n_allreduce = [0]

        def halo(V):
            """ghost rows of V (ordered as ``ghosts``) by gloo send/recv."""
            reqs = []
            for r, rows in send_rows.items():
                if rows.size:
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(V[rows])), r))
            G = np.zeros((ghosts.size, s))
            for r in range(world):
                if r != rank and recv_counts[r]:
                    buf = torch.zeros((int(recv_counts[r]), s), dtype=torch.float64)
                    dist.recv(buf, r)
                    G[recv_off[r]:recv_off[r + 1]] = buf.numpy()
            for q in reqs:
                q.wait()
            return np.vstack([V, G])

        def spmm_dist(V):
            return O.spmm(rp_loc, col_local, va_loc, halo(V))

        def allreduce(x):
            n_allreduce[0] += 1
            t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64))
            dist.all_reduce(t)
            return t.numpy()

        # (1) halo-extended local SpMM == global SpMM rows, bitwise
        V = np.random.default_rng(5).standard_normal((n, s))
        W_loc = spmm_dist(V[r0:r1])
        W_glob = O.spmm(rp, ci, va, V)
        assert np.array_equal(W_loc, W_glob[r0:r1])

        # (2) allreduced partial Gram == global Gram
        Xs = [V[r0:r1], W_loc]
        G = allreduce(O.ip_cl(Xs, W_loc))
        Gg = O.ip_cl([V, W_glob], W_glob)
        assert np.allclose(G, Gg, rtol=1e-13, atol=1e-13 * np.abs(Gg).max())

        # (3) K distributed BCGS-PIP steps, one halo + one allreduce each (Alg 3)
        n_allreduce[0] = 0
        Bl = B[r0:r1]
        beta_chk = O.chol_flag(O.sym(allreduce(O.gram(Bl, Bl))))      # IO: 1 sync
        beta, flag = beta_chk
        assert not flag
        Vs = [O.right_trsm_upper(Bl, beta)]
        Hbar = np.zeros(((K + 1) * s, K * s))
        for k in range(1, K + 1):
            W = spmm_dist(Vs[-1])                                       # halo
            Gk = allreduce(O.ip_cl(Vs + [W], W))                         # the single sync
            Hcol, Omega = Gk[:k * s], Gk[k * s:]
            R, flag = O.chol_flag(Omega - Hcol.T @ Hcol)
            assert not flag
            P = W - np.concatenate(Vs, axis=1) @ Hcol
            Vs.append(O.right_trsm_upper(P, R))
            Hbar[:k * s, (k - 1) * s:k * s] = Hcol
            Hbar[k * s:(k + 1) * s, (k - 1) * s:k * s] = R
        assert n_allreduce[0] == K + 1

        # (4) BMGS-CWY (Alg 6): after IO and loop iteration 1, every Arnoldi step is one halo
        # exchange + ONE allreduce of the two-block Gram <[V_1..V_k U], [U W]>
        n_allreduce[0] = 0
        Vc = [Vs[0]]
        W = spmm_dist(Vc[0])
        H11 = allreduce(O.ip_cl([Vc[0]], W))                           # iteration 1
        U = W - Vc[0] @ H11
        Hc = np.zeros(((K + 1) * s, K * s))
        Hc[:s, :s] = H11
        T = np.eye((K + 1) * s)
        for k in range(1, K + 1):
            W = spmm_dist(U)
            Gk = allreduce(O.ip_cl(Vc + [U], np.concatenate([U, W], axis=1)))   # the single sync
            Y, Z, Om, Pt = Gk[:k * s, :s], Gk[:k * s, s:], Gk[k * s:, :s], Gk[k * s:, s:]
            R, flag = O.chol_flag(Om)
            assert not flag
            Ri = O.right_trsm_upper(np.eye(s), R)
            P = np.linalg.solve(R.T, Pt)
            T[:k * s, k * s:(k + 1) * s] = -T[:k * s, :k * s] @ (Y @ Ri)
            Hn = T[:(k + 1) * s, :(k + 1) * s].T @ (np.vstack([Z, P]) @ Ri)
            Vc.append(U @ Ri)
            Hc[k * s:(k + 1) * s, (k - 1) * s:k * s] = R
            if k < K:
                Hc[:(k + 1) * s, k * s:(k + 1) * s] = Hn
            U = W @ Ri - np.concatenate(Vc, axis=1) @ Hn
        assert n_allreduce[0] == K + 1

        # (5) BCGS-IRO-LS (Alg 7, block DCGS2): the same lagged loop, still ONE allreduce of the
        # two-block Gram per step; Omega = Omega~ - Y^T Y, column k = J + Y, P = R^{-T}(P~ - Y^T Z),
        # J = ([Z; P] - H_{1:k+1,1:k} Y) R^{-1}
        n_allreduce[0] = 0
        Vi = [Vs[0]]
        W = spmm_dist(Vi[0])
        J = allreduce(O.ip_cl([Vi[0]], W))                             # iteration 1
        U = W - Vi[0] @ J
        Hi = np.zeros(((K + 1) * s, K * s))
        for k in range(1, K + 1):
            W = spmm_dist(U)
            Gk = allreduce(O.ip_cl(Vi + [U], np.concatenate([U, W], axis=1)))   # the single sync
            Y, Z, Omt, Pt = Gk[:k * s, :s], Gk[:k * s, s:], Gk[k * s:, :s], Gk[k * s:, s:]
            R, flag = O.chol_flag(Omt - Y.T @ Y)
            assert not flag
            Hi[:k * s, (k - 1) * s:k * s] = J + Y
            Hi[k * s:(k + 1) * s, (k - 1) * s:k * s] = R
            Ri = O.right_trsm_upper(np.eye(s), R)
            P = np.linalg.solve(R.T, Pt - Y.T @ Z)
            ZP = np.vstack([Z, P])
            J = (ZP - Hi[:(k + 1) * s, :k * s] @ Y) @ Ri
            Vn = (U - np.concatenate(Vi, axis=1) @ Y) @ Ri
            Vi.append(Vn)
            U = (W - np.concatenate(Vi, axis=1) @ ZP) @ Ri
        assert n_allreduce[0] == K + 1
        out[rank] = dict(H=Hbar, beta=beta, V=np.stack(Vs), rows=(r0, r1), Hc=Hc, Vc=np.stack(Vc),
                         Hi=Hi, Vi=np.stack(Vi))
    finally:
        dist.destroy_process_group()


def _run(world, kind, K):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, K, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
    codes = [p.exitcode for p in procs]
    res = dict(out)
    mgr.shutdown()
    assert codes == [0] * world, codes
    return res


@pytest.mark.parametrize("world,kind", [(2, "stencil"), (2, "random"), (3, "random")])
def test_distributed_pip_steps_match_single_rank(world, kind):
    import sys
    sys.path.insert(0, ROOT)
    from oracle import lsba_oracle as O
    K = 4
    res = _run(world, kind, K)
    A, B = _problem(kind)
    s = B.shape[1]
    arn = O.PipArnoldi(A, "cl", K, s)
    assert not arn.begin(B)
    for _ in range(K):
        assert not arn.step().flag
    cwy = O.CwyArnoldi(A, "cl", K, s)
    assert not cwy.begin(B)
    for _ in range(K):
        assert not cwy.step().flag
    iro = O.IrolsArnoldi(A, "cl", K, s)
    assert not iro.begin(B)
    for _ in range(K):
        assert not iro.step().flag
    for r in range(world):
        d = res[r]
        assert np.array_equal(d["Hc"], res[0]["Hc"]) and np.array_equal(d["Hi"], res[0]["Hi"])
        np.testing.assert_allclose(d["Hi"], iro.Hbar, rtol=0, atol=1e-11 * np.abs(iro.Hbar).max())
        for j in range(K + 1):
            r0, r1 = d["rows"]
            assert np.linalg.norm(d["Vi"][j] - iro.V[j][r0:r1]) <= 1e-11 * np.linalg.norm(iro.V[j])
        np.testing.assert_allclose(d["Hc"], cwy.Hbar, rtol=0, atol=1e-11 * np.abs(cwy.Hbar).max())
        for j in range(K + 1):
            r0, r1 = d["rows"]
            assert np.linalg.norm(d["Vc"][j] - cwy.V[j][r0:r1]) <= 1e-11 * np.linalg.norm(cwy.V[j])
        # replicated small state: identical on every rank (same allreduce results)
        assert np.array_equal(d["H"], res[0]["H"]) and np.array_equal(d["beta"], res[0]["beta"])
        np.testing.assert_allclose(d["H"], arn.Hbar, rtol=0, atol=1e-11 * np.abs(arn.Hbar).max())
        r0, r1 = d["rows"]
        for j in range(K + 1):
            vo = arn.V[j][r0:r1]
            assert np.linalg.norm(d["V"][j] - vo) <= 1e-11 * np.linalg.norm(arn.V[j])
