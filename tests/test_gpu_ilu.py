"""GPU parity of ILU(0) left preconditioning
through the C ABI against the oracle (oracle.lsba_oracle.ilu0 / Ilu0Factors / solve(prec=)):

  * factor values vs the oracle's IKJ ILU(0) at 1e-13 (same per-entry update order; FMA, R21)
    and the level counts of L and U exactly (integers);
  * lsba_ilu0_apply = U^{-1} L^{-1} X vs the oracle at 1e-12 normwise, bitwise repeatable over
    many launches (the sync-free solve sums every row in CSR order);
  * preconditioned restarted solves (BCGS-PIP and BMGS-CWY) vs the oracle's: converged in the
    preconditioned norm (checked with the oracle's arithmetic), cycles within one;
  * the exact-factorisation limit (tridiag: one step, happy breakdown), zero pivots;
  * BASELINE-size config 2 (2^20 rows, 2047 levels per factor): the defining property
    (L U)_ij = a_ij on pattern(A) and L (U Y) = X, checked with scipy.sparse products.
"""
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


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def twin(i):
    from lsba_inputs import make_twin
    return make_twin(i)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_factors_and_levels_vs_oracle(L, cfg):
    from oracle import lsba_oracle as O
    p = twin(cfg)
    F = O.ilu0(p.row_ptr, p.col_idx, p.vals)
    with L.Context(p.n, p.s, 4, p.row_ptr, p.col_idx, p.vals) as ctx:
        L.lsba_ilu0_setup(ctx.ctx, True)
        lu, (nlL, nlU) = L.lsba_copy_ilu0_factors(ctx.ctx, p.col_idx.size)
    scale = np.abs(F.lu).max()
    assert np.abs(lu - F.lu).max() <= 1e-13 * scale
    assert nlL == len(O._tri_plan(F, True)) and nlU == len(O._tri_plan(F, False))


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_apply_vs_oracle_and_repeatable(L, cfg):
    from oracle import lsba_oracle as O
    p = twin(cfg)
    F = O.ilu0(p.row_ptr, p.col_idx, p.vals)
    X = np.random.default_rng(cfg).standard_normal((p.n, p.s))
    Yo = F.solve(X)
    with L.Context(p.n, p.s, 4, p.row_ptr, p.col_idx, p.vals) as ctx:
        L.lsba_ilu0_setup(ctx.ctx, True)
        Xd = dev(X)
        Y0 = ctx.ilu0_apply(Xd).cpu().numpy()
        for _ in range(30):
            Y = ctx.ilu0_apply(Xd).cpu().numpy()
            assert np.array_equal(Y, Y0)
        Yd = Xd.clone()                                    # in place (X == Y)
        L.lsba_ilu0_apply(ctx.ctx, Yd, Yd)
        assert np.array_equal(Yd.cpu().numpy(), Y0)
    for c in range(p.s):
        assert np.linalg.norm(Y0[:, c] - Yo[:, c]) <= 1e-12 * np.linalg.norm(Yo[:, c])


def test_spmm_stays_plain_with_preconditioner(L):
    from oracle import lsba_oracle as O
    p = twin(3)
    V = np.random.default_rng(0).standard_normal((p.n, p.s))
    with L.Context(p.n, p.s, 4, p.row_ptr, p.col_idx, p.vals) as ctx:
        L.lsba_ilu0_setup(ctx.ctx, True)
        W = ctx.spmm(dev(V)).cpu().numpy()
    Wo = O.spmm(p.row_ptr, p.col_idx, p.vals, V)
    assert np.abs(W - Wo).max() <= 1e-14 * np.abs(Wo).max()       # A V, not M^{-1} A V


def test_arnoldi_steps_on_preconditioned_operator(L):
    """5 BCGS-PIP steps on M^{-1} A vs the oracle's PipArnoldi on IluOperator (1e-10, R16)."""
    from oracle import lsba_oracle as O
    p = twin(3)
    A = (p.row_ptr, p.col_idx, p.vals)
    F = O.ilu0(*A)
    K = 5
    with L.Context(p.n, p.s, K, *A) as ctx:
        L.lsba_ilu0_setup(ctx.ctx, True)
        assert ctx.begin(dev(p.B), "cl") == 0
        infos = [ctx.step() for _ in range(K)]
        assert all(i.chol_flag == 0 for i in infos)
        H = ctx.hessenberg(K, p.s)
        Vs = [ctx.basis_block(j).cpu().numpy() for j in range(1, K + 2)]
    arn = O.PipArnoldi(O.IluOperator(A, F), "cl", K, p.s)
    assert not arn.begin(p.B)
    amp = []
    for _ in range(K):
        r = arn.step()
        assert not r.flag
        # BCGS-PIP's Pythagorean step amplifies an operator error by (||W|| / sigma_min(R))^2
        # (its O(eps) kappa^2 bound).  The operator here carries the triangular
        # solves' own error (normwise <= 1e-12 vs the oracle, test_apply_vs_oracle): the
        # tolerance is that bound times the amplification, per step, and never below 1e-10
        amp.append((np.linalg.norm(r.W, 2) / np.linalg.svd(r.R, compute_uv=False)[-1]) ** 2)
    b = p.s
    for k in range(K):
        tol = max(1e-10, 1e-12 * max(amp[:k + 1]) * (k + 1))
        col, colo = H[:, k * b:(k + 1) * b], arn.Hbar[:(K + 1) * b, k * b:(k + 1) * b]
        assert np.linalg.norm(col - colo) <= tol * np.linalg.norm(colo), (k, amp)
    for j, (v, vo) in enumerate(zip(Vs, arn.V)):
        tol = max(1e-10, 1e-12 * max(amp[:max(j, 1)]) * max(j, 1))
        assert np.linalg.norm(v - vo) <= tol * np.linalg.norm(vo), (j, amp)


@pytest.mark.parametrize("cfg,ip,mod,skel", [(1, "cl", "gmres", "pip"), (1, "gl", "fom", "pip"),
                                             (2, "cl", "gmres", "pip"), (3, "cl", "gmres", "pip"),
                                             (3, "cl", "gmres", "cwy"), (4, "cl", "gmres", "pip"),
                                             (5, "cl", "gmres", "pip")])
def test_preconditioned_solve_vs_oracle(L, cfg, ip, mod, skel):
    from oracle import lsba_oracle as O
    p = twin(cfg)
    A = (p.row_ptr, p.col_idx, p.vals)
    F = O.ilu0(*A)
    Xo, io = O.solve(A, p.B, m=p.m, tol=p.tol, max_restarts=500, ip=ip, mod=mod, skel=skel, prec=F)
    with L.Context(p.n, p.s, p.m, *A) as ctx:
        X = dev(np.zeros_like(p.B))
        info = ctx.solve(dev(p.B), X, p.m, p.tol, 500, ip=ip, mod=mod, skel=skel, prec="ilu0")
        Xg = X.cpu().numpy()
    assert io.outcome == O.CONVERGED and info.outcome == L.LSBA_CONVERGED
    rel = np.linalg.norm(F.solve(p.B - O.spmm(*A, Xg))) / np.linalg.norm(F.solve(p.B))
    assert rel <= p.tol * (1 + 1e-6) and info.true_relres <= p.tol
    assert abs(rel - info.true_relres) <= 1e-6 * p.tol + 1e-9 * rel
    assert abs(info.cycles - io.cycles) <= 1
    if (info.cycles, info.iterations) == (io.cycles, io.iterations):
        assert np.linalg.norm(Xg - Xo) <= 1e-6 * np.linalg.norm(Xo)


def test_preconditioned_vs_plain_fewer_steps(L):
    p = twin(3)
    A = (p.row_ptr, p.col_idx, p.vals)
    with L.Context(p.n, p.s, p.m, *A) as ctx:
        X = dev(np.zeros_like(p.B))
        i0 = ctx.solve(dev(p.B), X, p.m, p.tol, 500)
        X.zero_()
        i1 = ctx.solve(dev(p.B), X, p.m, p.tol, 500, prec="ilu0")
        X.zero_()
        i2 = ctx.solve(dev(p.B), X, p.m, p.tol, 500)          # switched off again: plain operator
    assert i1.iterations < i0.iterations
    assert (i2.iterations, i2.cycles) == (i0.iterations, i0.cycles)


def test_exact_factorisation_one_step(L):
    from lsba_inputs import tridiag, tridiag_rhs
    n = 300
    A = tridiag(n)
    B = tridiag_rhs(n)
    with L.Context(n, 2, 10, *A) as ctx:
        X = dev(np.zeros_like(B))
        info = ctx.solve(dev(B), X, 10, 1e-10, 5, mod="fom", prec="ilu0")
        Xg = X.cpu().numpy()
    assert info.outcome == L.LSBA_CONVERGED and info.iterations == 1 and info.happy == 1
    D = np.zeros((n, n))
    for i in range(n):
        D[i, A[1][A[0][i]:A[0][i + 1]]] = A[2][A[0][i]:A[0][i + 1]]
    Xs = np.linalg.solve(D, B)
    assert np.linalg.norm(Xg - Xs) <= 1e-9 * np.linalg.norm(Xs)


def test_zero_pivot_is_reported(L):
    rp = np.array([0, 2, 4], dtype=np.int64)
    ci = np.array([0, 1, 0, 1], dtype=np.int32)
    va = np.array([1.0, 1.0, 1.0, 1.0])                   # [[1,1],[1,1]]: u_22 = 0
    with L.Context(2, 1, 2, rp, ci, va) as ctx:
        with pytest.raises(L.LsbaError) as e:
            L.lsba_ilu0_setup(ctx.ctx, True)
        assert e.value.status == L.LSBA_E_NUMERIC
        with pytest.raises(L.LsbaError):
            ctx.ilu0_apply(dev(np.ones((2, 1))))
    rp = np.array([0, 1, 2], dtype=np.int64)
    ci = np.array([1, 0], dtype=np.int32)                  # no diagonal at all
    with L.Context(2, 1, 2, rp, ci, np.array([1.0, 1.0])) as ctx:
        with pytest.raises(L.LsbaError) as e:
            L.lsba_ilu0_setup(ctx.ctx, True)
        assert e.value.status == L.LSBA_E_NUMERIC


def test_fullsize_config2_properties(L):
    """2^20 rows, natural order (2047 levels per factor): (L U)_ij = a_ij on pattern(A) and
    L (U Y) = X for Y = lsba_ilu0_apply(X), with scipy.sparse products on the host."""
    import scipy.sparse as sp
    from lsba_inputs import make_config
    p = make_config(2)
    n = p.n
    with L.Context(n, p.s, 4, p.row_ptr, p.col_idx, p.vals) as ctx:
        L.lsba_ilu0_setup(ctx.ctx, True)
        lu, (nlL, nlU) = L.lsba_copy_ilu0_factors(ctx.ctx, p.col_idx.size)
        X = np.random.default_rng(2).standard_normal((n, p.s))
        Y = ctx.ilu0_apply(dev(X)).cpu().numpy()
    assert nlL == nlU == 2 * 1024 - 1
    M = sp.csr_matrix((lu, p.col_idx, p.row_ptr), shape=(n, n))
    Lf = (sp.tril(M, -1) + sp.eye(n)).tocsr()
    Uf = sp.triu(M).tocsr()
    P = (Lf @ Uf).tocsr()
    A = sp.csr_matrix((p.vals, p.col_idx, p.row_ptr), shape=(n, n))
    rows = np.repeat(np.arange(n), np.diff(p.row_ptr))
    d = np.asarray(P[rows, p.col_idx]).ravel() - p.vals
    assert np.abs(d).max() <= 1e-12 * np.abs(p.vals).max()
    R = Lf @ (Uf @ Y) - X
    assert np.linalg.norm(R) <= 1e-12 * np.linalg.norm(X)


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_level_and_polling_solves_bitwise_equal(L, cfg, monkeypatch):
    """The level-synchronous solve on packed rows (default, LSBA_ILU_SOLVE=1) and the sync-free
    polling solve (LSBA_ILU_SOLVE=0) sum every row's dependencies in CSR order, then divide by
    the pivot: the same arithmetic, so the same bits (and both match the oracle, above)."""
    p = twin(cfg)
    X = np.random.default_rng(100 + cfg).standard_normal((p.n, p.s))
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("LSBA_ILU_SOLVE", mode)
        with L.Context(p.n, p.s, 4, p.row_ptr, p.col_idx, p.vals) as ctx:
            L.lsba_ilu0_setup(ctx.ctx, True)
            out[mode] = ctx.ilu0_apply(dev(X)).cpu().numpy()
    assert np.array_equal(out["1"], out["0"])
