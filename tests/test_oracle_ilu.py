"""Pins of the oracle's ILU(0) left preconditioning (
SPEC.md:512-528 for the interface): every check here is fixed by the mathematics, not by
re-running the oracle's own loops.

  I1  A upper triangular -> L = I, U = A exactly.
  I2  closed form: tridiag(-1, 2, -1) has no fill, so ILU(0) is its exact LU with
      u_ii = (i+1)/i, l_{i+1,i} = -i/(i+1) (1-based; the textbook Thomas recurrence).
  I3  the defining property: (L U)_ij = a_ij on pattern(A) for fixed-seed sparse matrices,
      to 1e-12, with L, U confined to pattern(A).
  I4  the triangular solves equal scipy.sparse.linalg.spsolve_triangular (library routine).
  I5  zero pivots (numerical and structural) raise ZeroPivot.
  I6  A = I -> M = I: the preconditioned operator is A itself.
  I7  exact-factorisation limit: on a no-fill matrix M^{-1} A = I, so the preconditioned solve
      ends after ONE step (the NaN-flag of Omega - H^T H = 0 is the happy breakdown, R7) with
      the exact solution.
  I8  linearity of the preconditioned operator.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import lsba_oracle as O  # noqa: E402


def csr_from_dense(D):
    rp, ci, va = [0], [], []
    for i in range(D.shape[0]):
        nz = np.nonzero(D[i])[0]
        ci.extend(nz.tolist())
        va.extend(D[i, nz].tolist())
        rp.append(len(ci))
    return np.array(rp, np.int64), np.array(ci, np.int64), np.array(va)


def to_dense(rp, ci, va, n):
    D = np.zeros((n, n))
    for i in range(n):
        D[i, ci[rp[i]:rp[i + 1]]] = va[rp[i]:rp[i + 1]]
    return D


def split_LU(F, n):
    LU = to_dense(F.row_ptr, F.col_idx, F.lu, n)
    return np.tril(LU, -1) + np.eye(n), np.triu(LU)


def random_sparse_dd(n, per_row, seed):
    """diagonally dominant random sparse matrix (nonsymmetric pattern)."""
    rng = np.random.default_rng(seed)
    D = np.zeros((n, n))
    for i in range(n):
        cols = rng.choice(n, size=per_row, replace=False)
        D[i, cols] = rng.uniform(-1, 1, size=per_row)
    np.fill_diagonal(D, 0.0)
    np.fill_diagonal(D, 1.5 * np.abs(D).sum(axis=1) + 1.0)
    return D


def test_I1_upper_triangular():
    rng = np.random.default_rng(3)
    D = np.triu(rng.uniform(-1, 1, (40, 40)) * (rng.random((40, 40)) < 0.2)) + 5 * np.eye(40)
    A = csr_from_dense(D)
    F = O.ilu0(*A)
    assert np.array_equal(F.lu, A[2])                   # L = I (no strictly-lower entries), U = A
    L, U = split_LU(F, 40)
    assert np.array_equal(L, np.eye(40)) and np.array_equal(U, D)


def test_I2_tridiag_closed_form():
    n = 200
    D = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    F = O.ilu0(*csr_from_dense(D))
    L, U = split_LU(F, n)
    i = np.arange(1, n + 1, dtype=np.float64)
    np.testing.assert_allclose(np.diag(U), (i + 1) / i, rtol=1e-14)
    np.testing.assert_allclose(np.diag(L, -1), -i[:-1] / (i[:-1] + 1), rtol=1e-14)
    np.testing.assert_array_equal(np.diag(U, 1), -np.ones(n - 1))
    np.testing.assert_allclose(L @ U, D, atol=1e-13)


@pytest.mark.parametrize("n,per_row,seed", [(60, 4, 0), (150, 6, 1), (300, 3, 2)])
def test_I3_pattern_restricted_product(n, per_row, seed):
    D = random_sparse_dd(n, per_row, seed)
    F = O.ilu0(*csr_from_dense(D))
    L, U = split_LU(F, n)
    pat = D != 0
    assert not np.any((L - np.eye(n))[~pat]) and not np.any(U[~pat])     # no fill
    P = L @ U
    np.testing.assert_allclose(P[pat], D[pat], rtol=0, atol=1e-12 * np.abs(D).max())
    # and it is NOT the exact LU when the pattern fills in (the product differs off-pattern)
    assert np.abs(P[~pat]).max() > 1e-6


def test_I3_stencil_twin():
    from lsba_inputs import make_twin
    p = make_twin(3)                                    # convection-diffusion 16^3, 7-point
    F = O.ilu0(p.row_ptr, p.col_idx, p.vals)
    import scipy.sparse as sp
    n = p.n
    M = sp.csr_matrix((F.lu, p.col_idx, p.row_ptr), shape=(n, n))
    L = sp.tril(M, -1) + sp.eye(n)
    U = sp.triu(M)
    P = (L @ U).tocsr()
    A = sp.csr_matrix((p.vals, p.col_idx, p.row_ptr), shape=(n, n))
    rows = np.repeat(np.arange(n), np.diff(p.row_ptr))
    d = np.asarray(P[rows, p.col_idx]).ravel() - np.asarray(A[rows, p.col_idx]).ravel()
    assert np.abs(d).max() <= 1e-12 * np.abs(p.vals).max()


def test_I4_triangular_solves_vs_scipy():
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    from lsba_inputs import make_twin
    for cfg in (2, 3, 4):
        p = make_twin(cfg)
        n = p.n
        F = O.ilu0(p.row_ptr, p.col_idx, p.vals)
        M = sp.csr_matrix((F.lu, p.col_idx, p.row_ptr), shape=(n, n))
        L = (sp.tril(M, -1) + sp.eye(n)).tocsr()
        U = sp.triu(M).tocsr()
        X = np.random.default_rng(cfg).standard_normal((n, 3))
        Y = F.lower_solve(X)
        Yr = sla.spsolve_triangular(L, X, lower=True)
        assert np.abs(Y - Yr).max() <= 1e-13 * np.abs(Yr).max()
        Z = F.upper_solve(Y)
        Zr = sla.spsolve_triangular(U, Yr, lower=False)
        assert np.abs(Z - Zr).max() <= 1e-12 * np.abs(Zr).max()


def test_I5_zero_pivots():
    with pytest.raises(O.ZeroPivot):
        O.ilu0(*csr_from_dense(np.array([[0.0, 1.0], [1.0, 0.0]])))
    # numerically zero pivot produced by the elimination: [[1, 1], [1, 1]] -> u_22 = 0
    with pytest.raises(O.ZeroPivot):
        O.ilu0(*csr_from_dense(np.array([[1.0, 1.0], [1.0, 1.0]])))
    # structurally missing diagonal entry
    rp, ci, va = np.array([0, 2, 3]), np.array([0, 1, 0]), np.array([1.0, 2.0, 3.0])
    with pytest.raises(O.ZeroPivot):
        O.ilu0(rp, ci, va)


def test_I6_identity():
    n = 30
    A = csr_from_dense(np.eye(n))
    F = O.ilu0(*A)
    X = np.random.default_rng(0).standard_normal((n, 2))
    op = O.IluOperator(A, F)
    assert np.array_equal(op(X), X) and np.array_equal(F.solve(X), X)


def test_I7_exact_factorisation_one_step():
    from lsba_inputs import tridiag, tridiag_rhs
    n = 300
    A = tridiag(n)                                      # tridiagonal, no fill
    B = tridiag_rhs(n)
    X, info = O.solve(A, B, m=10, tol=1e-10, max_restarts=5, ip="cl", mod="fom", prec="ilu0")
    assert info.outcome == O.CONVERGED and info.iterations == 1 and info.cycles == 1
    Xs = np.linalg.solve(to_dense(*A, n), B)
    assert np.linalg.norm(X - Xs) <= 1e-10 * np.linalg.norm(Xs)


def test_I8_linearity_and_preconditioned_solve():
    from lsba_inputs import make_twin
    p = make_twin(3)
    A = (p.row_ptr, p.col_idx, p.vals)
    F = O.ilu0(*A)
    op = O.IluOperator(A, F)
    rng = np.random.default_rng(7)
    X, Y = rng.standard_normal((p.n, 2)), rng.standard_normal((p.n, 2))
    np.testing.assert_allclose(op(2.0 * X - 3.0 * Y), 2.0 * op(X) - 3.0 * op(Y), rtol=0,
                               atol=1e-13 * np.abs(op(X)).max())
    # the preconditioned solve reaches tol in the preconditioned norm and needs fewer steps
    Xp, ip_ = O.solve(A, p.B, m=p.m, tol=p.tol, max_restarts=200, ip="cl", mod="gmres", prec=F)
    _, i0 = O.solve(A, p.B, m=p.m, tol=p.tol, max_restarts=200, ip="cl", mod="gmres")
    assert ip_.outcome == O.CONVERGED and ip_.iterations < i0.iterations
    R = F.solve(p.B - O.spmm(*A, Xp))
    assert np.linalg.norm(R) <= p.tol * np.linalg.norm(F.solve(p.B)) * (1 + 1e-9)
