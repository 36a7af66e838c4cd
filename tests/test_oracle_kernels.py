"""Oracle pins for the small kernels: Cholesky-with-flag, SpMM, the Gram, inner products, IO.

Each test pins the oracle to something other than itself: a worked example from SPEC.md,
a textbook/library routine on a special case, exact rational arithmetic, or a Def 2.1 axiom.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import lsba_oracle as O
from lsba_inputs import random_sparse, stencil, tridiag


def test_chol_spec_examples(golden_dir):
    """P1: SPEC.md:51-53 worked examples."""
    cases = json.load(open(os.path.join(golden_dir, "spec_chol_examples.json")))["cases"]
    for c in cases:
        R, flag = O.chol_flag(np.array(c["S"], dtype=float))
        assert flag == c["flag"]
        if not flag:
            np.testing.assert_allclose(R, np.array(c["R"], dtype=float), rtol=0, atol=1e-15)


@pytest.mark.parametrize("s", [1, 2, 4, 8, 16])
def test_chol_matches_lapack_on_spd(s):
    """Special case reducing to a library routine: LAPACK potrf (numpy.linalg.cholesky)."""
    rng = np.random.default_rng(s)
    X = rng.standard_normal((3 * s + 5, s))
    S = X.T @ X
    R, flag = O.chol_flag(S)
    assert not flag
    L = np.linalg.cholesky(S)
    np.testing.assert_allclose(R, L.T, rtol=1e-12, atol=1e-12)
    assert np.all(np.diag(R) > 0) and np.allclose(np.tril(R, -1), 0)


def test_chol_flags_nonpd_nan_inf():
    assert O.chol_flag(np.array([[1.0, 0], [0, 0.0]]))[1]          # semidefinite: pivot 0
    assert O.chol_flag(np.array([[1.0, 0], [0, -1e-300]]))[1]
    assert O.chol_flag(np.array([[np.nan, 0], [0, 1.0]]))[1]
    assert O.chol_flag(np.array([[1.0, np.inf], [np.inf, 1.0]]))[1]
    assert not O.chol_flag(np.array([[1e-300, 0], [0, 1e-300]]))[1]  # no relative threshold (R2)


def _dense(row_ptr, col_idx, vals, n):
    D = np.zeros((n, n))
    for i in range(n):
        for p in range(row_ptr[i], row_ptr[i + 1]):
            D[i, col_idx[p]] += vals[p]
    return D


@pytest.mark.parametrize("s", [1, 2, 3, 8, 16])
def test_spmm_vs_dense_random_csr_with_empty_rows(s):
    """Brute force: a dense matmul on a random CSR with empty and ragged rows."""
    rng = np.random.default_rng(7 + s)
    n = 57
    counts = rng.integers(0, 9, size=n)
    counts[[0, 5, 56]] = 0
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    cols = np.concatenate([np.sort(rng.choice(n, size=c, replace=False)) for c in counts]).astype(np.int32)
    vals = rng.standard_normal(row_ptr[-1])
    O.csr_check(n, row_ptr, cols, vals)
    V = rng.standard_normal((n, s))
    W = O.spmm(row_ptr, cols, vals, V, chunk_rows=13)
    np.testing.assert_allclose(W, _dense(row_ptr, cols, vals, n) @ V, rtol=1e-13, atol=1e-13)
    assert np.all(W[[0, 5, 56]] == 0)


def test_spmm_stencil_and_tridiag_rows():
    rp, ci, va = stencil(2, 4)                       # 2D Laplacian 4/-1
    D = _dense(rp, ci, va, 16)
    assert np.allclose(D, D.T) and np.allclose(np.diag(D), 4)
    assert D.sum(axis=1).max() == 2 and D.sum(axis=1).min() == 0   # corners / interior
    rp, ci, va = tridiag(3)                          # tridiag(3) e1 -> (-1, 1, 0)
    W = O.spmm(rp, ci, va, np.array([[1.0], [0.0], [0.0]]))
    np.testing.assert_array_equal(W[:, 0], [-1.0, 1.0, 0.0])


def test_csr_check_rejects_bad_input():
    rp = np.array([0, 2, 3], dtype=np.int64)
    with pytest.raises(ValueError):
        O.csr_check(2, rp, np.array([1, 0, 1], dtype=np.int32), np.ones(3))   # unsorted
    with pytest.raises(ValueError):
        O.csr_check(2, rp, np.array([0, 0, 1], dtype=np.int32), np.ones(3))   # duplicate
    with pytest.raises(ValueError):
        O.csr_check(2, rp, np.array([0, 2, 1], dtype=np.int32), np.ones(3))   # out of range
    with pytest.raises(ValueError):
        O.csr_check(2, np.array([0, 3, 2]), np.array([0, 1, 1], dtype=np.int32), np.ones(3))
    O.csr_check(2, rp, np.array([0, 1, 1], dtype=np.int32), np.ones(3))


def test_random_sparse_recipe():
    rp, ci, va = random_sparse(4096)
    n = 4096
    O.csr_check(n, rp, ci, va)
    assert np.all(np.diff(rp) == 16)
    rows = np.repeat(np.arange(n), 16)
    diag = ci == rows
    assert diag.sum() == n
    off = np.abs(va[~diag]).reshape(n, 15).sum(axis=1)
    np.testing.assert_allclose(va[diag], 1.1 * off, rtol=1e-15)
    band = (np.abs(ci.astype(np.int64) - rows) <= 64) & ~diag
    assert np.all(band.reshape(n, 16).sum(axis=1) >= 7)


def test_gram_near_exact_vs_rationals():
    """The extended-precision Gram equals the exactly-rounded X^T Y (Fractions) to <= 1 ulp
    on an ill-conditioned (cancelling) sum where plain fp64 is far off."""
    rng = np.random.default_rng(3)
    n = 2000
    x = rng.standard_normal(n) * 10.0 ** rng.integers(-8, 9, size=n)
    y = rng.standard_normal(n)
    X = np.stack([x, -x[::-1], x * 3], axis=1)
    Y = np.stack([y, y[::-1] * 1e-3], axis=1)
    G = O.gram(X, Y)
    G2 = O.gram_dot2(X, Y)
    for a in range(3):
        for b in range(2):
            exact = sum(Fraction(float(X[i, a])) * Fraction(float(Y[i, b])) for i in range(n))
            ref = float(exact)
            assert abs(G[a, b] - ref) <= 2 * np.spacing(abs(ref)) + 1e-300
            assert abs(G2[a, b] - ref) <= 2 * np.spacing(abs(ref)) + 1e-300


@pytest.mark.parametrize("ip", ["cl", "gl"])
def test_block_inner_product_axioms(ip):
    """P2: Def 2.1: S-linearity, symmetry, definiteness."""
    rng = np.random.default_rng(11)
    n, s = 200, 4
    X, Y, Z = (rng.standard_normal((n, s)) for _ in range(3))
    if ip == "cl":
        C = rng.standard_normal((s, s))
        lhs = O.ip_cl([X + Y], Z @ C)
        rhs = O.ip_cl([X], Z) @ C + O.ip_cl([Y], Z) @ C
        np.testing.assert_allclose(lhs, rhs, rtol=1e-12, atol=1e-11)
        np.testing.assert_allclose(O.ip_cl([X], Y), O.ip_cl([Y], X).T, rtol=1e-15)
        assert np.all(np.linalg.eigvalsh(O.ip_cl([X], X)) > 0)
    else:
        c = 1.7
        lhs = O.ip_gl([X + Y], Z * c)[0]
        assert math.isclose(lhs, (O.ip_gl([X], Z)[0] + O.ip_gl([Y], Z)[0]) * c, rel_tol=1e-12)
        assert O.ip_gl([X], Y)[0] == O.ip_gl([Y], X)[0]
        assert O.ip_gl([X], X)[0] > 0
    assert np.all(O.ip_cl([np.zeros((n, s))], np.zeros((n, s))) == 0)


def test_global_is_mean_of_classical_diagonal():
    """P2: the global block inner product is the mean of the classical
    block's diagonal."""
    rng = np.random.default_rng(5)
    X, Y = rng.standard_normal((300, 6)), rng.standard_normal((300, 6))
    assert math.isclose(O.ip_gl([X], Y)[0], np.trace(O.ip_cl([X], Y)) / 6, rel_tol=1e-14)


@pytest.mark.parametrize("ip", ["cl", "gl"])
def test_intra_ortho_scaling_quotient(ip):
    """P2 / Def 2.2: X = Q N(X) and <Q,Q> = I."""
    rng = np.random.default_rng(2)
    X = rng.standard_normal((500, 5))
    if ip == "cl":
        Q, R, flag = O.io_cl(X)
        assert not flag
        np.testing.assert_allclose(Q @ R, X, atol=1e-13)
        np.testing.assert_allclose(O.ip_cl([Q], Q), np.eye(5), atol=1e-14)
        # same R as a Householder QR with positive diagonal (library special case)
        Rq = np.linalg.qr(X, mode="r")
        Rq = np.diag(np.sign(np.diag(Rq))) @ Rq
        np.testing.assert_allclose(R, Rq, rtol=1e-12, atol=1e-12)
    else:
        Q, beta, flag = O.io_gl(X)
        assert not flag
        assert math.isclose(beta, np.linalg.norm(X) / math.sqrt(5), rel_tol=1e-15)
        assert math.isclose(O.ip_gl([Q], Q)[0], 1.0, rel_tol=1e-14)
    assert O.io_cl(np.zeros((10, 2)))[2] and O.io_gl(np.zeros((10, 2)))[2]


@pytest.mark.parametrize("ip", ["cl", "gl"])
@pytest.mark.parametrize("c", [0.0, 1e-9, 0.3, -0.45, 0.9])
def test_loss_of_orthogonality_closed_form(ip, c):
    """Eq loo, ||I - <Q,Q>||_2, on bases with a prescribed Gram matrix.
    (a) two blocks V_1 (orthonormal) and V_2 = V_1 cos(t) + P sin(t), P orthonormal and
        orthogonal to V_1: <Q,Q> = [[I, c I], [c I, I]], so LOO = |c|, c = cos(t);
    (b) three blocks with pairwise block inner product c I: <Q,Q> = ((1-c) I + c 1 1^T) (x) I_s,
        I - <Q,Q> = -c (1 1^T - I) (x) I_s with eigenvalues -2c and c: LOO = 2|c|;
    (c) one block scaled by a: LOO = |1 - a^2|.
    Both inner products give the same value (global: (1/s) tr of each s x s block)."""
    n, s = 400, 3
    rng = np.random.default_rng(17)
    U, _ = np.linalg.qr(rng.standard_normal((n, 4 * s)))
    blk = [U[:, i * s:(i + 1) * s] for i in range(4)]
    t = math.acos(c)
    V2 = blk[0] * c + blk[1] * math.sin(t)
    assert math.isclose(O.loss_of_orthogonality([blk[0], V2], ip), abs(c), rel_tol=1e-10, abs_tol=1e-14)
    Gt = (1 - c) * np.eye(3) + c * np.ones((3, 3))
    Lc = np.linalg.cholesky(Gt)                         # Gt = Lc Lc^T
    Vs = [sum(blk[q] * Lc[i, q] for q in range(3)) for i in range(3)]   # <V_i, V_j> = Gt_ij I
    assert math.isclose(O.loss_of_orthogonality(Vs, ip), 2 * abs(c), rel_tol=1e-10, abs_tol=1e-14)
    a = 1.0 + c / 3
    assert math.isclose(O.loss_of_orthogonality([a * blk[2]], ip), abs(1 - a * a), rel_tol=1e-10,
                        abs_tol=1e-14)
