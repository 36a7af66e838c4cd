"""ORACLE for the low-sync block Arnoldi hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import or execute anything under ``oracle/``.  The product path
(``paper_2208_09899_b200``) never imports it and fails loudly without its CUDA library.

What this is: a plain, slow, obviously-correct NumPy fp64 implementation of what the
paper's method computes, written in the paper's order and notation (Lund, arXiv 2208.09899,
/root/reference/PAPER.md; "PAPER.md:L" below is a line of that file):

* BCGS-PIP-Arnoldi, Alg 3, for the classical and global block inner
  products of Table 1;
* the CholQR / global intra-orthogonalisation ``IO`` used at line 1;
* the modified BFOM / BGMRES projected problem (Eq (Xm)), the cospatial
  residual relation and its norm (Thm 2.4), and restarts
  X^(2) = X_m + D_m;
* the adaptive restart of Sec 4 (NaN-flag: restart from the last safe block and reduce m,
  PAPER.md:405) plus this build's condition-threshold trigger (reading R8);
* BMGS-Arnoldi, Alg 2, used only as an independent cross-check (pin P5).

No blocking, fusion or reordering beyond what the paper states.  Library primitives used as
steps: ``numpy.linalg.solve`` (a textbook LU for the ks x ks projected systems) and
``numpy.linalg.inv`` for kappa_F on (k+1)s x (k+1)s triangular matrices.  The Gram
(block inner product) is accumulated in x87 80-bit extended precision (or, if the host has
no extended ``longdouble``, with Ogita-Rump-Oishi Dot2 compensated summation) so that it is
near-exactly rounded — the "parity note" of SURVEY.md 8(c) / DESIGN.md reading R23.

Readings where the paper is silent (R1..R23) are listed in DESIGN.md; each is cited inline.
Parity pins live in tests/test_oracle_*.py.  Functions without a pin say so.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --------------------------------------------------------------------------------------
# Sparse operator application (W = A V_k)
# --------------------------------------------------------------------------------------


def csr_check(n: int, row_ptr, col_idx, vals) -> None:
    """CSR invariants: row_ptr[0]=0, monotone, row_ptr[n]=nnz,
    columns in range and strictly increasing within each row.  Raises ValueError."""
    row_ptr = np.asarray(row_ptr)
    col_idx = np.asarray(col_idx)
    if row_ptr.shape != (n + 1,) or row_ptr[0] != 0:
        raise ValueError("row_ptr must have length n+1 and start at 0")
    if np.any(np.diff(row_ptr) < 0):
        raise ValueError("row_ptr not monotone")
    nnz = int(row_ptr[-1])
    if col_idx.shape != (nnz,) or np.asarray(vals).shape != (nnz,):
        raise ValueError("col_idx/vals length != nnz")
    if nnz and (col_idx.min() < 0 or col_idx.max() >= n):
        raise ValueError("column index out of range")
    if nnz > 1:
        inc = np.diff(col_idx.astype(np.int64))
        starts = row_ptr[1:-1]
        same_row = np.ones(nnz - 1, dtype=bool)
        same_row[starts[(starts > 0) & (starts < nnz)] - 1] = False
        if np.any(inc[same_row] <= 0):
            raise ValueError("columns not strictly increasing within a row")


def spmm(row_ptr, col_idx, vals, V, chunk_rows: int = 1 << 16) -> np.ndarray:
    """W = A V for CSR A and a row-major n x s block vector V (Alg 3 line 3).

    Explicit gather-and-accumulate: W[i,:] = sum_{p in row i} vals[p] * V[col_idx[p], :],
    summed in CSR order within each row (np.add.reduceat is a left-to-right loop)."""
    n = len(row_ptr) - 1
    V = np.asarray(V, dtype=np.float64)
    W = np.zeros((n, V.shape[1]))
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        p0, p1 = int(row_ptr[r0]), int(row_ptr[r1])
        if p1 == p0:
            continue
        contrib = vals[p0:p1, None] * V[col_idx[p0:p1]]
        starts = np.asarray(row_ptr[r0:r1], dtype=np.int64) - p0
        nonempty = np.diff(np.asarray(row_ptr[r0:r1 + 1])) > 0
        W[r0:r1][nonempty] = np.add.reduceat(contrib, starts[nonempty], axis=0)
    return W


# --------------------------------------------------------------------------------------
# ILU(0) left preconditioning ("an incomplete LU (ILU)
# preconditioner with no fill"; SPEC.md:512-528 for the interface and the side: LEFT, with
# every residual and tolerance in the preconditioned norm — DESIGN.md reading R28)
# --------------------------------------------------------------------------------------


class ZeroPivot(ValueError):
    """ILU(0) met a zero (or missing) pivot: the problem is reported unpreconditionable."""


@dataclass
class Ilu0Factors:
    """L (unit lower, strictly-lower entries) and U (upper incl. diagonal) stored together in
    the pattern of A: ``lu[p]`` for CSR position p (same row_ptr / col_idx as A)."""
    row_ptr: np.ndarray
    col_idx: np.ndarray
    lu: np.ndarray
    diag: np.ndarray          # CSR position of a_ii per row
    _plans: dict = field(default_factory=dict, repr=False)

    def lower_solve(self, X):
        """Y with L Y = X (unit diagonal): y_i = x_i - sum_{k<i} l_ik y_k (CSR order)."""
        return _tri_solve(self, X, lower=True)

    def upper_solve(self, Y):
        """Z with U Z = Y: z_i = (y_i - sum_{j>i} u_ij z_j) / u_ii (CSR order)."""
        return _tri_solve(self, Y, lower=False)

    def solve(self, X):
        """M^{-1} X = U^{-1} L^{-1} X."""
        return self.upper_solve(self.lower_solve(X))


def ilu0(row_ptr, col_idx, vals) -> Ilu0Factors:
    """ILU(0), the IKJ variant (Saad, Iterative Methods, Alg 10.4) restricted to pattern(A):
        for i = 2..n, for k < i with a_ik in the pattern (ascending):
            a_ik = a_ik / a_kk
            for j > k with a_ij in the pattern:  a_ij = a_ij - a_ik a_kj   (if a_kj is too)
    Zero or structurally missing pivot -> ZeroPivot.  Plain row loops."""
    n = len(row_ptr) - 1
    row_ptr = np.asarray(row_ptr, dtype=np.int64)
    col_idx = np.asarray(col_idx, dtype=np.int64)
    a = np.array(vals, dtype=np.float64)
    pos = []
    diag = np.full(n, -1, dtype=np.int64)
    for i in range(n):
        cols = col_idx[row_ptr[i]:row_ptr[i + 1]].tolist()
        pos.append({c: row_ptr[i] + t for t, c in enumerate(cols)})
        if i in pos[i]:
            diag[i] = pos[i][i]
    if np.any(diag < 0):
        raise ZeroPivot(f"structurally missing diagonal in row {int(np.argmax(diag < 0))}")
    for i in range(n):
        p0, p1 = int(row_ptr[i]), int(row_ptr[i + 1])
        for p in range(p0, p1):
            k = int(col_idx[p])
            if k >= i:
                break
            piv = a[diag[k]]
            if piv == 0.0 or not math.isfinite(piv):
                raise ZeroPivot(f"zero pivot u_{k}{k}")
            a[p] = a[p] / piv
            rk = pos[k]
            for q in range(p + 1, p1):
                r = rk.get(int(col_idx[q]))
                if r is not None:
                    a[q] = a[q] - a[p] * a[r]
        if a[diag[i]] == 0.0 or not math.isfinite(a[diag[i]]):
            raise ZeroPivot(f"zero pivot u_{i}{i}")
    return Ilu0Factors(row_ptr, col_idx, a, diag)


def _tri_plan(F: Ilu0Factors, lower: bool):
    """Level sets of the triangular factor (rows whose dependencies are all in earlier levels)
    and, per level, the off-diagonal CSR positions in CSR order.  Evaluating a level's rows
    together changes no row's arithmetic (each row sums its own terms in CSR order)."""
    if lower in F._plans:
        return F._plans[lower]
    rp, ci = F.row_ptr, F.col_idx
    n = len(rp) - 1
    lev = np.zeros(n, dtype=np.int64)
    rows = range(n) if lower else range(n - 1, -1, -1)
    for i in rows:
        cols = ci[rp[i]:rp[i + 1]]
        dep = cols[cols < i] if lower else cols[cols > i]
        lev[i] = 1 + int(lev[dep].max()) if dep.size else 0
    plan = []
    for L in range(int(lev.max()) + 1 if n else 0):
        R = np.nonzero(lev == L)[0]
        ps, starts, nz_rows = [], [], []
        for i in R:
            seg = np.arange(rp[i], rp[i + 1])
            seg = seg[ci[seg] < i] if lower else seg[ci[seg] > i]
            if seg.size:
                starts.append(sum(len(x) for x in ps))
                ps.append(seg)
                nz_rows.append(i)
        plan.append((R, np.concatenate(ps) if ps else np.zeros(0, np.int64),
                     np.array(starts, np.int64), np.array(nz_rows, np.int64)))
    F._plans[lower] = plan
    return plan


def _tri_solve(F: Ilu0Factors, X, lower: bool):
    X = np.asarray(X, dtype=np.float64)
    Y = X.copy()
    for R, ps, starts, nz_rows in _tri_plan(F, lower):
        if ps.size:
            contrib = F.lu[ps][:, None] * Y[F.col_idx[ps]]
            Y[nz_rows] = Y[nz_rows] - np.add.reduceat(contrib, starts, axis=0)
        if not lower:
            Y[R] = Y[R] / F.lu[F.diag[R]][:, None]
    return Y


class IluOperator:
    """The left-preconditioned operator X -> U^{-1} L^{-1} (A X)."""

    def __init__(self, A, factors: Ilu0Factors):
        self.A = A
        self.F = factors

    def __call__(self, V):
        return self.F.solve(spmm(*self.A, V))


def apply_A(A, V):
    """The operator of the Krylov method: A V for a CSR triple, M^{-1} A V for an IluOperator."""
    if isinstance(A, IluOperator):
        return A(V)
    return spmm(*A, V)


# --------------------------------------------------------------------------------------
# Near-exactly-rounded Gram  X^T Y  (parity note; R23)
# --------------------------------------------------------------------------------------

_LD = np.longdouble
HAVE_EXTENDED = bool(np.finfo(_LD).eps < 1e-18)


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _two_prod(a, b):
    p = a * b
    return p, np.fma(a, b, -p) if hasattr(np, "fma") else _dekker_err(a, b, p)


def _dekker_err(a, b, p):
    f = 134217729.0  # 2^27 + 1 (Veltkamp split)
    ca = f * a
    ah = ca - (ca - a)
    al = a - ah
    cb = f * b
    bh = cb - (cb - b)
    bl = b - bh
    return al * bl - (((p - ah * bh) - al * bh) - ah * bl)


def gram_dot2(X, Y, chunk_rows: int = 4096) -> np.ndarray:
    """X^T Y with Dot2 (Ogita, Rump, Oishi 2005) compensated fp64 accumulation:
    error-free products, a TwoSum cascade over rows; result as accurate as if computed
    in twice the working precision, then rounded."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    p, q = X.shape[1], Y.shape[1]
    S = np.zeros((p, q))
    C = np.zeros((p, q))
    for r0 in range(0, X.shape[0], chunk_rows):
        xs = X[r0:r0 + chunk_rows]
        ys = Y[r0:r0 + chunk_rows]
        for i in range(xs.shape[0]):
            pr, e = _two_prod(xs[i][:, None], ys[i][None, :])
            S, e2 = _two_sum(S, pr)
            C += e + e2
    return S + C


def gram(X, Y, chunk_rows: int = 1 << 15) -> np.ndarray:
    """Near-exactly rounded X^T Y (p x q) for X (n x p), Y (n x q)."""
    X = np.asarray(X, dtype=np.float64)
    Y = np.asarray(Y, dtype=np.float64)
    if not HAVE_EXTENDED:
        return gram_dot2(X, Y)
    acc = np.zeros((X.shape[1], Y.shape[1]), dtype=_LD)
    for r0 in range(0, X.shape[0], chunk_rows):
        xs = X[r0:r0 + chunk_rows].astype(_LD)
        ys = Y[r0:r0 + chunk_rows].astype(_LD)
        acc += xs.T @ ys
    return acc.astype(np.float64)


# --------------------------------------------------------------------------------------
# Block inner products and scaling quotients (Table 1)
# --------------------------------------------------------------------------------------


def ip_cl(Xs, Y) -> np.ndarray:
    """Classical <[X_1..X_p], Y> = [X_1..X_p]^T Y, a (p s) x s matrix (Table 1 row cl)."""
    Xcat = np.concatenate([np.asarray(x) for x in Xs], axis=1)
    return gram(Xcat, Y)


def ip_gl(Xs, Y) -> np.ndarray:
    """Global <X_j, Y> = (1/s) tr(X_j^T Y) I_s, returned as the p scalars (Table 1 row gl)."""
    s = Y.shape[1]
    y = np.asarray(Y, dtype=np.float64).reshape(-1, 1)
    out = np.empty(len(Xs))
    for j, x in enumerate(Xs):
        out[j] = gram(np.asarray(x, dtype=np.float64).reshape(-1, 1), y)[0, 0] / s
    return out


def sym(S: np.ndarray) -> np.ndarray:
    """Symmetrise: (S + S^T)/2 (reading R2)."""
    return 0.5 * (S + S.T)


def chol_flag(S: np.ndarray):
    """Upper Cholesky S = R^T R with a breakdown flag (Alg 3 line 5; "NaN-flag",
    PAPER.md:386, 405).  Reading R2: the input is symmetrised first; flag iff some pivot
    d_j = S_jj - sum_{i<j} R_ij^2 is not > 0 (so NaN/Inf also flag); no relative threshold
    (LAPACK dpotrf semantics).  Returns (R, flag); R is undefined when flag is True."""
    S = sym(np.asarray(S, dtype=np.float64))
    s = S.shape[0]
    R = np.zeros((s, s))
    for j in range(s):
        d = S[j, j] - sum(R[i, j] * R[i, j] for i in range(j))
        if not (d > 0.0) or not math.isfinite(d):
            return R, True
        R[j, j] = math.sqrt(d)
        for c in range(j + 1, s):
            R[j, c] = (S[j, c] - sum(R[i, j] * R[i, c] for i in range(j))) / R[j, j]
    if not np.all(np.isfinite(R)):
        return R, True
    return R, False


def right_trsm_upper(Y: np.ndarray, R: np.ndarray) -> np.ndarray:
    """Solve X R = Y for X, R upper triangular (column by column, written out)."""
    X = np.empty_like(Y, dtype=np.float64)
    for j in range(R.shape[0]):
        acc = Y[:, j].copy()
        for i in range(j):
            acc -= X[:, i] * R[i, j]
        X[:, j] = acc / R[j, j]
    return X


def io_cl(U: np.ndarray):
    """CholQR muscle (Alg 3 line 1 PAPER.md:265): G = <U,U> (one sync),
    R = chol(G), V = U R^{-1}.  Returns (V, R, flag)."""
    G = ip_cl([U], U)
    R, flag = chol_flag(G)
    if flag:
        return None, R, True
    return right_trsm_upper(U, R), R, False


def io_gl(U: np.ndarray):
    """Global muscle: N(U) = (1/sqrt(s)) ||U||_F (Table 1 row gl; reading R14).
    Returns (V, beta, flag) with V = U / beta; flag iff beta^2 is not > 0 (R3)."""
    b2 = ip_gl([U], U)[0]
    if not (b2 > 0.0) or not math.isfinite(b2):
        return None, 0.0, True
    beta = math.sqrt(b2)
    return U / beta, beta, False


# --------------------------------------------------------------------------------------
# One BCGS-PIP block Arnoldi step (Alg 3)
# --------------------------------------------------------------------------------------


@dataclass
class StepResult:
    Hcol: np.ndarray          # H_{1:k,k}  (k s x s classical; k scalars global)
    R: object                 # H_{k+1,k}  (s x s upper triangular classical; scalar global)
    V_next: np.ndarray | None  # V_{k+1}, None on flag
    flag: bool
    W: np.ndarray


def pip_step(A, Vs, ip: str, force_flag: bool = False) -> StepResult:
    """Lines 3-6 of Alg 3 for step k = len(Vs):
        W = A V_k;  [H_{1:k,k}; Omega] = <[V_k W], W>;  H_{k+1,k} = chol(Omega - H^* H);
        V_{k+1} = (W - V_k H_{1:k,k}) H_{k+1,k}^{-1}.
    Reading R1: Sec 3.1's "W - W H" is read as W - V_k H (line 6).
    Global (R3): H_{k+1,k} = sqrt(omega - sum_j h_j^2) I_s, flag iff radicand not > 0."""
    k = len(Vs)
    W = apply_A(A, Vs[-1])
    s = W.shape[1]
    if ip == "cl":
        G = ip_cl(list(Vs) + [W], W)                  # ONE call: the step's single sync
        Hcol, Omega = G[: k * s], G[k * s:]
        R, flag = chol_flag(Omega - Hcol.T @ Hcol)
        flag = flag or force_flag
        if flag:
            return StepResult(Hcol, R, None, True, W)
        P = W - np.concatenate(list(Vs), axis=1) @ Hcol          # W - V_k H_{1:k,k} (line 6)
        return StepResult(Hcol, R, right_trsm_upper(P, R), False, W)
    g = ip_gl(list(Vs) + [W], W)
    Hcol, omega = g[:k], g[k]
    rad = omega - float(np.dot(Hcol, Hcol))
    flag = (not (rad > 0.0)) or (not math.isfinite(rad)) or force_flag
    if flag:
        return StepResult(Hcol, float("nan"), None, True, W)
    r = math.sqrt(rad)
    P = W.copy()
    for j in range(k):
        P -= Vs[j] * Hcol[j]
    return StepResult(Hcol, r, P / r, False, W)


class PipArnoldi:
    """Alg 3 as a resumable object (exposes ``begin`` and ``step`` for step parity tests).

    State: the basis list ``V`` (V_1..V_{k+1}), the block Hessenberg ``Hbar``
    ((m+1)b x m b, b = s classical, 1 global) and ``beta`` (B = V_1 beta)."""

    def __init__(self, A, ip: str, m_max: int, s: int):
        self.A, self.ip, self.m_max, self.s = A, ip, m_max, s
        self.b = s if ip == "cl" else 1
        self.V: list[np.ndarray] = []
        self.Hbar = np.zeros(((m_max + 1) * self.b, m_max * self.b))
        self.beta = None
        self.k = 0

    def begin(self, B):
        """Line 1: [V_1, beta] = IO(B).  Returns flag."""
        if self.ip == "cl":
            V1, beta, flag = io_cl(B)
        else:
            V1, beta, flag = io_gl(B)
            beta = np.array([[beta]])
        self.V = [] if flag else [V1]
        self.beta = beta
        self.k = 0
        self.Hbar[:] = 0.0
        return flag

    def step(self, force_flag: bool = False) -> StepResult:
        res = pip_step(self.A, self.V, self.ip, force_flag)
        k, b = len(self.V), self.b
        Hcol = res.Hcol.reshape(k * b, b) if self.ip == "cl" else np.asarray(res.Hcol).reshape(k, 1)
        self.Hbar[: k * b, (k - 1) * b: k * b] = Hcol
        if not res.flag:
            Rm = res.R if self.ip == "cl" else np.array([[res.R]])
            self.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b] = Rm
            self.V.append(res.V_next)
            self.k = k
        return res


# --------------------------------------------------------------------------------------
# BMGS-CWY / BMGS-ICWY-Arnoldi, Alg 6, Sec 3.3 — the NEXT skeleton (§8(f) f1)
# --------------------------------------------------------------------------------------


class CwyArnoldi:
    """Alg 6 as a resumable object with the same interface as PipArnoldi.

    Alg 6 lags the normalisation by one iteration: loop iteration i >= 2 applies A to the
    unnormalised U (= V_i H_{i,i-1}), computes ONE block inner product
    [Y Z; Omega Pt] = <[V_1..V_{i-1} U], [U W]>, H_{i,i-1} = chol(Omega),
    P = H_{i,i-1}^{-*} Pt, the new block column of T (CWY: -T Y H^{-1}; ICWY: Y H^{-1}), the
    column H_{1:i,i} = T^* [Z; P] H^{-1} (CWY) or T^{-*} [Z; P] H^{-1} (ICWY), V_i = U H^{-1}
    and U = W H^{-1} - V_i-stack H_{1:i,i}.  Iteration 1 (W = A V_1,
    H_11 = <V_1, W>, U = W - V_1 H_11) is done by ``begin`` after IO, so ``step`` number k is
    Alg 6 iteration k+1: it completes Hessenberg column k (its subdiagonal H_{k+1,k}) and
    returns V_{k+1}.  Reading R24: Alg 6 line 15 writes V_{k-1} H_{1:k,k}; the k blocks of
    H_{1:k,k} need V_1..V_k (V_k set on line 14 of the same iteration), so it is read as the
    k-block stack.  Per cycle: m+1 A-applications and m+2 syncs (Table 1 PAPER.md:109-118;
    tridiag table).  Global inner product: scalars, chol = sqrt (R3)."""

    def __init__(self, A, ip: str, m_max: int, s: int, inverse: bool = False):
        self.A, self.ip, self.m_max, self.s = A, ip, m_max, s
        self.inverse = inverse                       # False: CWY, True: ICWY
        self.b = s if ip == "cl" else 1
        self.V: list[np.ndarray] = []
        self.Hbar = np.zeros(((m_max + 1) * self.b, m_max * self.b))
        self.T = np.eye((m_max + 1) * self.b)
        self.beta = None
        self.U = None
        self.k = 0

    def _ip(self, Xs, Y):
        if self.ip == "cl":
            return ip_cl(Xs, Y)
        return ip_gl(Xs, Y).reshape(-1, 1)

    def _mul(self, X, C):
        return X @ C if self.ip == "cl" else X * C[0, 0]

    def begin(self, B):
        """IO(B) (line 2), U = V_1 (line 3), and loop iteration 1 (lines 5-8)."""
        b = self.b
        if self.ip == "cl":
            V1, beta, flag = io_cl(B)
        else:
            V1, beta, flag = io_gl(B)
            beta = np.array([[beta]])
        self.beta = beta
        self.Hbar[:] = 0.0
        self.T = np.eye((self.m_max + 1) * b)
        self.k = 0
        if flag:
            self.V = []
            return flag
        self.V = [V1]
        W = apply_A(self.A, V1)                                # line 5
        H11 = self._ip([V1], W)                                # line 7 (its own sync)
        self.Hbar[:b, :b] = H11
        self.U = W - self._mul(V1, H11)                        # line 8
        return False

    def step(self, force_flag: bool = False) -> StepResult:
        """Alg 6 iteration k+1 for Arnoldi step k = len(V)."""
        b, k = self.b, len(self.V)
        Hcol = self.Hbar[: k * b, (k - 1) * b: k * b].copy()
        U = self.U
        W = apply_A(self.A, U)                                 # line 5
        G = self._ip(list(self.V) + [U], np.concatenate([U, W], axis=1)) if self.ip == "cl" else None
        if self.ip == "cl":
            s = self.s
            Y, Z = G[: k * s, :s], G[: k * s, s:]
            Omega, Pt = G[k * s:, :s], G[k * s:, s:]           # line 10: ONE block inner product
            R, flag = chol_flag(Omega)                         # line 11
        else:
            gU = ip_gl(list(self.V) + [U], U)
            gW = ip_gl(list(self.V) + [U], W)
            Y, Z = gU[:k].reshape(-1, 1), gW[:k].reshape(-1, 1)
            Omega, Pt = gU[k], gW[k]
            flag = not (Omega > 0.0) or not math.isfinite(Omega)
            R = np.array([[math.sqrt(Omega)]]) if not flag else np.array([[float("nan")]])
        flag = flag or force_flag
        if flag:
            return StepResult(Hcol, R if self.ip == "cl" else float("nan"), None, True, W)
        Rinv = right_trsm_upper(np.eye(b), R)                  # H_{k+1,k}^{-1}
        P = np.linalg.solve(R.T, Pt) if self.ip == "cl" else np.array([[Pt / R[0, 0]]])   # line 12
        T = self.T
        YR = Y @ Rinv
        if self.inverse:
            T[: k * b, k * b:(k + 1) * b] = YR                 # line 13 (ICWY)
        else:
            T[: k * b, k * b:(k + 1) * b] = -T[: k * b, : k * b] @ YR   # line 13 (CWY)
        ZP = np.vstack([Z, P]) @ Rinv
        Tk = T[:(k + 1) * b, :(k + 1) * b]
        Hnext = np.linalg.solve(Tk.T, ZP) if self.inverse else Tk.T @ ZP   # line 14
        Vn = self._mul(U, Rinv)                                # line 16: V_{k+1} = U H^{-1}
        self.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b] = R
        if k < self.m_max:
            self.Hbar[:(k + 1) * b, k * b:(k + 1) * b] = Hnext
        self.V.append(Vn)
        # line 17: U = W H^{-1} - [V_1..V_{k+1}] H_{1:k+1,k+1}  (reading R24)
        Un = self._mul(W, Rinv)
        for j, Vj in enumerate(self.V):
            Un = Un - self._mul(Vj, Hnext[j * b:(j + 1) * b])
        self.U = Un
        self.k = k
        return StepResult(Hcol, R if self.ip == "cl" else float(R[0, 0]), Vn, False, W)


class IrolsArnoldi(CwyArnoldi):
    """BCGS-IRO-LS-Arnoldi, Alg 7: the block DCGS2 — the same lagged loop and
    single block inner product <[V_1..V_k U], [U W]> as Alg 6, with the re-orthogonalisation
    folded into it: Omega = Omega~ - Y^* Y, H_{k+1,k} = chol(Omega), column k finalised as
    H_{1:k,k} = J + Y, P = H^{-*}(P~ - Y^* Z), J = ([Z; P] - H_{1:k+1,1:k} Y) H^{-1},
    V_{k+1} = (U - V Y) H^{-1}, U = (W - [V_1..V_{k+1}] [Z; P]) H^{-1}.  (Step k = loop
    iteration k+1, as in CwyArnoldi; J is the tentative next column.)  Per cycle m+1
    A-applications, m+2 syncs and 4 block evaluations per step."""

    def begin(self, B):
        flag = super().begin(B)
        if not flag:
            self.J = self.Hbar[: self.b, : self.b].copy()      # line 6: J = <U, W>, H_11 = J
        return flag

    def step(self, force_flag: bool = False) -> StepResult:
        b, k = self.b, len(self.V)
        U = self.U
        W = apply_A(self.A, U)                                 # line 4
        if self.ip == "cl":
            s = self.s
            G = ip_cl(list(self.V) + [U], np.concatenate([U, W], axis=1))   # line 10: one sync
            Y, Z = G[: k * s, :s], G[: k * s, s:]
            Om_t, Pt = G[k * s:, :s], G[k * s:, s:]
            R, flag = chol_flag(Om_t - Y.T @ Y)                # lines 11-12
        else:
            gU = ip_gl(list(self.V) + [U], U)
            gW = ip_gl(list(self.V) + [U], W)
            Y, Z = gU[:k].reshape(-1, 1), gW[:k].reshape(-1, 1)
            om = gU[k] - float(Y[:, 0] @ Y[:, 0])
            Pt = np.array([[gW[k]]])
            flag = not (om > 0.0) or not math.isfinite(om)
            R = np.array([[math.sqrt(om)]]) if not flag else np.array([[float("nan")]])
        Hcol = self.J + Y                                      # line 13: column k final
        self.Hbar[: k * b, (k - 1) * b: k * b] = Hcol
        flag = bool(flag) or force_flag
        if flag:
            return StepResult(Hcol, R if self.ip == "cl" else float("nan"), None, True, W)
        Rinv = right_trsm_upper(np.eye(b), R)
        P = np.linalg.solve(R.T, Pt - Y.T @ Z)                 # line 14
        self.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b] = R
        Hk = self.Hbar[:(k + 1) * b, : k * b]                  # H_{1:k+1,1:k}
        ZP = np.vstack([Z, P])
        self.J = (ZP - Hk @ Y) @ Rinv                          # line 15
        Vn = self._mul(U - _basis_combine(self.V, Y, b), Rinv)  # line 16
        self.V.append(Vn)
        self.U = self._mul(W - _basis_combine(self.V, ZP, b), Rinv)   # line 17
        self.k = k
        return StepResult(Hcol, R if self.ip == "cl" else float(R[0, 0]), Vn, False, W)


# --------------------------------------------------------------------------------------
# Comparison skeletons: BMGS-Arnoldi (Alg 2) and BCGS-PIO-Arnoldi (Alg 4)
# --------------------------------------------------------------------------------------


class BmgsArnoldi(PipArnoldi):
    """Alg 2 as a resumable object: per step k, k block inner products
    H_{j,k} = <V_j, W> each followed by W = W - V_j H_{j,k} (k syncs), then
    [V_{k+1}, H_{k+1,k}] = IO(W) (one more sync; CholQR for cl, the global norm for gl).
    A flag of that IO is the step's NaN-flag."""

    def step(self, force_flag: bool = False) -> StepResult:
        b, k = self.b, len(self.V)
        W = apply_A(self.A, self.V[-1])
        Hcol = np.zeros((k * b, b))
        for j in range(k):
            if self.ip == "cl":
                Hj = ip_cl([self.V[j]], W)
                W = W - self.V[j] @ Hj
            else:
                Hj = np.array([[ip_gl([self.V[j]], W)[0]]])
                W = W - self.V[j] * Hj[0, 0]
            Hcol[j * b:(j + 1) * b] = Hj
        self.Hbar[: k * b, (k - 1) * b: k * b] = Hcol
        if self.ip == "cl":
            Vn, R, flag = io_cl(W)
        else:
            Vn, R, flag = io_gl(W)
        flag = bool(flag) or force_flag
        if flag:
            return StepResult(Hcol, R, None, True, W)
        Rm = R if self.ip == "cl" else np.array([[R]])
        self.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b] = Rm
        self.V.append(Vn)
        self.k = k
        return StepResult(Hcol, R, Vn, False, W)


class PioArnoldi(PipArnoldi):
    """Alg 4, BCGS-PIO: H_{1:k,k} = <V_k-stack, W> (sync 1); the IO of
    diag(W, H_{1:k,k}) gives the R factors W~ = chol(<W, W>) (sync 2) and H~ = chol(H^* H)
    (replicated, no sync); H_{k+1,k} = chol(W~^* W~ - H~^* H~); V_{k+1} = (W - V H) H_{k+1,k}^{-1}.
    Reading R26: the IO muscle is CholQR (the paper's solver experiments use CholQR for the
    classical IO); a flag of any of the three Cholesky factorisations is the
    step's NaN-flag.  Global: W~ = ||W||_gl, H~ = ||H|| (Euclidean norm of the k scalars)."""

    def step(self, force_flag: bool = False) -> StepResult:
        b, k = self.b, len(self.V)
        W = apply_A(self.A, self.V[-1])
        if self.ip == "cl":
            Hcol = ip_cl(list(self.V), W)                       # line 4
            Wt, f1 = chol_flag(ip_cl([W], W))                    # line 5 (IO of W)
            Ht, f2 = chol_flag(Hcol.T @ Hcol)                    # line 5 (IO of H, local)
            R, f3 = chol_flag(Wt.T @ Wt - Ht.T @ Ht) if not (f1 or f2) else (Wt, True)   # line 6
            flag = f1 or f2 or f3 or force_flag
        else:
            Hcol = ip_gl(list(self.V), W)
            om = ip_gl([W], W)[0]
            hh = float(np.dot(Hcol, Hcol))
            wt = math.sqrt(om) if om > 0 else float("nan")
            ht = math.sqrt(hh) if hh > 0 else float("nan")
            rad = wt * wt - ht * ht
            flag = not (rad > 0.0) or not math.isfinite(rad) or force_flag
            R = math.sqrt(rad) if not flag else float("nan")
        b_ = self.b
        Hc = Hcol.reshape(k * b_, b_) if self.ip == "cl" else np.asarray(Hcol).reshape(k, 1)
        self.Hbar[: k * b_, (k - 1) * b_: k * b_] = Hc
        if flag:
            return StepResult(Hcol, R, None, True, W)
        if self.ip == "cl":
            P = W - np.concatenate(list(self.V), axis=1) @ Hcol
            Vn = right_trsm_upper(P, R)
            Rm = R
        else:
            P = W.copy()
            for j in range(k):
                P -= self.V[j] * Hcol[j]
            Vn = P / R
            Rm = np.array([[R]])
        self.Hbar[k * b_:(k + 1) * b_, (k - 1) * b_: k * b_] = Rm
        self.V.append(Vn)
        self.k = k
        return StepResult(Hcol, R, Vn, False, W)


# --------------------------------------------------------------------------------------
# BMGS-Arnoldi, Alg 2 — independent cross-check only (pin P5)
# --------------------------------------------------------------------------------------


def bmgs_arnoldi(A, B, m: int, ip: str):
    """Alg 2 with the CholQR (cl) or global (gl) muscle.  Returns (V list, Hbar, beta)."""
    s = B.shape[1]
    b = s if ip == "cl" else 1
    io = io_cl if ip == "cl" else io_gl
    V1, beta, flag = io(B)
    assert not flag
    V = [V1]
    Hbar = np.zeros(((m + 1) * b, m * b))
    for k in range(1, m + 1):
        W = apply_A(A, V[k - 1])
        for j in range(1, k + 1):
            if ip == "cl":
                Hjk = ip_cl([V[j - 1]], W)
                W = W - V[j - 1] @ Hjk
            else:
                Hjk = np.array([[ip_gl([V[j - 1]], W)[0]]])
                W = W - V[j - 1] * Hjk[0, 0]
            Hbar[(j - 1) * b: j * b, (k - 1) * b: k * b] = Hjk
        Vn, Rn, flag = io(W)
        assert not flag
        Rn = Rn if ip == "cl" else np.array([[Rn]])
        Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b] = Rn
        V.append(Vn)
    beta = beta if ip == "cl" else np.array([[beta]])
    return V, Hbar, beta


# --------------------------------------------------------------------------------------
# Projected problem: modified BFOM / BGMRES and Thm 2.4
# --------------------------------------------------------------------------------------


class SingularProjected(Exception):
    pass


def projected_solve(Hbar, beta, k: int, b: int, mod: str):
    """Xi_k = (H_k + M E_k^*)^{-1} E_1 beta with M = 0 (FOM) or
    M = H_k^{-*} E_k H_{k+1,k}^* H_{k+1,k} (GMRES; reading R11: computed
    literally as a modified BFOM).  Returns (Xi, M, cos) with cos = E_k^* Xi (the cospatial
    factor, Thm 2.4).  Raises SingularProjected if the ks x ks system is singular (R22)."""
    Hk = Hbar[: k * b, : k * b]
    Hk1 = Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b]
    E1B = np.zeros((k * b, b))
    E1B[:b] = beta
    M = np.zeros((k * b, b))
    try:
        if mod == "gmres":
            rhs = np.zeros((k * b, b))
            rhs[(k - 1) * b:] = Hk1.T @ Hk1
            M = np.linalg.solve(Hk.T, rhs)
        Hmod = Hk.copy()
        Hmod[:, (k - 1) * b:] += M
        Xi = np.linalg.solve(Hmod, E1B)
    except np.linalg.LinAlgError as e:  # exactly singular
        raise SingularProjected(str(e))
    if not (np.all(np.isfinite(Xi)) and np.all(np.isfinite(M))):
        raise SingularProjected("non-finite projected solution")
    cos = Xi[(k - 1) * b:]
    return Xi, M, cos


def residual_estimate(M, Hk1, cos, Cacc, s: int, b: int) -> float:
    """Eq (normF_Rm): ||[M; -H_{k+1,k}] (E_k^* Xi) C_acc||_F.
    For the global paradigm each scalar stands for a multiple of I_s with <V_i,V_j> =
    (1/s)tr(V_i^T V_j) = delta_ij, so the Frobenius norm of the n x s residual carries a
    factor sqrt(s) (reading R14)."""
    gen = np.vstack([M, -Hk1])
    val = np.linalg.norm(gen @ cos @ Cacc)
    return float(val) if b == s else float(math.sqrt(s) * val)


def kappa_F(beta, Hbar, k: int, b: int) -> float:
    """Reading R8: R_{k+1} := [E_1 beta, Hbar_k] ((k+1)b square, upper triangular) is the
    R factor of [U, A V_k] = V_{k+1} R_{k+1}; kappa_F = ||R||_F ||R^{-1}||_F >= kappa_2."""
    n = (k + 1) * b
    R = np.zeros((n, n))
    R[:b, :b] = beta
    R[:, b:] = Hbar[:n, : k * b]
    try:
        Ri = np.linalg.inv(R)
    except np.linalg.LinAlgError:
        return float("inf")
    return float(np.linalg.norm(R) * np.linalg.norm(Ri))


# --------------------------------------------------------------------------------------
# Restarted solver with adaptive restart
# --------------------------------------------------------------------------------------

CONVERGED, MAX_RESTARTS, DEAD = 0, 1, 2
OUTCOME_NAMES = {CONVERGED: "converged", MAX_RESTARTS: "max_restarts", DEAD: "dead"}


@dataclass
class SolveInfo:
    outcome: int = MAX_RESTARTS
    cycles: int = 0
    iterations: int = 0
    attempted_steps: int = 0
    nan_flags: int = 0
    cond_restarts: int = 0
    happy: int = 0
    false_convergences: int = 0
    m_final: int = 0
    true_relres: float = float("nan")
    res_est: float = float("nan")
    flags: list = field(default_factory=list)          # (cycle, k) of every NaN-flag
    cycle_lengths: list = field(default_factory=list)  # k_used per cycle
    history: list = field(default_factory=list)        # (cycle, k, res_est/normB, kappa_F)

    skel: str = "pip"

    # Paper accounting (PAPER.md:650 tables; pin P14): BCGS-PIP: sync = iterations + cycles,
    # A-ct = iterations, V-ct = 3 iterations; BMGS-(I)CWY: one
    # more A-application, sync and block evaluation per cycle (the lagged normalisation).
    # BMGS (Alg 2): k+1 syncs per step plus IO, A-ct = iterations, V-ct =
    # 2 iterations; BCGS-PIO (Alg 4): two syncs per step (Table 1).
    @property
    def syncs(self):
        if self.skel == "bmgs":
            return sum(k * (k + 3) // 2 for k in self.cycle_lengths) + self.cycles
        if self.skel == "pio":
            return 2 * self.iterations + self.cycles
        return self.iterations + (2 if self.skel in ("cwy", "icwy", "irols") else 1) * self.cycles

    @property
    def matvecs(self):
        return self.iterations + (self.cycles if self.skel in ("cwy", "icwy", "irols") else 0)

    @property
    def basis_evals(self):
        if self.skel == "bmgs":
            return 2 * self.iterations
        if self.skel == "irols":                  # 4 per step
            return 4 * self.iterations + self.cycles
        return 3 * self.iterations + (self.cycles if self.skel in ("cwy", "icwy") else 0)

    @property
    def restarts(self):
        return max(0, self.cycles - 1)


def solve(A, B, X0=None, m: int = 10, tol: float = 1e-8, max_restarts: int = 50,
          ip: str = "cl", mod: str = "gmres", cond_threshold: float = float("inf"),
          stop_on: str = "residual", X_star=None, force_flag_at=None,
          happy_check: bool = True, confirm_true: bool = True, record_kappa: bool = False,
          skel: str = "pip", prec=None):
    """Restarted modified BFOM/BGMRES with BCGS-PIP-Arnoldi (skel='pip', Alg 3) or
    BMGS-CWY / BMGS-ICWY-Arnoldi (skel='cwy' / 'icwy', Alg 6) and adaptive restart.
    ``prec='ilu0'`` (or an Ilu0Factors) runs the same method on M^{-1} A X = M^{-1} B with
    M = LU from ILU(0) (left preconditioning; tolerances in the preconditioned norm, R28).

    Follows SURVEY.md 8(c) "Step list" literally; readings cited inline.  ``A`` is the CSR
    triple (row_ptr, col_idx, vals).  ``stop_on='error'`` (test-only, pin P13) stops on
    ||X - X*||_F / ||X*||_F <= tol with X* given.  ``force_flag_at`` is
    the fault-injection hook (a NaN-flag at that step k of the first cycle reaching it).
    Returns (X, SolveInfo)."""
    n, s = B.shape
    b = s if ip == "cl" else 1
    B = np.asarray(B, dtype=np.float64)
    if prec is not None:      # left ILU(0): solve M^{-1} A X = M^{-1} B (R28)
        F = ilu0(*A) if isinstance(prec, str) else prec
        if isinstance(prec, str) and prec != "ilu0":
            raise ValueError(f"unknown preconditioner {prec!r}")
        A = IluOperator(A, F)
        B = F.solve(B)
    normB = math.sqrt(float(gram(B.reshape(-1, 1), B.reshape(-1, 1))[0, 0]))   # ||B||_F (R18)
    X = np.zeros_like(B) if X0 is None else np.array(X0, dtype=np.float64)
    if normB == 0.0:                               # B = 0: X = 0 is exact; nothing to do
        return np.zeros_like(B), SolveInfo(outcome=CONVERGED, true_relres=0.0, m_final=m)
    U = B.copy() if X0 is None else B - apply_A(A, X)                          # R13
    Cacc = np.eye(b)
    info = SolveInfo(skel=skel)
    m_cur = m
    if skel == "pip":
        arn = PipArnoldi(A, ip, m, s)
    elif skel in ("cwy", "icwy"):
        arn = CwyArnoldi(A, ip, m, s, inverse=(skel == "icwy"))
    elif skel == "irols":
        arn = IrolsArnoldi(A, ip, m, s)
    elif skel == "bmgs":
        arn = BmgsArnoldi(A, ip, m, s)
    elif skel == "pio":
        arn = PioArnoldi(A, ip, m, s)
    else:
        raise ValueError(f"unknown skeleton {skel!r}")
    forced_done = False

    def true_relres(Xc):
        Rr = B - apply_A(A, Xc)
        return float(np.linalg.norm(Rr)) / normB

    for cycle in range(1, max_restarts + 2):
        info.cycles = cycle
        if arn.begin(U):                           # IO flag: no safe block at all (R4)
            info.outcome = DEAD
            break
        k_used, why = 0, None
        last = None                                # (Xi, M, cos) of the last accepted step
        for k in range(1, m_cur + 1):
            info.attempted_steps += 1
            force = (force_flag_at is not None and not forced_done and k == force_flag_at)
            res = arn.step(force_flag=force)
            if force:
                forced_done = True
            flag = res.flag
            if not flag:
                try:
                    Xi, M, cos = projected_solve(arn.Hbar, arn.beta, k, b, mod)
                except SingularProjected:          # R22: FOM with singular H_k -> NaN-flag
                    flag = True
                    arn.V.pop()
                    arn.k = k - 1
            if flag:
                # R7: happy breakdown test — candidate with H_{k+1,k} := 0 (M = 0)
                if happy_check and not force:
                    Hsave = arn.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b].copy()
                    arn.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b] = 0.0
                    try:
                        Xi_h, _, _ = projected_solve(arn.Hbar, arn.beta, k, b, "fom")
                        Xc = X + _basis_combine(arn.V[:k], Xi_h @ Cacc, b)
                        if true_relres(Xc) <= tol:
                            X = Xc
                            info.iterations += 1
                            info.happy += 1
                            info.cycle_lengths.append(k)
                            info.true_relres = true_relres(X)
                            info.outcome = CONVERGED
                            info.m_final = m_cur
                            return X, info
                    except SingularProjected:
                        pass
                    arn.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b] = Hsave
                info.nan_flags += 1
                info.flags.append((cycle, k))
                k_used, why = k - 1, "flag"
                m_cur = k - 1                       # R6: m <- k-1 for all later cycles
                break
            info.iterations += 1
            last = (Xi, M, cos)
            Hk1 = arn.Hbar[k * b:(k + 1) * b, (k - 1) * b: k * b]
            est = residual_estimate(M, Hk1, cos, Cacc, s, b)
            info.res_est = est
            kap = kappa_F(arn.beta, arn.Hbar, k, b) if (record_kappa or math.isfinite(cond_threshold)) else float("nan")
            info.history.append((cycle, k, est / normB, kap))
            if stop_on == "error":
                Xc = X + _basis_combine(arn.V[:k], Xi @ Cacc, b)
                if np.linalg.norm(Xc - X_star) / np.linalg.norm(X_star) <= tol:
                    k_used, why = k, "error"
                    break
            elif est <= tol * normB:                 # R5: test after every accepted step
                k_used, why = k, "converged?"
                break
            if math.isfinite(cond_threshold) and kap > cond_threshold:   # R8
                info.cond_restarts += 1
                k_used, why = k, "kappa"
                break
            k_used, why = k, "m"
        info.cycle_lengths.append(k_used)
        if k_used == 0:
            info.outcome = DEAD
            break
        if why == "flag":
            Xi, M, cos = projected_solve(arn.Hbar, arn.beta, k_used, b, mod)
        else:
            Xi, M, cos = last
        X = X + _basis_combine(arn.V[:k_used], Xi @ Cacc, b)
        if why == "error":
            info.outcome = CONVERGED
            break
        if why == "converged?":
            tr = true_relres(X) if confirm_true else info.res_est / normB
            if tr <= tol:
                info.outcome = CONVERGED
                break
            # R19: the estimate drifted; restart from the true residual
            info.false_convergences += 1
            U = B - apply_A(A, X)
            Cacc = np.eye(b)
            continue
        # U = V_{k+1} [M; -H_{k+1,k}]  and  C_acc <- cos C_acc  (R10)
        Hk1 = arn.Hbar[k_used * b:(k_used + 1) * b, (k_used - 1) * b: k_used * b]
        U = _basis_combine(arn.V[: k_used + 1], np.vstack([M, -Hk1]), b)
        Cacc = cos @ Cacc
    info.m_final = m_cur
    info.true_relres = true_relres(X)
    return X, info


def _basis_combine(Vs, Y, b: int) -> np.ndarray:
    """sum_j V_j Y_j for block coefficients Y ((len(Vs) b) x b); global: scalars times V_j."""
    out = np.zeros_like(Vs[0])
    for j, Vj in enumerate(Vs):
        Yj = Y[j * b:(j + 1) * b]
        out += Vj @ Yj if b > 1 or Vj.shape[1] == 1 else Vj * Yj[0, 0]
    return out


def loss_of_orthogonality(Vs, ip: str) -> float:
    """||I - <Q,Q>||_2 (Eq loo) — diagnostic, exact SVD norm.  Pinned by
    closed forms in tests/test_oracle_kernels.py::test_loss_of_orthogonality_closed_form."""
    if ip == "cl":
        Q = np.concatenate(Vs, axis=1)
        G = gram(Q, Q)
    else:
        p = len(Vs)
        G = np.array([[ip_gl([Vs[i]], Vs[j])[0] for j in range(p)] for i in range(p)])
    return float(np.linalg.norm(np.eye(G.shape[0]) - G, 2))
