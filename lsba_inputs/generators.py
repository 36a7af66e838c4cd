"""Problem generators (inputs only; no method arithmetic).

Recipes (BASELINE.json ``configs``):

* stencil(dims, N, v): h^2-scaled first-order-upwind convection-diffusion  -Lap_h u + v.grad_h u
  on an N^d grid with homogeneous Dirichlet boundary eliminated, h = 1/(N+1), lexicographic
  ordering with x fastest (row i = x + N*y + N^2*z).  Entries: diagonal 2d + h*sum(v);
  backward neighbour in dimension d: -1 - h*v_d; forward neighbour: -1.  v = 0 is the
  5-/7-point Laplacian (4/-1 in 2D, 6/-1 in 3D).
* random_sparse(n): 16 stored entries per row: the diagonal, 7 distinct band columns
  (0 < |j-i| <= 64, 0 <= j < n, uniform over the valid offsets of that row) and 8 distinct
  uniform-random columns distinct from the row's other columns (collisions redrawn).
  Off-diagonal values U(-1,1); a_ii = 1.1 * sum_{j != i} |a_ij| (strictly diagonally
  dominant).  RNG numpy.random.default_rng(seed=1), rows drawn in chunks of 2^16.
* tridiag(n): PAPER.md:446 (Sec 5.1): 1 on the off-diagonals, -1, -2, ..., -n on the
  diagonal; B has two columns, the first all 1/sqrt(n), the second 1, 2, ..., n.
* rhs(n, s): numpy.random.default_rng(0).standard_normal((n, s)), fp64, C order
  (row-major n x s, which is also the device layout).

CSR convention: row_ptr int64 of length n+1, row_ptr[0] = 0, monotone;
col_idx int32 sorted strictly increasing within a row; vals float64.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np


@dataclass
class Problem:
    name: str
    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray
    B: np.ndarray
    m: int
    tol: float
    max_restarts: int
    ips: tuple = ("cl",)
    mods: tuple = ("gmres",)
    cond_threshold: float = float("inf")
    meta: dict = field(default_factory=dict)

    @property
    def s(self) -> int:
        return self.B.shape[1]

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])


def _compress(cols: np.ndarray, vals: np.ndarray, mask: np.ndarray):
    """Dense (rows, w) candidate arrays with validity mask -> CSR pieces (row-major order)."""
    counts = mask.sum(axis=1).astype(np.int64)
    return counts, cols[mask].astype(np.int32), vals[mask]


def stencil(dims: int, N: int, v=None, chunk_rows: int = 1 << 20, shape=None, rows=None):
    """h^2-scaled upwind convection-diffusion stencil on an N^dims grid (see module doc).

    shape: optional grid extents per dimension (x fastest), default (N,)*dims (h = 1/(N+1)).
    rows: optional (r0, r1): build only those rows (global column indices), for row-partitioned
    multi-GPU runs; row_ptr then starts at 0 for row r0."""
    if v is None:
        v = (0.0,) * dims
    v = tuple(float(x) for x in v)
    assert len(v) == dims and all(x >= 0 for x in v)
    h = 1.0 / (N + 1)
    shape = tuple(shape) if shape is not None else (N,) * dims
    assert len(shape) == dims
    n = int(np.prod(shape))
    strides = [int(np.prod(shape[:d])) for d in range(dims)]
    lo, hi = (0, n) if rows is None else (int(rows[0]), int(rows[1]))
    diag = 2.0 * dims + h * sum(v)
    # column order for sorted rows: backward z, y, x; centre; forward x, y, z
    offs = [-strides[d] for d in reversed(range(dims))] + [0] + [strides[d] for d in range(dims)]
    coef = [-1.0 - h * v[d] for d in reversed(range(dims))] + [diag] + [-1.0] * dims
    which = [d for d in reversed(range(dims))] + [-1] + list(range(dims))
    sign = [-1] * dims + [0] + [1] * dims
    w = len(offs)
    counts_all, cols_all, vals_all = [], [], []
    for r0 in range(lo, hi, chunk_rows):
        r1 = min(hi, r0 + chunk_rows)
        rows_ = np.arange(r0, r1, dtype=np.int64)
        coord = [(rows_ // strides[d]) % shape[d] for d in range(dims)]
        cols = np.empty((r1 - r0, w), dtype=np.int64)
        vals = np.empty((r1 - r0, w), dtype=np.float64)
        mask = np.ones((r1 - r0, w), dtype=bool)
        for t in range(w):
            cols[:, t] = rows_ + offs[t]
            vals[:, t] = coef[t]
            if sign[t] < 0:
                mask[:, t] = coord[which[t]] > 0
            elif sign[t] > 0:
                mask[:, t] = coord[which[t]] < shape[which[t]] - 1
        c, ci, vv = _compress(cols, vals, mask)
        counts_all.append(c)
        cols_all.append(ci)
        vals_all.append(vv)
    counts = np.concatenate(counts_all) if counts_all else np.zeros(0, dtype=np.int64)
    row_ptr = np.zeros(hi - lo + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    if not cols_all:
        return row_ptr, np.zeros(0, dtype=np.int32), np.zeros(0)
    return row_ptr, np.concatenate(cols_all), np.concatenate(vals_all)


def random_sparse(n: int, seed: int = 1, band: int = 64, n_band: int = 7, n_rand: int = 8,
                  chunk_rows: int = 1 << 16):
    """Random nonsymmetric strictly diagonally dominant matrix (see module doc)."""
    assert n > 2 * band, "n too small for the band recipe"
    rng = np.random.default_rng(seed)
    per_row = 1 + n_band + n_rand
    cand = np.concatenate([np.arange(-band, 0), np.arange(1, band + 1)])  # 2*band offsets
    row_ptr = np.arange(n + 1, dtype=np.int64) * per_row
    col_idx = np.empty(n * per_row, dtype=np.int32)
    vals = np.empty(n * per_row, dtype=np.float64)
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        rows = np.arange(r0, r1, dtype=np.int64)
        nr = r1 - r0
        # band part: uniform sample without replacement over this row's valid offsets
        keys = rng.random((nr, cand.size))
        tgt = rows[:, None] + cand[None, :]
        keys[(tgt < 0) | (tgt >= n)] = np.inf
        pick = np.argpartition(keys, n_band - 1, axis=1)[:, :n_band]
        bcols = np.take_along_axis(tgt, pick, axis=1)
        # random part: 8 distinct uniform columns, distinct from diagonal and band columns
        rcols = rng.integers(0, n, size=(nr, n_rand), dtype=np.int64)
        while True:
            allc = np.concatenate([rows[:, None], bcols, rcols], axis=1)
            srt = np.sort(allc, axis=1)
            dup_rows = np.any(srt[:, 1:] == srt[:, :-1], axis=1)
            if not dup_rows.any():
                break
            idx = np.nonzero(dup_rows)[0]
            # redraw every random column of the offending rows that collides with an earlier column
            for i in idx:
                row_cols = list(allc[i, : 1 + n_band])
                new = []
                for c in rcols[i]:
                    while c in row_cols or c in new:
                        c = int(rng.integers(0, n))
                    new.append(c)
                rcols[i] = new
        offv = rng.uniform(-1.0, 1.0, size=(nr, n_band + n_rand))
        diagv = 1.1 * np.abs(offv).sum(axis=1)
        allc = np.concatenate([rows[:, None], bcols, rcols], axis=1)
        allv = np.concatenate([diagv[:, None], offv], axis=1)
        order = np.argsort(allc, axis=1, kind="stable")
        allc = np.take_along_axis(allc, order, axis=1)
        allv = np.take_along_axis(allv, order, axis=1)
        col_idx[r0 * per_row: r1 * per_row] = allc.reshape(-1)
        vals[r0 * per_row: r1 * per_row] = allv.reshape(-1)
    return row_ptr, col_idx, vals


def tridiag(n: int):
    """PAPER.md:446 (Sec 5.1): off-diagonals 1, diagonal -1, -2, ..., -n."""
    rows = []
    for i in range(n):
        c = [j for j in (i - 1, i, i + 1) if 0 <= j < n]
        rows.append(c)
    counts = np.array([len(c) for c in rows], dtype=np.int64)
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    col_idx = np.array([j for c in rows for j in c], dtype=np.int32)
    vals = np.array([(-(i + 1.0) if j == i else 1.0) for i, c in enumerate(rows) for j in c])
    return row_ptr, col_idx, vals


def tridiag_rhs(n: int):
    """first column identical elements 1/sqrt(n), second column 1, 2, ..., n."""
    B = np.empty((n, 2))
    B[:, 0] = 1.0 / np.sqrt(n)
    B[:, 1] = np.arange(1, n + 1, dtype=np.float64)
    return B


def laplacian_1d(n: int):
    """1D Dirichlet Laplacian tridiag(-1, 2, -1) (closed-form eigenvalues 2 - 2cos(j pi/(n+1)))."""
    return stencil(1, n)


def identity(n: int):
    row_ptr = np.arange(n + 1, dtype=np.int64)
    return row_ptr, np.arange(n, dtype=np.int32), np.ones(n)


def rhs(n: int, s: int, seed: int = 0):
    return np.random.default_rng(seed).standard_normal((n, s))


def sketch_chunks(n: int, width: int = 8, seed: int = 11, chunk: int = 1 << 20):
    """Seeded Gaussian test matrix R (n x width, N(0,1) entries), yielded in row chunks
    (r0, r1, R[r0:r1]) so that it is never held whole at n = 2^24.  Chunk c is drawn from
    default_rng([seed, c]).  (A random input for full-size checks: E||R^T D||_F^2 =
    width ||D||_F^2 for any n x s matrix D.)"""
    for c, r0 in enumerate(range(0, n, chunk)):
        r1 = min(n, r0 + chunk)
        yield r0, r1, np.random.default_rng([seed, c]).standard_normal((r1 - r0, width))


def sample_rows(n: int, count: int = 1024, seed: int = 5) -> np.ndarray:
    """Seeded sorted sample of distinct row indices, always including the first and last row."""
    rng = np.random.default_rng(seed)
    rows = rng.choice(n, size=min(count, n), replace=False) if n > count else np.arange(n)
    return np.unique(np.concatenate([[0, n - 1], rows])).astype(np.int64)


def csr_sha256(row_ptr, col_idx, vals) -> str:
    h = hashlib.sha256()
    for a in (row_ptr, col_idx, vals):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


# BASELINE.json configs (index 0..4 = the JSON list order); SURVEY.md 8(d) table.
CONFIGS = {
    1: dict(name="tiny_cd2d_16", kind="stencil", dims=2, N=16, v=(10.0, 10.0), s=2, m=10,
            tol=1e-8, max_restarts=50, ips=("cl",), mods=("gmres",), tau=float("inf")),
    2: dict(name="lapl2d_1024", kind="stencil", dims=2, N=1024, v=None, s=4, m=20,
            tol=1e-8, max_restarts=20000, ips=("cl",), mods=("fom", "gmres"), tau=float("inf")),
    3: dict(name="cd3d_128", kind="stencil", dims=3, N=128, v=(50.0, 25.0, 12.5), s=8, m=30,
            tol=1e-8, max_restarts=20000, ips=("cl",), mods=("gmres",), tau=1e8),
    4: dict(name="random_4M", kind="random", n=1 << 22, s=16, m=25,
            tol=1e-8, max_restarts=20000, ips=("gl", "cl"), mods=("gmres",), tau=float("inf")),
    5: dict(name="lapl3d_256", kind="stencil", dims=3, N=256, v=None, s=8, m=40,
            tol=1e-8, max_restarts=20000, ips=("cl",), mods=("gmres",), tau=1e8),
}

# CPU-affordable scaled twins
TWINS = {
    2: dict(CONFIGS[2], name="lapl2d_64", N=64),
    3: dict(CONFIGS[3], name="cd3d_16", N=16),
    4: dict(CONFIGS[4], name="random_16K", n=1 << 14),
    5: dict(CONFIGS[5], name="lapl3d_24", N=24),
}


def _build(spec: dict, s_override=None) -> Problem:
    s = s_override or spec["s"]
    if spec["kind"] == "stencil":
        rp, ci, va = stencil(spec["dims"], spec["N"], spec["v"])
    else:
        rp, ci, va = random_sparse(spec["n"])
    n = rp.size - 1
    B = rhs(n, s)
    return Problem(spec["name"], n, rp, ci, va, B, spec["m"], spec["tol"], spec["max_restarts"],
                   spec["ips"], spec["mods"], spec["tau"], meta=dict(spec))


def make_config(i: int) -> Problem:
    """BASELINE.json configs[i-1] at full size."""
    return _build(CONFIGS[i])


def make_twin(i: int) -> Problem:
    """CPU-affordable scaled twin of config i (1 returns the tiny config itself)."""
    return _build(CONFIGS[1] if i == 1 else TWINS[i])
