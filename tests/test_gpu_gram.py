"""Kernel-level parity of the SHIPPED streaming Gram (the step's single sync, Alg 3 line 4,
PAPER.md:268-269; Table 1's classical and global block inner products; the
two-block Gram of BMGS-(I)CWY, Alg 6 line 10): k_gram_v7 / k_gram_gl2 run on the
context's basis slots through lsba_basis_inner_product, i.e. the exact kernels, per-J
configuration tables, multi-pass splits (J > 8 GMAX) and the two-level ticket reduction the
solver uses (not the DFMA fallback that lsba_block_inner_product takes for caller buffers).

1. Integer data (entries in [-7, 7], n = 200,003 rows: every partial sum is an integer below
   2^53, so every summation order is exact): the GPU Gram must equal the exact Gram BIT FOR BIT
   for every J = 1 .. m_max + 1, Y aliased to the last block (the solver's case) and not, the
   two-block variant, and every LSBA_G7-forced configuration.  A dropped or doubled row, a
   transposed operand or a wrong block index changes integers, not rounding.
2. Random N(0,1) data (rounding): element by element against the oracle's near-exactly
   rounded oracle.gram within 256 eps |X|^T |Y| (the sequential-run + tree depth of the kernel
   is well below 256 additions at these sizes).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = np.finfo(float).eps


@pytest.fixture(scope="module")
def L():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device")
    import paper_2208_09899_b200 as L
    return L


def identity_csr(n):
    return np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32), np.ones(n)


class Slots:
    """A context whose basis slots hold seeded test blocks (V_1 .. V_{m_max+2})."""

    def __init__(self, L, n, s, m_max, kind, seed, env=None):
        import torch
        old = {k: os.environ.get(k) for k in (env or {})}
        os.environ.update(env or {})
        try:
            self.ctx = L.Context(n, s, m_max, *identity_csr(n))
        finally:
            for k, v in old.items():
                if v is None:
                    os.environ.pop(k, None)
                else:
                    os.environ[k] = v
        rng = np.random.default_rng(seed)
        self.blocks = []
        for j in range(1, m_max + 3):
            if kind == "int":
                V = rng.integers(-7, 8, size=(n, s)).astype(np.float64)
            else:
                V = rng.standard_normal((n, s))
            self.blocks.append(V)
            L.lsba_set_basis_block(self.ctx.ctx, j, torch.from_numpy(V).cuda())
        self.L, self.n, self.s, self.m_max = L, n, s, m_max

    def gram(self, j0, J, y, y2=0, ip="cl"):
        return self.L.lsba_basis_inner_product(self.ctx.ctx, j0, J, y, y2, ip=ip, s=self.s)

    def close(self):
        self.ctx.close()


def exact_gram(blocks, ys, ip, s):
    """Exact for integer data (every partial sum is an integer < 2^53): the reference the
    GPU must equal bit for bit.  Classical: [X_1..X_J]^T [Y (Y2)]; global: (1/s) tr(X_j^T Y)."""
    X = np.concatenate(blocks, axis=1)
    Y = np.concatenate(ys, axis=1)
    G = X.T @ Y
    if ip == "cl":
        return G
    J, w = len(blocks), len(ys)
    out = np.array([[np.trace(G[j * s:(j + 1) * s, q * s:(q + 1) * s]) / s for q in range(w)] for j in range(J)])
    return out[:, 0] if w == 1 else out


def check_all_J(sl, ip, Js, two_block=True):
    s, top = sl.s, sl.m_max + 2
    for J in Js:
        for y in sorted({J, top}):                 # aliased (the solver's case) and not
            G = sl.gram(1, J, y, ip=ip)
            ref = exact_gram(sl.blocks[:J], [sl.blocks[y - 1]], ip, s)
            assert np.array_equal(G, ref), (ip, s, J, y, np.abs(G - ref).max())
        if two_block and J + 1 <= top:
            G = sl.gram(1, J, J, J + 1, ip=ip)
            ref = exact_gram(sl.blocks[:J], [sl.blocks[J - 1], sl.blocks[J]], ip, s)
            assert np.array_equal(G, ref), (ip, s, J, "two-block", np.abs(G - ref).max())


# m_max per s: s = 16 reaches J = 27 > 8 GMAX = 24 (multi-pass); s = 8 reaches J = 41 (config 5)
CASES = [(2, 12), (4, 21), (8, 40), (16, 26)]


@pytest.mark.parametrize("s,m_max", CASES)
@pytest.mark.parametrize("ip", ["cl", "gl"])
def test_gram_v7_exact_every_J(L, s, m_max, ip):
    sl = Slots(L, 200003, s, m_max, "int", seed=100 + s)
    try:
        check_all_J(sl, ip, range(1, m_max + 2))
        # a window that does not start at slot 1 (BMGS uses single-block Grams at V_j)
        G = sl.gram(3, 2, 7, ip=ip)
        assert np.array_equal(G, exact_gram(sl.blocks[2:4], [sl.blocks[6]], ip, s))
    finally:
        sl.close()


G7_CASES = [(4, c) for c in range(1, 9)] + [(8, c) for c in range(1, 9)] + [(16, c) for c in range(1, 5)]


@pytest.mark.parametrize("s,cfg", G7_CASES)
def test_gram_v7_forced_configurations_exact(L, s, cfg):
    """Every (GMAX, U, CTAs/SM) configuration LSBA_G7 can force, at small, mid and max J."""
    m_max = 26 if s == 16 else 20
    sl = Slots(L, 100003, s, m_max, "int", seed=7 * cfg + s, env={"LSBA_G7": str(cfg)})
    try:
        check_all_J(sl, "cl", [1, 2, 5, 9, m_max + 1], two_block=(s != 16 or cfg <= 4))
    finally:
        sl.close()


@pytest.mark.parametrize("n", [1000, 8, 30011])
@pytest.mark.parametrize("s", [2, 4, 8, 16])
def test_gram_v7_rounding_vs_oracle(L, s, n):
    """Random real data: element by element against oracle.gram (near-exactly rounded)."""
    from oracle import lsba_oracle as O
    if n < s:
        pytest.skip("n < s")
    m_max = 26 if s == 16 else 8
    sl = Slots(L, n, s, m_max, "real", seed=900 + s + n)
    try:
        for J in sorted({1, 3, m_max + 1}):
            X = sl.blocks[:J]
            Y = sl.blocks[J - 1]
            G = sl.gram(1, J, J, ip="cl")
            Go = O.ip_cl(X, Y)
            bound = 256 * EPS * (np.abs(np.concatenate(X, axis=1)).T @ np.abs(Y))
            assert np.all(np.abs(G - Go) <= bound), (s, n, J)
            g = sl.gram(1, J, J, ip="gl")
            go = O.ip_gl(X, Y)
            gb = 256 * EPS * np.array([np.sum(np.abs(x) * np.abs(Y)) / s for x in X])
            assert np.all(np.abs(g - go) <= gb), (s, n, J)
    finally:
        sl.close()
