"""CPU tests of the boundary: liblsba.so loads, exports every symbol include/lsba.h declares,
and its host-only entry points (CSR validation, ghost plan) behave (no GPU needed)."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    txt = open(os.path.join(ROOT, "include", "lsba.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lsba_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    import paper_2208_09899_b200 as L
    syms = _declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L.lib, s)]
    assert not missing, missing
    # and the Python binding exposes the same names
    assert not [s for s in syms if not hasattr(L, s)]


def test_library_is_in_tree_sm100a():
    import paper_2208_09899_b200 as L
    assert L.library_path.startswith(ROOT)
    out = os.popen(f"cuobjdump --list-elf {L.library_path} 2>/dev/null").read()
    if out:
        assert "sm_100a" in out


def test_status_strings():
    import paper_2208_09899_b200 as L
    assert L.lsba_status_str(0) == "LSBA_OK"
    assert L.lsba_status_str(5) == "LSBA_E_STATE"


def test_csr_validate_matches_oracle_rules():
    import paper_2208_09899_b200 as L
    from oracle import lsba_oracle as O
    rng = np.random.default_rng(0)
    for trial in range(60):
        n = int(rng.integers(1, 12))
        counts = np.minimum(rng.integers(0, 4, size=n), n)
        row_ptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=row_ptr[1:])
        cols = rng.integers(-1, n + 1, size=row_ptr[-1]).astype(np.int32)
        if trial % 2:
            cols = np.concatenate([np.sort(rng.choice(n, size=c, replace=False)) for c in counts]).astype(np.int32) \
                if row_ptr[-1] else cols
        st, msg = L.lsba_csr_validate(n, n, row_ptr, cols)
        try:
            O.csr_check(n, row_ptr, cols, np.ones(cols.size))
            ok = True
        except ValueError:
            ok = False
        assert (st == 0) == ok, (row_ptr, cols, msg)


def test_ghost_plan_brute_force():
    """Host-only ghost plan vs a brute-force construction."""
    import paper_2208_09899_b200 as L
    from lsba_inputs import random_sparse, stencil
    for rp, ci, va in (stencil(2, 12), random_sparse(1024)):
        n = rp.size - 1
        for P in (2, 3, 4):
            part = np.linspace(0, n, P + 1).astype(np.int64)
            for r in range(P):
                r0, r1 = part[r], part[r + 1]
                cols = ci[rp[r0]:rp[r1]]
                cl, gg, rc = L.lsba_ghost_plan(r0, r1, cols, part)
                remote = np.unique(cols[(cols < r0) | (cols >= r1)])
                np.testing.assert_array_equal(gg, remote)
                owners = np.searchsorted(part, remote, side="right") - 1
                np.testing.assert_array_equal(rc, np.bincount(owners, minlength=P))
                assert rc[r] == 0
                # remapped columns address the same global column
                gidx = np.clip(cl.astype(np.int64) - (r1 - r0), 0, max(gg.size - 1, 0))
                back = np.where(cl < r1 - r0, cl + r0, np.concatenate([gg, [0]])[gidx])
                np.testing.assert_array_equal(back, cols)


def test_create_rejects_bad_arguments_without_gpu_work():
    """Argument validation happens before any device call (s out of range, bad CSR)."""
    import paper_2208_09899_b200 as L
    rp = np.array([0, 1, 2], dtype=np.int64)
    ci = np.array([0, 1], dtype=np.int32)
    va = np.ones(2)
    with pytest.raises(L.LsbaError) as e:
        L.lsba_create(2, 17, 4, rp, ci, va)
    assert e.value.status == 1
    with pytest.raises(L.LsbaError):
        L.lsba_create(2, 1, 4, rp, np.array([1, 0], dtype=np.int32)[::-1].copy() * 0 + 5, va)
    with pytest.raises(L.LsbaError):
        L.lsba_create(2, 1, 0, rp, ci, va)
