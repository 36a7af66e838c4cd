"""CPU checks of bench.py's workload plumbing (no GPU): the strong-scaling partition gives every
rank whole z-planes of the SAME global problem (PAPER.md:57 row-partitioned block vectors;
SURVEY.md 8(e)), and the algorithmic-bytes accounting matches ROOF(k) of SURVEY.md 8(d)."""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_partition_whole_units_cover():
    import bench
    for n, unit, world in [(256 ** 3, 256 * 256, 8), (256 ** 3, 256 * 256, 3), (1024 * 1024, 1024, 7), (100, 1, 3)]:
        parts = [bench.partition(n, world, r, unit) for r in range(world)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        for (a0, a1), (b0, b1) in zip(parts, parts[1:]):
            assert a1 == b0
        assert all(r0 % unit == 0 and r1 % unit == 0 for r0, r1 in parts)
        sizes = [r1 - r0 for r0, r1 in parts]
        assert max(sizes) - min(sizes) <= unit


@pytest.mark.parametrize("world", [2, 3])
def test_strong_scaling_slices_of_one_problem(world, monkeypatch):
    """Twin-sized stand-in for config 5: the ranks' CSR rows and B rows are exactly the global
    problem's rows."""
    import bench
    import lsba_inputs
    from lsba_inputs import CONFIGS, rhs, stencil
    small = dict(CONFIGS[5], N=12)
    monkeypatch.setitem(lsba_inputs.CONFIGS, 5, small)
    monkeypatch.setattr(lsba_inputs.generators, "CONFIGS", lsba_inputs.CONFIGS)
    rp, ci, va = stencil(3, 12, None)
    Bg = rhs(12 ** 3, 8)
    seen = 0
    for r in range(world):
        wl = bench.build_workload(5, r, world, need_sha=False)
        r0, r1 = wl["row_begin"], wl["row_end"]
        assert r0 == seen and r0 % 144 == 0
        seen = r1
        lrp, lci, lva = wl["A"]
        assert np.array_equal(lrp, rp[r0:r1 + 1] - rp[r0])
        assert np.array_equal(lci, ci[rp[r0]:rp[r1]]) and np.array_equal(lva, va[rp[r0]:rp[r1]])
        assert np.array_equal(wl["B"], Bg[r0:r1])
        assert wl["nnz"] == rp[-1] and wl["n_global"] == 12 ** 3
    assert seen == 12 ** 3


def test_rank_proxy_slab_has_a_rank_s_share(monkeypatch):
    """--rank-proxy P (one-GPU diagnostic): the slab problem has exactly the rows of one rank of
    the P-rank partition, and each row keeps that rank's in-slab entries (the entries reaching
    into the neighbours' planes are cut off)."""
    import bench
    import lsba_inputs
    from lsba_inputs import CONFIGS
    small = dict(CONFIGS[5], N=12)
    monkeypatch.setitem(lsba_inputs.CONFIGS, 5, small)
    monkeypatch.setattr(lsba_inputs.generators, "CONFIGS", lsba_inputs.CONFIGS)
    P = 3
    wl = bench.build_workload(5, 0, 1, rank_proxy=P)
    mid = bench.build_workload(5, 1, P, need_sha=False)          # an interior rank of the real run
    r0, r1 = mid["row_begin"], mid["row_end"]
    assert wl["n_global"] == r1 - r0 == 12 * 12 * 4 and wl["B"].shape == (r1 - r0, 8)
    assert wl["name"].endswith("_slab_1of3_proxy")
    prp, pci, pva = wl["A"]
    rp, ci, va = mid["A"]
    assert wl["nnz"] == prp[-1] == rp[-1] - 2 * 144             # two cut-off planes of ghost entries
    for i in (0, 5, 143, 144, 300, 12 * 12 * 4 - 1):
        cols = ci[rp[i]:rp[i + 1]]
        keep = (cols >= r0) & (cols < r1)
        assert np.array_equal(pci[prp[i]:prp[i + 1]], cols[keep] - r0)
        assert np.array_equal(pva[prp[i]:prp[i + 1]], va[rp[i]:rp[i + 1]][keep])


def test_algorithmic_bytes_is_sum_of_roof():
    import bench
    nnz, n, s, m = 1000, 100, 4, 7
    iters, cycles = 2 * m, 2
    gram_blocks = 2 * sum(k + 1 for k in range(1, m + 1))
    expect = 2 * (sum(bench.roof_step(nnz, n, s, k) for k in range(1, m + 1)) + bench.roof_cycle_extra(n, s, m))
    assert bench.algorithmic_bytes(nnz, n, s, iters, cycles, gram_blocks) == pytest.approx(expect, rel=1e-14)


def test_reference_arm_line_contract():
    """`bench.py --impl reference` (the oracle timed on the host cores) prints ONE JSON line with
    the contract's keys; its `config` is what the GPU arm prints for the same workload."""
    import json
    import subprocess
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0 and d["n_gpus"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"] == d["e2e"]["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    import bench
    wl = bench.build_workload(1, 0, 1, need_sha=False)
    assert d["config"] == json.loads(json.dumps(bench.workload_config(wl, 1)))
    assert "Infinity" not in lines[0] and "NaN" not in lines[0]          # strict JSON
