#!/usr/bin/env python
"""Write the full-size parity goldens under tests/golden/fullsize/ — ORACLE ONLY.

This script imports nothing but ``oracle/`` and the seeded input generators ``lsba_inputs``;
no value it stores comes from the CUDA path.  The GPU tests (tests/test_gpu_fullsize.py) load
these files so that the oracle never has to run on the GPU box at BASELINE sizes.

  python tools/oracle_goldens.py --case c5_cl_steps   (one case; see CASES)
  python tools/oracle_goldens.py --all                 (every case, one process each)

Per "steps" case (BASELINE config, inner product, K = 5 free-running BCGS-PIP steps of the
oracle, Alg 3, north star "H_k and the basis agree to relative 1e-10 over the
first 5 block steps"):
  beta, Hbar ((K+1) b x K b), vnorm[j] = ||V_j||_F over all rows, V_j on sample_rows(n),
  sketch[j] = R^T V_j for the seeded Gaussian R of lsba_inputs.sketch_chunks (width 8).
Per "solve" case (config 4, the one full-size solve the oracle affords):
  the counts (cycles, iterations, NaN-flags), true relres, X on sample_rows(n), R^T X, ||X||_F.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from lsba_inputs import make_config, sample_rows, sketch_chunks  # noqa: E402
from oracle import lsba_oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "fullsize")
K = 5
CASES = {
    "c2_cl_steps": (2, "cl", "steps"),
    "c3_cl_steps": (3, "cl", "steps"),
    "c4_cl_steps": (4, "cl", "steps"),
    "c4_gl_steps": (4, "gl", "steps"),
    "c5_cl_steps": (5, "cl", "steps"),
    "c4_cl_solve": (4, "cl", "solve"),
    "c4_gl_solve": (4, "gl", "solve"),
    # the NEXT skeletons at full size: 5 free-running steps
    "c5_cl_cwy_steps": (5, "cl", "steps", "cwy"),
    "c3_cl_icwy_steps": (3, "cl", "steps", "icwy"),
    "c3_cl_irols_steps": (3, "cl", "steps", "irols"),
    "c4_gl_cwy_steps": (4, "gl", "steps", "cwy"),
    "c3_cl_pio_steps": (3, "cl", "steps", "pio"),
    "c3_cl_bmgs_steps": (3, "cl", "steps", "bmgs"),
}


def arnoldi(skel, A, ip, K, s):
    """The oracle's skeleton objects (same begin/step/V/Hbar/beta interface)."""
    if skel == "pip":
        return O.PipArnoldi(A, ip, K, s)
    if skel in ("cwy", "icwy"):
        return O.CwyArnoldi(A, ip, K, s, inverse=(skel == "icwy"))
    if skel == "irols":
        return O.IrolsArnoldi(A, ip, K, s)
    if skel == "pio":
        return O.PioArnoldi(A, ip, K, s)
    if skel == "bmgs":
        return O.BmgsArnoldi(A, ip, K, s)
    raise ValueError(skel)


def sketch(V):
    n = V.shape[0]
    out = np.zeros((8, V.shape[1]))
    for r0, r1, R in sketch_chunks(n):
        out += R.T @ V[r0:r1]
    return out


def run_case(name):
    cfg, ip, kind = CASES[name][:3]
    skel = CASES[name][3] if len(CASES[name]) > 3 else "pip"
    t0 = time.time()
    p = make_config(cfg)
    A = (p.row_ptr, p.col_idx, p.vals)
    n, s = p.B.shape
    b = s if ip == "cl" else 1
    rows = sample_rows(n)
    meta = {"case": name, "config": cfg, "workload": p.name, "ip": ip, "skel": skel, "n": n, "s": s, "m": p.m,
            "nnz": int(p.row_ptr[-1]), "written_by": "tools/oracle_goldens.py (oracle/ only)"}
    if kind == "steps":
        arn = arnoldi(skel, A, ip, K, s)
        assert not arn.begin(p.B)
        for k in range(K):
            assert not arn.step().flag, k
        Vs = arn.V
        out = dict(beta=np.asarray(arn.beta, dtype=np.float64), Hbar=arn.Hbar[:(K + 1) * b, :K * b].copy(),
                   vnorm=np.array([np.linalg.norm(v) for v in Vs]), rows=rows,
                   Vrows=np.stack([v[rows] for v in Vs]), sketch=np.stack([sketch(v) for v in Vs]))
        meta.update(K=K, cite={"pip": "Alg 3 PAPER.md:262-275", "cwy": "Alg 6 PAPER.md:316-348",
                               "icwy": "Alg 6 PAPER.md:316-348", "irols": "Alg 7 PAPER.md:350-379",
                               "pio": "Alg 4 PAPER.md:277-290", "bmgs": "Alg 2 PAPER.md:164-178"}[skel]
                    + "; north star 5-step parity (BASELINE.json)")
    else:
        X, info = O.solve(A, p.B, m=p.m, tol=p.tol, max_restarts=p.max_restarts, ip=ip, mod="gmres",
                          cond_threshold=p.cond_threshold)
        assert info.outcome == O.CONVERGED, info
        out = dict(rows=rows, Xrows=X[rows], Xsketch=sketch(X), xnorm=np.array(np.linalg.norm(X)),
                   counts=np.array([info.cycles, info.iterations, info.nan_flags, info.cond_restarts]),
                   true_relres=np.array(info.true_relres))
        meta.update(cycles=info.cycles, iterations=info.iterations, nan_flags=info.nan_flags,
                    flags=info.flags, cycle_lengths=info.cycle_lengths, true_relres=info.true_relres,
                    cite="restarted BGMRES, PAPER.md:186-219; north star full-solve parity")
    meta["oracle_seconds"] = round(time.time() - t0, 1)
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    with open(os.path.join(OUT, name + ".json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(json.dumps(meta), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", choices=sorted(CASES))
    ap.add_argument("--all", action="store_true")
    args = ap.parse_args()
    if args.case:
        run_case(args.case)
        return
    if args.all:
        procs = [subprocess.Popen([sys.executable, __file__, "--case", c]) for c in CASES]
        sys.exit(max(p.wait() for p in procs))
    ap.print_help()


if __name__ == "__main__":
    main()
