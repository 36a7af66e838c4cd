#!/usr/bin/env python
"""The paper's skeleton comparison (Appendix tables) on one B200: for each
problem, every skeleton's full solve — time, cycles, iterations, A-ct, V-ct, sync-ct, NaN-flags.

  python tools/skeleton_report.py [--out profiles/r01_skeletons.md] [--problems tridiag tiny c3 c4 c5]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SKELS = {"pip": "BCGS-PIP", "cwy": "BMGS-CWY", "icwy": "BMGS-ICWY", "irols": "BCGS-IRO-LS", "pio": "BCGS-PIO", "bmgs": "BMGS"}


def problems(names):
    from lsba_inputs import make_config, tridiag, tridiag_rhs
    for nm in names:
        if nm == "tridiag":
            A = tridiag(1000)
            # PAPER.md:446 (Sec 5.1) with Table 3's parameters: s = 2, m = 70, FOM, tol 1e-10
            yield nm, A, tridiag_rhs(1000), 70, 1e-10, [("cl", "fom"), ("gl", "fom")], float("inf"), list(SKELS)
        else:
            i = {"tiny": 1, "c2": 2, "c3": 3, "c4": 4, "c5": 5}[nm]
            p = make_config(i)
            skels = list(SKELS) if i in (1, 3, 4) else ["pip", "cwy", "icwy", "irols", "pio"]
            yield (p.name, (p.row_ptr, p.col_idx, p.vals), p.B, p.m, p.tol,
                   [(ip, md) for ip in p.ips for md in p.mods], p.cond_threshold, skels)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--problems", nargs="*", default=["tridiag", "tiny", "c3", "c4", "c5"])
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_2208_09899_b200 as L
    rows = []
    for name, A, B, m, tol, methods, tau, skels in problems(args.problems):
        n, s = B.shape
        with L.Context(n, s, m, *A) as ctx:
            Bd = torch.from_numpy(B).cuda()
            for ip, mod in methods:
                for sk in skels:
                    X = torch.zeros_like(Bd)
                    ctx.solve(Bd, X, m, tol, 20000, ip=ip, mod=mod, cond_threshold=tau, skel=sk)   # warm-up
                    X.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record()
                    info = ctx.solve(Bd, X, m, tol, 20000, ip=ip, mod=mod, cond_threshold=tau, skel=sk)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                    out = {0: "converged", 1: "max restarts", 2: "dead"}[info.outcome]
                    rows.append(f"| {name} | {ip}-{SKELS[sk]}-{mod.upper()} | {out} | {ms:.1f} | {info.cycles} | "
                                f"{info.iterations} | {info.matvecs} | {info.basis_evals} | {info.syncs} | "
                                f"{info.nan_flags} | {info.true_relres:.1e} |")
                    print(rows[-1], flush=True)
        torch.cuda.empty_cache()
    head = ("# Skeleton comparison on one B200 (the paper's Appendix tables, PAPER.md:646-790)\n\n"
            "`python tools/skeleton_report.py`: device time of one full solve from X0 = 0 after a warm-up solve; "
            "counters as the paper's (A-ct, V-ct, sync-ct).  tridiag = PAPER.md:446 with n = 1000, s = 2, "
            "m = 70, tol 1e-10 (Table 3); the others are the BASELINE.json configs.\n\n"
            "| problem | method | outcome | ms | cycles | iterations | A-ct | V-ct | sync-ct | NaN-flags | true relres |\n"
            "|---|---|---|---|---|---|---|---|---|---|---|\n")
    txt = head + "\n".join(rows) + "\n"
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
