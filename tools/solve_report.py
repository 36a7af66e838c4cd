#!/usr/bin/env python
"""Time-to-solution of full solves at the BASELINE sizes (SURVEY.md 8(d) "Separately, run the
full solve to tol 1e-8 and report time-to-solution, cycles and iterations").

  python tools/solve_report.py [--configs 1 2 3 4 5] [--out profiles/r01_solves.md]

Each solve starts from X0 = 0 with the config's (m, tol, tau); one warm-up solve first; the
device time of the solve call is measured with CUDA events; the true residual is the library's
explicit one (the GPU tests check it against the oracle's SpMM)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="*", default=[1, 2, 3, 4, 5])
    ap.add_argument("--out", default=None)
    ap.add_argument("--prec", default="none", choices=["none", "ilu0"],
                    help="left ILU(0): tol is then relative in the preconditioned norm (R28)")
    args = ap.parse_args()
    prec = None if args.prec == "none" else args.prec
    import torch
    import paper_2208_09899_b200 as L
    from lsba_inputs import make_config
    rows = []
    for cfg in args.configs:
        p = make_config(cfg)
        for ip in p.ips:
            for mod in p.mods:
                with L.Context(p.n, p.s, p.m, p.row_ptr, p.col_idx, p.vals) as ctx:
                    B = torch.from_numpy(p.B).cuda()
                    X = torch.zeros_like(B)
                    ctx.solve(B, X, p.m, p.tol, p.max_restarts, ip=ip, mod=mod, cond_threshold=p.cond_threshold,
                              prec=prec)
                    X.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda.synchronize()
                    e0.record()
                    info = ctx.solve(B, X, p.m, p.tol, p.max_restarts, ip=ip, mod=mod,
                                     cond_threshold=p.cond_threshold, prec=prec)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1)
                out = {0: "converged", 1: "max restarts", 2: "dead"}[info.outcome]
                rows.append(f"| {cfg} | {p.name} | {ip}-{mod}{'' if prec is None else ' + ILU(0)'} | {p.m} | {p.cond_threshold:g} | {out} | "
                            f"{info.cycles} | {info.iterations} | {info.nan_flags} | {info.cond_restarts} | "
                            f"{info.m_final} | {info.true_relres:.2e} | {ms:.1f} | "
                            f"{1e3 * info.iterations / ms:.0f} |")
                print(rows[-1], flush=True)
                torch.cuda.empty_cache()
        del p
    head = ("# Full solves at the BASELINE sizes (one B200, X0 = 0, tol 1e-8"
            + (", left ILU(0): tol in the preconditioned norm" if prec else "") + ")\n\n"
            "`python tools/solve_report.py`; device time of one `lsba_*_solve` call after a warm-up solve.\n\n"
            "| cfg | workload | method | m | tau | outcome | cycles | iterations | NaN-flags | kappa restarts "
            "| m_final | true relres | ms | block steps/s |\n|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    txt = head + "\n".join(rows) + "\n"
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt)
    print(txt)


if __name__ == "__main__":
    main()
