#!/usr/bin/env python
"""Time lsba_ilu0_apply (two sync-free triangular solves) on the BASELINE configs' matrices:
us per apply and us per dependency level.   python tools/ilu_apply_bench.py [--configs 2 3 5]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="*", type=int, default=[2, 3, 5])
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    import numpy as np
    import torch
    import paper_2208_09899_b200 as L
    from lsba_inputs import make_config
    for cfg in args.configs:
        p = make_config(cfg)
        with L.Context(p.n, p.s, 2, p.row_ptr, p.col_idx, p.vals) as ctx:
            L.lsba_ilu0_setup(ctx.ctx, True)
            _, (nlL, nlU) = L.lsba_copy_ilu0_factors(ctx.ctx, 0)
            X = torch.from_numpy(p.B).cuda()
            Y = torch.empty_like(X)
            L.lsba_ilu0_apply(ctx.ctx, X, Y)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.reps):
                L.lsba_ilu0_apply(ctx.ctx, X, Y)
            e1.record()
            torch.cuda.synchronize()
            us = 1e3 * e0.elapsed_time(e1) / args.reps
            print(f"config {cfg} ({p.name}, n={p.n}, s={p.s}): levels L {nlL} U {nlU}: "
                  f"{us:.0f} us per apply, {us / (nlL + nlU):.2f} us per level "
                  f"("
                  f"LSBA_ILU_CTAS={os.environ.get('LSBA_ILU_CTAS', '1')})", flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
