#!/usr/bin/env python
"""Per-launch timeline of restart cycles (CUDA events around every launch, both streams).

  python tools/timeline.py [--config 2] [--cycles 2] [--out gpurun_out/timeline_c2.txt]

Prints, for the profiled cycles: each launch (kernel, start, duration, gap to the previous
launch's end on the main stream) and a summary: busy time per kernel, total idle gaps on the
main stream, cycle time."""
import argparse
import collections
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--cycles", type=int, default=2)
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--out", default=None)
    ap.add_argument("--cold", action="store_true", help="profile a full solve from X0 = 0")
    ap.add_argument("--ip", default="cl")
    ap.add_argument("--skel", default="pip")
    args = ap.parse_args()
    import torch
    import paper_2208_09899_b200 as L
    import bench
    wl = bench.build_workload(args.config, 0, 1)
    ctx = L.Context(wl["n_global"], wl["s"], wl["m"], *wl["A"])
    L.lsba_set_kernel_variant(ctx.ctx, args.variant)
    B = torch.from_numpy(wl["B"]).cuda()
    X = torch.zeros_like(B)
    L.lsba_bgmres_solve(ctx.ctx, B, X, wl["m"], wl["tol"], 0, ip=args.ip, skel=args.skel)
    torch.cuda.synchronize()
    if args.cold:
        X.zero_()
    L.lsba_profile_enable(ctx.ctx, True)
    info = L.lsba_bgmres_solve(ctx.ctx, B, X, wl["m"], wl["tol"], 200 if args.cold else args.cycles - 1, ip=args.ip,
                               skel=args.skel)
    print("solve:", info.as_dict())
    tl = L.lsba_profile_timeline(ctx.ctx)
    L.lsba_profile_enable(ctx.ctx, False)
    lines = []
    busy = collections.defaultdict(float)
    cnt = collections.Counter()
    gaps = collections.defaultdict(float)
    prev_end = None
    for name, a, b in tl:
        gap = None
        if name != "step_update":
            gap = (a - prev_end) if prev_end is not None else 0.0
            prev_end = max(prev_end or 0.0, b)
            gaps[name] += gap
        busy[name] += b - a
        cnt[name] += 1
        lines.append(f"{name:14s} start {a * 1e3:10.1f} us  dur {1e3 * (b - a):8.1f} us" +
                     (f"  gap {1e3 * gap:7.1f} us" if gap is not None else "  (stream 2)"))
    total = tl[-1][2] - tl[0][1] if tl else 0.0
    lines.append(f"\nconfig {args.config} ({wl['name']}): {args.cycles} cycles in {total:.3f} ms")
    lines.append(f"{'kernel':14s} {'launches':>8s} {'busy us':>10s} {'us/launch':>10s} {'gaps before, us':>16s}")
    for k in busy:
        lines.append(f"{k:14s} {cnt[k]:8d} {1e3 * busy[k]:10.1f} {1e3 * busy[k] / cnt[k]:10.1f} {1e3 * gaps.get(k, 0.0):16.1f}")
    lines.append(f"main-stream idle (sum of gaps): {1e3 * sum(gaps.values()):.1f} us")
    txt = "\n".join(lines)
    print(txt)
    if args.out:
        with open(args.out, "w") as f:
            f.write(txt + "\n")
    ctx.close()


if __name__ == "__main__":
    main()
