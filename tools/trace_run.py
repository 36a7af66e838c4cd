#!/usr/bin/env python
"""Timeline of one restart cycle from a trace build (LSBA_NVCC_EXTRA=-DLSBA_TAIL_TRACE):
per block step, when block 0 of the SpMM / Gram / projection became resident (entry, before its
PDL wait) and when its wait returned, and the Gram's tail stamps, all relative to the step's
SpMM wait-return.

  python tools/trace_run.py --config 2"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_09899_b200 as L  # noqa: E402
from paper_2208_09899_b200 import _lib  # noqa: E402

NAMES = {8: "spmm.last_exit", 9: "proj.last_exit", 2: "spmm.entry", 3: "spmm.wait", 4: "gram.entry", 5: "gram.wait", 6: "proj.entry", 7: "proj.wait",
         10: "tail.loop_end", 11: "tail.grp_last", 12: "tail.final", 13: "tail.small_start", 14: "tail.end",
         20: "sc.entry", 21: "sc.G", 22: "sc.S", 23: "sc.chol", 24: "sc.end"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    a = ap.parse_args()
    dump = _lib.lib.lsba_trace_dump
    dump.restype = C.c_int
    dump.argtypes = [C.c_void_p, C.c_int]
    torch.cuda.set_device(0)
    wl = bench.build_workload(a.config, 0, 1, need_sha=False)
    B = torch.from_numpy(wl["B"]).cuda()
    X = torch.zeros_like(B)
    ctx = L.Context(wl["n_global"], wl["s"], wl["m"], *wl["A"])
    L.lsba_bgmres_solve(ctx.ctx, B, X, wl["m"], wl["tol"], 0, cond_threshold=wl["tau"])
    dump(None, 0)
    X.zero_()
    L.lsba_bgmres_solve(ctx.ctx, B, X, wl["m"], wl["tol"], 0, cond_threshold=wl["tau"])
    buf = np.zeros(1 << 18, dtype=np.uint64)
    n = dump(buf.ctypes.data, buf.size)
    rec = buf[:n].reshape(-1, 2)
    ev = sorted((int(t), int(w) >> 32, int(w) & 0xffffffff) for t, w in rec)
    t0 = ev[0][0]
    steps, cur = [], None
    for t, tag, J in ev:
        if tag == 3:                           # a step starts at its SpMM's wait-return
            cur = {"t": t}
            steps.append(cur)
        if cur is not None:
            cur.setdefault(NAMES.get(tag, str(tag)), t)
    print(f"config {a.config}: {len(ev)} records, {len(steps)} steps; times in us from the step's SpMM wait-return")
    cols = ["spmm.last_exit", "gram.entry", "gram.wait", "tail.loop_end", "tail.final", "tail.small_start",
            "tail.end", "proj.entry", "proj.wait", "proj.last_exit"]
    print("step " + " ".join(f"{c:>15s}" for c in cols) + "      next spmm.wait")
    for i, st in enumerate(steps):
        nxt = steps[i + 1]["t"] if i + 1 < len(steps) else None
        vals = [(st[c] - st["t"]) / 1e3 if c in st else float("nan") for c in cols]
        print(f"{i:4d} " + " ".join(f"{v:15.2f}" for v in vals) +
              (f"  {(nxt - st['t']) / 1e3:15.2f}" if nxt else ""))
    gaps = [(st["proj.wait"] - st["tail.end"]) / 1e3 for st in steps if "proj.wait" in st and "tail.end" in st]
    if gaps:
        gaps.sort()
        print(f"median gap tail.end -> proj.wait {gaps[len(gaps) // 2]:.2f} us")
    g2 = sorted((st["gram.wait"] - st["spmm.last_exit"]) / 1e3 for st in steps if "spmm.last_exit" in st and "gram.wait" in st)
    if g2:
        print(f"median gap spmm.last_exit -> gram.wait {g2[len(g2) // 2]:.2f} us")
    g3 = []
    for i in range(len(steps) - 1):
        a, b = steps[i], steps[i + 1]
        if "proj.last_exit" in a:          # (stamped before the next step's SpMM wait-return)
            g3.append((b["t"] - a["proj.last_exit"]) / 1e3)
    if g3:
        g3.sort()
        print(f"median gap proj.last_exit -> spmm.wait {g3[len(g3) // 2]:.2f} us")
    sc = [st for st in steps if "sc.end" in st and "sc.entry" in st]
    if sc:
        print("fused small step phases (us): G->smem  S  chol+Rinv  coef+stores  (median over steps)")
        keys = ["sc.entry", "sc.G", "sc.S", "sc.chol", "sc.end"]
        med = []
        for a, b in zip(keys, keys[1:]):
            v = sorted((st[b] - st[a]) / 1e3 for st in sc if a in st and b in st)
            med.append(v[len(v) // 2] if v else float("nan"))
        print("   " + "  ".join(f"{x:.2f}" for x in med))
    ctx.close()


if __name__ == "__main__":
    main()
