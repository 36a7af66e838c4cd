#!/usr/bin/env python
"""In-situ A/B of library switches read at lsba_create (environment variables), interleaved in
ONE process so every variant sees the same box, clock regime and workload.

  python tools/ab_env.py --config 2 --cycles 3 --rounds 3 "LSBA_PROJ_PF_MB=0" "LSBA_PROJ_PF_MB=24"

Per round and variant: a fresh context with the variant's environment, one warm-up cycle, then
K cycles of the real solve from X0 = 0 in one lsba_bgmres_solve call, timed with CUDA events on
the library's stream; GB/s = bench.algorithmic_bytes / time (the bench's numerator)."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2208_09899_b200 as L  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--cycles", type=int, default=3)
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--ip", default="cl")
    ap.add_argument("variants", nargs="+", help='"VAR=V,VAR2=W" per variant ("-" = defaults)')
    a = ap.parse_args()
    torch.cuda.set_device(0)
    wl = bench.build_workload(a.config, 0, 1, need_sha=False)
    B = torch.from_numpy(wl["B"]).cuda()
    X = torch.zeros_like(B)
    stream = torch.cuda.current_stream()
    full = a.config in (1, 4)
    res = {v: [] for v in a.variants}
    base_env = dict(os.environ)
    for r in range(a.rounds):
        for v in a.variants:
            os.environ.clear()
            os.environ.update(base_env)
            if v != "-":
                for kv in v.split(","):
                    k, val = kv.split("=", 1)
                    os.environ[k] = val
            ctx = L.Context(wl["n_global"], wl["s"], wl["m"], *wl["A"], stream=stream.cuda_stream)

            def solve(mr):
                return L.lsba_bgmres_solve(ctx.ctx, B, X, wl["m"], wl["tol"], mr, ip=a.ip,
                                           cond_threshold=wl["tau"])
            X.zero_()
            solve(0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            X.zero_()
            e0.record(stream)
            it = cy = gb = 0
            for i in range(a.cycles if full else 1):
                if i:
                    X.zero_()
                inf = solve(200 if full else a.cycles - 1)
                it += inf.iterations
                cy += inf.cycles
                gb += inf.gram_blocks
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            gbs = bench.algorithmic_bytes(wl["nnz"], wl["n_global"], wl["s"], it, cy, gb) / (ms / 1e3) / 1e9
            res[v].append(gbs)
            print(f"round {r} {v:40s} {gbs:8.1f} GB/s  {ms:9.3f} ms  it {it} cy {cy}", flush=True)
            ctx.close()
            torch.cuda.synchronize()
    os.environ.clear()
    os.environ.update(base_env)
    for v in a.variants:
        print(f"config {a.config} {v:40s} mean {statistics.mean(res[v]):8.1f}  max {max(res[v]):8.1f}  "
              f"all {[round(x) for x in res[v]]}")


if __name__ == "__main__":
    main()
