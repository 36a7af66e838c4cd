#!/usr/bin/env python
"""Benchmark: restarted cl-BGMRES with BCGS-PIP block Arnoldi on B200 (BASELINE.json metric
"block Arnoldi steps/s and fp64 HBM GB/s (% roofline) at 1/2/4/8 B200").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]

* Workload: BASELINE.json configs[4] = config 5, the 3D 7-point Laplacian on a 256^3 grid
  (n = 16,777,216, s = 8, m = 40, tau = 1e8), the largest configuration and the one BASELINE
  quotes at 1/2/4/8 GPUs.  --config 2/3/4 bench the other BASELINE configs.
* A bench "step" is one restart cycle of the solver: IO(U) + m block Arnoldi steps (SpMM,
  fused single-sync Gram, Cholesky, projection, estimates) + the cycle-end projected solve and
  the X/U update, i.e. every row of SURVEY.md 8(a).  K cycles run inside ONE
  lsba_bgmres_solve call (max_restarts = K-1) from X0 = 0 at the real tol 1e-8 (config 5 needs
  ~88 cycles, so none of the timed cycles converges).  Configs 1
  and 4 converge in a few cycles: there a step is one full solve.
* value = whole-job algorithmic fp64 GB/s: sum over steps of ROOF(k) = 12 nnz + 4(n+1)
  + 8 n s (2k+3) plus 8 n s (k+7) per cycle, divided by the max-over-ranks
  device time.  block_steps_per_s is reported beside it.
* N > 1: STRONG scaling of the same global problem: contiguous row ranges (whole z-planes for
  the stencils), each rank holding its rows of A, B and the basis; per block step one halo
  exchange and exactly one Gram allreduce.
* --impl reference: the oracle (oracle/, NumPy fp64, as it stands) on this box's host cores,
  on a bounded sample of the same workload per step (no reference implementation exists:
  /root/reference holds only the paper's text).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "block Arnoldi steps/s and fp64 HBM GB/s (% roofline) at 1/2/4/8 B200"
SAMPLE_ROWS = 1 << 20      # oracle samples: the leading 2^20 rows (16 planes of 256^2 for config 5)


def roof_step(nnz, n, s, k):
    """Algorithmic bytes of block step k: CSR A + basis read twice around the
    single sync + W written and read + V_{k+1} written."""
    return 12.0 * nnz + 4.0 * (n + 1) + 8.0 * n * s * (2 * k + 3)


def roof_cycle_extra(n, s, k_used):
    return 8.0 * n * s * (k_used + 7)


def ilu_bytes(nnz, n, s, iters):
    """ILU(0) left preconditioning (--prec ilu0): per operator application two triangular
    solves, each ~12 B per stored factor entry of its half (6 nnz in total), row pointers and
    the level order (8 B per row) and the block read + written once (16 ns)."""
    return iters * 2.0 * (6.0 * nnz + 8.0 * (n + 1) + 16.0 * n * s)


def l2_resident_csr(nnz, world):
    """Whether liblsba keeps this CSR in the persisting L2 set-aside (its rule: one rank, and
    col_idx + vals fit in the set-aside and in half of L2; LSBA_L2PERSIST=0 disables)."""
    if world != 1 or os.environ.get("LSBA_L2PERSIST") == "0":
        return False
    try:
        from cuda.bindings import runtime as rt
        _, maxp = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0)
        _, l2 = rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize, 0)
    except Exception:
        return False
    csr = 12 * nnz + 256
    return csr <= maxp and csr <= l2 // 2


def algorithmic_bytes(nnz, n, s, iters, cycles, gram_blocks, skel="pip"):
    """sum_steps ROOF(k) + per-cycle bytes, from the solver's counters (gram_blocks = sum over
    accepted steps of k+1).  BCGS-PIP: ROOF(k) = A + 8ns(2k+3), + 8ns(k_used+7) per cycle.
    BMGS-(I)CWY (Alg 6) and BCGS-IRO-LS (Alg 7): per step the SpMM of U (2 blocks), the Gram over [V_1..V_k U] and W
    (k+2) and the two-output pass (k+2 reads, 2 writes): A + 8ns(2k+8); per cycle IO (3), loop
    iteration 1 (7) and the cycle end (k_used+4): 8ns(k_used+14)."""
    A = 12.0 * nnz + 4.0 * (n + 1)
    blk = 8.0 * n * s
    if skel == "pip":
        return iters * (A + blk) + 2 * blk * gram_blocks + blk * (iters + 7 * cycles)
    if skel == "bmgs":     # per step: SpMM 2, k x (Gram 2 + update of W 3), IO 3: A + 8ns(5k+5)
        return iters * A + 5 * blk * gram_blocks + blk * (iters + 7 * cycles)
    if skel == "pio":      # per step: SpMM 2, Gram k+1, <W,W> 1, projection k+2: A + 8ns(2k+5)
        return iters * (A + 3 * blk) + 2 * blk * gram_blocks + blk * (iters + 7 * cycles)
    return iters * (A + 6 * blk) + 2 * blk * gram_blocks + blk * (iters + 14 * cycles)


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# --------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,power.draw")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(p[0]) for p in self.samples if p[0].replace(".", "").isdigit()]
        mx = [float(p[1]) for p in self.samples if p[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in self.samples for i in range(4) if p[2 + i].lower().startswith("active")})
        pw = []
        for p in self.samples:
            try:
                pw.append(float(p[6]))
            except (IndexError, ValueError):
                pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples),
                "power_w": statistics.median(pw) if pw else None}


# --------------------------------------------------------------------------- workload
def partition(n_global, world, rank, unit=1):
    """Contiguous row range of `rank`: whole units (z-planes for the stencils) split as evenly
    as possible, the first (units % world) ranks taking one more."""
    units = n_global // unit
    q, r = divmod(units, world)
    u0 = rank * q + min(rank, r)
    u1 = u0 + q + (1 if rank < r else 0)
    return u0 * unit, u1 * unit


def build_workload(config, rank, world, need_sha=True, rank_proxy=0):
    """The GLOBAL problem of BASELINE config `config` (strong scaling: the same A and B at
    every N), and this rank's rows of it.

    rank_proxy = P > 1 (one GPU, stencils only; tools/gpu_rank_proxy.sh): NOT a BASELINE
    workload -- the stencil on one rank's slab of a P-rank run (N^(d-1) x N/P grid, the same
    rows, nonzeros per row and block sizes as that rank's share; the neighbours' planes are
    cut off instead of exchanged), run as a one-rank problem so that one GPU can time the
    per-rank kernels at the P-rank size."""
    from lsba_inputs import CONFIGS, csr_sha256, random_sparse, rhs, stencil
    spec = dict(CONFIGS[config])
    s, m = spec["s"], spec["m"]
    sha = None
    if rank_proxy > 1:
        assert world == 1 and spec["kind"] == "stencil" and spec["N"] % rank_proxy == 0
        dims, N = spec["dims"], spec["N"]
        shape = (N,) * (dims - 1) + (N // rank_proxy,)
        A = stencil(dims, N, spec["v"], shape=shape)
        n = int(np.prod(shape))
        spec["name"] = f"{spec['name']}_slab_1of{rank_proxy}_proxy"
        return dict(name=spec["name"], n_global=n, row_begin=0, row_end=n, A=A,
                    B=np.ascontiguousarray(rhs(n, s)), s=s, m=m, tol=spec["tol"], tau=spec["tau"],
                    nnz=int(A[0][-1]), spec=spec, sha=csr_sha256(*A) if need_sha else None)
    if spec["kind"] == "stencil":
        dims, N = spec["dims"], spec["N"]
        n = N ** dims
        plane = N ** (dims - 1)                # rows of one slowest-dimension plane
        r0, r1 = partition(n, world, rank, plane)
        A = stencil(dims, N, spec["v"], rows=(r0, r1))
        nnz = n * (2 * dims + 1) - 2 * dims * (n // N)      # closed form
    else:
        n = spec["n"]
        r0, r1 = partition(n, world, rank)
        rp, ci, va = random_sparse(n)        # every rank builds the same matrix (seeded)
        nnz = int(rp[-1])
        A = (rp[r0:r1 + 1] - rp[r0], ci[rp[r0]:rp[r1]], va[rp[r0]:rp[r1]])
    if need_sha:
        sha = csr_sha256(*A)                 # = the global CSR's at N = 1
    B = np.ascontiguousarray(rhs(n, s)[r0:r1])   # this rank's rows of the global B
    return dict(name=spec["name"], n_global=n, row_begin=r0, row_end=r1, A=A, B=B, s=s, m=m,
                tol=spec["tol"], tau=spec["tau"], nnz=nnz, spec=spec, sha=sha)


def strict_json(o):
    """The line must be strict JSON: non-finite floats (a residual that was never computed, an
    infinite threshold) become null."""
    if isinstance(o, float):
        return o if np.isfinite(o) else None
    if isinstance(o, dict):
        return {k: strict_json(v) for k, v in o.items()}
    if isinstance(o, (list, tuple)):
        return [strict_json(v) for v in o]
    if isinstance(o, np.generic):
        return strict_json(o.item())
    return o


def workload_config(wl, n_gpus, ip="cl", skel="pip", prec="none"):
    """`config` of the JSON line: what identifies the workload and the method, identical in
    both arms (ours and --impl reference); what is specific to an arm goes under `run`."""
    n, s, m = wl["n_global"], wl["s"], wl["m"]
    return {"workload": wl["name"], "n": n, "nnz": int(wl["nnz"]), "s": s, "m": m, "tol": wl["tol"],
            "tau": wl["tau"] if np.isfinite(wl["tau"]) else None,     # None = no kappa_F trigger
            "method": f"{ip}-BGMRES, " + {"pip": "BCGS-PIP", "cwy": "BMGS-CWY", "icwy": "BMGS-ICWY",
                                          "irols": "BCGS-IRO-LS", "bmgs": "BMGS", "pio": "BCGS-PIO"}[skel]
                      + " skeleton, " + ("CholQR IO" if ip == "cl" else "global IO")
                      + (", left ILU(0)" if prec == "ilu0" else ""),
            "parallelism": f"rows-dp{n_gpus} (strong scaling: the same global problem, "
                           f"{'slabs of whole slowest-dimension planes' if wl['spec']['kind'] == 'stencil' else 'row blocks'})",
            "l2": f"inputs larger than L2 (the workload's basis: {8 * n * s * (m + 1) / 1e9:.2f} GB)"}


# --------------------------------------------------------------------------- oracle timing
def oracle_sample_problem(wl):
    """The bounded CPU sample: the leading principal submatrix of A on the first SAMPLE_ROWS
    rows (whole z-planes of the stencils: the same operator on a thinner slab) and those rows of
    B.  Returns (A_sample, B_sample, n_sample, nnz_sample, description)."""
    rp, ci, va = wl["A"]
    n = wl["B"].shape[0]
    ns = min(n, SAMPLE_ROWS)
    if ns == n:
        return (rp, ci, va), wl["B"], n, int(rp[-1]), f"all {n} rows"
    p1 = int(rp[ns])
    keep = ci[:p1] < ns
    rows = np.repeat(np.arange(ns), np.diff(rp[:ns + 1]))
    counts = np.bincount(rows[keep], minlength=ns)
    rps = np.zeros(ns + 1, dtype=np.int64)
    np.cumsum(counts, out=rps[1:])
    A = (rps, ci[:p1][keep], va[:p1][keep])
    return A, np.ascontiguousarray(wl["B"][:ns]), ns, int(rps[-1]), \
        f"leading principal {ns} x {ns} submatrix ({ns / n:.4g} of the rows) and those rows of B"


def oracle_sample(A, B, nnz, m, budget_s, plain_gram=False):
    """Time the oracle (as it stands) on a bounded sample: IO(B) and the first block steps of one
    cycle until ~budget_s.  plain_gram: the same oracle with its near-exactly rounded Gram
    replaced by one BLAS X^T Y (the fair CPU speed variant of BASELINE.md 3)."""
    from oracle import lsba_oracle as O
    n, s = B.shape
    g0 = O.gram
    if plain_gram:
        O.gram = lambda X, Y, chunk_rows=0: np.asarray(X, dtype=np.float64).T @ np.asarray(Y, dtype=np.float64)
    try:
        arn = O.PipArnoldi(A, "cl", m, s)
        t0 = time.perf_counter()
        arn.begin(B)
        steps, byts = 0, roof_cycle_extra(n, s, 0)
        while steps < m:
            arn.step()
            steps += 1
            byts += roof_step(nnz, n, s, steps)
            if time.perf_counter() - t0 > budget_s:
                break
        dt = time.perf_counter() - t0
    finally:
        O.gram = g0
    return dict(seconds=dt, steps=steps, bytes=byts)


def cpu_baseline_legs(wl, budget_s=6.0):
    """the oracle on this host with BLAS threads = all cores and = 1, with the
    accurate (parity) Gram and the plain-BLAS Gram, plus the full tiny-config solve."""
    from threadpoolctl import threadpool_limits
    from lsba_inputs import make_twin
    from oracle import lsba_oracle as O
    A, B, ns, nnz_s, desc = oracle_sample_problem(wl)
    cores = host_cores()
    legs = {}
    for gram_kind in ("plain", "accurate"):
        for thr in (cores, 1):
            with threadpool_limits(thr):
                r = oracle_sample(A, B, nnz_s, wl["m"], budget_s, plain_gram=(gram_kind == "plain"))
            legs[f"{gram_kind}_gram_{'all' if thr == cores else 1}_threads"] = {
                "GBps": r["bytes"] / r["seconds"] / 1e9, "block_steps_per_s": r["steps"] / r["seconds"],
                "s_per_block_step": r["seconds"] / max(1, r["steps"]), "threads": thr,
                "seconds": round(r["seconds"], 2), "steps": r["steps"]}
    p = make_twin(1)
    t0 = time.perf_counter()
    _, io = O.solve((p.row_ptr, p.col_idx, p.vals), p.B, m=p.m, tol=p.tol, max_restarts=p.max_restarts,
                    ip="cl", mod="gmres")
    tiny = {"seconds": time.perf_counter() - t0, "cycles": io.cycles, "iterations": io.iterations,
            "workload": p.name, "outcome": int(io.outcome)}
    # the fair CPU speed baseline: the plain-BLAS Gram, at the faster of its two thread counts
    fair_name = max(("plain_gram_all_threads", "plain_gram_1_threads"), key=lambda k: legs[k]["GBps"])
    fair = legs[fair_name]
    return {"value": fair["GBps"], "unit": "GB/s", "cores": fair["threads"], "kind": "oracle",
            "host_cores": cores, "fair_leg": fair_name,
            "block_steps_per_s": fair["block_steps_per_s"], "cpu_model": cpu_model(),
            "sample": f"oracle IO + first block steps of one cycle (~{budget_s:.0f} s per leg) on the {desc} "
                      f"of {wl['name']}; GB/s with the same ROOF(k) numerator at the sample's n, nnz",
            "legs": legs, "tiny_full_solve": tiny}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    wl = build_workload(args.config, 0, 1, need_sha=False)
    A, B, ns, nnz_s, desc = oracle_sample_problem(wl)
    per_step_budget = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    tot_s, tot_b, tot_steps = 0.0, 0.0, 0
    for _ in range(args.warmup):
        oracle_sample(A, B, nnz_s, wl["m"], per_step_budget / 4)
    for _ in range(args.steps):                 # the oracle as it stands, default BLAS threads
        r = oracle_sample(A, B, nnz_s, wl["m"], per_step_budget)
        tot_s += r["seconds"]
        tot_b += r["bytes"]
        tot_steps += r["steps"]
    gbs = tot_b / tot_s / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "block_steps_per_s": tot_steps / tot_s,
        "config": workload_config(wl, args.gpus),
        "run": {"implementation": "cl-BCGS-PIP block Arnoldi (oracle, NumPy fp64, accurate Gram)",
                "timed_unit": f"bounded sample: IO + the first block steps of one cycle on the {desc}"},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": host_cores(), "kind": "oracle",
                         "cpu_model": cpu_model(),
                         "sample": f"{tot_steps} block steps over {args.steps} samples of config {args.config} "
                                   f"({desc})"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(strict_json(line), allow_nan=False), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--repeats", type=int, default=5, help="timed regions of K steps (PAPER.md:424: mean of 5)")
    ap.add_argument("--variant", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the fixed-k step sweep")
    ap.add_argument("--no-tts", action="store_true", help="skip the full time-to-solution run")
    ap.add_argument("--rank-proxy", type=int, default=0,
                    help="one-GPU diagnostic, not a BASELINE workload: time one rank's slab of a P-rank "
                         "stencil run as a one-rank problem (see build_workload)")
    ap.add_argument("--ip", default="cl", choices=["cl", "gl"], help="block inner product (Table 1)")
    ap.add_argument("--prec", default="none", choices=["none", "ilu0"],
                    help="left ILU(0) preconditioning (SURVEY 8(f) f4); factored before the timed region")
    ap.add_argument("--skel", default="pip", choices=["pip", "cwy", "icwy", "irols", "bmgs", "pio"],
                    help="Gram-Schmidt skeleton: BCGS-PIP (Alg 3), BMGS-CWY / -ICWY (Alg 6), BCGS-IRO-LS "
                         "(Alg 7), or the comparison baselines BMGS (Alg 2) and BCGS-PIO (Alg 4)")
    args = ap.parse_args()
    assert args.warmup >= 0 and args.steps >= 1 and args.repeats >= 1

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    import paper_2208_09899_b200 as L
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    wl = build_workload(args.config, rank, world, rank_proxy=args.rank_proxy)
    nccl_id = None
    if world > 1:
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(L.lsba_get_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().numpy().tobytes())
    stream = torch.cuda.current_stream()
    ctx = L.Context(wl["n_global"], wl["s"], wl["m"], *wl["A"], row_begin=wl["row_begin"],
                    row_end=wl["row_end"], rank=rank, nranks=world, nccl_id=nccl_id, device=local,
                    stream=stream.cuda_stream)
    L.lsba_set_kernel_variant(ctx.ctx, args.variant)
    L.lsba_set_skeleton(ctx.ctx, args.skel)
    if args.prec == "ilu0":
        L.lsba_ilu0_setup(ctx.ctx, True)
    B = torch.from_numpy(wl["B"]).cuda()
    X = torch.zeros_like(B)
    m, tol, s, tau = wl["m"], wl["tol"], wl["s"], wl["tau"]
    n_loc, n_glob = wl["row_end"] - wl["row_begin"], wl["n_global"]

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def solve(max_restarts):
        return L.lsba_bgmres_solve(ctx.ctx, B, X, m, tol, max_restarts, ip=args.ip, cond_threshold=tau,
                                   skel=args.skel)

    # warm-up: W cycles (one solve call), not timed
    if args.warmup:
        X.zero_()
        solve(args.warmup - 1)
    barrier()

    # configs 1 and 4 converge in a few cycles: a bench step is then one full solve from X0 = 0
    full_solve = wl["spec"].get("max_restarts", 0) <= 50 or args.config == 4

    def timed_cycles(profile):
        """K cycles in one solve call from X0 = 0 (or K full solves), CUDA events on the
        library's stream, max over ranks.  Returns (iterations, cycles, ms, profile, info)."""
        L.lsba_profile_enable(ctx.ctx, profile)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        X.zero_()
        barrier()
        e0.record(stream)
        it = cy = nl = gb = 0
        for i in range(args.steps if full_solve else 1):
            if full_solve and i:
                X.zero_()
            inf = solve(200 if full_solve else args.steps - 1)
            it += inf.iterations
            cy += inf.cycles
            nl += inf.kernel_launches
            gb += inf.gram_blocks
        timed_cycles.launches = nl
        timed_cycles.gram_blocks = gb
        e1.record(stream)
        torch.cuda.synchronize()
        t_ms = max_over_ranks(e0.elapsed_time(e1))
        pr = {k: L.lsba_profile_read(ctx.ctx, k) for k in L.KERNEL_IDS} if profile else None
        L.lsba_profile_enable(ctx.ctx, False)
        return it, cy, t_ms, pr, inf

    def region_bytes(iters, cycles, gram_blocks):
        b = algorithmic_bytes(wl["nnz"], n_glob, s, iters, cycles, gram_blocks, args.skel)
        if args.prec == "ilu0":
            b += ilu_bytes(wl["nnz"], n_glob, s, iters)
        return b

    # headline: un-instrumented (a CUDA event around every launch costs ~2 us of GPU idle each);
    # then args.repeats - 1 more identical regions (mean / min); then the same K
    # cycles once more with per-launch events for the per-kernel times behind `roofline`
    clocks = ClockSampler(local)
    clocks.start()
    iters, cycles, ms, _, info = timed_cycles(False)
    launches = timed_cycles.launches
    total_bytes = region_bytes(iters, cycles, timed_cycles.gram_blocks)
    reps = [total_bytes / (ms / 1e3) / 1e9]
    reps_ms = [ms]
    for _ in range(args.repeats - 1):
        it_r, cy_r, ms_r, _, _ = timed_cycles(False)
        reps.append(region_bytes(it_r, cy_r, timed_cycles.gram_blocks) / (ms_r / 1e3) / 1e9)
        reps_ms.append(ms_r)
    clk = clocks.stop()
    _, _, ms_prof, prof, _ = timed_cycles(True)
    if not full_solve:
        assert cycles == args.steps, f"expected {args.steps} cycles, ran {cycles} (outcome {info.outcome})"
    gbs = reps[0]
    steps_per_s = iters / (ms / 1e3)
    peak, peak_kind = measured_peaks()

    # dominant kernel roofline (local rank's launches; per-launch averages)
    # the step's time = the kernels of the main stream, which run back to back; the update
    # kernel runs concurrently on stream 2 and its event pair brackets its wait for the Gram,
    # so its "time" is not part of the step (the ncu launch list, which serialises every
    # launch, gives it ~1% of the step)
    tot_ms = sum(v[1] for k, v in prof.items() if k != "step_update")
    # dominant kernel: the largest summed time among the kernels that move the step's bytes
    # (the 1-CTA update kernel runs concurrently on stream 2, off the critical path)
    dom = max((k for k in prof if prof[k][2] > 0), key=lambda k: prof[k][1])
    dn, dms, dbytes = prof[dom]
    achieved = dbytes / (dms / 1e3) / 1e9 if dms > 0 else 0.0
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic_per_launch.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(f"config{args.config}", {}).get(dom)
        except Exception:
            traffic = None

    # fixed-k step sweep: one Arnoldi cycle through the step API (one
    # lsba_block_arnoldi_step call per step, each reading its status word), CUDA events around
    # every step; ROOF(k) / time at k = 1, m/2, m
    sweep = None
    if not args.no_sweep and args.skel == "pip" and args.prec == "none":
        L.lsba_set_skeleton(ctx.ctx, "pip")
        X.zero_()
        barrier()
        ctx.begin(B, args.ip)
        per_k = {}
        for k in range(1, m + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            si = ctx.step()
            e1.record(stream)
            torch.cuda.synchronize()
            if si.chol_flag:
                break
            per_k[k] = max_over_ranks(e0.elapsed_time(e1))
        sweep = {}
        for k in sorted({1, max(1, m // 2), m}):
            if k in per_k:
                t = per_k[k]
                sweep[f"k={k}"] = {"ms": round(t, 4), "GBps": roof_step(wl["nnz"], n_glob, s, k) / (t / 1e3) / 1e9,
                                   "roof_bytes": roof_step(wl["nnz"], n_glob, s, k)}
        sweep["note"] = ("one step of the step API per k (its status read after each step adds "
                         "~10 us of launch latency per step); ROOF(k) / step time")

    # e2e through the public API with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e:
        Bh = torch.from_numpy(wl["B"]).pin_memory().numpy()
        Xh = torch.zeros(B.shape, dtype=torch.float64).pin_memory().numpy()
        # untimed warm-up call: allocates the library's device staging buffers once
        L.lsba_solve_host(ctx.ctx, Bh, Xh, m, tol, 0, ip=args.ip, cond_threshold=tau)
        Xh[:] = 0.0
        barrier()
        t0 = time.perf_counter()
        e2e_iters = e2e_cycles = e2e_gb = 0
        e2e_calls = []
        for _ in range(args.steps):
            if full_solve:
                Xh[:] = 0.0
            ih = L.lsba_solve_host(ctx.ctx, Bh, Xh, m, tol, 200 if full_solve else 0, ip=args.ip,
                                   cond_threshold=tau)
            e2e_calls.append(ih.seconds)
            e2e_iters += ih.iterations
            e2e_cycles += ih.cycles
            e2e_gb += ih.gram_blocks
        torch.cuda.synchronize()
        dt = max_over_ranks(time.perf_counter() - t0)
        e2e = {"value": region_bytes(e2e_iters, e2e_cycles, e2e_gb) / dt / 1e9, "unit": "GB/s",
               "block_steps_per_s": e2e_iters / dt,
               "h2d_bytes_per_step": 2 * n_glob * s * 8, "d2h_bytes_per_step": n_glob * s * 8,
               "api": "lsba_solve_host (" + ("one full solve per step, X0 = 0" if full_solve
                                             else "1 cycle per call, X0 = previous X") + ")",
               "ms_per_call": [round(1e3 * x, 3) for x in e2e_calls]}

    # time to solution: one full solve from X0 = 0 to tol (SURVEY.md 8(d) "separately, run the
    # full solve"); at N > 1 its counts must match N = 1's within the R20 rule
    tts = None
    if not args.no_tts and not full_solve:
        X.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        it = solve(wl["spec"]["max_restarts"])
        e1.record(stream)
        torch.cuda.synchronize()
        t = max_over_ranks(e0.elapsed_time(e1)) / 1e3
        tts = {"seconds": t, "outcome": int(it.outcome), "cycles": it.cycles, "iterations": it.iterations,
               "nan_flags": it.nan_flags, "cond_restarts": it.cond_restarts, "true_relres": it.true_relres,
               "block_steps_per_s": it.iterations / t,
               "GBps": region_bytes(it.iterations, it.cycles, it.gram_blocks) / t / 1e9}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_legs(wl)

    if rank == 0:
        line = {
            "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "block_steps_per_s": steps_per_s, "ms_per_block_step": ms / iters,
            "pct_roofline": {"of_measured_hbm": gbs / (peak * world), "of_8TBps_nominal": gbs / (8000.0 * world),
                             # the algorithmic bytes count A once per step; when the CSR is served
                             # from the persisting L2 set-aside those bytes never reach HBM
                             **({"of_measured_hbm_excluding_l2_resident_csr":
                                 gbs * (1.0 - 12.0 * wl["nnz"] * iters / total_bytes) / (peak * world)}
                                if l2_resident_csr(wl["nnz"], world) else {})},
            "repeats": {"n": len(reps), "GBps": [round(x, 1) for x in reps], "mean": statistics.mean(reps),
                        "min": min(reps), "max": max(reps),
                        "ms_per_step": [round(x / args.steps, 3) for x in reps_ms]},
            "config": workload_config(wl, world, args.ip, args.skel, args.prec),
            "run": {"implementation": "liblsba.so (sm_100a CUDA) through the C ABI",
                    "csr_sha256": wl["sha"] if world == 1 else None,
                    "csr_sha256_rank0_rows": wl["sha"] if world > 1 else None,
                    "timed_unit": (f"full solve to tol {tol} from X0 = 0 ({cycles / args.steps:.1f} cycles, "
                                   f"{iters / args.steps:.1f} block steps)") if full_solve
                                  else f"restart cycle = IO + {m} block steps + cycle end (K cycles from X0 = 0)",
                    "rows_rank0": [wl["row_begin"], wl["row_end"]],
                    "l2": f"inputs larger than L2 (basis {8 * n_loc * s * (m + 1) / 1e9:.2f} GB per rank)"
                          + (f"; the CSR ({12 * wl['nnz'] / 1e6:.0f} MB) is kept in the persisting L2 set-aside"
                             if l2_resident_csr(wl["nnz"], world) else "")},
            "roofline": {"bound": "hbm", "kernel": dom,
                         **({"note": "level-scheduled triangular solves: latency-bound (one dependency "
                                     "level after another), reported against the HBM roof"}
                            if dom == "ilu_solve" else {}), "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_kind,
                         "peak_note": "peak = the measured COPY bandwidth (read + write); a read-mostly "
                                      "stream can exceed it (pure-read ceiling measured at 7.3 TB/s, "
                                      "profiles/r01_microbench.txt), so frac may pass 1",
                         "launches": dn, "kernel_share_of_step": dms / tot_ms if tot_ms else None,
                         "measured_in": "instrumented re-run of the same K cycles (per-launch CUDA events "
                                        f"on the launching streams; {ms_prof / args.steps:.3f} ms per cycle)"},
            "kernel_times_ms": {k: round(v[1], 3) for k, v in prof.items() if v[0]},
            "kernel_gbs": {k: round(v[2] / (v[1] / 1e3) / 1e9, 1) for k, v in prof.items() if v[1] > 0 and v[2] > 0},
            "step_sweep": sweep,
            "gpu_launches": int(launches),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "time_to_solution": tts,
            "solver": {"cycles": cycles, "iterations": iters, "nan_flags": info.nan_flags,
                       "res_est_rel": info.res_est, "true_relres": info.true_relres},
        }
        print(json.dumps(strict_json(line), allow_nan=False), flush=True)
    ctx.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
