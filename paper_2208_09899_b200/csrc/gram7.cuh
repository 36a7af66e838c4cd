// gram7.cuh — the single-sync Gram pass G = <[X_0 .. X_{J-1}], Y> (Alg 3 line 4,
// PAPER.md:268-269) as a latency-tuned streaming kernel on the FP64 tensor cores.
//
// Design rules measured on B200 (tools/microbench.cu, profiles/r01_microbench.md):
//   * DMMA m8n8k4.f64 and DFMA both run at 64 MAC/clk/SM (37 TF/s): DMMA is used for its
//     register efficiency (an 8x8 fp64 accumulator is 2 doubles per lane), not for flops;
//   * a read stream reaches 7.3 TB/s only with >= 64 KB in flight per SM spread over
//     >= 16 warps; 8 warps per SM cap it near 3.9 TB/s whatever the unroll.
// So: no shared-memory tiles and no barriers in the main loop; each warp keeps U 4-row steps
// of loads in flight (issued together, then consumed), register budget sized for MINB CTAs of
// 256 threads per SM; the CTA partial is reduced through shared memory in one ordered pass
// and the cross-CTA reduction is a deterministic two-level ticketed tree.
//
// Fragment mapping (as v5/v6): lane (r4 = lane & 3, c8 = lane >> 2) loads a 16-byte column
// pair (2cp, 2cp+1) of row r4 of a block and feeds two DMMAs (M tile "even" columns, M tile
// "odd" columns); a group packs PB = 16/S blocks (S <= 8) into the 8 M rows; W (B operand) is
// W[r4][c8 (+8 tn)].  Inputs are basis slots (rows padded to kRowPad with zero rows).
#pragma once
#include <algorithm>

#include <nccl.h>
#include <nccl_device.h>

#include "dmma.cuh"
#include "small.cuh"

namespace lsba {

constexpr int kMaxGramPasses = 64;  // ticket sets allocated per context (one per pass)

// Fused small step: on a single rank the Gram's last-finishing CTA goes straight on with
// Alg 3 line 5 (S = Omega - H^T H, Cholesky + NaN-flag, R^-1, projection coefficients;
// step_coef_body of small.cuh) instead of a separate 1-CTA launch.
// The fused small step as a real call for s = 16: inlined, its 16 x 16 register arrays would
// raise the register demand (and spills) of the streaming loop above it.
template <int B>
__device__ __noinline__ void step_coef_noinline(const SmallState2& st, const double* G, double* Gs, int k,
                                                const CycleParams& prm, bool g_ready, int pre_force) {
  step_coef_body<B>(st, G, Gs, k, prm, 1.0, g_ready, pre_force);
}

#ifdef LSBA_TAIL_TRACE
// diagnostics build only: stamps of the Gram's tail, recorded by the CTA that runs the small step
#define G7T(i) do { if (tid == 0) tt[i] = gtime(); } while (0)
#else
#define G7T(i) do { } while (0)
#endif

// Ordered sum over c < cnt of p[c * stride] (c ascending, the same rounding as a plain loop);
// the loads are issued BATCH at a time so the sum costs a few L2 round trips, not cnt of them
// (the final level's 37 group partials: 2 round trips with batches of 20 instead of 3 with 16).
template <int BATCH = 16>
__device__ __forceinline__ double ordered_partial_sum(const double* p, size_t stride, int cnt) {
  double s = 0.0;
  for (int c0 = 0; c0 < cnt; c0 += BATCH) {
    double v[BATCH];
#pragma unroll
    for (int c = 0; c < BATCH; ++c) v[c] = (c0 + c < cnt) ? __ldcg(p + (size_t)(c0 + c) * stride) : 0.0;
#pragma unroll
    for (int c = 0; c < BATCH; ++c)
      if (c0 + c < cnt) s += v[c];
  }
  return s;
}

// Ticket increment with acquire-release semantics at GPU scope, by one thread after a CTA
// barrier: the release half publishes every write the CTA made before the barrier (barrier
// cumulativity), the acquire half (for the CTA that draws the last ticket) makes the other
// CTAs' published partials visible to this CTA after the next barrier.  Replaces a full
// __threadfence in every thread on both sides (the cooperative-groups grid-sync pattern).
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* p) {
  unsigned r;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(r) : "l"(p) : "memory");
  return r;
}

struct GramFuse {
  SmallState2 st;
  CycleParams prm;
  int k;    // step index (0 = IO)
  int on;   // 0: plain Gram
  // f2: the P > 1 allreduce folded into the tail (NCCL device API; LSBA_DEVAR=1)
  int ar;                 // 1: sum the ranks' G through the symmetric window below
  size_t woff;            // byte offset of this Gram's slot in the window (alternating slots)
  ncclWindow_t win;
  const ncclDevComm* dcomm;   // device copy (a pointer: the kernel parameter block stays small
                              // and is never addressed, which would copy it to local memory)
  // Device-side join of the previous step's update kernel (stream 2; one rank, v7 only): the
  // main stream does not wait on its event, so this Gram launches programmatically behind the
  // SpMM; the CTA that runs the small step acquires *upd_done >= upd_seq first.  Until then
  // the cycle control may still change, so CTAs that see the cycle ended skip their rows but
  // keep the ticket protocol, and the tail re-reads the control after the join.
  int upd_wait;
  unsigned upd_seq;
  const unsigned* upd_done;
};

// Spin (one thread) until the update kernel carrying sequence `seq` has exited.  The update
// kernel was made ready before this Gram's SpMM and runs on a high-priority stream, so it
// holds an SM long before this tail; the bound only turns a broken invariant into a fault
// instead of a hang.
__device__ __noinline__ void wait_update_seq(const unsigned* done, unsigned seq) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
  if ((int)(v - seq) >= 0) return;
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    __nanosleep(64);
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done) : "memory");
    if ((int)(v - seq) >= 0) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > 4000000000ull) __trap();
  }
}

// f2: the step's single sync folded into the Gram's tail
// through the NCCL device API.  The CTA that holds this rank's final G publishes it in its slot
// of a symmetric window, meets the other ranks at an LSA barrier (the NVLink load/store domain:
// one NVSwitch box), then sums every rank's G in rank order straight from their windows over
// NVLink — identical bits on every rank (equal to ncclAllReduce's for two ranks), no separate
// collective launch, and the small step stays fused into the same CTA as on one rank.  Slots
// alternate per call, so a rank never overwrites a slot a peer may still be reading (it passes
// the next call's barrier only after every peer has finished reading this one).
__device__ __noinline__ void gram_tail_allreduce(const ncclDevComm* dc, ncclWindow_t win, size_t woff, double* G,
                                                double* sm, int E, bool to_smem) {
  const int tid = threadIdx.x, nt = blockDim.x;
  double* mine = static_cast<double*>(ncclGetLsaPointer(win, woff, dc->lsaRank));
  for (int e = tid; e < E; e += nt) mine[e] = __ldcg(G + e);
  {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), *dc, ncclTeamTagLsa(), 0);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
  }
  const int P = dc->lsaSize;
  for (int e = tid; e < E; e += nt) {
    double t = 0.0;
    for (int r = 0; r < P; ++r)
      t += __ldcv(static_cast<const double*>(ncclGetLsaPointer(win, woff, r)) + e);
    G[e] = t;
    if (to_smem) sm[e] = t;
  }
  __syncthreads();
}

template <int S, int GMAX_, int U_, int MINB_, int NY_ = 1>
struct G7Cfg {
  static constexpr int PB = S >= 16 ? 1 : 16 / S;
  static constexpr int NY = NY_;                       // B-operand blocks: G = X^T [Y (Y2)]
  static constexpr int NCOL = NY * S;
  static constexpr int NT = (NCOL + 7) / 8;
  static constexpr int GMAX = GMAX_;
  static constexpr int U = U_;
  static constexpr int MINB = MINB_;
  static constexpr int NW = 8;
  static constexpr int NTHR = 256;
};

// Block groups of a J-block Gram: the J blocks (the last one is Y itself when y_alias) are
// packed PB per group in order; a launch covers the groups in `passes` contiguous ranges of
// at most 8 GMAX groups (blockIdx.x = pass + passes * row_chunk, so a chunk's passes run side
// by side and share the W rows through L2).
template <int S>
__host__ __device__ inline int g7_groups(int J) {
  constexpr int PB = S >= 16 ? 1 : 16 / S;
  return (J + PB - 1) / PB;
}
__host__ __device__ inline int g7_passes(int NG, int GMAX) { return (NG + 8 * GMAX - 1) / (8 * GMAX); }
__host__ __device__ inline int g7_qw(int ngp, int GMAX) {
  int QW = 1;
  while (QW < 8 && (ngp + QW - 1) / QW > GMAX) QW *= 2;
  return QW;
}

template <int S, int GMAX, int U, int MINB, bool WIN = true, int NY = 1>
__global__ void __launch_bounds__(256, MINB)
k_gram_v7(GramArgs g, GramFuse f) {
  using C = G7Cfg<S, GMAX, U, MINB, NY>;
  static_assert(S == 2 || S == 4 || S == 8 || S == 16, "v7 Gram: s in {2,4,8,16}");
  PDL_TRACE_ENTRY
  pdl_launch();
  extern __shared__ __align__(16) double sm7[];     // [RW][pass entries] row-slice partials
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = g.J, E = J * S * C::NCOL;
  const int NG = g7_groups<S>(J);
  const int passes = g7_passes(NG, C::GMAX);
  const int pass = blockIdx.x % passes, chunk = blockIdx.x / passes, nchunks = gridDim.x / passes;
  const int gp0 = (NG * pass) / passes, gp1 = (NG * (pass + 1)) / passes;
  const int QW = g7_qw(gp1 - gp0, C::GMAX);
  const int RW = C::NW / QW;
  const int rs = warp % RW, qs = warp / RW;
  const int gA = gp0 + ((gp1 - gp0) * qs) / QW, gB = gp0 + ((gp1 - gp0) * (qs + 1)) / QW;
  const int ng = gB - gA;
  const int jlo = gp0 * C::PB, jhi = min(J, gp1 * C::PB);   // blocks (entries) of this pass
  const long NS = ((long)g.n + 3) / 4;                 // 4-row steps (rows padded)
  if (g.pf_batches > 0 && tid == 0) {
    // Pre-wait prefetch: a CTA becomes resident as the SpMM drains; before waiting on it, the
    // rows of the basis blocks (constant during the step; not W, which the SpMM is writing)
    // that this CTA streams in its first pf_batches batches go to L2, so the stream starts at
    // once instead of after the SpMM's last CTA.  L2 only: never stale (kernels.cuh).
    const long bsteps = (long)C::U * RW;
    for (int i = 0; i < g.pf_batches; ++i) {
      const long st0 = WIN ? ((long)i * nchunks + chunk) * bsteps
                           : NS * chunk / nchunks + (long)i * bsteps;
      const long st1 = min(NS, min(st0 + bsteps, WIN ? NS : NS * (chunk + 1) / nchunks));
      if (st1 <= st0) break;
      for (int j = jlo; j < jhi; ++j) {
        const double* xj = g.X + (size_t)j * g.xstride;
        if (xj == g.Y) continue;
        bulk_prefetch_l2(xj + (size_t)st0 * 4 * S, 32L * S * (st1 - st0));
      }
    }
  }
  pdl_wait();
  PDL_TRACE_WAITED(kTrGram, J);
  TRACE_PREV_EXIT(0, 8);
  bool skip = false;                    // (device join: this CTA's rows are not needed)
  if (g.active && *g.active == 0) {     // speculative launch after the cycle ended: no-op
    if (!f.upd_wait) {
      if (f.on && blockIdx.x == 0 && threadIdx.x == 0) *f.st.flag_dev = 1;   // (projection no-ops)
      return;
    }
    skip = true;
  }
  // the fused small step's fault-injection state, read now (off the tail's critical path)
  int pre_force = (f.on && f.k > 0) ? ((f.k == f.st.ctl->force_k && !f.st.ctl->forced_done) ? 1 : 0) : 0;
#ifdef LSBA_TAIL_TRACE
  unsigned long long tt[8] = {};
#endif
  const uint64_t xpol = l2pol(c_l2hint & 2, false);
  const int e0 = jlo * S * C::NCOL, EP = (jhi - jlo) * S * C::NCOL;
  const int r4 = lane & 3, c8 = lane >> 2;
  constexpr int LPB = S >= 16 ? 8 : S / 2;
  const int jj = c8 / LPB, cp = c8 % LPB;

  const double* src[C::GMAX];
#pragma unroll
  for (int gi = 0; gi < C::GMAX; ++gi) {
    const int j = (gA + gi) * C::PB + (S >= 16 ? 0 : jj);
    src[gi] = (gi < ng && j < J) ? g.X + (size_t)j * g.xstride + r4 * S + 2 * cp : nullptr;
  }
  // B operand column tn*8 + c8 of [Y (Y2)] at row r4 of a step (nullptr: zero column)
  const double* wsrc[C::NT];
#pragma unroll
  for (int tn = 0; tn < C::NT; ++tn) {
    const int col = tn * 8 + c8;
    wsrc[tn] = (col < S) ? g.Y + r4 * S + col
                         : ((NY == 2 && col < 2 * S) ? g.Y2 + r4 * S + (col - S) : nullptr);
  }
  double acc[C::GMAX][2][C::NT][2];
#pragma unroll
  for (int a = 0; a < C::GMAX; ++a)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int tn = 0; tn < C::NT; ++tn) acc[a][e][tn][0] = acc[a][e][tn][1] = 0.0;

  // Row order ("windowed"): warp slice rs of chunk c takes the U consecutive steps starting at
  // ((i nchunks + c) RW + rs) U in its i-th batch, so the whole grid sweeps one moving window
  // of rows (few open DRAM pages, 16-row contiguous runs per block and warp).  Measured 3-8%
  // faster than per-CTA contiguous chunks with steps strided by RW (tools/gram_bench.cu).
  const long BS = (long)C::U * RW;                     // steps per chunk-batch
  const long GS = BS * nchunks;                        // steps per grid-batch
  (void)BS;
  // U 4-row steps per batch: load the batch's fragments, then run its DMMAs.
  auto mma_step = [&](const double2 (&av)[C::GMAX], const double (&bw)[C::NT]) {
#pragma unroll
    for (int gi = 0; gi < C::GMAX; ++gi) {
      if (gi >= ng) continue;
#pragma unroll
      for (int tn = 0; tn < C::NT; ++tn) {
        dmma(acc[gi][0][tn][0], acc[gi][0][tn][1], av[gi].x, bw[tn]);
        dmma(acc[gi][1][tn][0], acc[gi][1][tn][1], av[gi].y, bw[tn]);
      }
    }
  };
  if (skip) {
  } else if constexpr (WIN) {
    // windowed order (above): U consecutive steps per batch, the grid sweeping one window
    for (long st = ((long)chunk * RW + rs) * C::U; st < NS; st += GS) {
      double2 av[C::U][C::GMAX];
      double bw[C::U][C::NT];
      if (st + C::U <= NS) {                           // full batch: unpredicated loads
#pragma unroll
        for (int u = 0; u < C::U; ++u) {
          const size_t off = (size_t)(st + u) * 4 * S;
#pragma unroll
          for (int tn = 0; tn < C::NT; ++tn)
            bw[u][tn] = wsrc[tn] ? __ldg(wsrc[tn] + off) : 0.0;
#pragma unroll
          for (int gi = 0; gi < C::GMAX; ++gi)
            av[u][gi] = src[gi] ? ldh2(src[gi] + off, xpol) : make_double2(0.0, 0.0);
        }
      } else {                                         // the grid's last, ragged batch
#pragma unroll
        for (int u = 0; u < C::U; ++u) {
          const bool ok = st + u < NS;
          const size_t off = (size_t)(ok ? st + u : st) * 4 * S;
#pragma unroll
          for (int tn = 0; tn < C::NT; ++tn)
            bw[u][tn] = (ok && wsrc[tn]) ? __ldg(wsrc[tn] + off) : 0.0;
#pragma unroll
          for (int gi = 0; gi < C::GMAX; ++gi)
            av[u][gi] = (ok && src[gi]) ? ldh2(src[gi] + off, xpol)
                                        : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < C::U; ++u) mma_step(av[u], bw[u]);
    }
  } else {
    // per-CTA contiguous chunk, the steps of a batch strided by RW (s = 16: its DMMA load is 4x
    // that of s <= 8 and this order measured faster there)
    const long s0 = NS * chunk / nchunks, s1 = NS * (chunk + 1) / nchunks;
    long st = s0 + rs;
    for (; st + (long)(C::U - 1) * RW < s1; st += (long)C::U * RW) {
      double2 av[C::U][C::GMAX];
      double bw[C::U][C::NT];
#pragma unroll
      for (int u = 0; u < C::U; ++u) {
        const size_t off = (size_t)(st + (long)u * RW) * 4 * S;
#pragma unroll
        for (int tn = 0; tn < C::NT; ++tn)
          bw[u][tn] = wsrc[tn] ? __ldg(wsrc[tn] + off) : 0.0;
#pragma unroll
        for (int gi = 0; gi < C::GMAX; ++gi)
          av[u][gi] = src[gi] ? ldh2(src[gi] + off, xpol) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < C::U; ++u) mma_step(av[u], bw[u]);
    }
    for (; st < s1; st += RW) {                        // remainder steps, one at a time
      const size_t off = (size_t)st * 4 * S;
      double2 av[C::GMAX];
      double bw[C::NT];
#pragma unroll
      for (int tn = 0; tn < C::NT; ++tn) bw[tn] = wsrc[tn] ? __ldg(wsrc[tn] + off) : 0.0;
#pragma unroll
      for (int gi = 0; gi < C::GMAX; ++gi)
        av[gi] = src[gi] ? ldh2(src[gi] + off, xpol) : make_double2(0.0, 0.0);
      mma_step(av, bw);
    }
  }
  // CTA partial: each row slice writes its own slot (group sets are disjoint and cover the
  // pass), then one ordered sum over the RW slots (deterministic)
  for (int e = tid; e < RW * EP; e += C::NTHR) sm7[e] = 0.0;
  __syncthreads();
  double* mine = sm7 + (size_t)rs * EP - e0;
#pragma unroll
  for (int gi = 0; gi < C::GMAX; ++gi) {
    if (gi >= ng) continue;
    const int j = (gA + gi) * C::PB + (S >= 16 ? 0 : jj);
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int tn = 0; tn < C::NT; ++tn)
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int a = 2 * cp + e;
          const int bcol = tn * 8 + 2 * r4 + i;
          if (bcol < C::NCOL && j < J) mine[(j * S + a) * C::NCOL + bcol] = acc[gi][e][tn][i];
        }
  }
  __syncthreads();
  const int ngroups = (nchunks + kGramGroup - 1) / kGramGroup;
  const int grpi = chunk / kGramGroup;
  const int gsize = min(kGramGroup, nchunks - grpi * kGramGroup);
  unsigned* tk = g.tickets + (size_t)pass * (ngroups + 1);
  for (int e = tid; e < EP; e += C::NTHR) {
    double t = sm7[e];
    for (int r = 1; r < RW; ++r) t += sm7[(size_t)r * EP + e];
    g.part[(size_t)chunk * E + e0 + e] = t;
  }
  // ---- deterministic two-level reduction across the row chunks of this pass
  G7T(0);
  __syncthreads();
  __shared__ unsigned ticket7;
  if (tid == 0) ticket7 = ticket_acq_rel(&tk[grpi]);
  __syncthreads();
  if (ticket7 != (unsigned)(gsize - 1)) return;
  G7T(1);
  for (int e = e0 + tid; e < e0 + EP; e += C::NTHR)
    g.gpart[(size_t)grpi * E + e] = ordered_partial_sum(g.part + (size_t)grpi * kGramGroup * E + e, E, gsize);
  if (tid == 0) tk[grpi] = 0u;
  __syncthreads();
  if (tid == 0) ticket7 = ticket_acq_rel(&tk[ngroups]);
  __syncthreads();
  if (ticket7 != (unsigned)(ngroups - 1)) return;
  G7T(2);
  // one pass (and a fused small step): the final sums also go straight into shared memory,
  // where the small step reads G (no global round trip)
  const bool g_smem = f.on && passes == 1 && NY == 1;
  // device join (one pass): the CTA's last thread (idle in the final level when E < 256) waits
  // for the update and reads the control the small step needs while the others sum
  __shared__ int join7[2];
  const int jt = C::NTHR - 1;
  auto join_update = [&]() {
    wait_update_seq(f.upd_done, f.upd_seq);
    join7[0] = *(volatile const int*)g.active;
    join7[1] = (f.k > 0) ? ((f.k == f.st.ctl->force_k && !f.st.ctl->forced_done) ? 1 : 0) : 0;
  };
  if (f.upd_wait && passes == 1 && tid == jt) join_update();
  for (int e = e0 + tid; e < e0 + EP; e += C::NTHR) {
    const double s2 = ordered_partial_sum<20>(g.gpart + e, E, ngroups);
    g.G[e] = s2;
    if (g_smem) sm7[e] = s2;
  }
  if (tid == 0) tk[ngroups] = 0u;
  if (!f.on) return;
  // ---- fused small step, run by the CTA that completes the last pass
  if (passes > 1) {
    __syncthreads();
    unsigned* tpass = g.tickets + (size_t)kMaxGramPasses * (ngroups + 1);
    if (tid == 0) ticket7 = ticket_acq_rel(tpass);
    __syncthreads();
    if (ticket7 != (unsigned)(passes - 1)) return;
    if (tid == 0) *tpass = 0u;
  }
  if (f.upd_wait) {
    if (passes > 1 && tid == jt) join_update();
    __syncthreads();
    if (join7[0] == 0) {                 // the update ended the cycle meanwhile
      if (tid == 0) *f.st.flag_dev = 1;
      return;
    }
    pre_force = join7[1];
  }
  G7T(3);
  if (f.ar) {
    __syncthreads();
    gram_tail_allreduce(f.dcomm, f.win, f.woff, g.G, sm7, E, g_smem);
  }
  if constexpr (NY == 1) {
    if constexpr (S >= 16) step_coef_noinline<S>(f.st, g.G, sm7, f.k, f.prm, g_smem, pre_force);
    else step_coef_body<S>(f.st, g.G, sm7, f.k, f.prm, 1.0, g_smem, pre_force);
  }
#ifdef LSBA_TAIL_TRACE
  __syncthreads();
  if (tid == 0) {
    const unsigned long long t4 = gtime();
    for (int i = 0; i < 4; ++i) trace_rec(kTrTail + i, (unsigned)J, tt[i]);
    trace_rec(kTrTail + 4, (unsigned)J, t4);
  }
#endif
}

// ------------------------------------------------------------------------------------------
// Global block inner product (Table 1): g_j = (1/s) tr(X_j^T Y) = (1/s) sum of
// the elementwise products of two n x s blocks, for the J blocks of a step in ONE pass.  Each
// thread streams 16-byte pieces of Y and of up to JM blocks (the grid sweeps one window of the
// flattened blocks), keeping JM dot-product partials in registers; blocks beyond JM run as
// further passes over Y.  CTA partials: warp shuffle + ordered warp sum; cross-CTA: the same
// deterministic two-level ticketed tree as k_gram_v7; the small step can be fused the same way.
// Inputs are basis slots (rows padded to kRowPad with zero rows); S even.
// ------------------------------------------------------------------------------------------
constexpr int kGlJM = 8;

template <int S, int NY = 1>
__global__ void __launch_bounds__(256, 3)
k_gram_gl2(GramArgs g, GramFuse f) {
  static_assert(S % 2 == 0, "gl2: even s");
  pdl_begin();
  if (g.active && *g.active == 0) {
    if (f.on && blockIdx.x == 0 && threadIdx.x == 0) *f.st.flag_dev = 1;
    return;
  }
  __shared__ double red[8][kGlJM * NY];
  __shared__ double gsm[4 * kGlJM];     // fused small step (b = 1): (k+1) <= ... handled below
  __shared__ unsigned ticket;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = g.J, E = J * NY;                      // G[j NY + y] = <X_j, Y_y>
  const long npad = ((long)g.n + kRowPad - 1) / kRowPad * kRowPad;
  const long N2 = npad * S / 2;                       // double2 per block
  const long gstride = (long)gridDim.x * blockDim.x;
  const int P = gridDim.x;
  const int ngroups = (P + kGramGroup - 1) / kGramGroup;
  const int grpi = blockIdx.x / kGramGroup;
  const int gsize = min(kGramGroup, P - grpi * kGramGroup);
  const double2* Ya = reinterpret_cast<const double2*>(g.Y);
  const double2* Yb = reinterpret_cast<const double2*>(NY == 2 ? g.Y2 : g.Y);
  for (int j0 = 0; j0 < J; j0 += kGlJM) {
    const int nb = min(kGlJM, J - j0);
    double acc[kGlJM][NY];
#pragma unroll
    for (int q = 0; q < kGlJM; ++q)
#pragma unroll
      for (int y = 0; y < NY; ++y) acc[q][y] = 0.0;
    for (long e = (long)blockIdx.x * blockDim.x + tid; e < N2; e += gstride) {
      double2 yv[NY];
      yv[0] = __ldg(Ya + e);
      if constexpr (NY == 2) yv[NY - 1] = __ldg(Yb + e);
      double2 x0[kGlJM];
#pragma unroll
      for (int q = 0; q < kGlJM; ++q) {
        const double2* Xq = reinterpret_cast<const double2*>(g.X + (size_t)(j0 + q) * g.xstride);
        x0[q] = (q < nb) ? __ldg(Xq + e) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int q = 0; q < kGlJM; ++q)
#pragma unroll
        for (int y = 0; y < NY; ++y) {
          acc[q][y] = fma(x0[q].x, yv[y].x, acc[q][y]);
          acc[q][y] = fma(x0[q].y, yv[y].y, acc[q][y]);
        }
    }
#pragma unroll
    for (int q = 0; q < kGlJM; ++q)
#pragma unroll
      for (int y = 0; y < NY; ++y) {
        const double v = warp_sum(acc[q][y]);
        if (lane == 0) red[warp][q * NY + y] = v;
      }
    __syncthreads();
    if (tid < nb * NY) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w][tid];
      g.part[(size_t)blockIdx.x * E + j0 * NY + tid] = t;
    }
    __syncthreads();
  }
  __syncthreads();
  if (tid == 0) ticket = ticket_acq_rel(&g.tickets[grpi]);
  __syncthreads();
  if (ticket != (unsigned)(gsize - 1)) return;
  for (int e = tid; e < E; e += blockDim.x)
    g.gpart[(size_t)grpi * E + e] = ordered_partial_sum(g.part + (size_t)grpi * kGramGroup * E + e, E, gsize);
  if (tid == 0) g.tickets[grpi] = 0u;
  __syncthreads();
  if (tid == 0) ticket = ticket_acq_rel(&g.tickets[ngroups]);
  __syncthreads();
  if (ticket != (unsigned)(ngroups - 1)) return;
  for (int e = tid; e < E; e += blockDim.x)
    g.G[e] = ordered_partial_sum<20>(g.gpart + e, E, ngroups) * (1.0 / S);   // Table 1: (1/s) tr(X^T Y)
  if (tid == 0) g.tickets[ngroups] = 0u;
  (void)gsm;
  if (NY != 1 || !f.on) return;
  __syncthreads();                                    // (G written by this CTA: visible after the barrier)
  if (f.ar) gram_tail_allreduce(f.dcomm, f.win, f.woff, g.G, nullptr, E, false);
  extern __shared__ double gl2_dyn[];                 // (k+1) doubles for the small step
  step_coef_body<1>(f.st, g.G, gl2_dyn, f.k, f.prm, sqrt((double)S));
}

// launch geometry of k_gram_v7: grid (a multiple of the pass count) and dynamic smem bytes
template <int S, int GMAX, int NY = 1>
struct G7Launch {
  int passes, grid;
  size_t smem;
  G7Launch(int n, int J, int ctas_per_sm, int sms, bool fuse = false) {
    const int NG = g7_groups<S>(J);
    passes = g7_passes(NG, GMAX);
    int maxEP = 0, maxRW = 1;
    for (int p = 0; p < passes; ++p) {
      const int gp0 = NG * p / passes, gp1 = NG * (p + 1) / passes;
      const int ep = (std::min(J, gp1 * (S >= 16 ? 1 : 16 / S)) - gp0 * (S >= 16 ? 1 : 16 / S)) * S * S * NY;
      maxEP = std::max(maxEP, ep);
      maxRW = std::max(maxRW, 8 / g7_qw(gp1 - gp0, GMAX));
    }
    smem = sizeof(double) * (size_t)maxRW * maxEP;
    if (fuse) smem = std::max(smem, sizeof(double) * (size_t)J * S * S * NY);   // step_coef_body's Gs
    const long steps = ((long)n + 3) / 4;
    int chunks = std::max(1, ctas_per_sm * sms / passes);
    chunks = (int)std::max(1L, std::min<long>(chunks, (steps + 63) / 64));
    grid = chunks * passes;
  }
};

}  // namespace lsba
