// dmma.cuh — the two HBM passes of a BCGS-PIP step on the FP64 tensor cores (DMMA,
// mma.sync.aligned.m8n8k4.f64; tcgen05 has no fp64 kind).
//
//   k_spmm_gram<S>   pass 1: W = A V_k (CSR gather, W tile kept in shared memory and
//                    written once to its basis slot) fused with the single Gram
//                    G = [V_1 .. V_k W]^T W over the same rows (Alg 3 lines 3-4,
//                    PAPER.md:267-268), partial Gram per CTA, deterministic two-level
//                    cross-CTA reduction inside the kernel (fixed order: bitwise
//                    reproducible run to run and independent of CTA arrival order).
//   k_project_dmma<S> pass 2: out0 = base0 + sum_j X_j C0_j, out1 = sum_j X_j C1_j
//                    (Alg 3 line 6: V_{k+1} = [V_k W][-H R^-1; R^-1]; cycle end:
//                    X += V_k Xi C_acc, U = V_{k+1}[M; -H]), in place over an input block.
//
// Fragment layouts of m8n8k4.f64 (PTX ISA): A (8x4, row) a0 = A[lane/4][lane%4];
// B (4x8, col) b0 = B[lane%4][lane/4]; C/D (8x8) {c0,c1} = C[lane/4][2(lane%4) + {0,1}].
#pragma once
#include "kernels.cuh"

namespace lsba {

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int S>
struct GramCfg {
  static constexpr int JP = S >= 8 ? 1 : 8 / S;        // blocks j packed into one mma's M
  static constexpr int MT = S >= 8 ? S / 8 : 1;        // M tiles per block
  static constexpr int NT = S >= 8 ? S / 8 : 1;        // N tiles
  static constexpr int T = S >= 8 ? 64 : 512 / S;      // rows per tile
  static constexpr int L = S >= 2 ? S / 2 : 1;         // SpMM lanes per row
  static constexpr int NWG = 8;                        // tensor-core (Gram) warps
  static constexpr int NWS = 4;                        // gather (SpMM) warps
  static constexpr int NTHR = 32 * (NWG + NWS);
  static constexpr int RPP = 32 * NWS / L;             // SpMM rows per pass
  static constexpr int JMAX = S >= 16 ? 5 : 7;         // j-groups per Gram warp (registers)
  static constexpr int UF = S >= 16 ? 4 : 8;           // 4-row steps per unrolled batch
  static constexpr int NSTEP = T / 4;
};
// basis slots are padded to a multiple of this many rows (zero rows): branch-free tiles
constexpr int kRowPad = 512;

constexpr int kGramGroup = 16;  // CTAs per first-level reduction group

struct GramArgs {
  int n;
  const int* rp; const int* ci; const double* va;   // CSR (local rows)
  const double* Vk;        // SpMM input block (fused mode) or nullptr (W = Y given)
  const double* Vghost;
  const double* X;         // blocks X_0..X_{NVB-1} at X + j*xstride (rows padded to kRowPad)
  size_t xstride;
  int J;                   // total blocks in the Gram (including W if y_alias)
  int y_alias;             // 1: block J-1 is Y itself (taken from the W tile in smem)
  double* Y;               // W (written in fused mode; read otherwise; rows padded)
  const double* zeros;     // >= 16 zero doubles (padding lanes of packed groups)
  double* part;            // [cta][E]
  double* gpart;           // [group][E]
  unsigned* tickets;       // [ngroups + 1], zero-initialised, reset by the last CTA
  double* G;               // result, E = J S S doubles, row-major [(j S + a) S + b]
  const int* active;       // nullable: skip when *active == 0
  const double* Y2 = nullptr;  // k_gram_v7<.., NY = 2>: second B-operand block, G = X^T [Y Y2]
};

__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

// W rows of one tile by CSR gather, executed by the NWS gather warps (thread index gt).
// Lane group of L lanes per row, 2 columns per lane; up to 8 nonzeros' indices are loaded
// before their V rows.  Rows >= n produce zeros.
template <int S>
__device__ __forceinline__ void spmm_tile(const GramArgs& g, int row0, double* Ws, int gt) {
  using C = GramCfg<S>;
  const int n = g.n;
#pragma unroll 1
  for (int pass = 0; pass < (C::T + C::RPP - 1) / C::RPP; ++pass) {
    const int rl = pass * C::RPP + gt / C::L;
    const int ell = gt % C::L;
    if (rl >= C::T) continue;
    const int row = row0 + rl;
    double a0 = 0.0, a1 = 0.0;
    if (row < n) {
      const int p0 = __ldg(g.rp + row), p1 = __ldg(g.rp + row + 1);
      for (int p = p0; p < p1; p += 8) {
        int cc[8];
        double av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          cc[u] = (p + u < p1) ? __ldg(g.ci + p + u) : -1;
          av[u] = (p + u < p1) ? __ldg(g.va + p + u) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (cc[u] >= 0) {
            const double* src = (cc[u] < n) ? (g.Vk + (size_t)cc[u] * S) : (g.Vghost + (size_t)(cc[u] - n) * S);
            if constexpr (S >= 2) {
              const double2 v = __ldg(reinterpret_cast<const double2*>(src) + ell);
              a0 = fma(av[u], v.x, a0);
              a1 = fma(av[u], v.y, a1);
            } else {
              a0 = fma(av[u], __ldg(src), a0);
            }
          }
        }
      }
      if constexpr (S >= 2)
        reinterpret_cast<double2*>(g.Y + (size_t)row * S)[ell] = make_double2(a0, a1);
      else
        g.Y[row] = a0;
    }
    if constexpr (S >= 2) {
      reinterpret_cast<double2*>(Ws + rl * S)[ell] = make_double2(a0, a1);
    } else {
      Ws[rl] = a0;
    }
  }
}

// grid: persistent over row tiles; block NTHR = 384 (8 Gram warps + 4 gather warps);
// dyn smem (2 T S + J S S) doubles.  The gather warps produce W tile t+1 (double buffer)
// while the Gram warps run tile t on the tensor cores (named barriers 1-4).  A tile's
// Gram work = NG j-groups x NSTEP 4-row steps, split into 8 equal contiguous ranges.
template <int S>
__global__ void __launch_bounds__(GramCfg<S>::NTHR, (S >= 16 ? 1 : 2))
k_spmm_gram(GramArgs g) {
  using C = GramCfg<S>;
  if (g.active && *g.active == 0) return;
  extern __shared__ double smem[];
  double* Wbuf = smem;                     // 2 x (T x S)
  double* Gp = smem + 2 * C::T * S;        // J S S CTA partial
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = g.n, J = g.J;
  const int E = J * S * S;
  const int ntiles = (n + C::T - 1) / C::T;
  for (int e = tid; e < E; e += C::NTHR) Gp[e] = 0.0;
  __syncthreads();

  if (warp >= C::NWG) {
    // ======================= gather (SpMM) warps: producers of W tiles =======================
    const int gt = tid - 32 * C::NWG;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      if (it >= 2) named_sync(3 + b, C::NTHR);          // Gram warps released buffer b
      double* Ws = Wbuf + b * C::T * S;
      if (g.Vk) {
        spmm_tile<S>(g, t * C::T, Ws, gt);
      } else {
        for (int e = gt; e < C::T * S; e += 32 * C::NWS) Ws[e] = g.Y[(size_t)t * C::T * S + e];
      }
      __threadfence_block();
      named_arrive(1 + b, C::NTHR);                     // W tile of buffer b is full
    }
    // drain the outstanding "empty" arrivals of the last (up to) two tiles
    for (int k2 = (it >= 2 ? it - 2 : 0); k2 < it; ++k2) named_sync(3 + (k2 & 1), C::NTHR);
  } else {
    // ======================= Gram warps: consumers on the tensor cores =======================
    const int NVB = J - (g.y_alias ? 1 : 0);           // blocks read from global memory
    const int NGV = (NVB + C::JP - 1) / C::JP;
    const int NG = NGV + (g.y_alias ? 1 : 0);
    const int U = NG * C::NSTEP;
    const int u0 = (warp * U) / C::NWG, u1 = ((warp + 1) * U) / C::NWG;
    const int gfirst = u0 / C::NSTEP;
    const int glast = (u1 > u0) ? (u1 - 1) / C::NSTEP : gfirst - 1;
    const int r4 = lane & 3, c8 = lane >> 2;
    double acc[C::JMAX][C::MT][C::NT][2];
#pragma unroll
    for (int a = 0; a < C::JMAX; ++a)
#pragma unroll
      for (int bb = 0; bb < C::MT; ++bb)
#pragma unroll
        for (int c = 0; c < C::NT; ++c) acc[a][bb][c][0] = acc[a][bb][c][1] = 0.0;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int b = it & 1;
      named_sync(1 + b, C::NTHR);                       // wait for W tile t
      const double* Ws = Wbuf + b * C::T * S;
      const size_t row0 = (size_t)t * C::T;
#pragma unroll 1
      for (int gi = 0; gi < C::JMAX; ++gi) {
        const int grp = gfirst + gi;
        if (grp > glast) break;
        const int st0 = max(u0 - grp * C::NSTEP, 0);
        const int st1 = min(u1 - grp * C::NSTEP, C::NSTEP);
        double tacc[C::MT][C::NT][2];
#pragma unroll
        for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
          for (int tn = 0; tn < C::NT; ++tn) tacc[tm][tn][0] = tacc[tm][tn][1] = 0.0;
        if (grp < NGV) {
          // A fragments from global memory (branch-free: padded rows, zero source for
          // padding lanes of packed groups)
          const double* src[C::MT];
          int rstride[C::MT];
#pragma unroll
          for (int tm = 0; tm < C::MT; ++tm) {
            int j, col;
            if constexpr (S >= 8) { j = grp; col = tm * 8 + c8; }
            else { j = grp * C::JP + c8 / S; col = c8 % S; }
            if (j < NVB) {
              src[tm] = g.X + (size_t)j * g.xstride + (row0 + r4) * S + col;
              rstride[tm] = 4 * S;
            } else {
              src[tm] = g.zeros;
              rstride[tm] = 0;
            }
          }
#pragma unroll 1
          for (int st = st0; st < st1; st += C::UF) {
            double av[C::UF][C::MT], bf[C::UF][C::NT];
#pragma unroll
            for (int u = 0; u < C::UF; ++u) {
              const int s2 = min(st + u, st1 - 1);      // clamp (duplicates masked below)
#pragma unroll
              for (int tm = 0; tm < C::MT; ++tm) av[u][tm] = __ldg(src[tm] + s2 * rstride[tm]);
#pragma unroll
              for (int tn = 0; tn < C::NT; ++tn) {
                const int col = tn * 8 + c8;
                bf[u][tn] = (col < S && st + u < st1) ? Ws[(s2 * 4 + r4) * S + col] : 0.0;
              }
            }
#pragma unroll
            for (int u = 0; u < C::UF; ++u)
#pragma unroll
              for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
                for (int tn = 0; tn < C::NT; ++tn)
                  dmma(tacc[tm][tn][0], tacc[tm][tn][1], av[u][tm], bf[u][tn]);
          }
        } else {
          // the W block itself (y_alias): both operands from the shared-memory tile; in a
          // packed group (S < 8) only the first S rows of M carry W
#pragma unroll 1
          for (int st = st0; st < st1; ++st) {
            const int rl = st * 4 + r4;
#pragma unroll
            for (int tm = 0; tm < C::MT; ++tm) {
              double a;
              if constexpr (S >= 8) a = Ws[rl * S + tm * 8 + c8];
              else a = (c8 < S) ? Ws[rl * S + c8] : 0.0;
#pragma unroll
              for (int tn = 0; tn < C::NT; ++tn) {
                const int col = tn * 8 + c8;
                const double bv = (col < S) ? Ws[rl * S + col] : 0.0;
                dmma(tacc[tm][tn][0], tacc[tm][tn][1], a, bv);
              }
            }
          }
        }
        // fold into the per-group accumulator (static register indexing)
#pragma unroll
        for (int q = 0; q < C::JMAX; ++q)
          if (q == gi) {
#pragma unroll
            for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
              for (int tn = 0; tn < C::NT; ++tn) {
                acc[q][tm][tn][0] += tacc[tm][tn][0];
                acc[q][tm][tn][1] += tacc[tm][tn][1];
              }
          }
      }
      named_arrive(3 + b, C::NTHR);                     // buffer b may be refilled
    }
    // CTA partial: Gram warps add their fragments in warp order (deterministic)
    for (int w = 0; w < C::NWG; ++w) {
      if (warp == w) {
#pragma unroll
        for (int gi = 0; gi < C::JMAX; ++gi) {
          const int grp = gfirst + gi;
          if (grp > glast) break;
#pragma unroll
          for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
            for (int tn = 0; tn < C::NT; ++tn)
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int m = c8, nn = 2 * r4 + i;
                int j, a, bcol;
                bool ok;
                if (grp < NGV) {
                  if constexpr (S >= 8) { j = grp; a = tm * 8 + m; bcol = tn * 8 + nn; }
                  else { j = grp * C::JP + m / S; a = m % S; bcol = nn; }
                  ok = (j < NVB) && (bcol < S);
                } else {
                  j = J - 1;
                  if constexpr (S >= 8) { a = tm * 8 + m; bcol = tn * 8 + nn; ok = true; }
                  else { a = m; bcol = nn; ok = (m < S) && (nn < S); }
                }
                if (ok) Gp[(j * S + a) * S + bcol] += acc[gi][tm][tn][i];
              }
        }
      }
      named_sync(5, 32 * C::NWG);
    }
  }
  __syncthreads();
  // ---- deterministic two-level reduction across CTAs
  const int P = gridDim.x;
  const int ngroups = (P + kGramGroup - 1) / kGramGroup;
  const int grp = blockIdx.x / kGramGroup;
  const int gsize = min(kGramGroup, P - grp * kGramGroup);
  for (int e = tid; e < E; e += C::NTHR) g.part[(size_t)blockIdx.x * E + e] = Gp[e];
  __threadfence();
  __syncthreads();
  __shared__ unsigned ticket;
  if (tid == 0) ticket = atomicAdd(&g.tickets[grp], 1u);
  __syncthreads();
  if (ticket != (unsigned)(gsize - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s = 0.0;
    for (int c = 0; c < gsize; ++c) s += __ldcg(g.part + (size_t)(grp * kGramGroup + c) * E + e);
    g.gpart[(size_t)grp * E + e] = s;
  }
  if (tid == 0) g.tickets[grp] = 0u;
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(&g.tickets[ngroups], 1u);
  __syncthreads();
  if (ticket != (unsigned)(ngroups - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s = 0.0;
    for (int c = 0; c < ngroups; ++c) s += __ldcg(g.gpart + (size_t)c * E + e);
    g.G[e] = s;
  }
  if (tid == 0) g.tickets[ngroups] = 0u;
}

// ------------------------------------------------------------------------------------------
// TMA (cp.async.bulk) + mbarrier helpers
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------------------------------------
// pass 1, Gram on the tensor cores with TMA-staged tiles.  One producer warp streams, per
// row tile, the W tile (B operand, its own 2-deep ring) and then the V blocks in groups of
// JP (A operand, an R-deep ring of stages) with 1D bulk copies completing on mbarriers;
// NWG consumer warps run DMMA from shared memory.  Work of a tile = NG groups x NSTEP
// 4-row steps split into NWG contiguous ranges; every consumer warp releases every stage.
// Inputs must be basis slots (rows padded to kRowPad, zero pad rows).
// ------------------------------------------------------------------------------------------
template <int S>
struct TmaCfg {
  static constexpr int JP = GramCfg<S>::JP, MT = GramCfg<S>::MT, NT = GramCfg<S>::NT;
  static constexpr int T = GramCfg<S>::T;
  static constexpr int NSTEP = T / 4;
  static constexpr int NWG = 8;                               // consumer warps
  static constexpr int NTHR = 32 * (NWG + 1);
  static constexpr int TILE_BYTES = T * S * 8;                // one block's tile
  static constexpr int STAGE_BYTES = JP * TILE_BYTES;
  static constexpr int R = (96 * 1024) / STAGE_BYTES;         // stage ring depth
  static constexpr int WR = 2;                                // W ring depth
  static constexpr int JMAX = S >= 16 ? 5 : 7;
};

template <int S>
__global__ void __launch_bounds__(TmaCfg<S>::NTHR, 1)
k_gram_tma(GramArgs g) {
  using C = TmaCfg<S>;
  if (g.active && *g.active == 0) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double* stages = reinterpret_cast<double*>(smem_raw);                              // R x STAGE
  double* wbuf = reinterpret_cast<double*>(smem_raw + (size_t)C::R * C::STAGE_BYTES); // WR x TILE
  double* Gp = wbuf + (size_t)C::WR * C::T * S;                                      // E
  __shared__ __align__(8) uint64_t full[C::R], empty[C::R], wfull[C::WR], wempty[C::WR];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = g.J, E = J * S * S;
  const int NVB = J - (g.y_alias ? 1 : 0);
  const int NGV = (NVB + C::JP - 1) / C::JP;
  const int NG = NGV + (g.y_alias ? 1 : 0);
  const int ntiles = (g.n + C::T - 1) / C::T;
  for (int e = tid; e < E; e += C::NTHR) Gp[e] = 0.0;
  if (tid == 0) {
    for (int i = 0; i < C::R; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], C::NWG); }
    for (int i = 0; i < C::WR; ++i) { mbar_init(&wfull[i], 1); mbar_init(&wempty[i], C::NWG); }
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == C::NWG) {
    // ================= producer warp (one elected lane issues the bulk copies) =================
    if (lane == 0) {
      uint32_t q = 0;
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
        const size_t off = (size_t)t * C::T * S;
        const int wb = it % C::WR, wu = it / C::WR;
        if (wu > 0) mbar_wait(&wempty[wb], (wu - 1) & 1);
        mbar_expect_tx(&wfull[wb], C::TILE_BYTES);
        tma_load_1d(wbuf + (size_t)wb * C::T * S, g.Y + off, C::TILE_BYTES, &wfull[wb]);
        for (int gr = 0; gr < NGV; ++gr, ++q) {
          const int slot = q % C::R, use = q / C::R;
          if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
          const int nb = min(C::JP, NVB - gr * C::JP);
          mbar_expect_tx(&full[slot], nb * C::TILE_BYTES);
          for (int jj = 0; jj < nb; ++jj)
            tma_load_1d(stages + (size_t)slot * C::JP * C::T * S + (size_t)jj * C::T * S,
                        g.X + (size_t)(gr * C::JP + jj) * g.xstride + off, C::TILE_BYTES, &full[slot]);
        }
      }
    }
  } else {
    // ================= consumer warps: DMMA from shared memory =================
    const int U = NG * C::NSTEP;
    const int u0 = (warp * U) / C::NWG, u1 = ((warp + 1) * U) / C::NWG;
    const int gfirst = u0 / C::NSTEP;
    const int glast = (u1 > u0) ? (u1 - 1) / C::NSTEP : gfirst - 1;
    const int r4 = lane & 3, c8 = lane >> 2;
    double acc[C::JMAX][C::MT][C::NT][2];
#pragma unroll
    for (int a = 0; a < C::JMAX; ++a)
#pragma unroll
      for (int b = 0; b < C::MT; ++b)
#pragma unroll
        for (int c = 0; c < C::NT; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;
    uint32_t q = 0;
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int wb = it % C::WR, wu = it / C::WR;
      mbar_wait(&wfull[wb], wu & 1);
      const double* Ws = wbuf + (size_t)wb * C::T * S;
      for (int gr = 0; gr < NG; ++gr) {
        const bool vgroup = gr < NGV;
        int slot = 0;
        if (vgroup) {
          slot = q % C::R;
          mbar_wait(&full[slot], (q / C::R) & 1);
        }
        if (gr >= gfirst && gr <= glast) {
          const int gi = gr - gfirst;
          const int st0 = max(u0 - gr * C::NSTEP, 0);
          const int st1 = min(u1 - gr * C::NSTEP, C::NSTEP);
          double tacc[C::MT][C::NT][2];
#pragma unroll
          for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
            for (int tn = 0; tn < C::NT; ++tn) tacc[tm][tn][0] = tacc[tm][tn][1] = 0.0;
          if (vgroup) {
            const double* stg = stages + (size_t)slot * C::JP * C::T * S;
            int aoff[C::MT];
            bool aval[C::MT];
#pragma unroll
            for (int tm = 0; tm < C::MT; ++tm) {
              if constexpr (S >= 8) { aoff[tm] = tm * 8 + c8; aval[tm] = true; }
              else {
                const int jj = c8 / S;
                aoff[tm] = jj * C::T * S + c8 % S;
                aval[tm] = (gr * C::JP + jj) < NVB;
              }
            }
#pragma unroll 4
            for (int st = st0; st < st1; ++st) {
              const int rl = st * 4 + r4;
              double bf[C::NT];
#pragma unroll
              for (int tn = 0; tn < C::NT; ++tn) {
                const int col = tn * 8 + c8;
                bf[tn] = (col < S) ? Ws[rl * S + col] : 0.0;
              }
#pragma unroll
              for (int tm = 0; tm < C::MT; ++tm) {
                const double a = aval[tm] ? stg[rl * S + aoff[tm]] : 0.0;
#pragma unroll
                for (int tn = 0; tn < C::NT; ++tn) dmma(tacc[tm][tn][0], tacc[tm][tn][1], a, bf[tn]);
              }
            }
          } else {
            for (int st = st0; st < st1; ++st) {
              const int rl = st * 4 + r4;
#pragma unroll
              for (int tm = 0; tm < C::MT; ++tm) {
                double a;
                if constexpr (S >= 8) a = Ws[rl * S + tm * 8 + c8];
                else a = (c8 < S) ? Ws[rl * S + c8] : 0.0;
#pragma unroll
                for (int tn = 0; tn < C::NT; ++tn) {
                  const int col = tn * 8 + c8;
                  const double bv = (col < S) ? Ws[rl * S + col] : 0.0;
                  dmma(tacc[tm][tn][0], tacc[tm][tn][1], a, bv);
                }
              }
            }
          }
#pragma unroll
          for (int qq = 0; qq < C::JMAX; ++qq)
            if (qq == gi) {
#pragma unroll
              for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
                for (int tn = 0; tn < C::NT; ++tn) {
                  acc[qq][tm][tn][0] += tacc[tm][tn][0];
                  acc[qq][tm][tn][1] += tacc[tm][tn][1];
                }
            }
        }
        if (vgroup) {
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[slot]);
          ++q;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&wempty[wb]);
    }
    // CTA partial: consumer warps add their fragments in warp order (deterministic)
    for (int w = 0; w < C::NWG; ++w) {
      if (warp == w) {
#pragma unroll
        for (int gi = 0; gi < C::JMAX; ++gi) {
          const int gr = gfirst + gi;
          if (gr > glast) break;
#pragma unroll
          for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
            for (int tn = 0; tn < C::NT; ++tn)
#pragma unroll
              for (int i = 0; i < 2; ++i) {
                const int m = c8, nn = 2 * r4 + i;
                int j, a, bcol;
                bool ok;
                if (gr < NGV) {
                  if constexpr (S >= 8) { j = gr; a = tm * 8 + m; bcol = tn * 8 + nn; }
                  else { j = gr * C::JP + m / S; a = m % S; bcol = nn; }
                  ok = (j < NVB) && (bcol < S);
                } else {
                  j = J - 1;
                  if constexpr (S >= 8) { a = tm * 8 + m; bcol = tn * 8 + nn; ok = true; }
                  else { a = m; bcol = nn; ok = (m < S) && (nn < S); }
                }
                if (ok) Gp[(j * S + a) * S + bcol] += acc[gi][tm][tn][i];
              }
        }
      }
      named_sync(5, 32 * C::NWG);
    }
  }
  __syncthreads();
  // ---- deterministic two-level reduction across CTAs
  const int P = gridDim.x;
  const int ngroups = (P + kGramGroup - 1) / kGramGroup;
  const int grp = blockIdx.x / kGramGroup;
  const int gsize = min(kGramGroup, P - grp * kGramGroup);
  for (int e = tid; e < E; e += C::NTHR) g.part[(size_t)blockIdx.x * E + e] = Gp[e];
  __threadfence();
  __syncthreads();
  __shared__ unsigned ticket;
  if (tid == 0) ticket = atomicAdd(&g.tickets[grp], 1u);
  __syncthreads();
  if (ticket != (unsigned)(gsize - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s2 = 0.0;
    for (int c = 0; c < gsize; ++c) s2 += __ldcg(g.part + (size_t)(grp * kGramGroup + c) * E + e);
    g.gpart[(size_t)grp * E + e] = s2;
  }
  if (tid == 0) g.tickets[grp] = 0u;
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(&g.tickets[ngroups], 1u);
  __syncthreads();
  if (ticket != (unsigned)(ngroups - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s2 = 0.0;
    for (int c = 0; c < ngroups; ++c) s2 += __ldcg(g.gpart + (size_t)c * E + e);
    g.G[e] = s2;
  }
  if (tid == 0) g.tickets[ngroups] = 0u;
}

// ------------------------------------------------------------------------------------------
// pass 1 (unfused mode), register-staged v5: each lane loads a 16-byte column pair of a block
// row and feeds two DMMAs (M tile 0 = even columns, M tile 1 = odd columns), so a warp-load
// moves 512 B; a group packs PB = 16/S blocks (S <= 8) into the 8 M rows.  W tiles (B
// operand) are double-buffered in shared memory through a register prefetch of the next
// tile.  Requires S in {2,4,8,16} and basis-slot inputs (rows padded to kRowPad).
// ------------------------------------------------------------------------------------------
template <int S>
struct G5Cfg {
  static constexpr int PB = S >= 16 ? 1 : 16 / S;     // blocks per group
  static constexpr int NT = S >= 8 ? S / 8 : 1;       // N tiles (W columns)
  static constexpr int T = S >= 8 ? 64 : 512 / S;     // rows per tile
  static constexpr int NSTEP = T / 4;
  static constexpr int NW = 8;
  static constexpr int NTHR = 256;
  static constexpr int JMAX = S >= 16 ? 5 : 5;        // groups per warp (registers)
  static constexpr int UF = S >= 16 ? 4 : 8;          // steps per unrolled batch
  static constexpr int WPT = T * S / (2 * NTHR);      // W-tile double2 per thread (>= 1)
};

template <int S>
__global__ void __launch_bounds__(256, 2)
k_gram_v5(GramArgs g) {
  using C = G5Cfg<S>;
  static_assert(S == 2 || S == 4 || S == 8 || S == 16, "v5 Gram: s in {2,4,8,16}");
  if (g.active && *g.active == 0) return;
  extern __shared__ __align__(16) double smem5[];
  double* Wb = smem5;                            // 2 x T x S
  double* Gp = smem5 + 2 * C::T * S;             // E
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = g.J, E = J * S * S;
  const int NVB = J - (g.y_alias ? 1 : 0);
  const int NGV = (NVB + C::PB - 1) / C::PB;
  const int NG = NGV + (g.y_alias ? 1 : 0);
  const int U = NG * C::NSTEP;
  const int u0 = (warp * U) / C::NW, u1 = ((warp + 1) * U) / C::NW;
  const int gfirst = u0 / C::NSTEP;
  const int glast = (u1 > u0) ? (u1 - 1) / C::NSTEP : gfirst - 1;
  const int ntiles = (g.n + C::T - 1) / C::T;
  const int r4 = lane & 3, c8 = lane >> 2;
  constexpr int LPB = S >= 16 ? 8 : S / 2;        // lanes (c8 values) per block
  const int jj = c8 / LPB;                        // block within the group (S <= 8)
  const int cp = c8 % LPB;                        // column pair
  for (int e = tid; e < E; e += C::NTHR) Gp[e] = 0.0;
  double acc[C::JMAX][2][C::NT][2];
#pragma unroll
  for (int a = 0; a < C::JMAX; ++a)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int tn = 0; tn < C::NT; ++tn) acc[a][e][tn][0] = acc[a][e][tn][1] = 0.0;
  // prefetch the first W tile
  double2 wreg[C::WPT];
  int t = blockIdx.x;
  if (t < ntiles) {
#pragma unroll
    for (int i = 0; i < C::WPT; ++i)
      wreg[i] = __ldg(reinterpret_cast<const double2*>(g.Y + (size_t)t * C::T * S) + tid + i * C::NTHR);
  }
  int it = 0;
  for (; t < ntiles; t += gridDim.x, ++it) {
    double* Ws = Wb + (it & 1) * C::T * S;
#pragma unroll
    for (int i = 0; i < C::WPT; ++i) reinterpret_cast<double2*>(Ws)[tid + i * C::NTHR] = wreg[i];
    __syncthreads();
    const int tn_ = t + gridDim.x;
    if (tn_ < ntiles) {
#pragma unroll
      for (int i = 0; i < C::WPT; ++i)
        wreg[i] = __ldg(reinterpret_cast<const double2*>(g.Y + (size_t)tn_ * C::T * S) + tid + i * C::NTHR);
    }
    const size_t row0 = (size_t)t * C::T;
#pragma unroll 1
    for (int gi = 0; gi < C::JMAX; ++gi) {
      const int grp = gfirst + gi;
      if (grp > glast) break;
      const int st0 = max(u0 - grp * C::NSTEP, 0);
      const int st1 = min(u1 - grp * C::NSTEP, C::NSTEP);
      double tacc[2][C::NT][2];
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int tn = 0; tn < C::NT; ++tn) tacc[e][tn][0] = tacc[e][tn][1] = 0.0;
      if (grp < NGV) {
        const int j = grp * C::PB + (S >= 16 ? 0 : jj);
        const double* src;
        int rstr;
        if (j < NVB) {
          src = g.X + (size_t)j * g.xstride + (row0 + r4) * S + 2 * cp;
          rstr = 4 * S;
        } else {
          src = g.zeros;
          rstr = 0;
        }
#pragma unroll 1
        for (int st = st0; st < st1; st += C::UF) {
          double2 av[C::UF];
          double bf[C::UF][C::NT];
#pragma unroll
          for (int u = 0; u < C::UF; ++u) {
            const int s2 = min(st + u, st1 - 1);
            av[u] = __ldg(reinterpret_cast<const double2*>(src + s2 * rstr));
#pragma unroll
            for (int tn = 0; tn < C::NT; ++tn) {
              const int col = tn * 8 + c8;
              bf[u][tn] = (col < S && st + u < st1) ? Ws[(s2 * 4 + r4) * S + col] : 0.0;
            }
          }
#pragma unroll
          for (int u = 0; u < C::UF; ++u)
#pragma unroll
            for (int tn = 0; tn < C::NT; ++tn) {
              dmma(tacc[0][tn][0], tacc[0][tn][1], av[u].x, bf[u][tn]);
              dmma(tacc[1][tn][0], tacc[1][tn][1], av[u].y, bf[u][tn]);
            }
        }
      } else {
        // the W block (y_alias) from shared memory; in packed groups only block slot 0
#pragma unroll 1
        for (int st = st0; st < st1; ++st) {
          const int rl = st * 4 + r4;
          double2 a = make_double2(0.0, 0.0);
          if (S >= 16 || jj == 0) a = *reinterpret_cast<const double2*>(Ws + rl * S + 2 * cp);
#pragma unroll
          for (int tn = 0; tn < C::NT; ++tn) {
            const int col = tn * 8 + c8;
            const double bv = (col < S) ? Ws[rl * S + col] : 0.0;
            dmma(tacc[0][tn][0], tacc[0][tn][1], a.x, bv);
            dmma(tacc[1][tn][0], tacc[1][tn][1], a.y, bv);
          }
        }
      }
#pragma unroll
      for (int qq = 0; qq < C::JMAX; ++qq)
        if (qq == gi) {
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int tn = 0; tn < C::NT; ++tn) {
              acc[qq][e][tn][0] += tacc[e][tn][0];
              acc[qq][e][tn][1] += tacc[e][tn][1];
            }
        }
    }
    __syncthreads();
  }
  // CTA partial: warps add their fragments in warp order (deterministic).  D row m = c8 of
  // M tile e is block jj' = c8 / LPB, column 2 (c8 % LPB) + e; D column = W column.
  for (int w = 0; w < C::NW; ++w) {
    if (warp == w) {
#pragma unroll
      for (int gi = 0; gi < C::JMAX; ++gi) {
        const int grp = gfirst + gi;
        if (grp > glast) break;
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int tn = 0; tn < C::NT; ++tn)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int a = 2 * cp + e;
              const int bcol = tn * 8 + 2 * r4 + i;
              int j;
              bool ok = bcol < S;
              if (grp < NGV) {
                j = grp * C::PB + (S >= 16 ? 0 : jj);
                ok = ok && (j < NVB);
              } else {
                j = J - 1;
                ok = ok && (S >= 16 || jj == 0);
              }
              if (ok) Gp[(j * S + a) * S + bcol] += acc[gi][e][tn][i];
            }
      }
    }
    __syncthreads();
  }
  // ---- deterministic two-level reduction across CTAs
  const int P = gridDim.x;
  const int ngroups = (P + kGramGroup - 1) / kGramGroup;
  const int grpi = blockIdx.x / kGramGroup;
  const int gsize = min(kGramGroup, P - grpi * kGramGroup);
  for (int e = tid; e < E; e += C::NTHR) g.part[(size_t)blockIdx.x * E + e] = Gp[e];
  __threadfence();
  __syncthreads();
  __shared__ unsigned ticket;
  if (tid == 0) ticket = atomicAdd(&g.tickets[grpi], 1u);
  __syncthreads();
  if (ticket != (unsigned)(gsize - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s2 = 0.0;
    for (int c = 0; c < gsize; ++c) s2 += __ldcg(g.part + (size_t)(grpi * kGramGroup + c) * E + e);
    g.gpart[(size_t)grpi * E + e] = s2;
  }
  if (tid == 0) g.tickets[grpi] = 0u;
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(&g.tickets[ngroups], 1u);
  __syncthreads();
  if (ticket != (unsigned)(ngroups - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s2 = 0.0;
    for (int c = 0; c < ngroups; ++c) s2 += __ldcg(g.gpart + (size_t)c * E + e);
    g.G[e] = s2;
  }
  if (tid == 0) g.tickets[ngroups] = 0u;
}

// ------------------------------------------------------------------------------------------
// pass 1 (unfused), v6: barrier-free streaming Gram.  Warp (rs, qs) of a CTA owns the 4-row
// steps rs, rs+RW, ... of the CTA's contiguous step range and the block groups of set qs
// (QW sets x RW row slices = 8 warps).  Per step it loads the W (B) fragment from global
// memory (shared through L1 with the QW-1 sibling warps) and one 16-byte A fragment per
// group (even/odd column DMMA tiles, PB = 16/S blocks per group as in v5); two steps per
// iteration keep ~2 (GMAX + 1) independent loads in flight per warp.  No shared-memory
// tiles, no barriers until the final deterministic reduction.
// ------------------------------------------------------------------------------------------
template <int S>
struct G6Cfg {
  static constexpr int PB = S >= 16 ? 1 : 16 / S;
  static constexpr int NT = S >= 8 ? S / 8 : 1;
  static constexpr int GMAX = S >= 16 ? 4 : 6;
  static constexpr int NW = 8;
  static constexpr int NTHR = 256;
  static constexpr int U = 2;                      // steps per iteration
};

template <int S>
__global__ void __launch_bounds__(256, 2)
k_gram_v6(GramArgs g) {
  using C = G6Cfg<S>;
  static_assert(S == 2 || S == 4 || S == 8 || S == 16, "v6 Gram: s in {2,4,8,16}");
  if (g.active && *g.active == 0) return;
  extern __shared__ __align__(16) double Gp6[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = g.J, E = J * S * S;
  const int NVB = J - (g.y_alias ? 1 : 0);
  const int NGV = (NVB + C::PB - 1) / C::PB;
  const int NG = NGV + (g.y_alias ? 1 : 0);
  int QW = 1;
  while (QW < C::NW && (NG + QW - 1) / QW > C::GMAX) QW *= 2;
  const int RW = C::NW / QW;
  const int rs = warp % RW, qs = warp / RW;
  const int gA = (qs * NG) / QW, gB = ((qs + 1) * NG) / QW;
  const int ng = gB - gA;
  const int r4 = lane & 3, c8 = lane >> 2;
  constexpr int LPB = S >= 16 ? 8 : S / 2;
  const int jj = c8 / LPB, cp = c8 % LPB;
  for (int e = tid; e < E; e += C::NTHR) Gp6[e] = 0.0;

  // per-group A source of this lane (row r4 of step 0; + 4 S per step)
  const double* src[C::GMAX];
  int rstr[C::GMAX];
#pragma unroll
  for (int gi = 0; gi < C::GMAX; ++gi) {
    const int grp = gA + gi;
    src[gi] = g.zeros;
    rstr[gi] = 0;
    if (gi < ng) {
      if (grp < NGV) {
        const int j = grp * C::PB + (S >= 16 ? 0 : jj);
        if (j < NVB) { src[gi] = g.X + (size_t)j * g.xstride + r4 * S + 2 * cp; rstr[gi] = 4 * S; }
      } else if (S >= 16 || jj == 0) {      // the W block itself
        src[gi] = g.Y + r4 * S + 2 * cp;
        rstr[gi] = 4 * S;
      }
    }
  }
  double acc[C::GMAX][2][C::NT][2];
#pragma unroll
  for (int a = 0; a < C::GMAX; ++a)
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
      for (int tn = 0; tn < C::NT; ++tn) acc[a][e][tn][0] = acc[a][e][tn][1] = 0.0;

  const long NS = ((long)g.n + 3) / 4;                 // 4-row steps (rows padded)
  const long s0 = NS * blockIdx.x / gridDim.x, s1 = NS * (blockIdx.x + 1) / gridDim.x;
  for (long st = s0 + rs; st < s1; st += (long)C::U * RW) {
    double2 av[C::U][C::GMAX];
    double bw[C::U][C::NT];
#pragma unroll
    for (int u = 0; u < C::U; ++u) {
      const long su = st + (long)u * RW;
      const bool ok = su < s1;
      const long sc = ok ? su : st;
#pragma unroll
      for (int tn = 0; tn < C::NT; ++tn) {
        const int col = tn * 8 + c8;
        bw[u][tn] = (ok && col < S) ? __ldg(g.Y + (size_t)(sc * 4 + r4) * S + col) : 0.0;
      }
#pragma unroll
      for (int gi = 0; gi < C::GMAX; ++gi)
        av[u][gi] = (gi < ng) ? __ldg(reinterpret_cast<const double2*>(src[gi] + (size_t)sc * rstr[gi]))
                              : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int u = 0; u < C::U; ++u)
#pragma unroll
      for (int gi = 0; gi < C::GMAX; ++gi) {
        if (gi >= ng) continue;
#pragma unroll
        for (int tn = 0; tn < C::NT; ++tn) {
          dmma(acc[gi][0][tn][0], acc[gi][0][tn][1], av[u][gi].x, bw[u][tn]);
          dmma(acc[gi][1][tn][0], acc[gi][1][tn][1], av[u][gi].y, bw[u][tn]);
        }
      }
  }
  __syncthreads();
  // CTA partial: row slices add in order rs = 0..RW-1 (group sets are disjoint)
  for (int r = 0; r < RW; ++r) {
    if (rs == r) {
#pragma unroll
      for (int gi = 0; gi < C::GMAX; ++gi) {
        if (gi >= ng) continue;
        const int grp = gA + gi;
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int tn = 0; tn < C::NT; ++tn)
#pragma unroll
            for (int i = 0; i < 2; ++i) {
              const int a = 2 * cp + e;
              const int bcol = tn * 8 + 2 * r4 + i;
              int j;
              bool ok = bcol < S;
              if (grp < NGV) {
                j = grp * C::PB + (S >= 16 ? 0 : jj);
                ok = ok && (j < NVB);
              } else {
                j = J - 1;
                ok = ok && (S >= 16 || jj == 0);
              }
              if (ok) Gp6[(j * S + a) * S + bcol] += acc[gi][e][tn][i];
            }
      }
    }
    __syncthreads();
  }
  // ---- deterministic two-level reduction across CTAs
  const int P = gridDim.x;
  const int ngroups = (P + kGramGroup - 1) / kGramGroup;
  const int grpi = blockIdx.x / kGramGroup;
  const int gsize = min(kGramGroup, P - grpi * kGramGroup);
  for (int e = tid; e < E; e += C::NTHR) g.part[(size_t)blockIdx.x * E + e] = Gp6[e];
  __threadfence();
  __syncthreads();
  __shared__ unsigned ticket;
  if (tid == 0) ticket = atomicAdd(&g.tickets[grpi], 1u);
  __syncthreads();
  if (ticket != (unsigned)(gsize - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s2 = 0.0;
    for (int c = 0; c < gsize; ++c) s2 += __ldcg(g.part + (size_t)(grpi * kGramGroup + c) * E + e);
    g.gpart[(size_t)grpi * E + e] = s2;
  }
  if (tid == 0) g.tickets[grpi] = 0u;
  __threadfence();
  __syncthreads();
  if (tid == 0) ticket = atomicAdd(&g.tickets[ngroups], 1u);
  __syncthreads();
  if (ticket != (unsigned)(ngroups - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += C::NTHR) {
    double s2 = 0.0;
    for (int c = 0; c < ngroups; ++c) s2 += __ldcg(g.gpart + (size_t)c * E + e);
    g.G[e] = s2;
  }
  if (tid == 0) g.tickets[ngroups] = 0u;
}

// ------------------------------------------------------------------------------------------
// pass 2 on the tensor cores (S in {4, 8, 16}).  A warp owns 8-row blocks (grid-stride);
// per block j: A = X_j rows (8 x 4 chunks), B = C_j (4 x 8 chunks, shared memory), D in
// registers.  out0/out1 may alias an input block (each warp reads its rows before writing).
// ------------------------------------------------------------------------------------------
template <int S>
__global__ void __launch_bounds__(256)
k_project_dmma(int n, const double* X, size_t xstride, int J0, const double* __restrict__ C0,
               const double* base0, double* out0, int J1, const double* __restrict__ C1, double* out1,
               const int* __restrict__ flag_ptr) {
  static_assert(S == 4 || S == 8 || S == 16, "DMMA projection for s in {4,8,16}");
  if (flag_ptr && *flag_ptr) return;
  constexpr int KC = S / 4;                 // K chunks
  constexpr int NT = S >= 8 ? S / 8 : 1;    // N tiles
  constexpr int RB = S >= 16 ? 2 : 4;       // 8-row blocks per warp iteration
  extern __shared__ double sm[];
  double* c0 = sm;
  double* c1 = sm + (size_t)J0 * S * S;
  for (int e = threadIdx.x; e < J0 * S * S; e += blockDim.x) c0[e] = C0[e];
  for (int e = threadIdx.x; e < J1 * S * S; e += blockDim.x) c1[e] = C1[e];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int r8 = lane >> 2, k4 = lane & 3;
  const int nsup = (n + 8 * RB - 1) / (8 * RB);
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int Jmax = max(J0, J1);
  for (int sb = gw; sb < nsup; sb += nwarps) {
    double d0[RB][NT][2], d1[RB][NT][2];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
      for (int tn = 0; tn < NT; ++tn) d0[rb][tn][0] = d0[rb][tn][1] = d1[rb][tn][0] = d1[rb][tn][1] = 0.0;
    for (int j = 0; j < Jmax; ++j) {
      const double* Xj = X + (size_t)j * xstride;
      double a[RB][KC];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        const int row = (sb * RB + rb) * 8 + r8;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) a[rb][kc] = (row < n) ? Xj[(size_t)row * S + kc * 4 + k4] : 0.0;
      }
      if (j < J0) {
        const double* cj = c0 + (size_t)j * S * S;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int tn = 0; tn < NT; ++tn) {
            const int col = tn * 8 + r8;
            const double b = (col < S) ? cj[(kc * 4 + k4) * S + col] : 0.0;
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) dmma(d0[rb][tn][0], d0[rb][tn][1], a[rb][kc], b);
          }
      }
      if (j < J1) {
        const double* cj = c1 + (size_t)j * S * S;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int tn = 0; tn < NT; ++tn) {
            const int col = tn * 8 + r8;
            const double b = (col < S) ? cj[(kc * 4 + k4) * S + col] : 0.0;
#pragma unroll
            for (int rb = 0; rb < RB; ++rb) dmma(d1[rb][tn][0], d1[rb][tn][1], a[rb][kc], b);
          }
      }
    }
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) {
      const int orow = (sb * RB + rb) * 8 + r8;
      if (orow >= n) continue;
#pragma unroll
      for (int tn = 0; tn < NT; ++tn) {
        const int col = tn * 8 + 2 * k4;
        if (col < S) {
          if (J0 > 0) {
            double2 v = make_double2(d0[rb][tn][0], d0[rb][tn][1]);
            if (base0) {
              const double2 bb = *reinterpret_cast<const double2*>(base0 + (size_t)orow * S + col);
              v.x += bb.x;
              v.y += bb.y;
            }
            *reinterpret_cast<double2*>(out0 + (size_t)orow * S + col) = v;
          }
          if (J1 > 0)
            *reinterpret_cast<double2*>(out1 + (size_t)orow * S + col) =
                make_double2(d1[rb][tn][0], d1[rb][tn][1]);
        }
      }
    }
  }
}

}  // namespace lsba
