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
  static constexpr int RPP = 256 / L;                  // SpMM rows per pass (256 threads)
  static constexpr int JMAX = S >= 16 ? 5 : 7;         // j-groups per warp (registers)
  static constexpr int UF = S >= 16 ? 2 : 4;           // 4-row steps per unrolled batch
  static constexpr int NW = 8;                         // warps per CTA
  static constexpr int NSTEP = T / 4;
};

constexpr int kGramGroup = 16;  // CTAs per first-level reduction group

struct GramArgs {
  int n;
  const int* rp; const int* ci; const double* va;   // CSR (local rows)
  const double* Vk;        // SpMM input block (fused mode) or nullptr (W = Y given)
  const double* Vghost;
  const double* X;         // blocks X_0..X_{J-1} at X + j*xstride
  size_t xstride;
  int J;
  double* Y;               // W (written in fused mode; read otherwise); block J-1 if it aliases
  double* part;            // [cta][E]
  double* gpart;           // [group][E]
  unsigned* tickets;       // [ngroups + 1], zero-initialised, reset by the last CTA
  double* G;               // result, E = J S S doubles, row-major [(j S + a) S + b]
  const int* active;       // nullable: skip when *active == 0
};

// W rows of one tile by CSR gather (row-local lane group of L lanes, 2 columns per lane);
// column indices and values of up to 8 nonzeros are loaded before their V rows (MLP).
template <int S>
__device__ __forceinline__ void spmm_tile(const GramArgs& g, int row0, double* Ws) {
  using C = GramCfg<S>;
  const int tid = threadIdx.x, n = g.n;
#pragma unroll
  for (int pass = 0; pass < (C::T + C::RPP - 1) / C::RPP; ++pass) {
    const int rl = pass * C::RPP + tid / C::L;
    const int ell = tid % C::L;
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
        double vx[8], vy[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          vx[u] = vy[u] = 0.0;
          if (cc[u] >= 0) {
            const double* src = (cc[u] < n) ? (g.Vk + (size_t)cc[u] * S) : (g.Vghost + (size_t)(cc[u] - n) * S);
            if constexpr (S >= 2) {
              const double2 v = __ldg(reinterpret_cast<const double2*>(src) + ell);
              vx[u] = v.x;
              vy[u] = v.y;
            } else {
              vx[u] = __ldg(src);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          a0 = fma(av[u], vx[u], a0);
          if constexpr (S >= 2) a1 = fma(av[u], vy[u], a1);
        }
      }
      if constexpr (S >= 2)
        reinterpret_cast<double2*>(g.Y + (size_t)row * S)[ell] = make_double2(a0, a1);
      else
        g.Y[row] = a0;
    }
    if constexpr (S >= 2) {
      Ws[rl * S + 2 * ell] = a0;
      Ws[rl * S + 2 * ell + 1] = a1;
    } else {
      Ws[rl] = a0;
    }
  }
}

// grid: any size (persistent over row tiles); block 256; dyn smem T*S + J*S*S doubles.
// Work of a tile = NG j-groups x NSTEP 4-row steps, split into 8 equal contiguous ranges
// (one per warp; a warp touches at most JMAX groups).
template <int S>
__global__ void __launch_bounds__(256, 2)
k_spmm_gram(GramArgs g) {
  using C = GramCfg<S>;
  if (g.active && *g.active == 0) return;
  extern __shared__ double smem[];
  double* Ws = smem;                       // T x S tile of W
  double* Gp = smem + C::T * S;            // J S S partial (CTA)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = g.n, J = g.J;
  const int E = J * S * S;
  const int NG = (J + C::JP - 1) / C::JP;
  const int U = NG * C::NSTEP;
  const int u0 = (warp * U) / C::NW, u1 = ((warp + 1) * U) / C::NW;
  const int gfirst = u0 / C::NSTEP;
  const int glast = (u1 > u0) ? (u1 - 1) / C::NSTEP : gfirst - 1;
  const int ntiles = (n + C::T - 1) / C::T;
  for (int e = tid; e < E; e += 256) Gp[e] = 0.0;

  double acc[C::JMAX][C::MT][C::NT][2];
#pragma unroll
  for (int a = 0; a < C::JMAX; ++a)
#pragma unroll
    for (int b = 0; b < C::MT; ++b)
#pragma unroll
      for (int c = 0; c < C::NT; ++c) acc[a][b][c][0] = acc[a][b][c][1] = 0.0;

  const int r4 = lane & 3, c8 = lane >> 2;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int row0 = t * C::T;
    if (g.Vk) {
      spmm_tile<S>(g, row0, Ws);
    } else {
      for (int e = tid; e < C::T * S; e += 256) {
        const size_t gi = (size_t)row0 * S + e;
        Ws[e] = (gi < (size_t)n * S) ? g.Y[gi] : 0.0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int gi = 0; gi < C::JMAX; ++gi) {
      const int grp = gfirst + gi;
      if (grp > glast) break;
      const int st0 = max(u0 - grp * C::NSTEP, 0);
      const int st1 = min(u1 - grp * C::NSTEP, C::NSTEP);
      // A-fragment source of this lane for each M tile (fixed for the group)
      const double* src[C::MT];
      bool alias[C::MT];
      int colA[C::MT];
#pragma unroll
      for (int tm = 0; tm < C::MT; ++tm) {
        int j;
        if constexpr (S >= 8) { j = grp; colA[tm] = tm * 8 + c8; }
        else { j = grp * C::JP + c8 / S; colA[tm] = c8 % S; }
        const double* Xj = (j < J) ? g.X + (size_t)j * g.xstride : nullptr;
        alias[tm] = (Xj == g.Y);
        src[tm] = Xj;
      }
      for (int st = st0; st < st1; st += C::UF) {
        double av[C::UF][C::MT], bf[C::UF][C::NT];
#pragma unroll
        for (int u = 0; u < C::UF; ++u) {
          const int rl = (st + u) * 4 + r4;
          const int row = row0 + rl;
          const bool in = (st + u < st1);
#pragma unroll
          for (int tn = 0; tn < C::NT; ++tn) {
            const int col = tn * 8 + c8;
            bf[u][tn] = (in && col < S) ? Ws[rl * S + col] : 0.0;
          }
#pragma unroll
          for (int tm = 0; tm < C::MT; ++tm) {
            double v = 0.0;
            if (in && src[tm] != nullptr) {
              if (alias[tm]) v = Ws[rl * S + colA[tm]];
              else if (row < n) v = __ldg(src[tm] + (size_t)row * S + colA[tm]);
            }
            av[u][tm] = v;
          }
        }
#pragma unroll
        for (int u = 0; u < C::UF; ++u)
#pragma unroll
          for (int tm = 0; tm < C::MT; ++tm)
#pragma unroll
            for (int tn = 0; tn < C::NT; ++tn) dmma(acc[gi][tm][tn][0], acc[gi][tm][tn][1], av[u][tm], bf[u][tn]);
      }
    }
    __syncthreads();
  }
  // ---- CTA partial: warps add their fragments in warp order (deterministic)
  for (int w = 0; w < C::NW; ++w) {
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
              int j, a, b;
              if constexpr (S >= 8) { j = grp; a = tm * 8 + m; b = tn * 8 + nn; }
              else { j = grp * C::JP + m / S; a = m % S; b = nn; }
              if (j < J && b < S) Gp[(j * S + a) * S + b] += acc[gi][tm][tn][i];
            }
      }
    }
    __syncthreads();
  }
  // ---- deterministic two-level reduction across CTAs
  const int P = gridDim.x;
  const int ngroups = (P + kGramGroup - 1) / kGramGroup;
  const int grp = blockIdx.x / kGramGroup;
  const int gsize = min(kGramGroup, P - grp * kGramGroup);
  for (int e = tid; e < E; e += 256) g.part[(size_t)blockIdx.x * E + e] = Gp[e];
  __threadfence();
  __syncthreads();
  __shared__ unsigned ticket;
  if (tid == 0) ticket = atomicAdd(&g.tickets[grp], 1u);
  __syncthreads();
  if (ticket != (unsigned)(gsize - 1)) return;
  __threadfence();
  for (int e = tid; e < E; e += 256) {
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
  for (int e = tid; e < E; e += 256) {
    double s = 0.0;
    for (int c = 0; c < ngroups; ++c) s += __ldcg(g.gpart + (size_t)c * E + e);
    g.G[e] = s;
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
