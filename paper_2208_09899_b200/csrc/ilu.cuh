// ilu.cuh — ILU(0) left preconditioning on the device ("an
// incomplete LU (ILU) preconditioner with no fill"; left side, IKJ variant).
//
//   k_ilu0_level   one level of the IKJ factorisation, a warp per row (setup, once per matrix)
//   k_ilu_pack     level-ordered packed rows of each factor half (setup)
//   k_ilu_trsv_level (default, round 2) level-synchronous solve on the packs, grid barriers
//   k_ilu_trsv_poll  (LSBA_ILU_SOLVE=0) sync-free sparse triangular solve Z = L^{-1} X or U^{-1} X, one
//                  thread per row (all s columns), rows in level order claimed 32 at a time by
//                  the warps of a persistent grid, dependencies detected by polling the data itself
//                  (sentinel-filled output); measured 4.3 / 11 / 12 us per level on configs
//                  2 / 3 / 5 vs 6.9 / 25 / 56 with per-row ready flags and 17 / 46 / 72 with
//                  one CTA per chunk (round-1 variants, removed; profiles/r01_ilu_apply.txt)
//
// Factor storage: lu[p] for CSR position p of the local matrix (row_ptr / col_idx of A):
// strictly-lower entries are L (unit diagonal implied), the rest U.  Columns >= n_local
// (ghost rows of other ranks) are not part of the factor: with P > 1 this is block-Jacobi
// ILU(0) of the local diagonal block, equal to ILU(0) of A on one rank.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lsba {

// One level of Saad's IKJ ILU(0) (Iterative Methods, Alg 10.4), a warp per row i of the level:
//   for k < i in row i (ascending):  l = a_ik / a_kk;  a_ik = l;
//                                    a_ij -= l a_kj  for j > k in row i with (k, j) in pattern
// Rows of earlier levels (every k above) are final.  Lane 0 owns a_ik, lanes stride the j's.
// Zero / non-finite pivot -> *bad = 1 (the factor is then unusable; the host reports it).
__global__ void __launch_bounds__(256)
k_ilu0_level(int cnt, const int* __restrict__ rows, const int* __restrict__ rp,
             const int* __restrict__ ci, const int* __restrict__ diag, int n_local, double* lu,
             int* bad) {
  const int w = (int)((blockIdx.x * (long)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (w >= cnt) return;
  const int i = rows[w];
  const int p0 = rp[i], p1 = rp[i + 1];
  for (int p = p0; p < p1; ++p) {
    const int k = ci[p];
    if (k >= n_local || k >= i) continue;          // ghost column, or not in the L part
    const double piv = lu[diag[k]];
    if (!(piv != 0.0) || !isfinite(piv)) {
      if (lane == 0) *bad = 1;
      return;
    }
    const double l = lu[p] / piv;
    __syncwarp();
    if (lane == 0) lu[p] = l;
    const int k0 = rp[k], k1 = rp[k + 1];
    for (int q = p + 1 + lane; q < p1; q += 32) {
      const int j = ci[q];
      if (j >= n_local) continue;
      for (int r = k0; r < k1; ++r)                 // a_kj (row k is short: linear scan)
        if (ci[r] == j) {
          lu[q] = fma(-l, lu[r], lu[q]);
          break;
        }
    }
    __syncwarp();                                   // a_ij updates visible to lane 0's next a_ik
  }
  if (lane == 0) {
    const double d = lu[diag[i]];
    if (!(d != 0.0) || !isfinite(d)) *bad = 1;
  }
}

// Data-polling variant (no flags): the output Z is pre-filled with a sentinel NaN pattern
// (kIluSentinel, never produced by arithmetic: quiet NaNs from fp64 ops carry a zero payload);
// a row's dependency y_k is ready when none of its S values is the sentinel.  One L2 round trip
// per dependency instead of two (flag, then data).  Out of place: Z != X.
constexpr unsigned long long kIluSentinel = 0x7ff4dead5e47ee11ull;
__device__ __forceinline__ double ld_volatile_d(const double* p) {
  double v;
  asm volatile("ld.volatile.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_volatile_d2(const double* p) {
  double2 v;
  asm volatile("ld.volatile.global.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ bool not_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) != kIluSentinel;
}
__global__ void k_fill_sentinel(long count, double* __restrict__ z) {
  const double v = __longlong_as_double((long long)kIluSentinel);
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < count; e += (long)gridDim.x * blockDim.x)
    z[e] = v;
}
// Persistent solve: each WARP claims the next chunk of 32 rows (level order) from a global
// counter — no CTA barrier, so a warp never waits for the slowest row of a 256-row chunk — and
// a row's dependencies are polled in batches of up to 4 at once (every S value of every
// dependency in the batch loaded together, retried until none is the sentinel), so a ready
// row costs one L2 round trip per batch instead of one per dependency.  Warps only wait on rows
// of earlier chunks, claimed by warps that are already running: no deadlock.  The arithmetic
// (CSR order over the dependencies, then the diagonal) is the round-1 kernel's.
template <int S, bool LOWER>
__global__ void __launch_bounds__(256)
k_ilu_trsv_poll(int nrows, const int* __restrict__ order, const int* __restrict__ rp,
                const int* __restrict__ ci, const double* __restrict__ lu, const int* __restrict__ diag,
                int n_local, const double* __restrict__ X, double* Z, unsigned* ctr,
                const int* __restrict__ active, int backoff_ns) {
  const bool live = !(active && *active == 0);
  const int lane = threadIdx.x & 31;
  const int nchunks = (nrows + 31) / 32;
  constexpr int DB = 4;                       // dependencies polled per batch
  // one chunk ahead: the next chunk is claimed, and its row index and row pointers loaded,
  // before this chunk's dependencies are polled (the claim -> order -> row pointer chain leaves
  // the critical path; a warp only ever waits inside its current, smaller chunk: no deadlock)
  auto claim = [&]() {
    int ch = 0;
    if (lane == 0) ch = live ? (int)atomicAdd(ctr, 1u) : nchunks;
    return __shfl_sync(0xffffffffu, ch, 0);
  };
  int nx = claim(), nx_i = 0, nx_p0 = 0, nx_p1 = 0;
  auto meta = [&](int ch, int& i, int& q0, int& q1) {
    const int t = ch * 32 + lane;
    if (ch < nchunks && t < nrows) {
      i = order[t];
      q0 = rp[i];
      q1 = rp[i + 1];
    }
  };
  meta(nx, nx_i, nx_p0, nx_p1);
  for (;;) {
    const int chunk = nx, i = nx_i, p0 = nx_p0, p1 = nx_p1;
    if (chunk >= nchunks) break;
    nx = claim();
    meta(nx, nx_i, nx_p0, nx_p1);
    const int t = chunk * 32 + lane;
    if (t < nrows) {
      double acc[S];
#pragma unroll
      for (int c = 0; c < S; ++c) acc[c] = 0.0;
      int p = p0;
      while (p < p1) {
        // next batch: up to DB dependency entries of this row (CSR order)
        int ent[DB], nb = 0;
        for (; p < p1 && nb < DB; ++p) {
          const int k = ci[p];
          if (k >= n_local || (LOWER ? k >= i : k <= i)) continue;
          ent[nb++] = p;
        }
        double y[DB][S];
        // (a failed poll may back off: LSBA_ILU_BACKOFF; measured neutral, default 0)
        for (int sleep_ns = backoff_ns;; sleep_ns = min(2 * sleep_ns, 1024)) {
          bool ok = true;
#pragma unroll
          for (int d = 0; d < DB; ++d) {
            if (d < nb) {
              const double* zk = Z + (size_t)ci[ent[d]] * S;
              if constexpr (S % 2 == 0) {
#pragma unroll
                for (int c = 0; c < S; c += 2) {
                  const double2 v = ld_volatile_d2(zk + c);
                  y[d][c] = v.x;
                  y[d][c + 1] = v.y;
                  ok = ok && not_sentinel(v.x) && not_sentinel(v.y);
                }
              } else {
#pragma unroll
                for (int c = 0; c < S; ++c) {
                  y[d][c] = ld_volatile_d(zk + c);
                  ok = ok && not_sentinel(y[d][c]);
                }
              }
            }
          }
          if (ok) break;
          if (sleep_ns > 0) __nanosleep(sleep_ns);
        }
#pragma unroll
        for (int d = 0; d < DB; ++d) {
          if (d < nb) {
            const double a = lu[ent[d]];
#pragma unroll
            for (int c = 0; c < S; ++c) acc[c] = fma(a, y[d][c], acc[c]);
          }
        }
      }
      const double dinv = LOWER ? 1.0 : lu[diag[i]];
      double* zi = Z + (size_t)i * S;
#pragma unroll
      for (int c = 0; c < S; ++c) {
        const double r = X[(size_t)i * S + c] - acc[c];
        __stcg(zi + c, LOWER ? r : r / dinv);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned e = atomicAdd(ctr + 1, 1u);
    if (e == gridDim.x - 1) {
      ctr[0] = 0u;
      ctr[1] = 0u;
    }
  }
}

// ---------------------------------------------------------------------------------------
// Level-synchronous solve on level-ordered packed rows (round 2; for matrices whose levels
// are wide, e.g. 3D stencils: 5-22 K rows per level).  Setup packs, for every position t of
// the level order, the row index, its first kIluW dependencies (columns and factor values, in
// CSR order), the CSR position after them (the rest, rare, is read from the CSR), and the
// pivot: structure-of-arrays, so a level's threads read them coalesced, in one round trip,
// independent of the solve's data.  A resident grid walks the levels with one grid barrier
// between them; thread g holds row r0 + g of the level.  Software-pipelined: the packed data
// of level l+1 is loaded before the barrier that ends level l-1 and used after the one ending
// level l, so a level costs the barrier plus one round trip for its dependency values and the
// store.  Dependencies summed in CSR order, then the diagonal: the same arithmetic as
// k_ilu_trsv_poll, bitwise.
// ---------------------------------------------------------------------------------------
constexpr int kIluW = 4;          // packed dependencies per row
constexpr int kThreadsIluLvl = 256;
struct IluPack {                  // level-ordered, n entries each ([q * n + t] for k, v)
  int* row;                       // row index
  int* rest;                      // CSR position after the kIluW-th dependency (p1 if fewer)
  int* k;                         // dependency columns (-1: none)
  double* v;                      // factor values of those entries
  double* piv;                    // U: the pivot (L: unused)
};
// build the pack of one factor half: thread per level-order position
template <bool LOWER>
__global__ void k_ilu_pack(int n, const int* __restrict__ order, const int* __restrict__ rp,
                           const int* __restrict__ ci, const double* __restrict__ lu, const int* __restrict__ diag,
                           int n_local, IluPack pk) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int i = order[t];
  const int p0 = rp[i], p1 = rp[i + 1];
  int nd = 0, p = p0;
  for (; p < p1 && nd < kIluW; ++p) {
    const int k = ci[p];
    if (k >= n_local || (LOWER ? k >= i : k <= i)) continue;
    pk.k[(size_t)nd * n + t] = k;
    pk.v[(size_t)nd * n + t] = lu[p];
    ++nd;
  }
  for (int q = nd; q < kIluW; ++q) {
    pk.k[(size_t)q * n + t] = -1;
    pk.v[(size_t)q * n + t] = 0.0;
  }
  pk.row[t] = i;
  pk.rest[t] = p;
  if (!LOWER) pk.piv[t] = lu[diag[i]];
}
#ifndef LSBA_BAR_NS
#define LSBA_BAR_NS 0
#endif
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" :: "l"(bar) : "memory");
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
      if ((int)(v - target) >= 0) break;
      __nanosleep(LSBA_BAR_NS);
    }
  }
  __syncthreads();
}
// 32-byte L2 (coherent) access: rows written by other CTAs during the solve never come from L1
__device__ __forceinline__ double4 ldcg4(const double* p) {
  double4 v;
  asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void stcg4(double* p, double4 v) {
  asm volatile("st.global.cg.v4.f64 [%0], {%1,%2,%3,%4};" :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w) : "memory");
}
struct IluLvlRow {
  int i, rest, p1;
  int k[kIluW];
  double v[kIluW];
  double piv;
};
template <bool LOWER>
__device__ __forceinline__ void ilu_pack_load(long t, int n, const IluPack& pk, const int* __restrict__ rp,
                                              IluLvlRow& r) {
  r.i = __ldcg(pk.row + t);
  r.rest = __ldcg(pk.rest + t);
#pragma unroll
  for (int q = 0; q < kIluW; ++q) {
    r.k[q] = __ldcg(pk.k + (size_t)q * n + t);
    r.v[q] = __ldcg(pk.v + (size_t)q * n + t);
  }
  r.piv = LOWER ? 1.0 : __ldcg(pk.piv + t);
  r.p1 = -1;            // (row end: loaded only when a row has more than kIluW dependencies)
}
template <int S, bool LOWER>
__device__ __forceinline__ void ilu_pack_finish(const IluLvlRow& r, const int* __restrict__ rp,
                                                const int* __restrict__ ci, const double* __restrict__ lu,
                                                int n_local, const double* __restrict__ X, double* Z) {
  double y[kIluW][S];
#pragma unroll
  for (int q = 0; q < kIluW; ++q)
    if (r.k[q] >= 0) {
      if constexpr (S % 4 == 0) {
#pragma unroll
        for (int c = 0; c < S; c += 4) {
          const double4 w = ldcg4(Z + (size_t)r.k[q] * S + c);
          y[q][c] = w.x;
          y[q][c + 1] = w.y;
          y[q][c + 2] = w.z;
          y[q][c + 3] = w.w;
        }
      } else if constexpr (S % 2 == 0) {
#pragma unroll
        for (int c = 0; c < S; c += 2) {
          const double2 w = __ldcg(reinterpret_cast<const double2*>(Z + (size_t)r.k[q] * S + c));
          y[q][c] = w.x;
          y[q][c + 1] = w.y;
        }
      } else {
#pragma unroll
        for (int c = 0; c < S; ++c) y[q][c] = __ldcg(Z + (size_t)r.k[q] * S + c);
      }
    }
  double acc[S];
#pragma unroll
  for (int c = 0; c < S; ++c) acc[c] = 0.0;
#pragma unroll
  for (int q = 0; q < kIluW; ++q)
    if (r.k[q] >= 0)
#pragma unroll
      for (int c = 0; c < S; ++c) acc[c] = fma(r.v[q], y[q][c], acc[c]);
  if (r.k[kIluW - 1] >= 0) {                      // (more dependencies than packed: CSR)
    const int p1 = rp[r.i + 1];
    for (int p = r.rest; p < p1; ++p) {
      const int k = ci[p];
      if (k >= n_local || (LOWER ? k >= r.i : k <= r.i)) continue;
      const double a = lu[p];
#pragma unroll
      for (int c = 0; c < S; ++c) acc[c] = fma(a, __ldcg(Z + (size_t)k * S + c), acc[c]);
    }
  }
  double* zi = Z + (size_t)r.i * S;
  if constexpr (S % 4 == 0) {
#pragma unroll
    for (int c = 0; c < S; c += 4) {
      const double4 xv = ldcg4(X + (size_t)r.i * S + c);
      double4 o;
      o.x = LOWER ? xv.x - acc[c] : (xv.x - acc[c]) / r.piv;
      o.y = LOWER ? xv.y - acc[c + 1] : (xv.y - acc[c + 1]) / r.piv;
      o.z = LOWER ? xv.z - acc[c + 2] : (xv.z - acc[c + 2]) / r.piv;
      o.w = LOWER ? xv.w - acc[c + 3] : (xv.w - acc[c + 3]) / r.piv;
      stcg4(zi + c, o);
    }
  } else if constexpr (S % 2 == 0) {
#pragma unroll
    for (int c = 0; c < S; c += 2) {
      const double2 xv = __ldcg(reinterpret_cast<const double2*>(X + (size_t)r.i * S + c));
      double2 o;
      o.x = LOWER ? xv.x - acc[c] : (xv.x - acc[c]) / r.piv;
      o.y = LOWER ? xv.y - acc[c + 1] : (xv.y - acc[c + 1]) / r.piv;
      __stcg(reinterpret_cast<double2*>(zi + c), o);
    }
  } else {
#pragma unroll
    for (int c = 0; c < S; ++c) {
      const double v = __ldcg(X + (size_t)r.i * S + c) - acc[c];
      __stcg(zi + c, LOWER ? v : v / r.piv);
    }
  }
}
// bar[0]: CTA arrivals (monotonic within a launch), bar[1]: CTA exits (the last resets both);
// *go: block 0's reading of the cycle control, published by barrier 0 (a uniform no-op).
template <int S, bool LOWER>
__global__ void __launch_bounds__(kThreadsIluLvl, 1)
k_ilu_trsv_level(int n, int nlev, const int* __restrict__ lvl, IluPack pk, const int* __restrict__ rp,
                 const int* __restrict__ ci, const double* __restrict__ lu, int n_local,
                 const double* __restrict__ X, double* Z, unsigned* bar, int* go, const int* __restrict__ active) {
  const long T = (long)gridDim.x * blockDim.x;
  const long g = (long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned nbar = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile int*)go = (active && *active == 0) ? 0 : 1;
  IluLvlRow cur, nxt;
  long c0 = 0, ccnt = 0;
  if (nlev > 0) {
    c0 = lvl[0];
    ccnt = lvl[1] - c0;
    if (g < ccnt) ilu_pack_load<LOWER>(c0 + g, n, pk, rp, cur);
  }
  grid_barrier(bar, (++nbar) * gridDim.x);
  if (*(volatile int*)go != 0) {
    for (int l = 0; l < nlev; ++l) {
      // the next level's packed rows: loaded now, used after the next barrier
      long n0 = 0, ncnt = 0;
      if (l + 1 < nlev) {
        n0 = lvl[l + 1];
        ncnt = lvl[l + 2] - n0;
        if (g < ncnt) ilu_pack_load<LOWER>(n0 + g, n, pk, rp, nxt);
      }
      if (g < ccnt) ilu_pack_finish<S, LOWER>(cur, rp, ci, lu, n_local, X, Z);
      for (long t = g + T; t < ccnt; t += T) {            // (levels wider than the grid)
        IluLvlRow r2;
        ilu_pack_load<LOWER>(c0 + t, n, pk, rp, r2);
        ilu_pack_finish<S, LOWER>(r2, rp, ci, lu, n_local, X, Z);
      }
      if (l + 1 < nlev) grid_barrier(bar, (++nbar) * gridDim.x);   // level l complete
      cur = nxt;
      c0 = n0;
      ccnt = ncnt;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned e = atomicAdd(bar + 1, 1u);
    if (e == gridDim.x - 1) {
      bar[0] = 0u;
      bar[1] = 0u;
    }
  }
}

// per-CTA partial sums of squares of x[0..count) (grid-stride; fixed order per CTA)
__global__ void __launch_bounds__(256)
k_sq_partials(long count, const double* __restrict__ x, double* __restrict__ part) {
  __shared__ double red[8];
  double t = 0.0;
  for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < count; e += (long)gridDim.x * blockDim.x) {
    const double v = x[e];
    t = fma(v, v, t);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) u += red[w];
    part[blockIdx.x] = u;
  }
}

}  // namespace lsba
