// kernels.cuh — sm_100a fp64 kernels of the BCGS-PIP block Arnoldi hot path.
//
// Data layout in HBM: every block vector (V_j, W, U, X, B) is a
// row-major n_local x s fp64 array (row i's s values contiguous, 8s bytes); the Krylov basis
// is m_max+1 such blocks back to back ("slots"); W = A V_k is written into slot k and
// projected in place (Remark 3.2).  A is CSR with int32 row_ptr/col_idx
// on the device; column indices >= n_local address the halo ("ghost") buffer.
//
// Kernel map:
//   a1  k_spmm            W = A V_k                                  (Alg 3 l.3)
//   a2  k_gram_*          partial <[V_1..V_k W], W> per CTA          (Alg 3 l.4)
//       k_gram_finalize   deterministic fixed-order sum of partials
//   a3/a5 k_small_step    S = Omega - H^T H, chol + NaN-flag, R^-1, coefficients,
//                         Hessenberg column, incremental QR (res_est), kappa_F (R8)
//   a4  k_project_*       V_{k+1} = [V_1..V_k W] [-H R^-1; R^-1]    (Alg 3 l.6)
//   a5/a6 k_cycle_solve   Xi, M, cos (Eq Xm / Thm 2.4) by LU, once per cycle
//   a6  k_project_* (2 outputs) X += V_k Xi C_acc ; U = V_{k+1}[M; -H]
//   -   k_residual        R = B - A X and ||R||_F^2 partials (reading R19)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace lsba {

constexpr int kThreads = 256;

// ------------------------------------------------------------------------------------------
// L2 eviction-priority hints (createpolicy + ld.global.nc.L2::cache_hint).  c_l2hint bits:
// 1 = the SpMM's CSR streams (row_ptr, col_idx, vals) evict_last, so A can stay L2-resident
// across the step while the basis streams through; 2 = the Gram's basis reads evict_first;
// 4 = the projection's basis reads evict_first; 8 = the SpMM output W and the projection output
// V_{k+1} stored evict_last (the next kernel re-reads them).  The product uses 14 (measured in
// round 1: config 2 +8%, config 5 +1.5%, configs 3/4 neutral; bit 1 lost); a compile-time
// constant so that no module-wide state is shared between contexts.
// ------------------------------------------------------------------------------------------
constexpr int c_l2hint = 14;

// Programmatic dependent launch (PDL): the hot kernels of a step (SpMM, Gram, projection) may
// be launched with programmatic stream serialisation, so the next kernel's CTAs are scheduled
// while this one drains.  Every such kernel first lets its dependents launch, then WAITS for
// its predecessor grid (completion + memory flush) before touching any input — and before any
// early exit, so completion stays transitive along the stream.  No-ops without PDL.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifdef LSBA_TAIL_TRACE
// Diagnostics build only (LSBA_NVCC_EXTRA=-DLSBA_TAIL_TRACE): globaltimer stamps appended to a
// device buffer (two words per record: time, tag << 32 | J), read back by lsba_trace_dump.
// (Device printf costs ~40 us per call and would distort the timeline it measures.)
constexpr unsigned kTraceWords = 1u << 18;
static __device__ unsigned long long g_trace[kTraceWords];
static __device__ unsigned g_trace_n;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_rec(unsigned tag, unsigned J, unsigned long long t) {
  const unsigned i = atomicAdd(&g_trace_n, 2u);
  if (i + 1 < kTraceWords) {
    g_trace[i] = t;
    g_trace[i + 1] = ((unsigned long long)tag << 32) | J;
  }
}
// block 0 of a kernel: its time at entry (before the PDL wait) and after the wait
#define PDL_TRACE_ENTRY const unsigned long long pdl_t_entry = (blockIdx.x == 0 && threadIdx.x == 0) ? gtime() : 0ull;
#define PDL_TRACE_WAITED(tag, J) do { if (blockIdx.x == 0 && threadIdx.x == 0) { \
  trace_rec(tag, (unsigned)(J), pdl_t_entry); trace_rec((tag) + 1, (unsigned)(J), gtime()); } } while (0)
// the latest CTA exit of the SpMM (slot 0) / projection (slot 1) as thread 0 of each CTA saw it,
// recorded by block 0 of the next kernel once its wait returned (tags 8: SpMM, 9: projection)
static __device__ unsigned long long g_trace_exit[2];
#define TRACE_EXIT(slot) do { if (threadIdx.x == 0) atomicMax(&g_trace_exit[slot], gtime()); } while (0)
#define TRACE_PREV_EXIT(slot, tag) do { if (blockIdx.x == 0 && threadIdx.x == 0) \
  trace_rec(tag, 0, *(volatile unsigned long long*)&g_trace_exit[slot]); } while (0)
#else
#define PDL_TRACE_ENTRY
#define PDL_TRACE_WAITED(tag, J) do { } while (0)
#define TRACE_EXIT(slot) do { } while (0)
#define TRACE_PREV_EXIT(slot, tag) do { } while (0)
#endif
// trace tags: 2/3 SpMM entry/waited, 4/5 Gram, 6/7 projection; 10..14 the Gram tail (gram7.cuh)
enum { kTrSpmm = 2, kTrGram = 4, kTrProj = 6, kTrTail = 10 };
__device__ __forceinline__ uint64_t l2pol(bool hint, bool last) {
  uint64_t p;
  if (!hint) asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  else if (last) asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int ldh(const int* p, uint64_t pol) {
  int v;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldh(const double* p, uint64_t pol) {
  double v;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ double ldh_rw(const double* p, uint64_t pol) {   // coherent (not .nc)
  double v;
  asm("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void sth2(double* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1,%2}, %3;" :: "l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
__device__ __forceinline__ double2 ldh2(const double* p, uint64_t pol) {
  double2 v;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

// ------------------------------------------------------------------------------------------
// row access helpers: S doubles per row, loaded as double2 when S is even
// ------------------------------------------------------------------------------------------
template <int S>
__device__ __forceinline__ void load_row(const double* __restrict__ p, double (&v)[S]) {
  if constexpr (S % 2 == 0) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int t = 0; t < S / 2; ++t) {
      double2 d = __ldg(q + t);
      v[2 * t] = d.x;
      v[2 * t + 1] = d.y;
    }
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) v[t] = __ldg(p + t);
  }
}

template <int S>
__device__ __forceinline__ void load_row_h(const double* __restrict__ p, double (&v)[S], uint64_t pol) {
  if constexpr (S % 2 == 0) {
#pragma unroll
    for (int t = 0; t < S / 2; ++t) {
      double2 d = ldh2(p + 2 * t, pol);
      v[2 * t] = d.x;
      v[2 * t + 1] = d.y;
    }
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) v[t] = ldh(p + t, pol);
  }
}

// plain (non-__ldg) load: used when the buffer may be written by the same kernel
template <int S>
__device__ __forceinline__ void load_row_rw(const double* p, double (&v)[S]) {
  if constexpr (S % 2 == 0) {
    const double2* q = reinterpret_cast<const double2*>(p);
#pragma unroll
    for (int t = 0; t < S / 2; ++t) {
      double2 d = q[t];
      v[2 * t] = d.x;
      v[2 * t + 1] = d.y;
    }
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) v[t] = p[t];
  }
}

template <int S>
__device__ __forceinline__ void store_row(double* p, const double (&v)[S]) {
  if constexpr (S % 2 == 0) {
    double2* q = reinterpret_cast<double2*>(p);
#pragma unroll
    for (int t = 0; t < S / 2; ++t) q[t] = make_double2(v[2 * t], v[2 * t + 1]);
  } else {
#pragma unroll
    for (int t = 0; t < S; ++t) p[t] = v[t];
  }
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

// ------------------------------------------------------------------------------------------
// a1: SpMM  W = A V   (and the residual variant R = B - A X with ||R||^2 partials)
// L lanes per row; lane l owns columns {2l, 2l+1} (S >= 2) -> coalesced 16-byte accesses.
// Summation over a row's nonzeros runs in CSR order (same order as the oracle).
//
// The kernel is latency-bound (one dependent index -> gather -> FMA chain per entry, few bytes
// in flight per warp), so thread 0 of every CTA issues bulk L2 prefetches
// (cp.async.bulk.prefetch.L2) for the CTA launched pf_dist CTAs later: its column indices and
// values, its own V rows (pf_v) and, one distance further, its row pointers.  When that CTA
// runs, its matrix stream comes from L2 (standalone, config 5: 884 -> 687 us, config 3: 117 ->
// 93 us; tools/spmm_tile_bench.cu, profiles/r02_spmm_prefetch_raw.txt).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void bulk_prefetch_l2(const void* p, long bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  for (uintptr_t q = a; q < e; q += 65536) {
    const unsigned sz = (unsigned)((e - q) < 65536 ? (e - q) : 65536);
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" :: "l"(q), "r"(sz) : "memory");
  }
}

// Projection pre-wait prefetch: a projection CTA launched early (PDL) sits on an SM the Gram
// has left while the Gram's serial tail (the last CTAs' reductions and the fused small step,
// ~7 us) runs and HBM idles.  Before waiting on the Gram, thread 0 of each of the first
// pf_ctas CTAs bulk-prefetches into L2 the rows of every input block that the CTA reads first,
// so that tail overlaps the projection's stream.  Only L2 is touched (the point of coherence):
// the data cannot be stale whatever the predecessor still writes.
__device__ __forceinline__ void prefetch_blocks_l2(int pf_ctas, const double* X, size_t xstride, int J,
                                                   long off, long bytes) {
  if ((int)blockIdx.x >= pf_ctas || threadIdx.x != 0 || bytes <= 0) return;
  for (int j = 0; j < J; ++j) bulk_prefetch_l2(X + (size_t)j * xstride + off, bytes);
}

// 32-byte vector access (sm_100a LDG.E.256 / STG.E.256)
__device__ __forceinline__ double4 ld4nc(const double* p) {
  double4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ void st4h(double* p, double4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f64 [%0], {%1,%2,%3,%4}, %5;"
               :: "l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w), "l"(pol) : "memory");
}

// Columns per lane of the row-lane SpMM: 4 (one 32-byte access) when s % 4 == 0, else 2
// (16 bytes) for even s, else 1.  Round 2: 32-byte lanes halve the lanes per row and with them
// the redundant index/value loads per entry (standalone, config 5: 852 -> 606 us = 6.0 TB/s;
// config 3: 115 -> 79 us; tools/spmm_tile_bench.cu, profiles/r02_spmm_q256_raw.txt).
template <int S>
struct SpmmLanes {
  static constexpr int C = (S % 4 == 0) ? 4 : ((S % 2 == 0) ? 2 : 1);
  static constexpr int L = S / C;      // lanes per row
};

// Rows [row0, row1) of the n local rows (the halo overlap runs the interior rows while the
// ghost rows are in flight, then the boundary rows); columns >= n address Vghost.
// CW: columns per lane (SpmmLanes<S>::C; 2 when a caller buffer is only 16-byte aligned).
// Register budget for 6 CTAs of 256 per SM (<= 40 registers): the compiler then keeps more
// entries' loads in flight than at its default 36 (interleaved standalone A/B:
// profiles/r02_spmm_ab_raw.txt: configs 3 / 5 -5% / -2% time, config 2 -6%)
template <int S, bool RESID, int CW = SpmmLanes<S>::C>
__global__ void __launch_bounds__(kThreads, 6)
k_spmm(int n, const int* __restrict__ rp, const int* __restrict__ ci,
       const double* __restrict__ va, const double* __restrict__ V,
       const double* __restrict__ Vghost, const double* __restrict__ Bm,
       double* __restrict__ W, double* __restrict__ sq_part, const int* __restrict__ active = nullptr,
       int pf_dist = 0, int pf_v = 0, int row0 = 0, int row1 = -1) {
  PDL_TRACE_ENTRY
  pdl_begin();
  PDL_TRACE_WAITED(kTrSpmm, 0);
  TRACE_PREV_EXIT(1, 9);
  if (active && *active == 0) return;
  constexpr int C = CW;                // columns per lane
  constexpr int L = S / CW;            // lanes per row
  constexpr int RPC = kThreads / L;    // rows per CTA
  if (row1 < 0) row1 = n;
  if (pf_dist > 0 && threadIdx.x == 0) {
    const long r0 = row0 + (long)(blockIdx.x + pf_dist) * RPC;
    if (r0 < row1) {
      const long r1 = r0 + RPC < row1 ? r0 + RPC : row1;
      const int q0 = __ldg(rp + r0), q1 = __ldg(rp + r1);
      bulk_prefetch_l2(ci + q0, 4L * (q1 - q0));
      bulk_prefetch_l2(va + q0, 8L * (q1 - q0));
      if (pf_v) bulk_prefetch_l2(V + r0 * S, 8L * S * (r1 - r0));
      const long r2 = row0 + (long)(blockIdx.x + 2L * pf_dist) * RPC;
      if (r2 < row1) bulk_prefetch_l2(rp + r2, 4L * ((r2 + RPC < row1 ? r2 + RPC : row1) - r2 + 1));
    }
  }
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = row0 + (int)(gt / L);
  const int lane = (int)(gt % L);
  double sq = 0.0;
  // row pointers: one coalesced load of the warp's 32/L + 1 pointers, then shuffles (instead
  // of 2 L redundant dependent loads per row)
  int p0, p1;
  {
    const int lane32 = threadIdx.x & 31;
    const int row_w = row0 + (int)(((long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / L);
    const int rr = row_w + lane32;
    const int pv = (lane32 <= 32 / L && rr <= row1) ? __ldg(rp + rr) : 0;
    if constexpr (L == 1) {            // 32 rows per warp: the 33rd pointer by a second load
      const int nx = __shfl_down_sync(0xffffffffu, pv, 1);
      p0 = pv;
      p1 = (lane32 < 31) ? nx : ((rr + 1 <= row1) ? __ldg(rp + rr + 1) : 0);
    } else {
      p0 = __shfl_sync(0xffffffffu, pv, lane32 / L);
      p1 = __shfl_sync(0xffffffffu, pv, lane32 / L + 1);
    }
  }
  if (row < row1) {
    double acc[C];
#pragma unroll
    for (int t = 0; t < C; ++t) acc[t] = 0.0;
    for (int p = p0; p < p1; ++p) {
      const int c = __ldg(ci + p);
      const double a = __ldg(va + p);
      const double* src = ((c < n) ? (V + (size_t)c * S) : (Vghost + (size_t)(c - n) * S)) + C * lane;
      if constexpr (C == 4) {
        const double4 v = ld4nc(src);
        acc[0] = fma(a, v.x, acc[0]);
        acc[1] = fma(a, v.y, acc[1]);
        acc[2] = fma(a, v.z, acc[2]);
        acc[3] = fma(a, v.w, acc[3]);
      } else if constexpr (C == 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(src));
        acc[0] = fma(a, v.x, acc[0]);
        acc[1] = fma(a, v.y, acc[1]);
      } else {
        acc[0] = fma(a, __ldg(src), acc[0]);
      }
    }
    double* dst = W + (size_t)row * S + C * lane;
    if constexpr (RESID) {
      const double* bsrc = Bm + (size_t)row * S + C * lane;
#pragma unroll
      for (int t = 0; t < C; ++t) {
        acc[t] = __ldg(bsrc + t) - acc[t];
        sq += acc[t] * acc[t];
      }
    }
    if constexpr (C == 4)
      st4h(dst, make_double4(acc[0], acc[1], acc[2], acc[3]), l2pol(c_l2hint & 8, true));
    else if constexpr (C == 2)
      sth2(dst, make_double2(acc[0], acc[1]), l2pol(c_l2hint & 8, true));
    else
      dst[0] = acc[0];
  }
  if constexpr (RESID) {
    __shared__ double red[kThreads / 32];
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      sq_part[blockIdx.x] = t;
    }
  }
  TRACE_EXIT(0);
}

// P > 1 without a contiguous interior block (config 4's random columns): the SpMM runs on the
// local-column part of A while the halo is in flight, then this kernel adds the ghost-column
// part of the rows that have one: W[row] += sum over the row's ghost entries (ghost index c,
// Vghost rows).  The row's sum is then local entries (CSR order) + ghost entries (CSR order).
template <int S>
__global__ void __launch_bounds__(kThreads)
k_spmm_ghost_acc(int ng, const int* __restrict__ rows, const int* __restrict__ rp, const int* __restrict__ ci,
                 const double* __restrict__ va, const double* __restrict__ Vghost, double* __restrict__ W,
                 const int* __restrict__ active) {
  pdl_begin();
  if (active && *active == 0) return;
  constexpr int C = (S % 2 == 0) ? 2 : 1;
  constexpr int L = S / C;
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int t = (int)(gt / L), lane = (int)(gt % L);
  if (t >= ng) return;
  double acc[C];
#pragma unroll
  for (int q = 0; q < C; ++q) acc[q] = 0.0;
  for (int p = rp[t]; p < rp[t + 1]; ++p) {
    const double a = __ldg(va + p);
    const double* src = Vghost + (size_t)__ldg(ci + p) * S + C * lane;
#pragma unroll
    for (int q = 0; q < C; ++q) acc[q] = fma(a, __ldg(src + q), acc[q]);
  }
  double* dst = W + (size_t)rows[t] * S + C * lane;
#pragma unroll
  for (int q = 0; q < C; ++q) dst[q] += acc[q];
}

// odd s: one thread per row, scalar column loads
template <int S, bool RESID>
__global__ void __launch_bounds__(kThreads)
k_spmm_odd(int n, const int* __restrict__ rp, const int* __restrict__ ci,
           const double* __restrict__ va, const double* __restrict__ V,
           const double* __restrict__ Vghost, const double* __restrict__ Bm,
           double* __restrict__ W, double* __restrict__ sq_part, const int* __restrict__ active = nullptr,
           int row0 = 0, int row1 = -1) {
  if (active && *active == 0) return;
  if (row1 < 0) row1 = n;
  const int row = row0 + blockIdx.x * blockDim.x + threadIdx.x;
  double sq = 0.0;
  if (row < row1) {
    double acc[S];
#pragma unroll
    for (int t = 0; t < S; ++t) acc[t] = 0.0;
    for (int p = rp[row]; p < rp[row + 1]; ++p) {
      const int c = __ldg(ci + p);
      const double a = __ldg(va + p);
      const double* src = (c < n) ? (V + (size_t)c * S) : (Vghost + (size_t)(c - n) * S);
#pragma unroll
      for (int t = 0; t < S; ++t) acc[t] = fma(a, __ldg(src + t), acc[t]);
    }
    if constexpr (RESID) {
#pragma unroll
      for (int t = 0; t < S; ++t) {
        acc[t] = __ldg(Bm + (size_t)row * S + t) - acc[t];
        sq += acc[t] * acc[t];
      }
    }
#pragma unroll
    for (int t = 0; t < S; ++t) W[(size_t)row * S + t] = acc[t];
  }
  if constexpr (RESID) {
    __shared__ double red[kThreads / 32];
    sq = warp_sum(sq);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
      sq_part[blockIdx.x] = t;
    }
  }
}

// *flag |= (any x[i] != 0) over count doubles (flag zeroed by the caller); used to take
// U = B without an SpMM when X0 = 0 (reading R13)
static __global__ void k_any_nonzero(long count, const double* __restrict__ x, int* __restrict__ flag) {
  int nz = 0;
  for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (long)gridDim.x * blockDim.x)
    nz |= (x[i] != 0.0);
  nz = __syncthreads_or(nz);
  if (threadIdx.x == 0 && nz) atomicOr(flag, 1);
}

// halo pack: send[i] = V[idx[i]] (rows)
template <int S>
__global__ void k_halo_pack(int cnt, const int* __restrict__ idx, const double* __restrict__ V,
                            double* __restrict__ out) {
  const long t = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long)cnt * S) return;
  const int r = (int)(t / S), c = (int)(t % S);
  out[t] = __ldg(V + (size_t)idx[r] * S + c);
}

// ------------------------------------------------------------------------------------------
// a2: block inner products, DFMA variant.  Partial Gram per CTA over a contiguous row range;
// fixed-order CTA reduction (warp butterfly, then warps in index order) -> deterministic.
// Classical: G_j = X_j^T Y (S x S) for blocks j = 0..J-1 at X + j*xstride.
// CTA (jt, p): block j = jt / (S/TA), output rows a0 = (jt % (S/TA))*TA .. +TA, rows of
// slice p.  part layout: [p][j][S][S].
// ------------------------------------------------------------------------------------------
template <int S>
struct GramTA {
  static constexpr int value = (S <= 8) ? S : (S % 4 == 0 ? 4 : (S % 3 == 0 ? 3 : (S % 2 == 0 ? 2 : 1)));
};

template <int S>
__global__ void __launch_bounds__(kThreads)
k_gram_cl(int n, const double* __restrict__ X, size_t xstride, int J,
          const double* __restrict__ Y, double* __restrict__ part, const int* __restrict__ active) {
  if (active && *active == 0) return;
  constexpr int TA = GramTA<S>::value;
  constexpr int NA = S / TA;
  const int j = blockIdx.x / NA;
  const int a0 = (blockIdx.x % NA) * TA;
  const int P = gridDim.y;
  const int chunk = (n + P - 1) / P;
  const int r0 = blockIdx.y * chunk;
  const int r1 = min(n, r0 + chunk);
  const double* Xj = X + (size_t)j * xstride;
  double acc[TA][S];
#pragma unroll
  for (int a = 0; a < TA; ++a)
#pragma unroll
    for (int b = 0; b < S; ++b) acc[a][b] = 0.0;
  for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double y[S];
    load_row<S>(Y + (size_t)i * S, y);
    double x[TA];
#pragma unroll
    for (int a = 0; a < TA; ++a) x[a] = __ldg(Xj + (size_t)i * S + a0 + a);
#pragma unroll
    for (int a = 0; a < TA; ++a)
#pragma unroll
      for (int b = 0; b < S; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
  }
  __shared__ double red[kThreads / 32][TA * S];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
  for (int a = 0; a < TA; ++a)
#pragma unroll
    for (int b = 0; b < S; ++b) {
      const double v = warp_sum(acc[a][b]);
      if (l == 0) red[w][a * S + b] = v;
    }
  __syncthreads();
  const int nw = blockDim.x >> 5;
  for (int e = threadIdx.x; e < TA * S; e += blockDim.x) {
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += red[q][e];
    const int a = e / S, b = e % S;
    part[((size_t)blockIdx.y * J + j) * S * S + (size_t)(a0 + a) * S + b] = t;
  }
}

// Global: g_j = sum_{i,a} X_j[i,a] Y[i,a];  part layout [p][j]
template <int S>
__global__ void __launch_bounds__(kThreads)
k_gram_gl(int n, const double* __restrict__ X, size_t xstride, int J,
          const double* __restrict__ Y, double* __restrict__ part, const int* __restrict__ active) {
  if (active && *active == 0) return;
  const int j = blockIdx.x;
  const int P = gridDim.y;
  const int chunk = (n + P - 1) / P;
  const int r0 = blockIdx.y * chunk;
  const int r1 = min(n, r0 + chunk);
  const double* Xj = X + (size_t)j * xstride;
  double acc = 0.0;
  for (int i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    double y[S], x[S];
    load_row<S>(Y + (size_t)i * S, y);
    load_row<S>(Xj + (size_t)i * S, x);
#pragma unroll
    for (int a = 0; a < S; ++a) acc = fma(x[a], y[a], acc);
  }
  __shared__ double red[kThreads / 32];
  const double v = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    part[(size_t)blockIdx.y * J + j] = t;
  }
}

// G[e] = scale * sum_{p=0..P-1} part[p][e]   (fixed order: deterministic, rank-independent)
static __global__ void k_gram_finalize(int P, int E, const double* __restrict__ part,
                                double* __restrict__ G, double scale, const int* __restrict__ active) {
  if (active && *active == 0) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double t = 0.0;
  for (int p = 0; p < P; ++p) t += part[(size_t)p * E + e];
  G[e] = t * scale;
}

// sum of partials -> out[0] (single thread block, fixed order)
static __global__ void k_sum_partials(int P, const double* __restrict__ part, double* __restrict__ out) {
  __shared__ double red[kThreads];
  double t = 0.0;
  const int chunk = (P + blockDim.x - 1) / blockDim.x;
  const int p0 = threadIdx.x * chunk, p1 = min(P, p0 + chunk);
  for (int p = p0; p < p1; ++p) t += part[p];
  red[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < (int)blockDim.x; ++q) s += red[q];
    out[0] = s;
  }
}

// ------------------------------------------------------------------------------------------
// a4/a6: multi-block projection ("basis_eval"), DFMA variant.
//   out0[i] = (base0 ? base0[i] : 0) + sum_{j<J0} X_j[i] C0_j        (S x S blocks C0_j)
//   out1[i] = sum_{j<J1} X_j[i] C1_j                                   (if J1 > 0)
// X_j at X + j*xstride.  Classical: C*_j are S x S row-major, [j][a][c].  Global: scalars.
// One thread per row; coefficients in shared memory (broadcast reads).  out0/out1 may alias
// an input block: every thread reads its row of all blocks before writing it.
// flag_ptr: if non-null and *flag_ptr != 0 the kernel does nothing (NaN-flagged step).
// ------------------------------------------------------------------------------------------
// Global inner product (Table 1): the projection coefficients are scalars, so
// a projection is an elementwise combination of whole blocks.  Flat over the n S doubles of a
// block (S even: 16-byte vectors, coalesced across the warp), up to 4 blocks in flight per
// thread, the same j-ascending fma chain as k_project (bitwise the same results).  A thread
// reads its elements of every block before writing them, so an output may alias an input block.
__device__ __forceinline__ double2 ldh2_co(const double* p, uint64_t pol) {   // coherent, 16 bytes
  double2 v;
  asm("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
static __global__ void __launch_bounds__(kThreads)
k_project_flat(long cnt2, const double* X, size_t xstride, int J0, const double* __restrict__ C0,
               const double* base0, double* out0, int J1, const double* __restrict__ C1, double* out1,
               const int* __restrict__ flag_ptr, int pf_ctas = 0) {
  PDL_TRACE_ENTRY
  pdl_launch();
  {
    const long e0 = (long)blockIdx.x * blockDim.x;
    prefetch_blocks_l2(pf_ctas, X, xstride, max(J0, J1), 2 * e0,
                       16L * (min(cnt2, e0 + (long)blockDim.x) - e0));
  }
  pdl_wait();
  PDL_TRACE_WAITED(kTrProj, max(J0, J1));
  if (flag_ptr && *flag_ptr) return;
  extern __shared__ double sm[];
  double* c0 = sm;
  double* c1 = sm + J0;
  for (int e = threadIdx.x; e < J0; e += blockDim.x) c0[e] = C0[e];
  for (int e = threadIdx.x; e < J1; e += blockDim.x) c1[e] = C1[e];
  __syncthreads();
  const int Jmax = max(J0, J1);
  const uint64_t xpol = l2pol(c_l2hint & 4, false), opol = l2pol(c_l2hint & 8, true);
  for (long e = (long)blockIdx.x * blockDim.x + threadIdx.x; e < cnt2; e += (long)gridDim.x * blockDim.x) {
    double2 o0 = make_double2(0.0, 0.0), o1 = make_double2(0.0, 0.0);
    int j = 0;
    for (; j + 4 <= Jmax; j += 4) {
      double2 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = ldh2_co(X + (size_t)(j + u) * xstride + 2 * e, xpol);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (j + u < J0) { o0.x = fma(x[u].x, c0[j + u], o0.x); o0.y = fma(x[u].y, c0[j + u], o0.y); }
        if (j + u < J1) { o1.x = fma(x[u].x, c1[j + u], o1.x); o1.y = fma(x[u].y, c1[j + u], o1.y); }
      }
    }
    for (; j < Jmax; ++j) {
      const double2 x = ldh2_co(X + (size_t)j * xstride + 2 * e, xpol);
      if (j < J0) { o0.x = fma(x.x, c0[j], o0.x); o0.y = fma(x.y, c0[j], o0.y); }
      if (j < J1) { o1.x = fma(x.x, c1[j], o1.x); o1.y = fma(x.y, c1[j], o1.y); }
    }
    if (base0) {
      const double2 b = *reinterpret_cast<const double2*>(base0 + 2 * e);
      o0.x += b.x;
      o0.y += b.y;
    }
    if (J0 > 0) sth2(out0 + 2 * e, o0, opol);
    if (J1 > 0) sth2(out1 + 2 * e, o1, opol);
  }
}

template <int S, bool GLOBAL>
__global__ void __launch_bounds__(kThreads)
k_project(int n, const double* X, size_t xstride, int J0, const double* __restrict__ C0,
          const double* base0, double* out0, int J1, const double* __restrict__ C1,
          double* out1, const int* __restrict__ flag_ptr, int pf_ctas = 0) {
  PDL_TRACE_ENTRY
  pdl_launch();
  {
    const long r0 = (long)blockIdx.x * blockDim.x;
    prefetch_blocks_l2(pf_ctas, X, xstride, max(J0, J1), r0 * S,
                       8L * S * (min((long)n, r0 + (long)blockDim.x) - r0));
  }
  pdl_wait();
  PDL_TRACE_WAITED(kTrProj, max(J0, J1));
  if (flag_ptr && *flag_ptr) return;
  extern __shared__ double sm[];
  constexpr int CB = GLOBAL ? 1 : S * S;   // coefficients per block
  double* c0 = sm;
  double* c1 = sm + (size_t)J0 * CB;
  for (int e = threadIdx.x; e < J0 * CB; e += blockDim.x) c0[e] = C0[e];
  for (int e = threadIdx.x; e < J1 * CB; e += blockDim.x) c1[e] = C1[e];
  __syncthreads();
  // grid-stride over rows on a resident grid: the coefficients are staged once per CTA, and the
  // CTAs the next kernel's early launch waits on all start together (config 2 +3% in situ,
  // profiles/r02_coef_flag_raw.txt)
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
  double o0[S], o1[S];
#pragma unroll
  for (int c = 0; c < S; ++c) { o0[c] = 0.0; o1[c] = 0.0; }
  if (J1 == 0 && !base0) {
    // the step projection (one output): blocks in batches of 4 so that a thread has four
    // rows in flight.  Every thread reads only its own row of every block before writing that
    // row (the output may be the last input block), so the read-only path is safe here.
    int j = 0;
    const uint64_t xpol = l2pol(c_l2hint & 4, false);
    for (; j + 4 <= J0; j += 4) {
      double x[4][S];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_row_h<S>(X + (size_t)(j + u) * xstride + (size_t)i * S, x[u], xpol);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if constexpr (GLOBAL) {
          const double cj = c0[j + u];
#pragma unroll
          for (int c = 0; c < S; ++c) o0[c] = fma(x[u][c], cj, o0[c]);
        } else {
          const double* cj = c0 + (size_t)(j + u) * S * S;
#pragma unroll
          for (int a = 0; a < S; ++a)
#pragma unroll
            for (int c = 0; c < S; ++c) o0[c] = fma(x[u][a], cj[a * S + c], o0[c]);
        }
      }
    }
    for (; j < J0; ++j) {
      double x[S];
      load_row<S>(X + (size_t)j * xstride + (size_t)i * S, x);
      if constexpr (GLOBAL) {
        const double cj = c0[j];
#pragma unroll
        for (int c = 0; c < S; ++c) o0[c] = fma(x[c], cj, o0[c]);
      } else {
        const double* cj = c0 + (size_t)j * S * S;
#pragma unroll
        for (int a = 0; a < S; ++a)
#pragma unroll
          for (int c = 0; c < S; ++c) o0[c] = fma(x[a], cj[a * S + c], o0[c]);
      }
    }
    if constexpr (S % 2 == 0) {
      const uint64_t opol = l2pol(c_l2hint & 8, true);
#pragma unroll
      for (int t = 0; t < S / 2; ++t) sth2(out0 + (size_t)i * S + 2 * t, make_double2(o0[2 * t], o0[2 * t + 1]), opol);
    } else {
      store_row<S>(out0 + (size_t)i * S, o0);
    }
    continue;
  }
  const int Jmax = max(J0, J1);
  for (int j = 0; j < Jmax; ++j) {
    double x[S];
    load_row_rw<S>(X + (size_t)j * xstride + (size_t)i * S, x);
    if (j < J0) {
      if constexpr (GLOBAL) {
        const double cj = c0[j];
#pragma unroll
        for (int c = 0; c < S; ++c) o0[c] = fma(x[c], cj, o0[c]);
      } else {
        const double* cj = c0 + (size_t)j * S * S;
#pragma unroll
        for (int a = 0; a < S; ++a)
#pragma unroll
          for (int c = 0; c < S; ++c) o0[c] = fma(x[a], cj[a * S + c], o0[c]);
      }
    }
    if (j < J1) {
      if constexpr (GLOBAL) {
        const double cj = c1[j];
#pragma unroll
        for (int c = 0; c < S; ++c) o1[c] = fma(x[c], cj, o1[c]);
      } else {
        const double* cj = c1 + (size_t)j * S * S;
#pragma unroll
        for (int a = 0; a < S; ++a)
#pragma unroll
          for (int c = 0; c < S; ++c) o1[c] = fma(x[a], cj[a * S + c], o1[c]);
      }
    }
  }
  if (base0) {
    double b[S];
    load_row_rw<S>(base0 + (size_t)i * S, b);
#pragma unroll
    for (int c = 0; c < S; ++c) o0[c] += b[c];
  }
  if (J0 > 0) store_row<S>(out0 + (size_t)i * S, o0);
  if (J1 > 0) store_row<S>(out1 + (size_t)i * S, o1);
  }
  TRACE_EXIT(1);
}

// ------------------------------------------------------------------------------------------
// small-state helpers shared with small.cuh
// ------------------------------------------------------------------------------------------
struct StepStatus {
  int32_t k;
  int32_t flag;          // Cholesky NaN-flag (or forced)
  int32_t proj_singular; // h~_k singular: FOM projected matrix singular (reading R22)
  int32_t pad;
  double res_gmres;      // ||g_{k+1} C_acc||_F * rfac
  double res_fom;        // ||H_{k+1,k} h~^{-1} g^_k C_acc||_F * rfac
  double kappa_F;        // ||R_{k+1}||_F ||R_{k+1}^{-1}||_F
  double normU2;         // IO only: ||U||_F^2 (k == 0)
};

// Device-side cycle control (one per context): the step kernel takes the continue /
// restart decision of SURVEY 8(c) step 2.2 on the device, so the host can enqueue a whole
// cycle and read this block once per cycle.
struct CycleCtl {
  int32_t active;        // 1 while the cycle continues (kernels of later steps no-op when 0)
  int32_t why;           // 0 running, 1 NaN-flag / singular FOM matrix, 2 res_est <= tol,
                         // 3 kappa_F > tau, 4 k == m_cur, 5 IO flagged
  int32_t k_used;        // accepted steps of this cycle
  int32_t k_flag;        // step index of the flag (why == 1)
  int32_t forced_here;   // the flag was injected (lsba_set_force_flag)
  int32_t force_k;       // fault-injection step (0 = off)
  int32_t forced_done;   // the injected flag already happened in this solve
  int32_t proj_singular; // why == 1 because h~_k was singular (reading R22)
  int32_t m_cur;         // step budget of this cycle
  int32_t gmres;         // 1: BGMRES estimate, 0: BFOM estimate
  int32_t need_kappa;    // 1: maintain kappa_F each step
  int32_t pad1;
  double tol_abs;        // tol * ||B||_F (negative: never converge)
  double tau;            // kappa_F threshold (inf: off)
  double res_est;        // estimate of the last accepted step (times C_acc)
  double kappa;          // kappa_F of the last accepted step
};

constexpr int kMaxB = 16;

// block-wide sum (blockDim multiple of 32, <= 1024); all threads get the result
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  const int nw = (blockDim.x + 31) >> 5;
  for (int q = 0; q < nw; ++q) t += red[q];
  return t;
}

static __global__ void k_set_identity(double* Cm, int b) {
  const int e = threadIdx.x;
  if (e < b * b) Cm[e] = (e % b == e / b) ? 1.0 : 0.0;
}

}  // namespace lsba
