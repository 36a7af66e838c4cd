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
// ------------------------------------------------------------------------------------------
template <int S, bool RESID>
__global__ void __launch_bounds__(kThreads)
k_spmm(int n, const int* __restrict__ rp, const int* __restrict__ ci,
       const double* __restrict__ va, const double* __restrict__ V,
       const double* __restrict__ Vghost, const double* __restrict__ Bm,
       double* __restrict__ W, double* __restrict__ sq_part) {
  constexpr int L = (S >= 2) ? S / 2 : 1;
  constexpr int C = (S >= 2) ? 2 : 1;  // columns per lane
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / L);
  const int lane = (int)(gt % L);
  double sq = 0.0;
  if (row < n) {
    const int p0 = rp[row], p1 = rp[row + 1];
    double a0 = 0.0, a1 = 0.0;
    for (int p = p0; p < p1; ++p) {
      const int c = __ldg(ci + p);
      const double a = __ldg(va + p);
      const double* src = (c < n) ? (V + (size_t)c * S) : (Vghost + (size_t)(c - n) * S);
      if constexpr (C == 2) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(src) + lane);
        a0 = fma(a, v.x, a0);
        a1 = fma(a, v.y, a1);
      } else {
        a0 = fma(a, __ldg(src), a0);
      }
    }
    double* dst = W + (size_t)row * S;
    if constexpr (RESID) {
      if constexpr (C == 2) {
        const double2 b = __ldg(reinterpret_cast<const double2*>(Bm + (size_t)row * S) + lane);
        a0 = b.x - a0;
        a1 = b.y - a1;
      } else {
        a0 = __ldg(Bm + row) - a0;
      }
      sq = a0 * a0 + (C == 2 ? a1 * a1 : 0.0);
    }
    if constexpr (C == 2)
      reinterpret_cast<double2*>(dst)[lane] = make_double2(a0, a1);
    else
      dst[0] = a0;
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

// odd s: one thread per row, scalar column loads
template <int S, bool RESID>
__global__ void __launch_bounds__(kThreads)
k_spmm_odd(int n, const int* __restrict__ rp, const int* __restrict__ ci,
           const double* __restrict__ va, const double* __restrict__ V,
           const double* __restrict__ Vghost, const double* __restrict__ Bm,
           double* __restrict__ W, double* __restrict__ sq_part) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  double sq = 0.0;
  if (row < n) {
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
          const double* __restrict__ Y, double* __restrict__ part) {
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
          const double* __restrict__ Y, double* __restrict__ part) {
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
__global__ void k_gram_finalize(int P, int E, const double* __restrict__ part,
                                double* __restrict__ G, double scale) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= E) return;
  double t = 0.0;
  for (int p = 0; p < P; ++p) t += part[(size_t)p * E + e];
  G[e] = t * scale;
}

// sum of partials -> out[0] (single thread block, fixed order)
__global__ void k_sum_partials(int P, const double* __restrict__ part, double* __restrict__ out) {
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
template <int S, bool GLOBAL>
__global__ void __launch_bounds__(kThreads)
k_project(int n, const double* X, size_t xstride, int J0, const double* __restrict__ C0,
          const double* base0, double* out0, int J1, const double* __restrict__ C1,
          double* out1, const int* __restrict__ flag_ptr) {
  if (flag_ptr && *flag_ptr) return;
  extern __shared__ double sm[];
  constexpr int CB = GLOBAL ? 1 : S * S;   // coefficients per block
  double* c0 = sm;
  double* c1 = sm + (size_t)J0 * CB;
  for (int e = threadIdx.x; e < J0 * CB; e += blockDim.x) c0[e] = C0[e];
  for (int e = threadIdx.x; e < J1 * CB; e += blockDim.x) c1[e] = C1[e];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double o0[S], o1[S];
#pragma unroll
  for (int c = 0; c < S; ++c) { o0[c] = 0.0; o1[c] = 0.0; }
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

// ------------------------------------------------------------------------------------------
// Small-state kernels (one CTA).  State layout (column-major small matrices, fp64):
//   Hbar  : ((m+1)b) x (m b), ld = ldH = (m+1)b         block upper Hessenberg (D3)
//   beta  : b x b                                        IO factor of the cycle's start block
//   coef  : ((k+1)b) x b row-major [j][a][c]             projection coefficients
//   qr_v  : m x b x 2b, qr_tau: m x b                    Householder reflectors of Hbar's QR
//   g     : ((m+1)b) x b, ld = ldH                       Q^T (E_1 beta) (reading R11)
//   Rinv  : ((m+1)b)^2, ld = ldH                         R_{k+1}^{-1}, R_{k+1} = [E_1 beta, Hbar_k] (R8)
//   sc[]  : scalars: [0] ||R||_F^2, [1] ||R^{-1}||_F^2
//   Cacc  : b x b                                        accumulated cospatial product (R10)
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

struct SmallState {
  double* Hbar; double* beta; double* coef; double* qr_v; double* qr_tau; double* g;
  double* Rinv; double* sc; double* Cacc; StepStatus* status; int* flag_dev;
  int ldH; int m; int b;
};

constexpr int kMaxB = 16;

// block-wide sum (blockDim multiple of 32, <= 1024); all threads get the result
__device__ double block_sum(double v, double* red) {
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

// Upper Cholesky with NaN-flag (reading R2), sequential; S symmetric b x b, column-major.
__device__ bool chol_upper(const double* S, double* R, int b) {
  for (int x = 0; x < b * b; ++x) R[x] = 0.0;
  for (int j = 0; j < b; ++j) {
    double d = S[j + j * b];
    for (int i = 0; i < j; ++i) d -= R[i + j * b] * R[i + j * b];
    if (!(d > 0.0) || !isfinite(d)) return true;
    const double r = sqrt(d);
    R[j + j * b] = r;
    for (int c = j + 1; c < b; ++c) {
      double t = S[j + c * b];
      for (int i = 0; i < j; ++i) t -= R[i + j * b] * R[i + c * b];
      R[j + c * b] = t / r;
    }
  }
  for (int x = 0; x < b * b; ++x)
    if (!isfinite(R[x])) return true;
  return false;
}

// Householder (LAPACK dlarfg convention): x (len) -> v (v[0]=1), tau, beta.
__device__ void house(const double* x, int len, double* v, double* tau, double* beta_out) {
  double alpha = x[0];
  double xn2 = 0.0;
  for (int i = 1; i < len; ++i) xn2 += x[i] * x[i];
  v[0] = 1.0;
  if (xn2 == 0.0) {
    *tau = 0.0;
    *beta_out = alpha;
    for (int i = 1; i < len; ++i) v[i] = 0.0;
    return;
  }
  double nrm = sqrt(alpha * alpha + xn2);
  double beta = (alpha >= 0.0) ? -nrm : nrm;
  *tau = (beta - alpha) / beta;
  const double sc = 1.0 / (alpha - beta);
  for (int i = 1; i < len; ++i) v[i] = x[i] * sc;
  *beta_out = beta;
}

// Solve the b x b system Hm X = Gm (column-major, in place copies) by Gaussian elimination
// with partial pivoting (sequential).  Returns true if singular.
__device__ bool small_solve(double* Hm, double* Gm, int b) {
  for (int p = 0; p < b; ++p) {
    int piv = p;
    double best = fabs(Hm[p + p * b]);
    for (int r = p + 1; r < b; ++r)
      if (fabs(Hm[r + p * b]) > best) { best = fabs(Hm[r + p * b]); piv = r; }
    if (!(best > 0.0) || !isfinite(best)) return true;
    if (piv != p) {
      for (int c = 0; c < b; ++c) { double t = Hm[p + c * b]; Hm[p + c * b] = Hm[piv + c * b]; Hm[piv + c * b] = t; }
      for (int c = 0; c < b; ++c) { double t = Gm[p + c * b]; Gm[p + c * b] = Gm[piv + c * b]; Gm[piv + c * b] = t; }
    }
    const double d = Hm[p + p * b];
    for (int r = p + 1; r < b; ++r) {
      const double f = Hm[r + p * b] / d;
      for (int c = p; c < b; ++c) Hm[r + c * b] -= f * Hm[p + c * b];
      for (int c = 0; c < b; ++c) Gm[r + c * b] -= f * Gm[p + c * b];
    }
  }
  for (int c = 0; c < b; ++c)
    for (int r = b - 1; r >= 0; --r) {
      double t = Gm[r + c * b];
      for (int q = r + 1; q < b; ++q) t -= Hm[r + q * b] * Gm[q + c * b];
      Gm[r + c * b] = t / Hm[r + r * b];
    }
  for (int x = 0; x < b * b; ++x)
    if (!isfinite(Gm[x])) return true;
  return false;
}

// a3 + a5: one block, blockDim = 256.  k >= 1: step k; k == 0: IO of the cycle's start block.
// G: ((k+1)b) x b row-major (classical) or k+1 scalars (global, already scaled by 1/s).
// rfac: sqrt(s) for global (residual norms), 1 for classical.
__global__ void __launch_bounds__(256)
k_small_step(SmallState st, const double* __restrict__ G, int k, int force_flag, double rfac) {
  const int b = st.b, ldH = st.ldH;
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double S_[kMaxB * kMaxB], R_[kMaxB * kMaxB], Ri_[kMaxB * kMaxB];
  __shared__ double col_[2 * kMaxB * kMaxB], tmpA[kMaxB * kMaxB], tmpB[kMaxB * kMaxB];
  __shared__ double red[32];
  __shared__ int flag_s;
  const int kb = k * b;
  // Hcol -> Hbar column block k-1 (rows 0..kb-1); G is row-major [(row) * b + col]
  if (k > 0)
    for (int e = tid; e < kb * b; e += nt) {
      const int r = e / b, c = e % b;
      st.Hbar[r + (size_t)((k - 1) * b + c) * ldH] = G[e];
    }
  // S = Omega - Hcol^T Hcol, symmetrised (R2); column-major b x b
  for (int e = tid; e < b * b; e += nt) {
    const int x = e % b, y = e / b;
    double t = G[(size_t)(kb + x) * b + y];
    for (int r = 0; r < kb; ++r) t -= G[(size_t)r * b + x] * G[(size_t)r * b + y];
    tmpA[x + y * b] = t;
  }
  __syncthreads();
  for (int e = tid; e < b * b; e += nt) {
    const int x = e % b, y = e / b;
    S_[x + y * b] = 0.5 * (tmpA[x + y * b] + tmpA[y + x * b]);
  }
  __syncthreads();
  if (tid == 0) {
    bool f = chol_upper(S_, R_, b);
    if (force_flag) f = true;
    flag_s = f ? 1 : 0;
    *st.flag_dev = flag_s;
    if (f && k > 0)  // flagged step: no H_{k+1,k}; keep Hbar's subdiagonal block clean
      for (int x = 0; x < b; ++x)
        for (int y = 0; y < b; ++y) st.Hbar[(kb + x) + (size_t)((k - 1) * b + y) * ldH] = 0.0;
    st.status->k = k;
    st.status->flag = flag_s;
    st.status->proj_singular = 0;
    st.status->res_gmres = st.status->res_fom = st.status->kappa_F = nan("");
    if (k == 0) {
      double tr = 0.0;
      for (int x = 0; x < b; ++x) tr += G[x * b + x];
      st.status->normU2 = tr * (rfac * rfac);
    }
  }
  __syncthreads();
  if (flag_s) return;
  // R^{-1} (upper triangular), column c by back substitution (threads over columns)
  if (tid < b) {
    const int c = tid;
    for (int r = b - 1; r >= 0; --r) {
      double t = (r == c) ? 1.0 : 0.0;
      for (int q = r + 1; q <= c; ++q) t -= R_[r + q * b] * Ri_[q + c * b];
      Ri_[r + c * b] = (r <= c) ? t / R_[r + r * b] : 0.0;
    }
    for (int r = c + 1; r < b; ++r) Ri_[r + c * b] = 0.0;
  }
  __syncthreads();
  // projection coefficients, row-major [(row)*b + c]: rows < kb: -Hcol R^{-1}; then R^{-1}
  for (int e = tid; e < (kb + b) * b; e += nt) {
    const int r = e / b, c = e % b;
    double t;
    if (r < kb) {
      t = 0.0;
      for (int q = 0; q <= c; ++q) t -= G[(size_t)r * b + q] * Ri_[q + c * b];
    } else {
      t = Ri_[(r - kb) + c * b];
    }
    st.coef[e] = t;
  }
  if (k == 0) {
    // IO: beta = R; QR / kappa state of the cycle start: g = E_1 beta, R_1^{-1} = beta^{-1}
    for (int e = tid; e < b * b; e += nt) {
      const int x = e % b, y = e / b;
      st.beta[e] = R_[e];
      st.Rinv[x + (size_t)y * ldH] = Ri_[e];
    }
    for (int e = tid; e < (st.m + 1) * b * b; e += nt) {
      const int r = e % ((st.m + 1) * b), c = e / ((st.m + 1) * b);
      st.g[r + (size_t)c * ldH] = (r < b) ? R_[r + c * b] : 0.0;
    }
    double nr = 0.0, ni = 0.0;
    for (int e = tid; e < b * b; e += nt) { nr += R_[e] * R_[e]; ni += Ri_[e] * Ri_[e]; }
    nr = block_sum(nr, red);
    ni = block_sum(ni, red);
    if (tid == 0) { st.sc[0] = nr; st.sc[1] = ni; st.status->kappa_F = sqrt(nr * ni); }
    return;
  }
  // store H_{k+1,k} = R into Hbar
  for (int e = tid; e < b * b; e += nt) {
    const int x = e % b, y = e / b;
    st.Hbar[(kb + x) + (size_t)((k - 1) * b + y) * ldH] = R_[e];
  }
  __syncthreads();
  // ---- incremental Householder QR of Hbar (reading R11) ----
  // new column c ((k+1)b x b) -> col_ local copy of the last two block rows after applying
  // reflectors 1..k-1 (reflector j acts on block rows j-1, j).  Thread per column of c.
  // We only need block rows k-1 and k of the transformed column at the end, but the
  // transformation sweeps down the column, so carry a 2b window.
  if (tid < b) {
    const int c = tid;
    // window holds rows [(j-1)b, (j+1)b) of the working column; start with j = 1
    double win[2 * kMaxB];
    for (int r = 0; r < 2 * b; ++r) {
      const int gr = r;
      win[r] = (gr < kb + b) ? st.Hbar[gr + (size_t)((k - 1) * b + c) * ldH] : 0.0;
    }
    for (int j = 1; j <= k - 1; ++j) {
      const double* V = st.qr_v + (size_t)(j - 1) * b * 2 * b;
      const double* T = st.qr_tau + (size_t)(j - 1) * b;
      for (int q = 0; q < b; ++q) {
        const double* v = V + (size_t)q * 2 * b;
        double d = 0.0;
        for (int r = q; r < 2 * b; ++r) d += v[r] * win[r];
        d *= T[q];
        for (int r = q; r < 2 * b; ++r) win[r] -= d * v[r];
      }
      // top block row of the window is final (an R entry, not needed): shift down by b
      for (int r = 0; r < b; ++r) win[r] = win[b + r];
      for (int r = 0; r < b; ++r) {
        const int gr = (j + 1) * b + r;
        win[b + r] = (gr < kb + b) ? st.Hbar[gr + (size_t)((k - 1) * b + c) * ldH] : 0.0;
      }
    }
    for (int r = 0; r < 2 * b; ++r) col_[r + c * 2 * b] = win[r];
  }
  __syncthreads();
  if (tid == 0) {
    // FOM estimate: h~ = col_ rows 0..b-1, g^ = g rows (k-1)b..kb-1 (before reflector k)
    for (int x = 0; x < b; ++x)
      for (int y = 0; y < b; ++y) {
        tmpA[x + y * b] = col_[x + y * 2 * b];
        tmpB[x + y * b] = st.g[((k - 1) * b + x) + (size_t)y * ldH];
      }
    const bool sing = small_solve(tmpA, tmpB, b);   // tmpB <- h~^{-1} g^
    st.status->proj_singular = sing ? 1 : 0;
    double rf = nan("");
    if (!sing) {
      // ||R cos C_acc||_F with R = H_{k+1,k} (upper) ; tmpA <- cos C_acc
      double acc2 = 0.0;
      for (int x = 0; x < b; ++x)
        for (int y = 0; y < b; ++y) {
          double t = 0.0;
          for (int q = 0; q < b; ++q) t += tmpB[x + q * b] * st.Cacc[q + y * b];
          tmpA[x + y * b] = t;
        }
      for (int x = 0; x < b; ++x)
        for (int y = 0; y < b; ++y) {
          double t = 0.0;
          for (int q = x; q < b; ++q) t += R_[x + q * b] * tmpA[q + y * b];
          acc2 += t * t;
        }
      rf = sqrt(acc2) * rfac;
    }
    st.status->res_fom = rf;
    // Householder QR of the 2b x b stack col_ -> reflectors for block column k
    double* Vk = st.qr_v + (size_t)(k - 1) * b * 2 * b;
    double* Tk = st.qr_tau + (size_t)(k - 1) * b;
    for (int q = 0; q < b; ++q) {
      double* v = Vk + (size_t)q * 2 * b;
      for (int r = 0; r < q; ++r) v[r] = 0.0;
      double tau, beta_;
      house(col_ + q + q * 2 * b, 2 * b - q, v + q, &tau, &beta_);
      Tk[q] = tau;
      // apply to remaining columns of the stack
      for (int c = q; c < b; ++c) {
        double d = 0.0;
        for (int r = q; r < 2 * b; ++r) d += v[r] * col_[r + c * 2 * b];
        d *= tau;
        for (int r = q; r < 2 * b; ++r) col_[r + c * 2 * b] -= d * v[r];
      }
      // apply to g rows (k-1)b .. (k+1)b-1
      for (int c = 0; c < b; ++c) {
        double* gc = st.g + (size_t)c * ldH + (k - 1) * b;
        double d = 0.0;
        for (int r = q; r < 2 * b; ++r) d += v[r] * gc[r];
        d *= tau;
        for (int r = q; r < 2 * b; ++r) gc[r] -= d * v[r];
      }
    }
    // GMRES estimate: ||g_{k+1} C_acc||_F
    double acc2 = 0.0;
    for (int x = 0; x < b; ++x)
      for (int y = 0; y < b; ++y) {
        double t = 0.0;
        for (int q = 0; q < b; ++q) t += st.g[(kb + x) + (size_t)q * ldH] * st.Cacc[q + y * b];
        acc2 += t * t;
      }
    st.status->res_gmres = sqrt(acc2) * rfac;
  }
  // ---- kappa_F update (reading R8): new block column of R_{k+1}^{-1} ----
  // T = R_k^{-1} Hcol (kb x b), X = -T R^{-1};  Rinv[:, kb..kb+b) = [X; R^{-1}]
  double part_r = 0.0, part_i = 0.0;
  for (int e = tid; e < kb * b; e += nt) {
    const int r = e % kb, c = e / kb;
    double t = 0.0;
    // row r of R_k^{-1} is nonzero for columns q >= r (upper triangular)
    for (int q = r; q < kb; ++q) t += st.Rinv[r + (size_t)q * ldH] * G[(size_t)q * b + c];
    // store T temporarily in Rinv's new column block (column-major), finished below
    st.Rinv[r + (size_t)(kb + c) * ldH] = t;
    part_r += G[(size_t)r * b + c] * G[(size_t)r * b + c];
  }
  __syncthreads();
  for (int e = tid; e < kb * b; e += nt) {
    const int r = e % kb, c = e / kb;
    // X[r][c] = - sum_q T[r][q] Ri[q][c], q <= c
    double t = 0.0;
    for (int q = 0; q <= c; ++q) t -= st.Rinv[r + (size_t)(kb + q) * ldH] * Ri_[q + c * b];
    // write into a scratch column-major buffer (qr g column space is busy; use coef tail)
    st.coef[(kb + b) * b + e] = t;
  }
  __syncthreads();
  for (int e = tid; e < kb * b; e += nt) {
    const int r = e % kb, c = e / kb;
    const double x = st.coef[(kb + b) * b + e];
    st.Rinv[r + (size_t)(kb + c) * ldH] = x;
    part_i += x * x;
  }
  for (int e = tid; e < b * b; e += nt) {
    const int x = e % b, y = e / b;
    st.Rinv[(kb + x) + (size_t)(kb + y) * ldH] = Ri_[e];
    part_i += Ri_[e] * Ri_[e];
    part_r += R_[e] * R_[e];
  }
  const double dr = block_sum(part_r, red);
  const double di = block_sum(part_i, red);
  if (tid == 0) {
    st.sc[0] += dr;
    st.sc[1] += di;
    st.status->kappa_F = sqrt(st.sc[0] * st.sc[1]);
  }
}

// ------------------------------------------------------------------------------------------
// a5/a6 at cycle end: projected solve by dense LU with partial pivoting (one CTA).
//   mode 0: FOM      M = 0
//   mode 1: GMRES    M = H_k^{-T} E_k H_{k+1,k}^T H_{k+1,k}
//   happy != 0: H_{k+1,k} := 0 (reading R7) -> FOM solution, C_acc not updated
// Outputs (row-major, [row][c]):  Y = Xi C_acc (kb x b);  Z = [M; -H_{k+1,k}] ((k+1)b x b);
// then C_acc <- cos C_acc (unless happy).  work: >= (kb)^2 + 2 kb b doubles.
// info[0] = 1 if singular.
// ------------------------------------------------------------------------------------------
__device__ void block_lu_solve(double* Am, int N, double* Bm, int nrhs, int* piv_s,
                               double* red, int* ired, bool* sing) {
  // Am column-major N x N (ld N), Bm column-major N x nrhs (ld N); solved in place.
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int p = 0; p < N; ++p) {
    // pivot search (thread-parallel argmax, deterministic tie-break on index)
    double best = -1.0;
    int bi = p;
    for (int r = p + tid; r < N; r += nt) {
      const double v = fabs(Am[r + (size_t)p * N]);
      if (v > best || (v == best && r < bi)) { best = v; bi = r; }
    }
    red[tid] = best;
    ired[tid] = bi;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (tid < o) {
        const double v2 = red[tid + o];
        const int i2 = ired[tid + o];
        if (v2 > red[tid] || (v2 == red[tid] && i2 < ired[tid])) { red[tid] = v2; ired[tid] = i2; }
      }
      __syncthreads();
    }
    const int pr = ired[0];
    const double pv = red[0];
    __syncthreads();
    if (!(pv > 0.0) || !isfinite(pv)) { *sing = true; return; }
    if (pr != p) {
      for (int c = tid; c < N; c += nt) {
        const double t = Am[p + (size_t)c * N];
        Am[p + (size_t)c * N] = Am[pr + (size_t)c * N];
        Am[pr + (size_t)c * N] = t;
      }
      for (int c = tid; c < nrhs; c += nt) {
        const double t = Bm[p + (size_t)c * N];
        Bm[p + (size_t)c * N] = Bm[pr + (size_t)c * N];
        Bm[pr + (size_t)c * N] = t;
      }
    }
    __syncthreads();
    const double d = Am[p + (size_t)p * N];
    for (int r = p + 1 + tid; r < N; r += nt) Am[r + (size_t)p * N] /= d;
    __syncthreads();
    const int rem = N - p - 1;
    const int tot = rem * (rem + nrhs);
    for (int e = tid; e < tot; e += nt) {
      const int r = p + 1 + e % rem;
      const int c = e / rem;  // 0..rem-1: matrix columns p+1+c; rem..: rhs columns
      const double l = Am[r + (size_t)p * N];
      if (c < rem) Am[r + (size_t)(p + 1 + c) * N] -= l * Am[p + (size_t)(p + 1 + c) * N];
      else         Bm[r + (size_t)(c - rem) * N] -= l * Bm[p + (size_t)(c - rem) * N];
    }
    __syncthreads();
  }
  // back substitution, column-parallel over rhs, row-sequential
  for (int r = N - 1; r >= 0; --r) {
    for (int c = tid; c < nrhs; c += nt) Bm[r + (size_t)c * N] /= Am[r + (size_t)r * N];
    __syncthreads();
    const int tot = r * nrhs;
    for (int e = tid; e < tot; e += nt) {
      const int q = e % r, c = e / r;
      Bm[q + (size_t)c * N] -= Am[q + (size_t)r * N] * Bm[r + (size_t)c * N];
    }
    __syncthreads();
  }
  for (int e = tid; e < N * nrhs; e += nt)
    if (!isfinite(Bm[e])) *sing = true;
  __syncthreads();
}

__global__ void __launch_bounds__(512)
k_cycle_solve(SmallState st, int k, int gmres, int happy, double* __restrict__ work,
              double* __restrict__ Y, double* __restrict__ Z, int* __restrict__ info) {
  const int b = st.b, ldH = st.ldH, kb = k * b;
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double red[512];
  __shared__ int ired[512];
  __shared__ bool sing;
  __shared__ double HtH[kMaxB * kMaxB], cosC[kMaxB * kMaxB];
  if (tid == 0) sing = false;
  double* Am = work;                         // kb x kb
  double* Mm = work + (size_t)kb * kb;       // kb x b  (column-major, ld kb)
  double* Xi = Mm + (size_t)kb * b;          // kb x b
  const double* Hk1 = st.Hbar + kb + (size_t)(k - 1) * b * ldH;  // (row kb, col (k-1)b)
  // HtH = H_{k+1,k}^T H_{k+1,k}  (zero if happy)
  for (int e = tid; e < b * b; e += nt) {
    const int x = e % b, y = e / b;
    double t = 0.0;
    if (!happy)
      for (int q = 0; q < b; ++q) t += Hk1[q + (size_t)x * ldH] * Hk1[q + (size_t)y * ldH];
    HtH[e] = t;
  }
  for (int e = tid; e < kb * b; e += nt) Mm[e] = 0.0;
  __syncthreads();
  if (gmres && !happy) {
    // A = H_k^T ; rhs = E_k HtH
    for (int e = tid; e < kb * kb; e += nt) {
      const int r = e % kb, c = e / kb;
      Am[e] = st.Hbar[c + (size_t)r * ldH];
    }
    for (int e = tid; e < kb * b; e += nt) {
      const int r = e % kb, c = e / kb;
      Mm[e] = (r >= kb - b) ? HtH[(r - (kb - b)) + c * b] : 0.0;
    }
    __syncthreads();
    block_lu_solve(Am, kb, Mm, b, nullptr, red, ired, &sing);
    __syncthreads();
  }
  // A = H_k + M E_k^T ; rhs = E_1 beta
  for (int e = tid; e < kb * kb; e += nt) {
    const int r = e % kb, c = e / kb;
    double t = st.Hbar[r + (size_t)c * ldH];
    if (c >= kb - b) t += Mm[r + (size_t)(c - (kb - b)) * kb];
    Am[e] = t;
  }
  for (int e = tid; e < kb * b; e += nt) {
    const int r = e % kb, c = e / kb;
    Xi[e] = (r < b) ? st.beta[r + c * b] : 0.0;
  }
  __syncthreads();
  block_lu_solve(Am, kb, Xi, b, nullptr, red, ired, &sing);
  __syncthreads();
  // Y = Xi C_acc (row-major), Z = [M; -H_{k+1,k}] (row-major)
  for (int e = tid; e < kb * b; e += nt) {
    const int r = e / b, c = e % b;
    double t = 0.0;
    for (int q = 0; q < b; ++q) t += Xi[r + (size_t)q * kb] * st.Cacc[q + c * b];
    Y[e] = t;
  }
  for (int e = tid; e < (kb + b) * b; e += nt) {
    const int r = e / b, c = e % b;
    Z[e] = (r < kb) ? Mm[r + (size_t)c * kb] : -Hk1[(r - kb) + (size_t)c * ldH];
  }
  __syncthreads();
  if (!happy) {
    // C_acc <- cos C_acc, cos = Xi rows kb-b..kb-1
    for (int e = tid; e < b * b; e += nt) {
      const int x = e % b, y = e / b;
      double t = 0.0;
      for (int q = 0; q < b; ++q) t += Xi[(kb - b + x) + (size_t)q * kb] * st.Cacc[q + y * b];
      cosC[e] = t;
    }
    __syncthreads();
    for (int e = tid; e < b * b; e += nt) st.Cacc[e] = cosC[e];
  }
  if (tid == 0) info[0] = sing ? 1 : 0;
}

__global__ void k_set_identity(double* Cm, int b) {
  const int e = threadIdx.x;
  if (e < b * b) Cm[e] = (e % b == e / b) ? 1.0 : 0.0;
}

}  // namespace lsba
