// spmm_bench.cu — standalone timing of SpMM kernel candidates (dev tool) on the stencil shapes
// of configs 2 (2D 5-point, n = 2^20, s = 4) and 5 (3D 7-point, n = 2^24, s = 8).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build_tools/spmm_bench tools/spmm_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include "../paper_2208_09899_b200/csrc/kernels.cuh"

using namespace lsba;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

// B: two rows per lane group (rows i and i + half), one joint loop
template <int S>
__global__ void __launch_bounds__(256)
k_spmm_2row(int n, int half, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
            const double* __restrict__ V, double* __restrict__ W) {
  constexpr int L = S / 2;
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int r1 = (int)(gt / L), lane = (int)(gt % L);
  const int r2 = r1 + half;
  if (r1 >= half) return;
  const bool has2 = r2 < n;
  const int p10 = __ldg(rp + r1), p11 = __ldg(rp + r1 + 1);
  const int p20 = has2 ? __ldg(rp + r2) : 0, p21 = has2 ? __ldg(rp + r2 + 1) : 0;
  double a0 = 0, a1 = 0, b0 = 0, b1 = 0;
  const int l1 = p11 - p10, l2 = p21 - p20;
  const int lm = max(l1, l2);
  for (int t = 0; t < lm; ++t) {
    if (t < l1) {
      const int c = __ldg(ci + p10 + t); const double a = __ldg(va + p10 + t);
      const double2 v = __ldg(reinterpret_cast<const double2*>(V + (size_t)c * S) + lane);
      a0 = fma(a, v.x, a0); a1 = fma(a, v.y, a1);
    }
    if (t < l2) {
      const int c = __ldg(ci + p20 + t); const double a = __ldg(va + p20 + t);
      const double2 v = __ldg(reinterpret_cast<const double2*>(V + (size_t)c * S) + lane);
      b0 = fma(a, v.x, b0); b1 = fma(a, v.y, b1);
    }
  }
  reinterpret_cast<double2*>(W + (size_t)r1 * S)[lane] = make_double2(a0, a1);
  if (has2) reinterpret_cast<double2*>(W + (size_t)r2 * S)[lane] = make_double2(b0, b1);
}

// C: current kernel with the entry loop unrolled by 8
template <int S>
__global__ void __launch_bounds__(256)
k_spmm_u8(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
          const double* __restrict__ V, double* __restrict__ W) {
  constexpr int L = S / 2;
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / L), lane = (int)(gt % L);
  if (row >= n) return;
  const int p0 = __ldg(rp + row), p1 = __ldg(rp + row + 1);
  double a0 = 0, a1 = 0;
#pragma unroll 8
  for (int p = p0; p < p1; ++p) {
    const int c = __ldg(ci + p); const double a = __ldg(va + p);
    const double2 v = __ldg(reinterpret_cast<const double2*>(V + (size_t)c * S) + lane);
    a0 = fma(a, v.x, a0); a1 = fma(a, v.y, a1);
  }
  reinterpret_cast<double2*>(W + (size_t)row * S)[lane] = make_double2(a0, a1);
}

// D: one thread per row, all S columns
template <int S>
__global__ void __launch_bounds__(256)
k_spmm_row(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
           const double* __restrict__ V, double* __restrict__ W) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const int p0 = __ldg(rp + row), p1 = __ldg(rp + row + 1);
  double acc[S];
#pragma unroll
  for (int t = 0; t < S; ++t) acc[t] = 0;
  for (int p = p0; p < p1; ++p) {
    const int c = __ldg(ci + p); const double a = __ldg(va + p);
    const double2* src = reinterpret_cast<const double2*>(V + (size_t)c * S);
#pragma unroll
    for (int t = 0; t < S / 2; ++t) { const double2 v = __ldg(src + t); acc[2 * t] = fma(a, v.x, acc[2 * t]); acc[2 * t + 1] = fma(a, v.y, acc[2 * t + 1]); }
  }
  double2* dst = reinterpret_cast<double2*>(W + (size_t)row * S);
#pragma unroll
  for (int t = 0; t < S / 2; ++t) dst[t] = make_double2(acc[2 * t], acc[2 * t + 1]);
}

// E: rows of a warp processed as a "column-major" walk: entry t of all rows of the lane group
// block before entry t+1 (same as A but with the row pointer pair loaded by a shuffle)
template <int S>
__global__ void __launch_bounds__(256)
k_spmm_shfl(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
            const double* __restrict__ V, double* __restrict__ W) {
  constexpr int L = S / 2;
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / L), lane = (int)(gt % L);
  const int lane32 = threadIdx.x & 31;
  // the warp's rows are row_w .. row_w + 32/L - 1: lane j loads rp[row_w + j] (j <= 32/L)
  const int row_w = (int)(((long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / L);
  const int rr = row_w + lane32;
  const int pv = (lane32 <= 32 / L && rr <= n) ? __ldg(rp + rr) : 0;
  const int me = lane32 / L;
  const int p0 = __shfl_sync(0xffffffffu, pv, me), p1 = __shfl_sync(0xffffffffu, pv, me + 1);
  if (row >= n) return;
  double a0 = 0, a1 = 0;
  for (int p = p0; p < p1; ++p) {
    const int c = __ldg(ci + p); const double a = __ldg(va + p);
    const double2 v = __ldg(reinterpret_cast<const double2*>(V + (size_t)c * S) + lane);
    a0 = fma(a, v.x, a0); a1 = fma(a, v.y, a1);
  }
  reinterpret_cast<double2*>(W + (size_t)row * S)[lane] = make_double2(a0, a1);
}

__device__ __forceinline__ int ld_pf_i(const int* p) {
  int v; asm volatile("ld.global.nc.L2::256B.b32 %0, [%1];" : "=r"(v) : "l"(p)); return v;
}
__device__ __forceinline__ double ld_pf_d(const double* p) {
  double v; asm volatile("ld.global.nc.L2::256B.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v;
}
__device__ __forceinline__ double2 ld_pf_d2(const double2* p) {
  double2 v; asm volatile("ld.global.nc.L2::256B.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p)); return v;
}
// F: shfl + 256-byte L2 prefetch on the index/value streams (G: and on the V gathers)
template <int S, bool PFV>
__global__ void __launch_bounds__(256)
k_spmm_pf(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
          const double* __restrict__ V, double* __restrict__ W) {
  constexpr int L = S / 2;
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / L), lane = (int)(gt % L);
  const int lane32 = threadIdx.x & 31;
  const int row_w = (int)(((long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / L);
  const int rr = row_w + lane32;
  const int pv = (lane32 <= 32 / L && rr <= n) ? ld_pf_i(rp + rr) : 0;
  const int me = lane32 / L;
  const int p0 = __shfl_sync(0xffffffffu, pv, me), p1 = __shfl_sync(0xffffffffu, pv, me + 1);
  if (row >= n) return;
  double a0 = 0, a1 = 0;
  for (int p = p0; p < p1; ++p) {
    const int c = ld_pf_i(ci + p); const double a = ld_pf_d(va + p);
    const double2* src = reinterpret_cast<const double2*>(V + (size_t)c * S) + lane;
    const double2 v = PFV ? ld_pf_d2(src) : __ldg(src);
    a0 = fma(a, v.x, a0); a1 = fma(a, v.y, a1);
  }
  reinterpret_cast<double2*>(W + (size_t)row * S)[lane] = make_double2(a0, a1);
}

// H: batched entries: per chunk of NB entries of the row, all index/value loads first, then all
// NB gathers, then the FMAs (NB independent gathers in flight per thread); register budget
// from MINB CTAs of 256 per SM.  NA: index/value loads bypass L1 allocation.
template <bool NA>
__device__ __forceinline__ int ld_i(const int* p) {
  if constexpr (NA) { int v; asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(v) : "l"(p)); return v; }
  else return __ldg(p);
}
template <bool NA>
__device__ __forceinline__ double ld_d(const double* p) {
  if constexpr (NA) { double v; asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p)); return v; }
  else return __ldg(p);
}
template <int S, int NB, int MINB, bool NA>
__global__ void __launch_bounds__(256, MINB)
k_spmm_batch(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
             const double* __restrict__ V, double* __restrict__ W) {
  constexpr int L = S / 2;
  const long gt = (long)blockIdx.x * blockDim.x + threadIdx.x;
  const int row = (int)(gt / L), lane = (int)(gt % L);
  const int lane32 = threadIdx.x & 31;
  const int row_w = (int)(((long)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / L);
  const int rr = row_w + lane32;
  const int pv = (lane32 <= 32 / L && rr <= n) ? __ldg(rp + rr) : 0;
  const int me = lane32 / L;
  const int p0 = __shfl_sync(0xffffffffu, pv, me), p1 = __shfl_sync(0xffffffffu, pv, me + 1);
  if (row >= n) return;
  double a0 = 0, a1 = 0;
  for (int p = p0; p < p1; p += NB) {
    int c[NB]; double a[NB]; double2 v[NB];
#pragma unroll
    for (int t = 0; t < NB; ++t) {
      const bool ok = p + t < p1;
      c[t] = ok ? ld_i<NA>(ci + p + t) : row;
      a[t] = ok ? ld_d<NA>(va + p + t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t < NB; ++t) v[t] = __ldg(reinterpret_cast<const double2*>(V + (size_t)c[t] * S) + lane);
#pragma unroll
    for (int t = 0; t < NB; ++t) { a0 = fma(a[t], v[t].x, a0); a1 = fma(a[t], v[t].y, a1); }
  }
  reinterpret_cast<double2*>(W + (size_t)row * S)[lane] = make_double2(a0, a1);
}

// P: persistent CTAs with a cp.async double-buffered shared-memory ring of the CSR slices
// (row pointers, column indices, values of one chunk of RPC rows) — the CSR stream runs ahead
// asynchronously; the compute warps read indices from shared memory and issue all of a row's
// gathers at once (up to NB per batch).  Chunks whose slice exceeds MAXE entries fall back to
// global index loads.
__device__ __forceinline__ void cpa4(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" :: "r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa8(void* dst, const void* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" :: "n"(N) : "memory"); }

template <int S, int MAXPR, int NB, int CPS>
__global__ void __launch_bounds__(256, CPS)
k_spmm_pipe(int n, const int* __restrict__ rp, const int* __restrict__ ci, const double* __restrict__ va,
            const double* __restrict__ V, double* __restrict__ W) {
  constexpr int L = S / 2, RPC = 256 / L, MAXE = MAXPR * RPC;
  __shared__ int srp[2][RPC + 1];
  __shared__ int sci[2][MAXE];
  __shared__ double sva[2][MAXE];
  const int nchunks = (n + RPC - 1) / RPC;
  const int tid = threadIdx.x;
  auto stage = [&](int chunk, int buf) {
    const int r0 = chunk * RPC, r1 = min(n, r0 + RPC);
    for (int e = tid; e <= r1 - r0; e += 256) cpa4(&srp[buf][e], rp + r0 + e);
    const int p0 = __ldg(rp + r0), p1 = __ldg(rp + r1);
    if (p1 - p0 <= MAXE) {
      for (int e = tid; e < p1 - p0; e += 256) {
        cpa4(&sci[buf][e], ci + p0 + e);
        cpa8(&sva[buf][e], va + p0 + e);
      }
    }
    cpa_commit();
  };
  int chunk = blockIdx.x;
  if (chunk < nchunks) stage(chunk, 0);
  for (int it = 0; chunk < nchunks; ++it, chunk += gridDim.x) {
    const int buf = it & 1;
    const int nxt = chunk + gridDim.x;
    if (nxt < nchunks) stage(nxt, buf ^ 1); else cpa_commit();
    cpa_wait<1>();
    __syncthreads();
    const int r0 = chunk * RPC;
    const int lr = tid / L, lane = tid % L;
    const int row = r0 + lr;
    if (row < n) {
      const int pb = srp[buf][0];
      const int q0 = srp[buf][lr] - pb, q1 = srp[buf][lr + 1] - pb;
      const bool in_smem = (srp[buf][min(RPC, n - r0)] - pb) <= MAXE;
      double a0 = 0, a1 = 0;
      for (int q = q0; q < q1; q += NB) {
        int c[NB]; double a[NB]; double2 v[NB];
#pragma unroll
        for (int t = 0; t < NB; ++t) {
          const bool ok = q + t < q1;
          c[t] = ok ? (in_smem ? sci[buf][q + t] : __ldg(ci + pb + q + t)) : row;
          a[t] = ok ? (in_smem ? sva[buf][q + t] : __ldg(va + pb + q + t)) : 0.0;
        }
#pragma unroll
        for (int t = 0; t < NB; ++t) v[t] = __ldg(reinterpret_cast<const double2*>(V + (size_t)c[t] * S) + lane);
#pragma unroll
        for (int t = 0; t < NB; ++t) { a0 = fma(a[t], v[t].x, a0); a1 = fma(a[t], v[t].y, a1); }
      }
      reinterpret_cast<double2*>(W + (size_t)row * S)[lane] = make_double2(a0, a1);
    }
    __syncthreads();
  }
  cpa_wait<0>();
}

template <typename F>
static double time_it(F launch) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) launch();
  cudaEventRecord(b); CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  return 1e3 * ms / 20;
}

template <int S>
static void run(int dims, int N) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long n = 1; for (int d = 0; d < dims; ++d) n *= N;
  std::vector<int> rp(n + 1), ci; std::vector<double> va;
  ci.reserve(n * (2 * dims + 1)); va.reserve(n * (2 * dims + 1));
  long stride[3] = {1, N, (long)N * N};
  for (long i = 0; i < n; ++i) {
    rp[i] = (int)ci.size();
    long coord[3] = {i % N, (i / N) % N, i / ((long)N * N)};
    for (int d = dims - 1; d >= 0; --d) if (coord[d] > 0) { ci.push_back((int)(i - stride[d])); va.push_back(-1.0); }
    ci.push_back((int)i); va.push_back(2.0 * dims);
    for (int d = 0; d < dims; ++d) if (coord[d] < N - 1) { ci.push_back((int)(i + stride[d])); va.push_back(-1.0); }
  }
  rp[n] = (int)ci.size();
  const long nnz = ci.size();
  int *drp, *dci; double *dva, *dV, *dW, *dW2;
  CK(cudaMalloc(&drp, 4 * (n + 1))); CK(cudaMalloc(&dci, 4 * nnz)); CK(cudaMalloc(&dva, 8 * nnz));
  CK(cudaMalloc(&dV, 8 * n * S)); CK(cudaMalloc(&dW, 8 * n * S)); CK(cudaMalloc(&dW2, 8 * n * S));
  CK(cudaMemcpy(drp, rp.data(), 4 * (n + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dci, ci.data(), 4 * nnz, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dva, va.data(), 8 * nnz, cudaMemcpyHostToDevice));
  std::vector<double> hv(n * S); for (long i = 0; i < n * S; ++i) hv[i] = std::sin(0.001 * i);
  CK(cudaMemcpy(dV, hv.data(), 8 * n * S, cudaMemcpyHostToDevice));
  const double bytes = 12.0 * nnz + 4.0 * (n + 1) + 16.0 * n * S;
  constexpr int L = S / 2;
  auto check = [&](const char* name, double us) {
    std::vector<double> a(n * S), b(n * S);
    CK(cudaMemcpy(a.data(), dW, 8 * n * S, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(b.data(), dW2, 8 * n * S, cudaMemcpyDeviceToHost));
    double md = 0; for (long i = 0; i < n * S; ++i) md = std::max(md, std::fabs(a[i] - b[i]));
    printf("  %-10s %8.1f us %7.0f GB/s  maxdiff %.1e\n", name, us, bytes / us / 1e3, md);
  };
  printf("dims %d N %d n %ld s %d nnz %ld (%.0f MB)\n", dims, N, n, S, nnz, bytes / 1e6);
  const int gA = (int)((n * L + 255) / 256);
  double us = time_it([&] { k_spmm<S, false><<<gA, 256>>>((int)n, drp, dci, dva, dV, nullptr, nullptr, dW, nullptr, nullptr); });
  CK(cudaMemcpy(dW2, dW, 8 * n * S, cudaMemcpyDeviceToDevice));
  check("current", us);
  const int half = (int)((n + 1) / 2);
  us = time_it([&] { k_spmm_u8<S><<<gA, 256>>>((int)n, drp, dci, dva, dV, dW); });
  check("unroll8", us);
  us = time_it([&] { k_spmm_shfl<S><<<gA, 256>>>((int)n, drp, dci, dva, dV, dW); });
  check("shfl", us);
  us = time_it([&] { k_spmm_pf<S, false><<<gA, 256>>>((int)n, drp, dci, dva, dV, dW); });
  check("pf", us);
  us = time_it([&] { k_spmm_pf<S, true><<<gA, 256>>>((int)n, drp, dci, dva, dV, dW); });
  check("pfV", us);
#define HB(NB, MINB, NA) \
  us = time_it([&] { k_spmm_batch<S, NB, MINB, NA><<<gA, 256>>>((int)n, drp, dci, dva, dV, dW); }); \
  check("b" #NB "m" #MINB #NA, us);
#undef HB
#define HP(MAXPR, NB, CPS, G) \
  us = time_it([&] { k_spmm_pipe<S, MAXPR, NB, CPS><<<sms * G, 256>>>((int)n, drp, dci, dva, dV, dW); }); \
  check("pipe" #MAXPR "_" #NB "_" #CPS "x" #G, us);
  HP(8, 4, 2, 2) HP(8, 8, 2, 2) HP(8, 4, 3, 3) HP(8, 8, 3, 3) HP(8, 4, 4, 4) HP(8, 8, 4, 4) HP(8, 4, 4, 8)
#undef HP
  cudaFree(drp); cudaFree(dci); cudaFree(dva); cudaFree(dV); cudaFree(dW); cudaFree(dW2);
}

int main() {
  run<4>(2, 1024);
  run<8>(3, 128);
  run<8>(3, 256);
  run<16>(3, 128);
  return 0;
}
