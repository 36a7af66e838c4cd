// microbench.cu — B200 measurements that decide the Gram/projection kernel design:
//   1. DFMA throughput (independent FMA chains, all SMs)
//   2. DMMA m8n8k4 f64 throughput (independent accumulator chains)
//   3. streaming-read bandwidth vs bytes in flight per thread (LDG.128, grid-stride)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench tools/microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_dfma(double* out, int iters, double a) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, 1.0);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters, double a) {
  double d[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) d[i][0] = d[i][1] = 0.0;
  double b = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma(d[i][0], d[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += d[i][0] + d[i][1];
  if (s == 1234.5) out[0] = s;
}

__global__ void k_mixed(double* out, int iters, double a) {
  double d[4][2];
  double x[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) d[i][0] = d[i][1] = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  double b = threadIdx.x * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) dmma(d[i][0], d[i][1], a, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, 1.0);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += d[i][0] + d[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

template <int U>
__global__ void k_read(const double2* __restrict__ p, size_t n2, double* out) {
  double2 acc = make_double2(0, 0);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n2; i += U * stride) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldg(p + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
  }
  for (; i < n2; i += stride) { double2 v = __ldg(p + i); acc.x += v.x; acc.y += v.y; }
  if (acc.x == 1234.5) out[0] = acc.y;
}

template <int U>
static float time_read(const double2* p, size_t n2, double* out, int grid, int block) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  k_read<U><<<grid, block>>>(p, n2, out);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_read<U><<<grid, block>>>(p, n2, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  for (int occ : {4, 8, 16}) {
    const int grid = sms * occ, block = 256;
    k_dfma<<<grid, block>>>(out, 16, 1.0000001);
    cudaEventRecord(a); k_dfma<<<grid, block>>>(out, iters, 1.0000001); cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fma_ = (double)grid * block * iters * 8;
    printf("DFMA  grid %5d: %.2f TFLOP/s (%.1f FMA/clk/SM)\n", grid, 2 * fma_ / ms / 1e9,
           fma_ / (ms * 1e-3) / sms / (clk * 1e3));
  }
  for (int occ : {4, 8, 16}) {
    const int grid = sms * occ, block = 256;
    k_dmma<<<grid, block>>>(out, 16, 1.0);
    cudaEventRecord(a); k_dmma<<<grid, block>>>(out, iters, 1.0); cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    double mac = (double)grid * (block / 32) * iters * 8 * 256;
    printf("DMMA  grid %5d: %.2f TFLOP/s (%.1f MAC/clk/SM)\n", grid, 2 * mac / ms / 1e9,
           mac / (ms * 1e-3) / sms / (clk * 1e3));
  }
  for (int occ : {8, 16}) {
    const int grid = sms * occ, block = 256;
    k_mixed<<<grid, block>>>(out, 16, 1.0);
    cudaEventRecord(a); k_mixed<<<grid, block>>>(out, iters, 1.0); cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b);
    // per warp-iteration: 4 DMMA (4 x 256 MAC) + 8 DFMA per lane (8 x 32 FMA)
    const double mac = (double)grid * (block / 32) * iters * (4.0 * 256 + 8.0 * 32);
    printf("MIXED grid %5d: %.1f MAC/clk/SM (DMMA share %.0f%%)\n", grid,
           mac / (ms * 1e-3) / sms / (clk * 1e3), 100.0 * 1024 / 1280);
  }
  const size_t bytes = (size_t)4 << 30;
  double2* p; CK(cudaMalloc(&p, bytes));
  CK(cudaMemset(p, 0, bytes));
  const size_t n2 = bytes / 16;
  for (int block : {256}) {
    for (int cps : {1, 2, 4, 8}) {
      const int grid = sms * cps;
      float t1 = time_read<1>(p, n2, out, grid, block);
      float t2 = time_read<2>(p, n2, out, grid, block);
      float t4 = time_read<4>(p, n2, out, grid, block);
      float t8 = time_read<8>(p, n2, out, grid, block);
      printf("read  %d CTA/SM x %d thr: U1 %.0f  U2 %.0f  U4 %.0f  U8 %.0f GB/s\n", cps, block,
             bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t4 / 1e6, bytes / t8 / 1e6);
    }
  }
  return 0;
}
