// gram_bench.cu — standalone timing of the Gram-pass kernel candidates on the bench shapes
// (dev tool; the product path is liblsba.so).  For (n, s, J): basis of J padded slots with the
// last slot aliased as W, G = [X_0..X_{J-1}]^T W.  Reports us/launch and algorithmic GB/s
// (8 n s J bytes), and the max relative difference of G against k_gram_v7<S, 2, 4, 3>.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o build_tools/gram_bench tools/gram_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>
#include "../paper_2208_09899_b200/csrc/gram7.cuh"

using namespace lsba;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed;
    x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
    p[i] = (double)x / 4294967296.0 - 0.5;
  }
}

struct Bufs {
  double *V, *part, *gpart, *G, *zeros;
  unsigned* tickets;
  size_t stride;
};

template <typename F>
static double time_it(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  return 1e3 * ms / reps;
}

static GramArgs args(const Bufs& B, int n, int J) {
  GramArgs a{};
  a.n = n; a.X = B.V; a.xstride = B.stride; a.J = J; a.y_alias = 1;
  a.Y = B.V + (size_t)(J - 1) * B.stride; a.zeros = B.zeros;
  a.part = B.part; a.gpart = B.gpart; a.tickets = B.tickets; a.G = B.G; a.active = nullptr;
  return a;
}

template <int S, int GMAX, int U, int MINB, bool WIN = true>
static std::vector<double> run_v7(const Bufs& B, int n, int J, double* us, int* grid_out) {
  GramArgs a = args(B, n, J);
  auto fn = k_gram_v7<S, GMAX, U, MINB, WIN>;
  G7Launch<S, GMAX> geo(n, J, MINB, 148);
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(geo.smem, 48 * 1024)));
  *grid_out = geo.grid;
  GramFuse nf{};
  *us = time_it([&] { fn<<<geo.grid, 256, geo.smem>>>(a, nf); }, 10);
  CK(cudaGetLastError());
  std::vector<double> G(J * S * S);
  CK(cudaMemcpy(G.data(), B.G, sizeof(double) * G.size(), cudaMemcpyDeviceToHost));
  return G;
}

// memory-only twin of k_gram_v7's access pattern: same chunks, same per-lane 16-byte loads of
// every block row (and the W fragment), summed instead of multiplied on the tensor cores
// memory-only twins of k_gram_v7's access pattern (16-byte loads of every block row, summed):
// WIN = false: each CTA streams its own contiguous chunk (as v7); WIN = true: the whole grid
// sweeps a moving window of rows (CTA b, warp w take U consecutive steps at ((i G + b) 8 + w) U)
template <int S, int U, bool WIN>
__global__ void __launch_bounds__(256, 3)
k_read_blocks(const double* X, size_t xstride, int J, int n, double* out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long NS = ((long)n + 3) / 4;
  constexpr int PB = S >= 16 ? 1 : 16 / S;
  const int NG = (J + PB - 1) / PB;
  const int r4 = lane & 3, c8 = lane >> 2;
  constexpr int LPB = S >= 16 ? 8 : S / 2;
  const int jj = c8 / LPB, cp = c8 % LPB;
  double acc = 0.0;
  for (int g0 = 0; g0 < NG; g0 += 4) {      // 4 groups at a time (registers)
    long s0, s1, stride, first;
    if (WIN) { s0 = 0; s1 = NS; first = ((long)blockIdx.x * 8 + warp) * U; stride = (long)gridDim.x * 8 * U; }
    else { s0 = NS * blockIdx.x / gridDim.x; s1 = NS * (blockIdx.x + 1) / gridDim.x; first = s0 + (long)warp * U; stride = 8L * U; }
    for (long st = first; st < s1; st += stride) {
      double2 v[U][4];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int j = (g0 + g) * PB + jj;
          const long su = st + u;
          v[u][g] = (g0 + g < NG && j < J && su < s1)
                        ? __ldg(reinterpret_cast<const double2*>(X + (size_t)j * xstride + (su * 4 + r4) * S + 2 * cp))
                        : make_double2(0.0, 0.0);
        }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int g = 0; g < 4; ++g) acc += v[u][g].x + v[u][g].y;
    }
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int S>
static void read_line(const Bufs& B, int n, int J, double bytes) {
  double us = time_it([&] { k_read_blocks<S, 4, false><<<444, 256>>>(B.V, B.stride, J, n, B.G); }, 10);
  printf("   read twin chunked  : %8.1f us %7.0f GB/s\n", us, bytes / us / 1e3);
  us = time_it([&] { k_read_blocks<S, 4, true><<<444, 256>>>(B.V, B.stride, J, n, B.G); }, 10);
  printf("   read twin windowed : %8.1f us %7.0f GB/s\n", us, bytes / us / 1e3);
}

static double reldiff(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) { num = std::max(num, std::fabs(a[i] - b[i])); den = std::max(den, std::fabs(b[i])); }
  return num / den;
}

template <int S, int GMAX, int U, int MINB, bool WIN = true>
static void v7_line(const Bufs& B, int n, int J, const std::vector<double>& ref, double bytes) {
  double us; int grid;
  auto G = run_v7<S, GMAX, U, MINB, WIN>(B, n, J, &us, &grid);
  int regs = 0;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_gram_v7<S, GMAX, U, MINB, WIN>); regs = fa.numRegs;
  printf("   v7<G%d,U%d,B%d,W%d> regs %3d grid %4d: %8.1f us %7.0f GB/s  diff %.1e\n", GMAX, U, MINB, (int)WIN, regs, grid, us,
         bytes / us / 1e3, reldiff(G, ref));
}

template <int S>
static void sweep(int n, std::vector<int> Js) {
  const int maxJ = *std::max_element(Js.begin(), Js.end());
  Bufs B;
  const size_t npad = ((size_t)n + kRowPad - 1) / kRowPad * kRowPad;
  B.stride = npad * S;
  CK(cudaMalloc(&B.V, sizeof(double) * B.stride * maxJ));
  CK(cudaMemset(B.V, 0, sizeof(double) * B.stride * maxJ));
  for (int j = 0; j < maxJ; ++j) k_fill<<<1024, 256>>>(B.V + j * B.stride, (size_t)n * S, 17 + j);
  const size_t E = (size_t)maxJ * S * S;
  CK(cudaMalloc(&B.part, sizeof(double) * E * 148 * 8));
  CK(cudaMalloc(&B.gpart, sizeof(double) * E * 148));
  CK(cudaMalloc(&B.G, sizeof(double) * E));
  CK(cudaMalloc(&B.zeros, 64 * sizeof(double)));
  CK(cudaMemset(B.zeros, 0, 64 * sizeof(double)));
  CK(cudaMalloc(&B.tickets, 4096 * sizeof(unsigned)));
  CK(cudaMemset(B.tickets, 0, 4096 * sizeof(unsigned)));
  for (int J : Js) {
    const double bytes = 8.0 * n * S * J;
    double us0;
    int grid0;
    auto ref = run_v7<S, 2, 4, 3>(B, n, J, &us0, &grid0);   // reference for the diffs
    printf("s=%d n=%d J=%d (%.0f MB)\n", S, n, J, bytes / 1e6);
    if constexpr (S == 16) {
      v7_line<S, 2, 4, 3, false>(B, n, J, ref, bytes);
      v7_line<S, 1, 4, 4, false>(B, n, J, ref, bytes);
      v7_line<S, 1, 8, 3, false>(B, n, J, ref, bytes);
      v7_line<S, 2, 2, 4, false>(B, n, J, ref, bytes);
      v7_line<S, 1, 2, 4, false>(B, n, J, ref, bytes);
      v7_line<S, 1, 4, 4, true>(B, n, J, ref, bytes);
      v7_line<S, 4, 2, 3, false>(B, n, J, ref, bytes);
      v7_line<S, 2, 6, 2, false>(B, n, J, ref, bytes);
    } else {
      v7_line<S, 3, 4, 3>(B, n, J, ref, bytes);
      v7_line<S, 2, 4, 3>(B, n, J, ref, bytes);
      v7_line<S, 3, 6, 2>(B, n, J, ref, bytes);
    }
    read_line<S>(B, n, J, bytes);
  }
  cudaFree(B.V); cudaFree(B.part); cudaFree(B.gpart); cudaFree(B.G); cudaFree(B.zeros); cudaFree(B.tickets);
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0 || which == 2) sweep<4>(1 << 20, {2, 6, 11, 16, 21});
  if (which == 0 || which == 3) sweep<8>(1 << 21, {2, 11, 21, 31});
  if (which == 0 || which == 5) sweep<8>(1 << 24, {2, 21, 41});
  if (which == 0 || which == 4) sweep<16>(1 << 22, {2, 7, 13, 19, 26});
  return 0;
}
