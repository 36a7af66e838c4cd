// gram_bench.cu — standalone timing of the Gram-pass kernel candidates on the bench shapes
// (dev tool; the product path is liblsba.so).  For (n, s, J): basis of J padded slots with the
// last slot aliased as W, G = [X_0..X_{J-1}]^T W.  Reports us/launch and algorithmic GB/s
// (8 n s J bytes), and the max relative difference of G against k_gram_v6.
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

template <int S>
static std::vector<double> run_v6(const Bufs& B, int n, int J, double* us) {
  using G6 = G6Cfg<S>;
  GramArgs a = args(B, n, J);
  const size_t smem = sizeof(double) * J * S * S;
  auto fn = k_gram_v6<S>;
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(smem, 48 * 1024)));
  int occ = 1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, G6::NTHR, smem));
  const int grid = std::max(1, std::min(std::min(occ, 4) * 148, (n / 4 + 63) / 64));
  *us = time_it([&] { fn<<<grid, G6::NTHR, smem>>>(a); }, 10);
  CK(cudaGetLastError());
  std::vector<double> G(J * S * S);
  CK(cudaMemcpy(G.data(), B.G, sizeof(double) * G.size(), cudaMemcpyDeviceToHost));
  return G;
}

template <int S, int GMAX, int U, int MINB, bool PIPE>
static std::vector<double> run_v7(const Bufs& B, int n, int J, double* us, int* grid_out) {
  GramArgs a = args(B, n, J);
  auto fn = k_gram_v7<S, GMAX, U, MINB, PIPE>;
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

static double reldiff(const std::vector<double>& a, const std::vector<double>& b) {
  double num = 0, den = 0;
  for (size_t i = 0; i < a.size(); ++i) { num = std::max(num, std::fabs(a[i] - b[i])); den = std::max(den, std::fabs(b[i])); }
  return num / den;
}

template <int S, int GMAX, int U, int MINB, bool PIPE = false>
static void v7_line(const Bufs& B, int n, int J, const std::vector<double>& ref, double bytes) {
  double us; int grid;
  auto G = run_v7<S, GMAX, U, MINB, PIPE>(B, n, J, &us, &grid);
  int regs = 0;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k_gram_v7<S, GMAX, U, MINB, PIPE>); regs = fa.numRegs;
  printf("   v7<G%d,U%d,B%d,P%d> regs %3d grid %4d: %8.1f us %7.0f GB/s  diff %.1e\n", GMAX, U, MINB, (int)PIPE, regs, grid, us,
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
    double us6;
    auto ref = run_v6<S>(B, n, J, &us6);
    printf("s=%d n=%d J=%d (%.0f MB)\n   v6               : %8.1f us %7.0f GB/s\n", S, n, J, bytes / 1e6, us6, bytes / us6 / 1e3);
    v7_line<S, 3, 4, 3>(B, n, J, ref, bytes);
    v7_line<S, 2, 8, 3>(B, n, J, ref, bytes);
    v7_line<S, 1, 16, 3>(B, n, J, ref, bytes);
    v7_line<S, 4, 4, 3>(B, n, J, ref, bytes);
    v7_line<S, 2, 4, 3>(B, n, J, ref, bytes);
    v7_line<S, 3, 6, 2>(B, n, J, ref, bytes);
    v7_line<S, 3, 2, 4>(B, n, J, ref, bytes);
    v7_line<S, 1, 8, 4>(B, n, J, ref, bytes);
    v7_line<S, 2, 6, 3>(B, n, J, ref, bytes);
    v7_line<S, 4, 2, 4>(B, n, J, ref, bytes);
  }
  cudaFree(B.V); cudaFree(B.part); cudaFree(B.gpart); cudaFree(B.G); cudaFree(B.zeros); cudaFree(B.tickets);
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  if (which == 0 || which == 2) sweep<4>(1 << 20, {3, 6, 9, 13, 17, 21});
  if (which == 0 || which == 3) sweep<8>(1 << 21, {2, 11, 21, 31});
  if (which == 0 || which == 5) sweep<8>(1 << 24, {2, 21, 41});
  if (which == 0 || which == 4) sweep<16>(1 << 22, {3, 7, 13, 19, 26});
  return 0;
}
