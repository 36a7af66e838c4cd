// small_inst.cu — compiled once per block size with -DLSBA_B=<1..16> (see build.sh).
#include "small.cuh"
#include "launch_small.h"

#ifndef LSBA_B
#error "compile with -DLSBA_B=<block size>"
#endif

namespace lsba {

template <>
cudaError_t launch_step_small<LSBA_B>(const SmallState2& st, const double* G, int k,
                                      const CycleParams& prm, double rfac, cudaStream_t stream) {
  constexpr int B = LSBA_B;
  const size_t smem = sizeof(double) * (size_t)(k + 1) * B * B;
  auto fn = k_step_coef<B>;
  if (smem > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  fn<<<1, 128, smem, stream>>>(st, G, k, prm, rfac);
  return cudaGetLastError();
}

template <>
cudaError_t launch_step_update<LSBA_B>(const SmallState2& st, const double* G, int k, double rfac,
                                       cudaStream_t stream) {
  constexpr int B = LSBA_B;
  const size_t km1 = k > 1 ? (size_t)(k - 1) : 0;
  const size_t smem = sizeof(double) * ((size_t)(k + 1) * B * B + km1 * B * 2 * B + km1 * B);
  auto fn = k_step_update<B>;
  if (smem > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  fn<<<1, 32 * (B + 2), smem, stream>>>(st, G, k, rfac);
  return cudaGetLastError();
}

template <>
cudaError_t launch_cycle_end<LSBA_B>(const SmallState2& st, int k, int gmres, int happy, int upd,
                                     double* Y, double* Z, int* info, const int* prior, int force_sing,
                                     cudaStream_t stream) {
  constexpr int B = LSBA_B;
  const size_t kb = (size_t)k * B;
  size_t smem = sizeof(double) * kb * B;
  const int stage_r = (smem + sizeof(double) * kb * kb <= 200 * 1024) ? 1 : 0;
  if (stage_r) smem += sizeof(double) * kb * kb;
  auto fn = k_cycle_end<B>;
  if (smem > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  fn<<<1, 32 * (B > 8 ? B : 8), smem, stream>>>(st, k, gmres, happy, upd, Y, Z, info, stage_r, prior,
                                                 force_sing);
  return cudaGetLastError();
}

template <>
cudaError_t launch_cwy_iter1<LSBA_B>(const SmallState2& st, const double* G, cudaStream_t stream) {
  k_cwy_iter1<LSBA_B><<<1, 128, 0, stream>>>(st, G);
  return cudaGetLastError();
}

template <>
cudaError_t launch_cwy_coef<LSBA_B>(const SmallState2& st, const double* G, int k, int inverse,
                                    cudaStream_t stream) {
  constexpr int B = LSBA_B;
  const size_t k1b = (size_t)(k + 1) * B;
  const size_t smem = sizeof(double) * (k1b * 2 * B + 2 * k1b * B);
  auto fn = k_cwy_coef<B>;
  if (smem > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  fn<<<1, 256, smem, stream>>>(st, G, k, inverse);
  return cudaGetLastError();
}

template <>
cudaError_t launch_irols_coef<LSBA_B>(const SmallState2& st, const double* G, int k, cudaStream_t stream) {
  constexpr int B = LSBA_B;
  const size_t k1b = (size_t)(k + 1) * B;
  const size_t smem = sizeof(double) * (k1b * 3 * B);
  auto fn = k_irols_coef<B>;
  if (smem > 32 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  fn<<<1, 256, smem, stream>>>(st, G, k);
  return cudaGetLastError();
}

template <>
cudaError_t launch_bmgs_h<LSBA_B>(const SmallState2& st, const double* G, int j, int k, cudaStream_t stream) {
  k_bmgs_h<LSBA_B><<<1, 64, 0, stream>>>(st, G, j, k);
  return cudaGetLastError();
}

template <>
cudaError_t launch_bmgs_r<LSBA_B>(const SmallState2& st, const double* G, int k, cudaStream_t stream) {
  k_bmgs_r<LSBA_B><<<1, 64, 0, stream>>>(st, G, k);
  return cudaGetLastError();
}

template <>
cudaError_t launch_pio_coef<LSBA_B>(const SmallState2& st, const double* G1, const double* G2, int k,
                                    cudaStream_t stream) {
  k_pio_coef<LSBA_B><<<1, 128, 0, stream>>>(st, G1, G2, k);
  return cudaGetLastError();
}

}  // namespace lsba
