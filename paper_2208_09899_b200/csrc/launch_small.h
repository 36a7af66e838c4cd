// launch_small.h — host launchers of the per-B small-state kernels (small.cuh).  Each B is
// compiled in its own translation unit (small_inst.cu with -DLSBA_B=B) so the 16 fully
// unrolled instantiations build in parallel.
#pragma once
#include <cuda_runtime.h>

namespace lsba {
struct SmallState2;
struct CycleParams;

template <int B>
cudaError_t launch_step_small(const SmallState2& st, const double* G, int k, const CycleParams& prm,
                              double rfac, cudaStream_t stream);
template <int B>
cudaError_t launch_step_update(const SmallState2& st, const double* G, int k, double rfac,
                               cudaStream_t stream);
template <int B>
cudaError_t launch_cycle_end(const SmallState2& st, int k, int gmres, int happy, int upd, double* Y,
                             double* Z, int* info, const int* prior, int force_sing, cudaStream_t stream);

template <int B>
cudaError_t launch_cwy_iter1(const SmallState2& st, const double* G, cudaStream_t stream);
template <int B>
cudaError_t launch_cwy_coef(const SmallState2& st, const double* G, int k, int inverse, cudaStream_t stream);
template <int B>
cudaError_t launch_irols_coef(const SmallState2& st, const double* G, int k, cudaStream_t stream);
template <int B>
cudaError_t launch_bmgs_h(const SmallState2& st, const double* G, int j, int k, cudaStream_t stream);
template <int B>
cudaError_t launch_bmgs_r(const SmallState2& st, const double* G, int k, cudaStream_t stream);
template <int B>
cudaError_t launch_pio_coef(const SmallState2& st, const double* G1, const double* G2, int k, cudaStream_t stream);

#define LSBA_DECL_SMALL(B)                                                                              \
  template <>                                                                                           \
  cudaError_t launch_step_small<B>(const SmallState2&, const double*, int, const CycleParams&, double,  \
                                   cudaStream_t);                                                        \
  template <>                                                                                           \
  cudaError_t launch_step_update<B>(const SmallState2&, const double*, int, double, cudaStream_t);     \
  template <>                                                                                           \
  cudaError_t launch_cycle_end<B>(const SmallState2&, int, int, int, int, double*, double*, int*,     \
                                  const int*, int, cudaStream_t);                                       \
  template <>                                                                                           \
  cudaError_t launch_cwy_iter1<B>(const SmallState2&, const double*, cudaStream_t);                    \
  template <>                                                                                           \
  cudaError_t launch_cwy_coef<B>(const SmallState2&, const double*, int, int, cudaStream_t);           \
  template <>                                                                                           \
  cudaError_t launch_irols_coef<B>(const SmallState2&, const double*, int, cudaStream_t);              \
  template <>                                                                                           \
  cudaError_t launch_bmgs_h<B>(const SmallState2&, const double*, int, int, cudaStream_t);             \
  template <>                                                                                           \
  cudaError_t launch_bmgs_r<B>(const SmallState2&, const double*, int, cudaStream_t);                  \
  template <>                                                                                           \
  cudaError_t launch_pio_coef<B>(const SmallState2&, const double*, const double*, int, cudaStream_t);
LSBA_DECL_SMALL(1) LSBA_DECL_SMALL(2) LSBA_DECL_SMALL(3) LSBA_DECL_SMALL(4)
LSBA_DECL_SMALL(5) LSBA_DECL_SMALL(6) LSBA_DECL_SMALL(7) LSBA_DECL_SMALL(8)
LSBA_DECL_SMALL(9) LSBA_DECL_SMALL(10) LSBA_DECL_SMALL(11) LSBA_DECL_SMALL(12)
LSBA_DECL_SMALL(13) LSBA_DECL_SMALL(14) LSBA_DECL_SMALL(15) LSBA_DECL_SMALL(16)
#undef LSBA_DECL_SMALL
}  // namespace lsba
