// dmma.cuh — FP64 tensor-core (DMMA, mma.sync.aligned.m8n8k4.f64; tcgen05 has no fp64 kind)
// building blocks of the two HBM passes of a block step: the dmma() wrapper, the Gram launch
// arguments shared by the Gram kernels (gram7.cuh), and the projection
//   k_project_dmma<S>: out0 = base0 + sum_j X_j C0_j, out1 = sum_j X_j C1_j (Alg 3 line 6:
//                      V_{k+1} = [V_k W][-H R^-1; R^-1]; Alg 6 lines 16-17; cycle end:
//                      X += V_k Xi C_acc, U = V_{k+1}[M; -H]), in place over an input block.
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

// basis slots are padded to a multiple of this many rows (zero rows): branch-free tiles
constexpr int kRowPad = 512;

constexpr int kGramGroup = 16;  // CTAs per first-level reduction group

struct GramArgs {
  int n;
  const int* rp; const int* ci; const double* va;   // CSR (local rows)
  const double* Vk;        // SpMM input block (fused mode) or nullptr (W = Y given)
  const double* Vghost;
  const double* X;         // blocks X_0..X_{NVB-1} at X + j*xstride (rows padded to kRowPad)
  size_t xstride;
  int J;                   // total blocks in the Gram (including W if y_alias)
  int y_alias;             // 1: block J-1 is Y itself (taken from the W tile in smem)
  double* Y;               // W (written in fused mode; read otherwise; rows padded)
  const double* zeros;     // >= 16 zero doubles (padding lanes of packed groups)
  double* part;            // [cta][E]
  double* gpart;           // [group][E]
  unsigned* tickets;       // [ngroups + 1], zero-initialised, reset by the last CTA
  double* G;               // result, E = J S S doubles, row-major [(j S + a) S + b]
  const int* active;       // nullable: skip when *active == 0
  const double* Y2 = nullptr;  // k_gram_v7<.., NY = 2>: second B-operand block, G = X^T [Y Y2]
  int pf_batches = 0;          // k_gram_v7: row batches of the basis blocks prefetched into L2
                               // before waiting on the SpMM (gram7.cuh)
};

// ------------------------------------------------------------------------------------------
// pass 2 on the tensor cores (S in {4, 8, 16}).  A warp owns 8-row blocks (grid-stride);
// per block j: A = X_j rows (8 x 4 chunks), B = C_j (4 x 8 chunks, shared memory), D in
// registers.  out0/out1 may alias an input block (each warp reads its rows before writing).
// ------------------------------------------------------------------------------------------
// K index of chunk kc, lane k4 (the column of X the lane's A value came from)
template <int S>
__device__ __forceinline__ int kmap(int kc, int k4) {
  return S == 16 ? 4 * k4 + kc : (S == 8 ? 2 * k4 + kc : kc * 4 + k4);
}
__device__ __forceinline__ double2 ldh2_rw(const double* p, uint64_t pol) {   // coherent, 16 bytes
  double2 v;
  asm("ld.global.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ double4 ldh4_rw(const double* p, uint64_t pol) {   // coherent, 32 bytes
  double4 v;
  asm("ld.global.L2::cache_hint.v4.f64 {%0,%1,%2,%3}, [%4], %5;"
      : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p), "l"(pol));
  return v;
}

template <int S>
__global__ void __launch_bounds__(256)
k_project_dmma(int n, const double* X, size_t xstride, int J0, const double* __restrict__ C0,
               const double* base0, double* out0, int J1, const double* __restrict__ C1, double* out1,
               const int* __restrict__ flag_ptr, int pf_ctas = 0) {
  static_assert(S == 4 || S == 8 || S == 16, "DMMA projection for s in {4,8,16}");
  constexpr int KC = S / 4;                 // K chunks
  constexpr int NT = S >= 8 ? S / 8 : 1;    // N tiles
  constexpr int RB = S >= 16 ? 2 : 4;       // 8-row blocks per warp iteration
  PDL_TRACE_ENTRY
  pdl_launch();
  {  // the CTA's first grid-stride iteration: its 8 warps' super-blocks are contiguous rows
    const long r0 = (long)blockIdx.x * (blockDim.x >> 5) * RB * 8;
    prefetch_blocks_l2(pf_ctas, X, xstride, max(J0, J1), r0 * S,
                       8L * S * (min((long)n, r0 + (long)(blockDim.x >> 5) * RB * 8) - r0));
  }
  pdl_wait();
  PDL_TRACE_WAITED(kTrProj, max(J0, J1));
  if (flag_ptr && *flag_ptr) return;
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
  const uint64_t xpol = l2pol(c_l2hint & 4, false);
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
        if constexpr (S == 16) {
          // one 32-byte load per lane covers a quarter row: K chunk kc takes column 4 k4 + kc
          // (the coefficient rows below use the same map), a quarter of the load instructions
          // of 8-byte loads (round 1: the L1 pipe was the limit at s = 16)
          const double4 v = (row < n) ? ldh4_rw(Xj + (size_t)row * S + 4 * k4, xpol) : make_double4(0, 0, 0, 0);
          a[rb][0] = v.x; a[rb][1] = v.y; a[rb][2] = v.z; a[rb][3] = v.w;
        } else if constexpr (S == 8) {
          // s = 8: one 16-byte load per lane, K chunk kc takes column 2 k4 + kc
          const double2 v = (row < n) ? ldh2_rw(Xj + (size_t)row * S + 2 * k4, xpol) : make_double2(0, 0);
          a[rb][0] = v.x; a[rb][1] = v.y;
        } else {
#pragma unroll
          for (int kc = 0; kc < KC; ++kc) a[rb][kc] = (row < n) ? ldh_rw(Xj + (size_t)row * S + kc * 4 + k4, xpol) : 0.0;
        }
      }
      if (j < J0) {
        const double* cj = c0 + (size_t)j * S * S;
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int tn = 0; tn < NT; ++tn) {
            const int col = tn * 8 + r8;
            const double b = (col < S) ? cj[kmap<S>(kc, k4) * S + col] : 0.0;
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
            const double b = (col < S) ? cj[kmap<S>(kc, k4) * S + col] : 0.0;
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
  TRACE_EXIT(1);
}

}  // namespace lsba
