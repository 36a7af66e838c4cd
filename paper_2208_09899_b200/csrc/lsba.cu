// lsba.cu — C-ABI (include/lsba.h) and the host engine around the sm_100a kernels.
//
// The engine is the restarted modified BFOM/BGMRES driver of PAPER.md:186-219 with the BCGS-PIP
// skeleton (Alg 3) and the adaptive restart of Sec 4,
// following the same step list as the oracle; every
// arithmetic step runs in a kernel of kernels.cuh (or the single NCCL allreduce / halo
// send-recv).  The host only sequences launches and reads one 48-byte status word per step
// (the convergence / restart check, the north star's single host round trip).
#include "../../include/lsba.h"

#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "kernels.cuh"
#include "small.cuh"  // SmallState2 / StepStatus layouts (kernels are in small_inst.cu)
#include "dmma.cuh"
#include "gram7.cuh"
#include "ilu.cuh"
#include "launch_small.h"
#include "comm.h"

using namespace lsba;

namespace {

struct EvPair { cudaEvent_t a, b; };

struct Prof {
  bool on = false;
  std::vector<EvPair> ev[LSBA_K_COUNT];
  size_t used[LSBA_K_COUNT] = {};
  double bytes[LSBA_K_COUNT] = {};
  int64_t launches[LSBA_K_COUNT] = {};
  std::vector<std::pair<int, size_t>> order;   // launch order: (kernel id, index into ev[kid])
};

constexpr int kGramCtas = 4 * 148 * 2;  // target CTAs of the partial-Gram grid

}  // namespace

struct lsba_ctx_ {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n_global = 0, row_begin = 0, row_end = 0;
  int n = 0;  // local rows
  int s = 0, m_max = 0, rank = 0, nranks = 1;
  int64_t nnz = 0;
  // CSR (device)
  int* d_rp = nullptr;
  int* d_ci = nullptr;
  double* d_va = nullptr;
  // basis: (m_max+1) slots of n x s
  double* d_V = nullptr;
  size_t slot = 0;         // elements per block (n_local x s)
  size_t slot_stride = 0;  // elements between consecutive basis slots (rows padded to kRowPad)
  double* d_zeros = nullptr;
  // halo
  int n_ghost = 0;
  double* d_ghost = nullptr;
  std::vector<int64_t> send_cnt, recv_cnt, send_off, recv_off;
  int* d_send_idx = nullptr;
  double* d_sendbuf = nullptr;
  int64_t n_send = 0;
  Comm* comm = nullptr;            // collectives (NCCL, or the loopback test group); null on one rank
  NcclComm* nccl = nullptr;        // == comm when it is NCCL
  bool devar_req = false;          // LSBA_DEVAR=1: fold the Gram allreduce into the Gram tail (f2)
  uint64_t ar_seq = 0;             // device-allreduce calls so far (alternating window slots)
  size_t ar_slot = 0;              // window bytes per slot
  // Gram
  double* d_part = nullptr;
  size_t part_cap = 0;
  double* d_G = nullptr;          // current Gram result (one of the two halves of d_Gbase)
  double* d_Gbase = nullptr;      // 2 x (m_max+1) s^2: step k uses half k & 1, so the Gram of
                                  // step k+1 never overwrites what the update of step k reads
  size_t g_half = 0;
  double* d_gpart = nullptr;     // DMMA Gram: first-level group partials
  unsigned* d_tickets = nullptr;  // DMMA Gram: CTA arrival counters (self-resetting)
  int gram_grid = 0;              // DMMA Gram: persistent grid size
  CycleCtl* d_ctl = nullptr;      // device-side cycle control
  cudaStream_t stream2 = nullptr;  // update kernels run here, concurrent with the projection
  cudaEvent_t ev_coef = nullptr, ev_upd = nullptr;
  CycleCtl* h_ctl = nullptr;      // pinned copy
  volatile int* h_prog = nullptr; // mapped pinned 2 k_done + active (see publish_progress)
  int n_sms = 148;
  // small state
  SmallState2 st{};
  double* d_small = nullptr;
  double* d_Y = nullptr;
  double* d_Z = nullptr;
  int* d_info = nullptr;
  StepStatus* h_status = nullptr;  // pinned
  int* h_info = nullptr;           // pinned
  double* h_scalar = nullptr;      // pinned
  double* d_Xc = nullptr;
  double* d_sq = nullptr;
  int sq_cap = 0;
  double* d_scalar = nullptr;
  double* d_Bh = nullptr;  // e2e staging
  double* d_Xh = nullptr;
  // state machine for the step API
  int ip = LSBA_IP_CLASSICAL;
  int b = 0;
  int k = -1;
  bool flagged = false;
  int force_flag_k = 0;
  bool forced_done = false;
  int variant = 0;
  bool no_fuse = false;          // diagnostics: LSBA_NO_FUSE=1 keeps the small step a separate launch
  // ILU(0) left preconditioning (ilu.cuh; lsba_ilu0_setup)
  bool prec = false;             // operator is M^{-1} A (every spmm / residual)
  bool ilu_ready = false;
  double* d_lu = nullptr;        // factor values in the CSR pattern of A
  int* d_diag = nullptr;         // CSR position of a_ii
  int* d_ordL = nullptr;         // rows by level of L (ascending dependencies)
  int* d_ordU = nullptr;         // rows by level of U
  int* d_lvlL = nullptr;         // level pointers into d_ordL (nlL + 1) and d_ordU (nlU + 1)
  int* d_lvlU = nullptr;
  IluPack packL{}, packU{};      // level-ordered packed rows (ilu.cuh k_ilu_trsv_level)
  int ilu_solve = 1;             // 1 level-synchronous on packed rows, 0 sync-free polling (LSBA_ILU_SOLVE)
  double* d_ilu_tmp = nullptr;   // n x s intermediate of the data-polling variant
  unsigned* d_ticket = nullptr;  // CTA start tickets (2: L and U solves)
  int ilu_levels[2] = {0, 0};
  int ilu_backoff = 0;           // ns of the first back-off after a failed dependency poll (LSBA_ILU_BACKOFF)
  int ilu_ctas = 1;              // persistent CTAs per SM (LSBA_ILU_CTAS)
  cudaEvent_t ev_status = nullptr;
  cudaStream_t cstream = nullptr;  // P > 1: halo exchange stream (overlaps the interior SpMM)
  cudaEvent_t ev_pack = nullptr, ev_halo = nullptr;
  int int0 = 0, int1 = 0;          // contiguous interior rows (no ghost columns); int1 > int0: overlap
  // no interior block (random columns): local/ghost split of A for the overlap (P > 1)
  bool split = false;
  int* d_rpL = nullptr; int* d_ciL = nullptr; double* d_vaL = nullptr;   // local columns, all rows
  int ng_rows = 0;
  int* d_rowsG = nullptr; int* d_rpG = nullptr; int* d_ciG = nullptr; double* d_vaG = nullptr;
  bool halo_ovl = true;            // LSBA_HALO_OVERLAP
  bool upd_main = false;         // diagnostics: LSBA_UPD_MAIN=1
  int devjoin = 1;               // Gram joins the update on the device: 0 never (stream event),
                                 // 1 for basis blocks <= 64 MB, 2 always (LSBA_DEVJOIN)
  bool spec_end = true;          // speculative cycle end before the status read (LSBA_SPEC_END)
  int spmm_pf = -1;              // SpMM L2 prefetch distance in CTAs (-1: 4 x SMs; LSBA_SPMM_PF)
  int spmm_pfv = 1;              // ... and of the CTA's V rows (LSBA_SPMM_PFV)
  bool spmm_lanes16 = false;     // diagnostics: LSBA_SPMM_LANES16=1 forces 16-byte SpMM lanes
  bool proj_dfma = false;        // diagnostics: LSBA_PROJ_DFMA=1 uses the DFMA projection at s = 8, 16
  long proj_pf = 12L << 20;      // projection pre-wait L2 prefetch budget in bytes (LSBA_PROJ_PF_MB)
  long gram_pf = 8L << 20;       // Gram pre-wait L2 prefetch budget in bytes (LSBA_GRAM_PF_MB)
  bool force_comm = false;       // LSBA_FORCE_COMM=1: one rank through the distributed code path
  int force_sing_cycle = 0;      // test hook: the cycle end of this cycle reports singular
  int cur_cycle = 0;
  size_t csr_bytes = 0;          // joint col_idx + vals allocation (d_va points into it)
  int l2persist = -1;            // SpMM CSR window persisting in L2: -1 auto, 0 off, 1 on (LSBA_L2PERSIST)
  size_t l2win = 0;
  float l2hit = 0.f;
  bool in_spmm = false;
  bool pdl_proj = true;          // PDL for the projection too (LSBA_PDL_PROJ)
  bool in_proj = false;
  int g7force = 0;               // diagnostics: LSBA_G7 forces a v7 Gram configuration (s = 4, 8)
  bool pdl = true;               // programmatic dependent launch of SpMM / Gram / projection (LSBA_PDL)
  bool pending_upd = false;   // the main stream must join ev_upd before the next Gram
  int skel = LSBA_SKEL_BCGS_PIP;          // skeleton of the running solve / Arnoldi process
  int skel_default = LSBA_SKEL_BCGS_PIP;  // lsba_set_skeleton: step API and lsba_solve_host
  int64_t launches = 0;
  int64_t ws_bytes = 0;
  lsba_allocator alloc{};          // lsba_create_with_allocator: the caller owns the workspace
  bool has_alloc = false;
  std::vector<void*> owned;
  std::string err;
  Prof prof;
};

// ------------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------------
static lsba_status fail(lsba_ctx c, lsba_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  return st;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(c, e_ == cudaErrorMemoryAllocation ? LSBA_E_OOM : LSBA_E_CUDA,          \
                  "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(e_));      \
  } while (0)

#define CKL()                                                                             \
  do {                                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess)                                                                \
      return fail(c, LSBA_E_CUDA, "%s:%d launch: %s", __FILE__, __LINE__,               \
                  cudaGetErrorString(e_));                                                \
  } while (0)

#define CKN(call)                                                                         \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess)                                                                \
      return fail(c, LSBA_E_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                  ncclGetErrorString(r_));                                                \
  } while (0)

#define TRYC(call)                                                                        \
  do {                                                                                    \
    const int e_ = (call);                                                                \
    if (e_) return fail(c, e_ == 2 ? LSBA_E_NCCL : LSBA_E_CUDA, "%s", c->comm->err.c_str()); \
  } while (0)

#define TRY(x)                        \
  do {                                \
    lsba_status s_ = (x);             \
    if (s_ != LSBA_OK) return s_;     \
  } while (0)

// profiling scope around one launch
struct LaunchScope {
  lsba_ctx c;
  int kid;
  EvPair* ev = nullptr;
  cudaStream_t strm;
  LaunchScope(lsba_ctx c_, int kid_, double bytes, cudaStream_t s_ = nullptr)
      : c(c_), kid(kid_), strm(s_ ? s_ : c_->stream) {
    c->launches++;
    if (!c->prof.on) return;
    Prof& p = c->prof;
    p.launches[kid]++;
    p.bytes[kid] += bytes;
    if (p.used[kid] == p.ev[kid].size()) {
      EvPair e;
      cudaEventCreate(&e.a);
      cudaEventCreate(&e.b);
      p.ev[kid].push_back(e);
    }
    p.order.emplace_back(kid, p.used[kid]);
    ev = &p.ev[kid][p.used[kid]++];
    cudaEventRecord(ev->a, strm);
  }
  ~LaunchScope() {
    if (ev) cudaEventRecord(ev->b, strm);
  }
};

// ------------------------------------------------------------------------------------------
// template dispatch over s = 1..16
// ------------------------------------------------------------------------------------------
#define LSBA_DISPATCH_S(s, FN, ...)         \
  switch (s) {                              \
    case 1: return FN<1>(__VA_ARGS__);      \
    case 2: return FN<2>(__VA_ARGS__);      \
    case 3: return FN<3>(__VA_ARGS__);      \
    case 4: return FN<4>(__VA_ARGS__);      \
    case 5: return FN<5>(__VA_ARGS__);      \
    case 6: return FN<6>(__VA_ARGS__);      \
    case 7: return FN<7>(__VA_ARGS__);      \
    case 8: return FN<8>(__VA_ARGS__);      \
    case 9: return FN<9>(__VA_ARGS__);      \
    case 10: return FN<10>(__VA_ARGS__);    \
    case 11: return FN<11>(__VA_ARGS__);    \
    case 12: return FN<12>(__VA_ARGS__);    \
    case 13: return FN<13>(__VA_ARGS__);    \
    case 14: return FN<14>(__VA_ARGS__);    \
    case 15: return FN<15>(__VA_ARGS__);    \
    case 16: return FN<16>(__VA_ARGS__);    \
    default: return LSBA_E_ARG;             \
  }

static inline int cdiv(long a, long b) { return (int)((a + b - 1) / b); }
static inline double* slotp(lsba_ctx c, int j) { return c->d_V + (size_t)j * c->slot_stride; }
// skeletons with Alg 6's lagged loop (iteration 1 after IO, the two-block Gram per step)
static inline bool lagged(int skel) {
  return skel == LSBA_SKEL_BMGS_CWY || skel == LSBA_SKEL_BMGS_ICWY || skel == LSBA_SKEL_BCGS_IROLS;
}
static inline bool in_basis(lsba_ctx c, const double* p) {
  return p >= c->d_V && p < c->d_V + (size_t)(c->m_max + 2) * c->slot_stride;
}

// ---------------------------------------------------------------- halo exchange (P > 1)
// Pack the rows peers need (main stream), then the grouped send/recv: on the main stream, or
// on the comm stream when the SpMM overlaps it (ovl: the interior rows run meanwhile; the
// caller joins ev_halo before the boundary rows).
template <int S>
static lsba_status halo_t(lsba_ctx c, const double* V, bool ovl = false) {
  if (!c->comm) return LSBA_OK;
  if (c->n_send > 0) {
    LaunchScope L(c, LSBA_K_HALO_PACK, 16.0 * c->n_send * S + 4.0 * c->n_send);
    const long tot = c->n_send * S;
    k_halo_pack<S><<<cdiv(tot, kThreads), kThreads, 0, c->stream>>>((int)c->n_send, c->d_send_idx, V,
                                                                     c->d_sendbuf);
    CKL();
  }
  std::vector<P2POp> ops;
  for (int r = 0; r < c->nranks; ++r) {
    if (r == c->rank || (c->send_cnt[r] == 0 && c->recv_cnt[r] == 0)) continue;
    ops.push_back({r, c->d_sendbuf + c->send_off[r] * S, sizeof(double) * (size_t)c->send_cnt[r] * S,
                   c->d_ghost + c->recv_off[r] * S, sizeof(double) * (size_t)c->recv_cnt[r] * S});
  }
  if (!ovl) {
    TRYC(c->comm->exchange(ops, c->stream));
    return LSBA_OK;
  }
  CK(cudaEventRecord(c->ev_pack, c->stream));
  CK(cudaStreamWaitEvent(c->cstream, c->ev_pack, 0));
  TRYC(c->comm->exchange(ops, c->cstream));
  CK(cudaEventRecord(c->ev_halo, c->cstream));
  return LSBA_OK;
}

// Launch with programmatic stream serialisation (PDL) when enabled: the kernel may be scheduled
// while its predecessor drains; it waits for it in-kernel (pdl_begin, kernels.cuh).
template <typename... P, typename... A>
static cudaError_t launch_k(lsba_ctx c, void (*kern)(P...), dim3 grid, dim3 block, size_t smem, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (c->pdl && (c->pdl_proj || !c->in_proj)) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (c->in_spmm && c->l2win > 0) {   // CSR arrays persisting in the L2 set-aside
    attr[na].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[na].val.accessPolicyWindow.base_ptr = (void*)c->d_ci;
    attr[na].val.accessPolicyWindow.num_bytes = c->l2win;
    attr[na].val.accessPolicyWindow.hitRatio = c->l2hit;
    attr[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<A>(args)...);
}

// ---------------------------------------------------------------- f4: ILU(0) apply
// Y <- U^{-1} L^{-1} Y in place (two sync-free triangular solves; ilu.cuh)
template <int S>
static lsba_status ilu_apply_t(lsba_ctx c, double* Y, const int* active) {
  if (!c->ilu_ready) return fail(c, LSBA_E_STATE, "ILU(0) preconditioner not set up");
  if (c->n == 0) return LSBA_OK;
  const int nblk = cdiv(c->n, kThreads);
  // algorithmic bytes per solve: the factor half (~12 B per stored entry + row pointers and
  // the row order) and Y read + written once
  const double by = 6.0 * c->nnz + 8.0 * (c->n + 1) + 16.0 * c->n * S;
  // level-synchronous on packed rows (default; LSBA_ILU_SOLVE=0: sync-free data polling)
  if (c->ilu_solve != 0) {
    auto fl = k_ilu_trsv_level<S, true>;
    auto fu = k_ilu_trsv_level<S, false>;
    int occ = 1, occ2 = 1;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fl, kThreadsIluLvl, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ2, fu, kThreadsIluLvl, 0));
    // every CTA resident (grid barriers): occupancy x SMs, less two slots for the 1-CTA kernels
    // of stream 2 that may hold part of an SM meanwhile
    const int lgrid = std::max(1, std::min(std::min(occ, occ2) * c->n_sms - 2, cdiv(c->n, kThreadsIluLvl)));
    unsigned* bar = c->d_ticket + 4;
    int* go = reinterpret_cast<int*>(c->d_ticket + 6);
    // cooperative launches: the runtime refuses a grid that cannot be co-resident (the grid
    // barriers would otherwise wait forever)
    auto coop = [&](auto fn, int nlev_h, const int* lvl, const IluPack& pk, const double* Xin, double* Zout) -> cudaError_t {
      int n_ = c->n, nl_ = nlev_h, nloc = c->n;
      const int* rp_ = c->d_rp;
      const int* ci_ = c->d_ci;
      const double* lu_ = c->d_lu;
      IluPack pk_ = pk;
      void* args[] = {&n_, &nl_, (void*)&lvl, &pk_, (void*)&rp_, (void*)&ci_, (void*)&lu_, &nloc, (void*)&Xin, (void*)&Zout,
                      (void*)&bar, (void*)&go, (void*)&active};
      return cudaLaunchCooperativeKernel((const void*)fn, dim3(lgrid), dim3(kThreadsIluLvl), args, 0, c->stream);
    };
    {
      LaunchScope Ls(c, LSBA_K_ILU_SOLVE, by);
      CK(coop(fl, c->ilu_levels[0], c->d_lvlL, c->packL, Y, c->d_ilu_tmp));
    }
    {
      LaunchScope Ls(c, LSBA_K_ILU_SOLVE, by);
      CK(coop(fu, c->ilu_levels[1], c->d_lvlU, c->packU, c->d_ilu_tmp, Y));
    }
    return LSBA_OK;
  }
  // data polling, out of place: Y -> T (L), T -> Y (U)
  const int grid = std::min(nblk, c->n_sms * c->ilu_ctas);
  const long cnt = (long)c->n * S;
  const int fgrid = std::min(4 * c->n_sms, (int)cdiv(cnt, kThreads));
  {
    LaunchScope Ls(c, LSBA_K_ILU_SOLVE, by);
    k_fill_sentinel<<<fgrid, kThreads, 0, c->stream>>>(cnt, c->d_ilu_tmp);
    k_ilu_trsv_poll<S, true><<<grid, kThreads, 0, c->stream>>>(c->n, c->d_ordL, c->d_rp, c->d_ci,
        c->d_lu, c->d_diag, c->n, Y, c->d_ilu_tmp, c->d_ticket, active, c->ilu_backoff);
    CKL();
  }
  {
    LaunchScope Ls(c, LSBA_K_ILU_SOLVE, by);
    k_fill_sentinel<<<fgrid, kThreads, 0, c->stream>>>(cnt, Y);
    k_ilu_trsv_poll<S, false><<<grid, kThreads, 0, c->stream>>>(c->n, c->d_ordU, c->d_rp, c->d_ci,
        c->d_lu, c->d_diag, c->n, c->d_ilu_tmp, Y, c->d_ticket + 2, active, c->ilu_backoff);
    CKL();
  }
  return LSBA_OK;
}
static lsba_status ilu_apply(lsba_ctx c, double* Y, const int* active = nullptr);

// ---------------------------------------------------------------- a1: SpMM / residual
template <int S>
static lsba_status spmm_t(lsba_ctx c, const double* V, double* W, const int* active) {
  const int n = c->n;
  // P > 1 with a contiguous interior block [int0, int1) (rows without ghost columns, e.g. all
  // but the boundary planes of a z-slab): the halo moves on the comm stream while the interior
  // rows compute; the boundary rows follow once it has arrived
  const bool ovl = c->comm && c->halo_ovl && c->int1 > c->int0;
  const bool split = c->split;
  TRY(halo_t<S>(c, V, ovl || split));
  // 32-byte lanes need 32-byte aligned rows (basis slots always are; caller buffers of
  // lsba_spmm / the residual may only be 16-byte aligned: then 16-byte lanes)
  constexpr int CW = SpmmLanes<S>::C;
  const bool a32 = CW != 4 || (!c->spmm_lanes16 && !((((uintptr_t)V) | ((uintptr_t)W) | ((uintptr_t)c->d_ghost)) & 31));
  {
    LaunchScope Ls(c, LSBA_K_SPMM, 12.0 * c->nnz + 4.0 * (n + 1) + 16.0 * n * S);
    if (n == 0) {
      if (ovl || split) CK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
      return LSBA_OK;
    }
    auto rows = [&](int r0, int r1, const int* rp, const int* ci, const double* va) -> lsba_status {
      if (r1 <= r0) return LSBA_OK;
      if constexpr (S % 2 == 0 || S == 1) {
        constexpr int CW2 = (CW == 4) ? 2 : CW;
        auto kern = a32 ? k_spmm<S, false, CW> : k_spmm<S, false, CW2>;
        const int L = S / (a32 ? CW : CW2);
        c->in_spmm = true;
        const cudaError_t le = launch_k(c, kern, dim3(cdiv((long)(r1 - r0) * L, kThreads)),
                    dim3(kThreads), 0, n, rp, ci, va, V,
                    (const double*)c->d_ghost, (const double*)nullptr, W, (double*)nullptr, active,
                    c->spmm_pf, c->spmm_pfv, r0, r1);
        c->in_spmm = false;
        CK(le);
      } else {
        k_spmm_odd<S, false><<<cdiv(r1 - r0, kThreads), kThreads, 0, c->stream>>>(
            n, rp, ci, va, V, c->d_ghost, nullptr, W, nullptr, active, r0, r1);
      }
      CKL();
      return LSBA_OK;
    };
    const int* rp = c->d_rp;
    const int* ci = c->d_ci;
    const double* va = c->d_va;
    if (!ovl && !split) {
      TRY(rows(0, n, rp, ci, va));
    } else if (ovl) {
      TRY(rows(c->int0, c->int1, rp, ci, va));
      CK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
      TRY(rows(0, c->int0, rp, ci, va));
      TRY(rows(c->int1, n, rp, ci, va));
    } else {                        // local columns of every row, then the ghost part
      TRY(rows(0, n, c->d_rpL, c->d_ciL, c->d_vaL));
      CK(cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
      if (c->ng_rows > 0) {
        constexpr int LG = (S % 2 == 0) ? S / 2 : S;
        CK(launch_k(c, k_spmm_ghost_acc<S>, dim3(cdiv((long)c->ng_rows * LG, kThreads)), dim3(kThreads), 0,
                    c->ng_rows, (const int*)c->d_rowsG, (const int*)c->d_rpG, (const int*)c->d_ciG,
                    (const double*)c->d_vaG, (const double*)c->d_ghost, W, active));
      }
    }
  }
  if (c->prec) TRY(ilu_apply_t<S>(c, W, active));
  return LSBA_OK;
}

// R = B - A X -> out; ||R||_F^2 (all ranks) -> d_scalar[0]
template <int S>
static lsba_status residual_t(lsba_ctx c, const double* Bm, const double* X, double* out) {
  TRY(halo_t<S>(c, X));
  constexpr int CW = SpmmLanes<S>::C, CW2 = (CW == 4) ? 2 : CW;
  const bool a32 = CW != 4 || !((((uintptr_t)X) | ((uintptr_t)out) | ((uintptr_t)c->d_ghost)) & 31);
  const int L = S / (a32 ? CW : CW2);
  int nblk = (S % 2 == 0 || S == 1) ? cdiv((long)c->n * L, kThreads) : cdiv(c->n, kThreads);
  if (nblk < 1) nblk = 1;
  if (nblk > c->sq_cap) return fail(c, LSBA_E_STATE, "residual partial buffer too small");
  {
    LaunchScope Ls(c, LSBA_K_RESIDUAL, 12.0 * c->nnz + 4.0 * (c->n + 1) + 24.0 * c->n * S);
    if (c->n == 0) {
      CK(cudaMemsetAsync(c->d_sq, 0, sizeof(double), c->stream));
    } else if constexpr (S % 2 == 0 || S == 1) {
      auto kern = a32 ? k_spmm<S, true, CW> : k_spmm<S, true, CW2>;
      kern<<<nblk, kThreads, 0, c->stream>>>(c->n, c->d_rp, c->d_ci, c->d_va, X, c->d_ghost, Bm, out,
                                               c->d_sq, nullptr, c->spmm_pf, c->spmm_pfv, 0, -1);
    } else {
      k_spmm_odd<S, true><<<nblk, kThreads, 0, c->stream>>>(c->n, c->d_rp, c->d_ci, c->d_va, X,
                                                              c->d_ghost, Bm, out, c->d_sq, nullptr);
    }
    CKL();
  }
  if (c->prec && c->n > 0) {   // preconditioned residual M^{-1}(B - A X) and its norm (R28)
    TRY(ilu_apply_t<S>(c, out, nullptr));
    LaunchScope Ls(c, LSBA_K_MISC, 8.0 * c->n * S);
    k_sq_partials<<<nblk, kThreads, 0, c->stream>>>((long)c->n * S, out, c->d_sq);
    CKL();
  }
  {
    LaunchScope Ls(c, LSBA_K_MISC, 8.0 * nblk);
    k_sum_partials<<<1, kThreads, 0, c->stream>>>(c->n == 0 ? 1 : nblk, c->d_sq, c->d_scalar);
    CKL();
  }
  if (c->comm) TRYC(c->comm->allreduce_sum_f64(c->d_scalar, 1, c->stream));
  return LSBA_OK;
}

// The previous step's update kernel (stream 2) overlaps this step's SpMM; everything after the
// SpMM reads its decision or the small state it writes, so the main stream joins it here.
static lsba_status wait_update(lsba_ctx c) {
  if (c->pending_upd) {
    CK(cudaStreamWaitEvent(c->stream, c->ev_upd, 0));
    c->pending_upd = false;
  }
  return LSBA_OK;
}

// ---------------------------------------------------------------- a2: v7 streaming Gram
// Tuned (GMAX groups per warp, U steps per batch, MINB CTAs per SM) per s and J from the
// standalone sweep in tools/gram_bench.cu (profiles/r01_gram_sweep*_raw.txt).
template <int S, int GMAX, int U, int MINB, bool WIN = true, int NY = 1>
static lsba_status gram_v7_launch(lsba_ctx c, const GramArgs& a, const GramFuse& f) {
  auto fn = k_gram_v7<S, GMAX, U, MINB, WIN, NY>;
  G7Launch<S, GMAX, NY> geo(c->n, a.J, MINB, c->n_sms, f.on != 0);
  if ((size_t)geo.grid * a.J * S * S * NY > c->part_cap || geo.passes > kMaxGramPasses)
    return fail(c, LSBA_E_STATE, "v7 Gram workspace too small (J=%d)", a.J);
  if (geo.smem > 32 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)geo.smem));
  GramArgs ap = a;
  {  // pre-wait L2 prefetch: whole batches of every basis block within the budget c->gram_pf
    const long per_batch = 8L * U * 4 * S * 8 * a.J * geo.grid;   // (upper bound: 8 row slices)
    ap.pf_batches = (c->pdl && c->gram_pf > 0) ? (int)std::min<long>(4, c->gram_pf / per_batch) : 0;
  }
  CK(launch_k(c, fn, dim3(geo.grid), dim3(256), geo.smem, ap, f));
  return LSBA_OK;
}

template <int S>
static lsba_status gram_v7(lsba_ctx c, const GramArgs& a, const GramFuse& f) {
  if constexpr (S == 4 || S == 8) {         // diagnostics: LSBA_G7=1..8 forces one configuration
    switch (c->g7force) {
      case 1: return gram_v7_launch<S, 1, 8, 4>(c, a, f);
      case 2: return gram_v7_launch<S, 2, 4, 3>(c, a, f);
      case 3: return gram_v7_launch<S, 3, 6, 2>(c, a, f);
      case 4: return gram_v7_launch<S, 2, 4, 2>(c, a, f);
      case 5: return gram_v7_launch<S, 1, 4, 3>(c, a, f);
      case 6: return gram_v7_launch<S, 1, 8, 2>(c, a, f);
      case 7: return gram_v7_launch<S, 3, 4, 2>(c, a, f);
      case 8: return gram_v7_launch<S, 3, 6, 1>(c, a, f);
      default: break;
    }
  } else if constexpr (S == 16) {
    switch (c->g7force) {
      case 1: return gram_v7_launch<S, 1, 4, 4, false>(c, a, f);
      case 2: return gram_v7_launch<S, 2, 4, 3, false>(c, a, f);
      case 3: return gram_v7_launch<S, 3, 6, 2, false>(c, a, f);
      case 4: return gram_v7_launch<S, 2, 4, 2, false>(c, a, f);
      default: break;
    }
  }
  // (GMAX, U, MINB) per J from in-situ per-launch timings of every configuration on configs
  // 2, 3 and 5 (tools/g7sweep.py over LSBA_G7-forced timelines; profiles/r01_g7_insitu.md):
  // the best choice alternates with the number of groups per pass
  // (the best choice follows the number of groups per pass: NG = ceil(J / (16 / s)))
  if constexpr (S == 2 || S == 4) {
    const int J = a.J;
    if (J <= 4) return gram_v7_launch<S, 1, 8, 4>(c, a, f);
    if (J <= 8 || (J >= 13 && J <= 16)) return gram_v7_launch<S, 2, 4, 3>(c, a, f);
    return gram_v7_launch<S, 3, 6, 2>(c, a, f);
  } else if constexpr (S == 8) {
    const int J = a.J;
    if (J <= 2) return gram_v7_launch<S, 1, 8, 4>(c, a, f);
    if ((J >= 3 && J <= 4) || (J >= 7 && J <= 8) || (J >= 13 && J <= 16) || (J >= 25 && J <= 32))
      return gram_v7_launch<S, 2, 4, 3>(c, a, f);
    return gram_v7_launch<S, 3, 6, 2>(c, a, f);
  } else if constexpr (S == 16) {            // (config 4, cold full solves, per J)
    const int J = a.J;
    if (J == 1) return gram_v7_launch<S, 1, 4, 4, false>(c, a, f);
    if (J == 2 || J == 4) return gram_v7_launch<S, 2, 4, 3, false>(c, a, f);
    if ((J >= 7 && J <= 8) || (J >= 13 && J <= 16)) return gram_v7_launch<S, 2, 4, 2, false>(c, a, f);
    return gram_v7_launch<S, 3, 6, 2, false>(c, a, f);
  } else {
    return fail(c, LSBA_E_STATE, "v7 Gram: s=%d unsupported", S);
  }
}

// BMGS-(I)CWY Gram: G = X^T [Y Y2] ((J s) x 2s) in one pass (v7 with two B-operand blocks)
template <int S>
static lsba_status gram2_v7(lsba_ctx c, const GramArgs& a) {
  const GramFuse f{};
  if constexpr (S == 4 || S == 8) {         // diagnostics: LSBA_G7=1..4 forces one configuration
    switch (c->g7force) {
      case 1: return gram_v7_launch<S, 1, 8, 4, true, 2>(c, a, f);
      case 2: return gram_v7_launch<S, 2, 4, 3, true, 2>(c, a, f);
      case 3: return gram_v7_launch<S, 3, 6, 2, true, 2>(c, a, f);
      case 4: return gram_v7_launch<S, 2, 4, 2, true, 2>(c, a, f);
      case 5: return gram_v7_launch<S, 1, 4, 3, true, 2>(c, a, f);
      case 6: return gram_v7_launch<S, 1, 8, 2, true, 2>(c, a, f);
      case 7: return gram_v7_launch<S, 2, 2, 2, true, 2>(c, a, f);
      case 8: return gram_v7_launch<S, 2, 4, 1, true, 2>(c, a, f);
      default: break;
    }
  }
  // per J from the in-situ sweep (profiles/r01_g7_insitu.md, BMGS-CWY rows)
  if constexpr (S == 2 || S == 4) {
    const int J = a.J;
    if (J <= 3) return gram_v7_launch<S, 1, 8, 4, true, 2>(c, a, f);
    if (J <= 8 || (J >= 12 && J <= 16)) return gram_v7_launch<S, 2, 4, 3, true, 2>(c, a, f);
    return gram_v7_launch<S, 3, 6, 2, true, 2>(c, a, f);
  } else if constexpr (S == 8) {
    const int J = a.J;
    if ((J >= 18 && J <= 20) || J >= 33) return gram_v7_launch<S, 1, 8, 2, true, 2>(c, a, f);
    return gram_v7_launch<S, 2, 4, 2, true, 2>(c, a, f);
  } else if constexpr (S == 16) {
    return gram_v7_launch<S, 1, 4, 2, false, 2>(c, a, f);
  } else {
    return fail(c, LSBA_E_STATE, "v7 Gram (2 blocks): s=%d unsupported", S);
  }
}

__global__ void k_interleave2(int R, int b, const double* __restrict__ G1, const double* __restrict__ G2,
                              double* __restrict__ G) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;   // G[r][0..2b) = [G1[r] G2[r]]
  if (e >= R * 2 * b) return;
  const int r = e / (2 * b), c = e % (2 * b);
  G[e] = (c < b) ? G1[(size_t)r * b + c] : G2[(size_t)r * b + c - b];
}

// ---------------------------------------------------------------- a1+a2: (SpMM +) Gram (+ allreduce)
// G (device, c->d_G) = <[X_0..X_{J-1}], Y>; classical (J s) x s row-major; global J scalars
// (scaled by 1/s).  If Vk != nullptr, Y = W is first computed as A Vk.  Exactly one allreduce
// when P > 1 (the step's single sync).  coef_k >= 0: the small step of step coef_k may be fused
// into the Gram's tail (one rank); *coef_fused says whether it was.
template <int S>
static lsba_status gram_t(lsba_ctx c, const double* X, size_t xstride, int J, double* Y, int ip,
                          const double* Vk, const int* active, int coef_k, const CycleParams* prm,
                          bool* coef_fused) {
  const bool gl = (ip == LSBA_IP_GLOBAL);
  const size_t E = gl ? (size_t)J : (size_t)J * S * S;
  if (coef_fused) *coef_fused = false;
  if (Vk) TRY(spmm_t<S>(c, Vk, Y, active));
  const bool y_is_block = (X + (size_t)(J - 1) * xstride == Y);
  const bool slots = c->variant == 0 && in_basis(c, X) && in_basis(c, Y) && c->d_tickets;
  constexpr bool v7_s = (S == 2 || S == 4 || S == 8 || S == 16);
  // one rank, a v7 Gram with the small step fused into its tail: the tail joins the previous
  // step's update kernel on the device (GramFuse::upd_wait) instead of the main stream
  // waiting on its event, which would keep this Gram from launching behind the SpMM (PDL)
  // Cost model: it saves ~2-4 us per step (the event join keeps the Gram from launching behind
  // the SpMM), but a Gram enqueued speculatively past a mid-cycle ending (convergence, kappa,
  // flag) may now stream before it sees the ending — a whole wasted Gram.  So by default only
  // for basis blocks <= 64 MB, where a step is short and a Gram cheap (config 2: +1.4%; config
  // 4's 537 MB blocks: -2%; configs 3 and 5 neutral; profiles/r02_devjoin_ab_raw.txt).
  const bool devjoin = (c->devjoin == 2 || (c->devjoin == 1 && 8.0 * c->n * S <= 64.0 * (1 << 20))) &&
                       c->pending_upd && !c->comm && !gl && v7_s && slots && c->n > 0 &&
                       coef_k > 0 && coef_fused && !c->no_fuse && E * sizeof(double) <= 64 * 1024 &&
                       !c->upd_main;
  if (devjoin) c->pending_upd = false;
  TRY(wait_update(c));
  bool ar_in_kernel = false;       // f2: the kernel's tail did the allreduce
  if (slots && ((!gl && v7_s) || (gl && S % 2 == 0))) {
    LaunchScope Ls(c, LSBA_K_GRAM, 8.0 * c->n * S * (J - (y_is_block ? 1 : 0)) + 8.0 * c->n * S);
    if (c->n > 0) {
      GramArgs a;
      a.n = c->n; a.rp = c->d_rp; a.ci = c->d_ci; a.va = c->d_va;
      a.Vk = nullptr; a.Vghost = c->d_ghost; a.X = X; a.xstride = xstride;
      // the J blocks X_0..X_{J-1} (the last is Y itself when y_is_block), Y as the B operand
      a.J = J; a.y_alias = y_is_block ? 1 : 0; a.Y = Y; a.zeros = c->d_zeros;
      a.part = c->d_part; a.gpart = c->d_gpart; a.tickets = c->d_tickets; a.G = c->d_G;
      a.active = active;
      GramFuse f{};
      // fuse the small step into the Gram tail on one rank (no allreduce in between), or on
      // P > 1 ranks when the allreduce itself runs in the tail (f2, LSBA_DEVAR), while its
      // Gram copy fits next to the partials (<= 64 KB of shared memory)
      const bool devar = c->nccl && c->nccl->devar;
      if (coef_k >= 0 && coef_fused && (!c->comm || devar) && !c->no_fuse && E * sizeof(double) <= 64 * 1024) {
        f.on = 1;
        f.st = c->st;
        f.k = coef_k;
        f.prm = prm ? *prm : CycleParams{};
        *coef_fused = true;
        if (devjoin) {
          f.upd_wait = 1;
          f.upd_seq = c->st.upd_seq;
          f.upd_done = c->st.upd_done;
        }
        if (devar) {
          f.ar = 1;
          f.woff = (size_t)(c->ar_seq++ & 1) * c->ar_slot;
          f.win = c->nccl->win;
          f.dcomm = c->nccl->d_dcomm;
          ar_in_kernel = true;
        }
      }
      if (!gl) {
        if constexpr (v7_s) TRY(gram_v7<S>(c, a, f));
      } else {
        if constexpr (S % 2 == 0) {
          // streaming global Gram (gram7.cuh)
          const int grid = std::max(1, std::min(3 * c->n_sms, cdiv(cdiv((long)c->slot, 2), 256)));
          k_gram_gl2<S><<<grid, 256, sizeof(double) * (J + 1), c->stream>>>(a, f);
          CKL();
        }
      }
    } else {
      CK(cudaMemsetAsync(c->d_G, 0, sizeof(double) * E, c->stream));
      if (coef_fused) *coef_fused = false;
    }
  } else {
    // DFMA fallback (odd s, s = 1, variant 1, non-slot inputs): per-CTA partials + fixed-order sum
    const int gx = gl ? J : J * (S / GramTA<S>::value);
    int P = std::max(1, std::min(cdiv(std::max(c->n, 1), 256), cdiv(kGramCtas, gx)));
    if ((size_t)P * E > c->part_cap) P = std::max(1, (int)(c->part_cap / E));
    {
      LaunchScope Ls(c, LSBA_K_GRAM, 8.0 * c->n * S * J + (y_is_block ? 0.0 : 8.0 * c->n * S));
      dim3 grid(gx, P);
      if (gl)
        k_gram_gl<S><<<grid, kThreads, 0, c->stream>>>(c->n, X, xstride, J, Y, c->d_part, active);
      else
        k_gram_cl<S><<<grid, kThreads, 0, c->stream>>>(c->n, X, xstride, J, Y, c->d_part, active);
      CKL();
    }
    {
      LaunchScope Ls(c, LSBA_K_GRAM_FINALIZE, 8.0 * P * E);
      k_gram_finalize<<<cdiv(E, 128), 128, 0, c->stream>>>(P, (int)E, c->d_part, c->d_G,
                                                           gl ? 1.0 / S : 1.0, active);
      CKL();
    }
  }
  if (c->comm && !ar_in_kernel) TRYC(c->comm->allreduce_sum_f64(c->d_G, E, c->stream));
  return LSBA_OK;
}

// ---------------------------------------------------------------- a4/a6: projection
// CTAs of a projection launch that prefetch their first rows into L2 before waiting on the
// Gram (kernels.cuh prefetch_blocks_l2): as many as the budget c->proj_pf covers.
static int proj_pf_ctas(lsba_ctx c, long bytes_per_cta, int grid) {
  if (!c->pdl || c->proj_pf <= 0 || bytes_per_cta <= 0) return 0;
  return (int)std::min<long>(grid, c->proj_pf / bytes_per_cta);
}
template <int S>
static lsba_status project_t(lsba_ctx c, const double* X, size_t xstride, int J0,
                             const double* C0, const double* base0, double* out0, int J1,
                             const double* C1, double* out1, const int* flag_ptr, int kid) {
  const bool gl = (c->ip == LSBA_IP_GLOBAL);
  const size_t CB = gl ? 1 : (size_t)S * S;
  const size_t smem = (size_t)(J0 + J1) * CB * sizeof(double);
  if (smem > 200 * 1024 && J0 > 0 && J1 > 0) {
    // too many coefficients for one CTA's shared memory: two passes
    TRY(project_t<S>(c, X, xstride, J0, C0, base0, out0, 0, nullptr, nullptr, flag_ptr, kid));
    return project_t<S>(c, X, xstride, 0, nullptr, nullptr, nullptr, J1, C1, out1, flag_ptr, kid);
  }
  const int Jmax = std::max(J0, J1);
  const int n = c->n;
  const double bytes = 8.0 * n * S * (Jmax + (J0 > 0) + (J1 > 0) + (base0 ? 1 : 0));
  LaunchScope Ls(c, kid, bytes);
  if (n == 0) return LSBA_OK;
  // s = 4: the DFMA kernel streams faster than the DMMA one (5.8 vs 5.0 TB/s on config 2,
  // tools/gpu_variants.sh); s = 8, 16: DMMA (6.65 TB/s on configs 3 and 5)
  if constexpr (S == 8 || S == 16) {
    if (!gl && c->variant == 0 && !c->proj_dfma) {
      auto fn = k_project_dmma<S>;
      if (smem > 32 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int occ = 1;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, 256, smem));
      const int rows_per_warp = (S >= 16 ? 16 : 32);
      const int grid = std::max(1, std::min(cdiv(cdiv(n, rows_per_warp), 8), occ * c->n_sms));
      CK(launch_k(c, fn, dim3(grid), dim3(256), smem, n, X, xstride, J0, C0, base0, out0, J1, C1,
                  out1, flag_ptr, proj_pf_ctas(c, 8L * rows_per_warp * S * 8 * Jmax, grid)));
      return LSBA_OK;
    }
  }
  if (gl && S % 2 == 0) {           // flat elementwise combination (scalar coefficients)
    const long cnt2 = (long)n * S / 2;
    const int grid = std::max(1, std::min(cdiv(cnt2, kThreads), 8 * c->n_sms));
    CK(launch_k(c, k_project_flat, dim3(grid), dim3(kThreads), smem, cnt2, X, xstride, J0, C0, base0,
                out0, J1, C1, out1, flag_ptr, proj_pf_ctas(c, 16L * kThreads * Jmax, grid)));
    return LSBA_OK;
  }
  // one-row-per-thread kernel on a resident (grid-stride) grid
  auto resident_grid = [&](auto fn) -> int {
    int occ = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kThreads, smem) != cudaSuccess || occ < 1) occ = 1;
    return std::max(1, std::min(cdiv(n, kThreads), occ * c->n_sms));
  };
  if (gl) {
    auto fn = k_project<S, true>;
    if (smem > 32 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    fn<<<resident_grid(fn), kThreads, smem, c->stream>>>(n, X, xstride, J0, C0, base0, out0,
                                                          J1, C1, out1, flag_ptr, 0);
  } else {
    auto fn = k_project<S, false>;
    if (smem > 32 * 1024) CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = resident_grid(fn);
    CK(launch_k(c, fn, dim3(grid), dim3(kThreads), smem, n, X, xstride, J0, C0,
                base0, out0, J1, C1, out1, flag_ptr, proj_pf_ctas(c, 8L * kThreads * S * Jmax, grid)));
  }
  CKL();
  return LSBA_OK;
}

// dispatch wrappers (runtime s)
static lsba_status spmm(lsba_ctx c, const double* V, double* W, const int* active = nullptr) {
  LSBA_DISPATCH_S(c->s, spmm_t, c, V, W, active);
}
static lsba_status residual(lsba_ctx c, const double* Bm, const double* X, double* out) {
  LSBA_DISPATCH_S(c->s, residual_t, c, Bm, X, out);
}
static lsba_status ilu_apply(lsba_ctx c, double* Y, const int* active) {
  LSBA_DISPATCH_S(c->s, ilu_apply_t, c, Y, active);
}
static lsba_status gram(lsba_ctx c, const double* X, size_t xstride, int J, double* Y, int ip,
                        const double* Vk = nullptr, const int* active = nullptr, int coef_k = -1,
                        const CycleParams* prm = nullptr, bool* coef_fused = nullptr) {
  LSBA_DISPATCH_S(c->s, gram_t, c, X, xstride, J, Y, ip, Vk, active, coef_k, prm, coef_fused);
}
// BMGS-(I)CWY block inner product <[X_0..X_{J-1}], [Y Y2]> ((J b) x 2b, row-major; global:
// J pairs) into c->d_G, one pass and one allreduce (Alg 6 line 10).
template <int S>
static lsba_status gram2_t(lsba_ctx c, const double* X, size_t xstride, int J, const double* Y,
                           const double* Y2, int ip, const int* active) {
  const bool gl = (ip == LSBA_IP_GLOBAL);
  const size_t E = gl ? 2 * (size_t)J : 2 * (size_t)J * S * S;
  const bool slots = in_basis(c, X) && in_basis(c, Y) && in_basis(c, Y2) && c->d_tickets;
  bool done = false;
  if (c->variant == 0 && slots) {
    LaunchScope Ls(c, LSBA_K_GRAM, 8.0 * c->n * S * (J + 1));
    GramArgs a;
    a.n = c->n; a.rp = c->d_rp; a.ci = c->d_ci; a.va = c->d_va;
    a.Vk = nullptr; a.Vghost = c->d_ghost; a.X = X; a.xstride = xstride;
    a.J = J; a.y_alias = 0; a.Y = const_cast<double*>(Y); a.Y2 = Y2; a.zeros = c->d_zeros;
    a.part = c->d_part; a.gpart = c->d_gpart; a.tickets = c->d_tickets; a.G = c->d_G;
    a.active = active;
    if (c->n == 0) {
      CK(cudaMemsetAsync(c->d_G, 0, sizeof(double) * E, c->stream));
      done = true;
    } else if (!gl) {
      if constexpr (S == 2 || S == 4 || S == 8 || S == 16) {
        TRY(gram2_v7<S>(c, a));
        done = true;
      }
    } else {
      if constexpr (S % 2 == 0) {
        const int grid = std::max(1, std::min(3 * c->n_sms, cdiv(cdiv((long)c->slot, 2), 256)));
        k_gram_gl2<S, 2><<<grid, 256, 0, c->stream>>>(a, GramFuse{});
        CKL();
        done = true;
      }
    }
  }
  if (done) {
    if (c->comm) TRYC(c->comm->allreduce_sum_f64(c->d_G, E, c->stream));
    return LSBA_OK;
  }
  // fallback (odd s, DFMA variant, non-slot inputs): two block inner products (two syncs on
  // P > 1), interleaved; the other half of the G double buffer is free in a CWY step
  double* const Gdst = c->d_G;
  double* const T1 = (Gdst == c->d_Gbase) ? c->d_Gbase + c->g_half : c->d_Gbase;
  double* const T2 = T1 + E / 2;
  c->d_G = T1;
  TRY(gram_t<S>(c, X, xstride, J, const_cast<double*>(Y), ip, nullptr, active, -1, nullptr, nullptr));
  c->d_G = T2;
  TRY(gram_t<S>(c, X, xstride, J, const_cast<double*>(Y2), ip, nullptr, active, -1, nullptr, nullptr));
  c->d_G = Gdst;
  {
    LaunchScope Ls(c, LSBA_K_MISC, 16.0 * E);
    const int bb = gl ? 1 : S;
    k_interleave2<<<cdiv((long)E, 256), 256, 0, c->stream>>>(J * bb, bb, T1, T2, Gdst);
    CKL();
  }
  return LSBA_OK;
}
static lsba_status gram2(lsba_ctx c, const double* X, size_t xstride, int J, const double* Y,
                         const double* Y2, int ip, const int* active) {
  LSBA_DISPATCH_S(c->s, gram2_t, c, X, xstride, J, Y, Y2, ip, active);
}

template <int S>
static lsba_status project_tp(lsba_ctx c, const double* X, size_t xstride, int J0, const double* C0,
                              const double* base0, double* out0, int J1, const double* C1, double* out1,
                              const int* flag_ptr, int kid) {
  c->in_proj = true;
  const lsba_status st = project_t<S>(c, X, xstride, J0, C0, base0, out0, J1, C1, out1, flag_ptr, kid);
  c->in_proj = false;
  return st;
}
static lsba_status project(lsba_ctx c, const double* X, size_t xstride, int J0, const double* C0,
                           const double* base0, double* out0, int J1, const double* C1, double* out1,
                           const int* flag_ptr, int kid) {
  LSBA_DISPATCH_S(c->s, project_tp, c, X, xstride, J0, C0, base0, out0, J1, C1, out1, flag_ptr, kid);
}


template <int B>
static lsba_status small_step_t(lsba_ctx c, int k, const CycleParams& prm) {
  LaunchScope Ls(c, LSBA_K_SMALL_STEP, 0.0);
  const double rfac = (c->ip == LSBA_IP_GLOBAL) ? std::sqrt((double)c->s) : 1.0;
  CK(launch_step_small<B>(c->st, c->d_G, k, prm, rfac, c->stream));
  return LSBA_OK;
}
static lsba_status small_step(lsba_ctx c, int k, const CycleParams& prm) {
  LSBA_DISPATCH_S(c->b, small_step_t, c, k, prm);
}

template <int B>
static lsba_status step_update_t(lsba_ctx c, int k, const double* G) {
  // (diagnostics: LSBA_UPD_MAIN=1 serialises it on the main stream to time it alone)
  cudaStream_t st = c->upd_main ? c->stream : c->stream2;
  LaunchScope Ls(c, LSBA_K_STEP_UPDATE, 0.0, st);
  const double rfac = (c->ip == LSBA_IP_GLOBAL) ? std::sqrt((double)c->s) : 1.0;
  ++c->st.upd_seq;   // released to st.upd_done when this launch exits (device-side join)
  CK(launch_step_update<B>(c->st, G, k, rfac, st));
  return LSBA_OK;
}
static lsba_status step_update(lsba_ctx c, int k, const double* G) {
  LSBA_DISPATCH_S(c->b, step_update_t, c, k, G);
}

// ---------------------------------------------------------------- BMGS-(I)CWY small kernels
template <int B>
static lsba_status cwy_iter1_t(lsba_ctx c) {
  LaunchScope Ls(c, LSBA_K_SMALL_STEP, 0.0);
  CK(launch_cwy_iter1<B>(c->st, c->d_G, c->stream));
  return LSBA_OK;
}
template <int B>
static lsba_status cwy_coef_t(lsba_ctx c, int k) {
  LaunchScope Ls(c, LSBA_K_SMALL_STEP, 0.0);
  CK(launch_cwy_coef<B>(c->st, c->d_G, k, c->skel == LSBA_SKEL_BMGS_ICWY ? 1 : 0, c->stream));
  return LSBA_OK;
}
template <int B>
static lsba_status irols_coef_t(lsba_ctx c, int k) {
  LaunchScope Ls(c, LSBA_K_SMALL_STEP, 0.0);
  CK(launch_irols_coef<B>(c->st, c->d_G, k, c->stream));
  return LSBA_OK;
}
static lsba_status cwy_iter1_small(lsba_ctx c) { LSBA_DISPATCH_S(c->b, cwy_iter1_t, c); }
static lsba_status cwy_coef(lsba_ctx c, int k) {
  if (c->skel == LSBA_SKEL_BCGS_IROLS) { LSBA_DISPATCH_S(c->b, irols_coef_t, c, k); }
  LSBA_DISPATCH_S(c->b, cwy_coef_t, c, k);
}

// ---------------------------------------------------------------- BMGS / BCGS-PIO small kernels
template <int B>
static lsba_status bmgs_h_t(lsba_ctx c, int j, int k) {
  LaunchScope Ls(c, LSBA_K_SMALL_STEP, 0.0);
  CK(launch_bmgs_h<B>(c->st, c->d_G, j, k, c->stream));
  return LSBA_OK;
}
template <int B>
static lsba_status bmgs_r_t(lsba_ctx c, int k) {
  LaunchScope Ls(c, LSBA_K_SMALL_STEP, 0.0);
  CK(launch_bmgs_r<B>(c->st, c->d_G, k, c->stream));
  return LSBA_OK;
}
template <int B>
static lsba_status pio_coef_t(lsba_ctx c, const double* G1, const double* G2, int k) {
  LaunchScope Ls(c, LSBA_K_SMALL_STEP, 0.0);
  CK(launch_pio_coef<B>(c->st, G1, G2, k, c->stream));
  return LSBA_OK;
}
static lsba_status bmgs_h(lsba_ctx c, int j, int k) { LSBA_DISPATCH_S(c->b, bmgs_h_t, c, j, k); }
static lsba_status bmgs_r(lsba_ctx c, int k) { LSBA_DISPATCH_S(c->b, bmgs_r_t, c, k); }
static lsba_status pio_coef(lsba_ctx c, const double* G1, const double* G2, int k) {
  LSBA_DISPATCH_S(c->b, pio_coef_t, c, G1, G2, k);
}

static lsba_status read_status(lsba_ctx c, StepStatus* out, CycleCtl* ctl) {
  CK(cudaMemcpyAsync(c->h_status, c->st.status, sizeof(StepStatus), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(CycleCtl), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(c->h_info + 1, c->d_info + 1, 7 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (out) *out = *c->h_status;
  if (ctl) *ctl = *c->h_ctl;
  return LSBA_OK;
}

// IO(U) with U in slot 0: Gram (1 sync), chol, scale in place (Alg 3 line 1).  Resets the
// device cycle control with this cycle's parameters.  Asynchronous.
static lsba_status io_begin_async(lsba_ctx c, const CycleParams& prm) {
  bool fused = false;
  TRY(gram(c, slotp(c, 0), c->slot_stride, 1, slotp(c, 0), c->ip, nullptr, nullptr, 0, &prm, &fused));
  if (!fused) TRY(small_step(c, 0, prm));
  TRY(project(c, slotp(c, 0), c->slot_stride, 1, c->st.coef, nullptr, slotp(c, 0), 0, nullptr, nullptr,
              c->st.flag_dev, LSBA_K_PROJECT));
  return LSBA_OK;
}

// One Alg-3 step k (1-based), asynchronous; every kernel no-ops once the device cycle
// control says the cycle has ended (speculative enqueue of a whole cycle).
static lsba_status pip_step_async(lsba_ctx c, int k) {
  const CycleParams none{};   // (k > 0 launches read their parameters from the device control)
  // The SpMM of step k runs while the update kernel of step k-1 (stream 2) is still taking
  // the continue/restart decision: it only writes slot k, scratch if the cycle ended at step
  // k-1.  The Gram (and the small step fused into its tail) waits for the update: its tail
  // acquires the update's exit on the device when fused (GramFuse::upd_wait), else the main
  // stream joins the update's event (wait_update).
  c->d_G = c->d_Gbase + (size_t)(k & 1) * c->g_half;
  c->pending_upd = (k > 1);
  bool fused = false;
  TRY(gram(c, slotp(c, 0), c->slot_stride, k + 1, slotp(c, k), c->ip, slotp(c, k - 1),
           &c->d_ctl->active, k, &none, &fused));                                // lines 3-4 (+5)
  TRY(wait_update(c));
  if (!fused) TRY(small_step(c, k, none));                                       // line 5
  // estimates / kappa_F / decision on stream 2, concurrent with the projection
  CK(cudaEventRecord(c->ev_coef, c->stream));
  CK(cudaStreamWaitEvent(c->stream2, c->ev_coef, 0));
  TRY(step_update(c, k, c->d_G));
  CK(cudaEventRecord(c->ev_upd, c->stream2));
  TRY(project(c, slotp(c, 0), c->slot_stride, k + 1, c->st.coef, nullptr, slotp(c, k), 0, nullptr,
              nullptr, c->st.flag_dev, LSBA_K_PROJECT));                         // line 6
  return LSBA_OK;
}

// Host-side lookahead bound for the speculative enqueue of a cycle: step k is enqueued once
// the device has decided step k - kLookahead (polling the mapped progress word 2 k + active).
// Returns false once no more steps of this cycle are to be enqueued.
//  * One rank: stop as soon as the device has ended the cycle (flag, convergence, kappa).
//  * P > 1 ranks: every step carries a halo exchange and the Gram allreduce, so all ranks must
//    enqueue the same steps.  The end step k_end is a replicated device decision (bitwise-equal
//    allreduce results), and no host is ever more than kLookahead steps past the decided step,
//    so every rank enqueues exactly steps 1 .. min(m, k_end + kLookahead) and stops there.
constexpr int kLookahead = 3;
static bool throttle(lsba_ctx c, int k) {
  const bool single = !c->comm;
  for (;;) {
    const int v = c->h_prog[0];
    const int done = v < 0 ? -1 : (v >> 1), act = v < 0 ? 1 : (v & 1);
    if (done >= 0 && act == 0) return single ? false : (k <= done + kLookahead);
    if (k <= kLookahead || done >= k - kLookahead) return true;
    // device drained (no stall possible) or failed (the error surfaces at the next CUDA call):
    // stop polling.  (On P > 1 a drained stream has decided every enqueued step, so the
    // conditions above already hold unless the device failed.)
    if (cudaStreamQuery(c->stream) != cudaErrorNotReady) return true;
  }
}

// BMGS-(I)CWY (Alg 6): loop iteration 1 after IO(U): W = A V_1 (slot 1),
// H_11 = <V_1, W>, U = W - V_1 H_11 over W (slot 1).  Asynchronous.
static lsba_status cwy_iter1_async(lsba_ctx c) {
  const int* act = &c->d_ctl->active;
  TRY(spmm(c, slotp(c, 0), slotp(c, 1), act));                                    // line 5
  TRY(gram(c, slotp(c, 0), c->slot_stride, 2, slotp(c, 1), c->ip, nullptr, act));  // line 7
  TRY(cwy_iter1_small(c));
  TRY(project(c, slotp(c, 0), c->slot_stride, 2, c->st.coef, nullptr, slotp(c, 1), 0, nullptr, nullptr,
              c->st.flag_dev, LSBA_K_PROJECT));                                     // line 8
  return LSBA_OK;
}

// Arnoldi step k >= 1 = Alg 6 loop iteration k+1: U (unnormalised V_{k+1}) sits in slot k.
// W = A U -> slot k+1; ONE block inner product <[V_1..V_k U], [U W]> (+ one allreduce); the
// small step (chol, T column, H_{1:k+1,k+1}, coefficients); the update kernel (QR, estimates,
// decision) on stream 2 for the now complete Hessenberg column k; and one two-output pass
// V_{k+1} = U H^{-1} (over slot k), U' = W H^{-1} - V H_{1:k+1,k+1} (over slot k+1; skipped on
// the cycle's last step).  Asynchronous.
static lsba_status cwy_step_async(lsba_ctx c, int k, bool last) {
  const int* act = &c->d_ctl->active;
  const size_t bb = (size_t)c->b * c->b;
  c->d_G = c->d_Gbase + (size_t)(k & 1) * c->g_half;
  c->pending_upd = (k > 1);
  TRY(spmm(c, slotp(c, k), slotp(c, k + 1), act));                                 // line 5
  TRY(wait_update(c));
  TRY(gram2(c, slotp(c, 0), c->slot_stride, k + 1, slotp(c, k), slotp(c, k + 1), c->ip, act));  // line 10
  TRY(cwy_coef(c, k));                                                              // lines 11-14
  CK(cudaEventRecord(c->ev_coef, c->stream));
  CK(cudaStreamWaitEvent(c->stream2, c->ev_coef, 0));
  TRY(step_update(c, k, c->st.gpip));
  CK(cudaEventRecord(c->ev_upd, c->stream2));
  TRY(project(c, slotp(c, 0), c->slot_stride, k + 1, c->st.coef, nullptr, slotp(c, k), last ? 0 : k + 2,
              c->st.coef + (size_t)(k + 1) * bb, slotp(c, k + 1), c->st.flag_dev, LSBA_K_PROJECT));  // 16-17
  return LSBA_OK;
}

// BMGS-Arnoldi step k (Alg 2; comparison baseline):
// W = A V_k; for j = 1..k: H_{j,k} = <V_j, W> (a sync each), W = W - V_j H_{j,k}; then
// [V_{k+1}, H_{k+1,k}] = IO(W) (one more sync).  Asynchronous.
static lsba_status bmgs_step_async(lsba_ctx c, int k) {
  const int* act = &c->d_ctl->active;
  c->d_G = c->d_Gbase + (size_t)(k & 1) * c->g_half;
  c->pending_upd = (k > 1);
  TRY(spmm(c, slotp(c, k - 1), slotp(c, k), act));                                 // line 3
  TRY(wait_update(c));
  for (int j = 1; j <= k; ++j) {
    TRY(gram(c, slotp(c, j - 1), c->slot_stride, 1, slotp(c, k), c->ip, nullptr, act));   // line 5
    TRY(bmgs_h(c, j, k));
    TRY(project(c, slotp(c, j - 1), (size_t)(k - j + 1) * c->slot_stride, 2, c->st.coef, nullptr,
                slotp(c, k), 0, nullptr, nullptr, c->st.flag_dev, LSBA_K_PROJECT));   // line 6
  }
  TRY(gram(c, slotp(c, k), c->slot_stride, 1, slotp(c, k), c->ip, nullptr, act));  // line 7: IO
  TRY(bmgs_r(c, k));
  CK(cudaEventRecord(c->ev_coef, c->stream));
  CK(cudaStreamWaitEvent(c->stream2, c->ev_coef, 0));
  TRY(step_update(c, k, c->st.gpip));
  CK(cudaEventRecord(c->ev_upd, c->stream2));
  TRY(project(c, slotp(c, k), c->slot_stride, 1, c->st.coef, nullptr, slotp(c, k), 0, nullptr, nullptr,
              c->st.flag_dev, LSBA_K_PROJECT));
  return LSBA_OK;
}

// BCGS-PIO step k (Alg 4; comparison baseline): W = A V_k; H = <[V_1..V_k], W>
// (sync 1); <W, W> (sync 2); H_{k+1,k} = chol(W~^T W~ - H~^T H~); V_{k+1} as BCGS-PIP.
static lsba_status pio_step_async(lsba_ctx c, int k) {
  const int* act = &c->d_ctl->active;
  double* const G1 = c->d_Gbase + (size_t)(k & 1) * c->g_half;
  double* const G2 = G1 + (size_t)k * c->b * c->b;
  c->pending_upd = (k > 1);
  c->d_G = G1;
  TRY(spmm(c, slotp(c, k - 1), slotp(c, k), act));                                 // line 3
  TRY(wait_update(c));
  TRY(gram(c, slotp(c, 0), c->slot_stride, k, slotp(c, k), c->ip, nullptr, act));  // line 4
  c->d_G = G2;
  TRY(gram(c, slotp(c, k), c->slot_stride, 1, slotp(c, k), c->ip, nullptr, act));  // line 5 (IO of W)
  c->d_G = G1;
  TRY(pio_coef(c, G1, G2, k));                                                      // lines 5-6
  CK(cudaEventRecord(c->ev_coef, c->stream));
  CK(cudaStreamWaitEvent(c->stream2, c->ev_coef, 0));
  TRY(step_update(c, k, G1));
  CK(cudaEventRecord(c->ev_upd, c->stream2));
  TRY(project(c, slotp(c, 0), c->slot_stride, k + 1, c->st.coef, nullptr, slotp(c, k), 0, nullptr,
              nullptr, c->st.flag_dev, LSBA_K_PROJECT));                           // line 7
  return LSBA_OK;
}

static lsba_status step_async(lsba_ctx c, int k, bool last) {
  switch (c->skel) {
    case LSBA_SKEL_BCGS_PIP: return pip_step_async(c, k);
    case LSBA_SKEL_BMGS_CWY:
    case LSBA_SKEL_BMGS_ICWY:
    case LSBA_SKEL_BCGS_IROLS: return cwy_step_async(c, k, last);
    case LSBA_SKEL_BMGS: return bmgs_step_async(c, k);
    case LSBA_SKEL_BCGS_PIO: return pio_step_async(c, k);
    default: return fail(c, LSBA_E_ARG, "bad skeleton");
  }
}

// join stream 2 (the last step's update) into the main stream
static lsba_status join_update(lsba_ctx c) {
  CK(cudaStreamWaitEvent(c->stream, c->ev_upd, 0));
  return LSBA_OK;
}

static lsba_status set_identity(lsba_ctx c) {
  LaunchScope Ls(c, LSBA_K_MISC, 0.0);
  k_set_identity<<<1, 256, 0, c->stream>>>(c->st.Cacc, c->b);
  CKL();
  return LSBA_OK;
}

template <int B>
static lsba_status cycle_end_t(lsba_ctx c, int k, int gmres, int happy, int upd, int* info,
                               const int* prior) {
  LaunchScope Ls(c, LSBA_K_CYCLE_SOLVE, 0.0);
  const int force = (!happy && c->force_sing_cycle > 0 && c->cur_cycle == c->force_sing_cycle) ? 1 : 0;
  CK(launch_cycle_end<B>(c->st, k, gmres, happy, upd, c->d_Y, c->d_Z, info, prior, force, c->stream));
  return LSBA_OK;
}
static lsba_status cycle_end(lsba_ctx c, int k, int gmres, int happy, int upd, int* info,
                             const int* prior = nullptr) {
  LSBA_DISPATCH_S(c->b, cycle_end_t, c, k, gmres, happy, upd, info, prior);
}

// Enqueue the cycle-end projected solve; its singular flag goes to d_info[1] and guards the
// combine that follows (no host round trip; the flag is read with the next cycle's status).
static lsba_status cycle_solve_async(lsba_ctx c, int k, int gmres) {
  return cycle_end(c, k, gmres, 0, 1, c->d_info + 1);
}

// The speculative cycle end (one rank): enqueued with k = m before the host reads the cycle's
// status; runs only if the cycle ended at k = m and the previous cycle end (guard `prior`, if
// one is pending) was not singular (k_cycle_end's guard).  Ping-pong flag slots per cycle
// parity: d_info[4 + par] = singular / combine guard, d_info[6 + par] = skipped.
static lsba_status cycle_solve_spec(lsba_ctx c, int k, int gmres, int par, const int* prior) {
  return cycle_end(c, k, gmres, 0, 2, c->d_info + 4 + par, prior);
}

static lsba_status cycle_solve(lsba_ctx c, int k, int gmres, int happy, int* singular, int upd = 1) {
  TRY(cycle_end(c, k, gmres, happy, upd, c->d_info));
  CK(cudaMemcpyAsync(c->h_info, c->d_info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *singular = c->h_info[0];
  return LSBA_OK;
}

static lsba_status read_scalar(lsba_ctx c, double* v) {
  CK(cudaMemcpyAsync(c->h_scalar, c->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *v = *c->h_scalar;
  return LSBA_OK;
}

// ------------------------------------------------------------------------------------------
// the restarted solver (mirrors oracle.solve step by step)
// ------------------------------------------------------------------------------------------
static void set_ip(lsba_ctx c, int ip) {
  c->ip = ip;
  c->b = (ip == LSBA_IP_GLOBAL) ? 1 : c->s;
}

static lsba_status solve_impl(lsba_ctx c, const double* B, double* X, int m, double tol,
                              int max_restarts, int gmres, int ip, double tau,
                              lsba_solve_info* info, int skel = LSBA_SKEL_BCGS_PIP) {
  if (!c) return LSBA_E_ARG;
  if (!info) return fail(c, LSBA_E_ARG, "info is NULL");
  if (m < 1 || m > c->m_max) return fail(c, LSBA_E_ARG, "m=%d outside [1, m_max=%d]", m, c->m_max);
  if (!(tol > 0.0)) return fail(c, LSBA_E_ARG, "tol must be > 0");
  if (max_restarts < 0) return fail(c, LSBA_E_ARG, "max_restarts < 0");
  if (ip != LSBA_IP_CLASSICAL && ip != LSBA_IP_GLOBAL) return fail(c, LSBA_E_ARG, "bad inner product");
  if (c->n > 0 && (!B || !X)) return fail(c, LSBA_E_ARG, "B/X is NULL");
  if (((uintptr_t)B | (uintptr_t)X) & 15) return fail(c, LSBA_E_ARG, "B/X not 16-byte aligned");
  CK(cudaSetDevice(c->device));
  const auto t0 = std::chrono::steady_clock::now();
  const int64_t launches0 = c->launches;
  std::memset(info, 0, sizeof *info);
  info->true_relres = NAN;
  info->res_est = NAN;
  if (skel < LSBA_SKEL_BCGS_PIP || skel > LSBA_SKEL_BCGS_IROLS) return fail(c, LSBA_E_ARG, "bad skeleton");
  set_ip(c, ip);
  c->skel = skel;
  c->forced_done = false;
  c->k = -1;
  c->flagged = false;
  auto finish = [&]() {
    // the paper's counters (PAPER.md:650 tables): BMGS-(I)CWY applies A, syncs and evaluates
    // one more block per cycle than BCGS-PIP (the lagged normalisation)
    const bool cwy = lagged(skel);
    const int64_t extra = cwy ? info->cycles : 0;
    info->restarts = info->cycles > 0 ? info->cycles - 1 : 0;
    info->syncs = (int64_t)info->iterations + info->cycles + extra;
    info->matvecs = info->iterations + extra;
    info->basis_evals = 3 * (int64_t)info->iterations + extra;
    if (skel == LSBA_SKEL_BMGS) {          // k+1 syncs per step
      info->syncs = info->gram_blocks + info->cycles;
      info->basis_evals = 2 * (int64_t)info->iterations;
    } else if (skel == LSBA_SKEL_BCGS_PIO) {   // two syncs per step (Table 1)
      info->syncs = 2 * (int64_t)info->iterations + info->cycles;
    } else if (skel == LSBA_SKEL_BCGS_IROLS) { // 4 block evaluations per step
      info->basis_evals = 4 * (int64_t)info->iterations + info->cycles;
    }
    info->kernel_launches = c->launches - launches0;
    info->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  };

  // ||B||_F^2 = s * <B,B>_gl  (R18: tolerance relative to ||B||_F); preconditioned (R28):
  // the method runs on M^{-1} A X = M^{-1} B, so the reference norm is ||M^{-1} B||_F and
  // slot 0 keeps M^{-1} B (= U when X0 = 0)
  if (c->prec && c->n > 0) {
    CK(cudaMemcpyAsync(slotp(c, 0), B, sizeof(double) * c->slot, cudaMemcpyDeviceToDevice, c->stream));
    TRY(ilu_apply(c, slotp(c, 0)));
  }
  {  // sum of squares: per-CTA partials in a fixed order, then one fixed-order sum (+ allreduce)
    const double* Bn = c->prec ? slotp(c, 0) : B;
    const long cnt = (long)c->n * c->s;
    const int nblk = std::max(1, std::min<int>(c->sq_cap, std::min<long>(4L * c->n_sms, cdiv(cnt, kThreads))));
    LaunchScope Ls(c, LSBA_K_MISC, 8.0 * cnt);
    if (c->n > 0) {
      k_sq_partials<<<nblk, kThreads, 0, c->stream>>>(cnt, Bn, c->d_sq);
      CKL();
      k_sum_partials<<<1, kThreads, 0, c->stream>>>(nblk, c->d_sq, c->d_scalar);
      CKL();
    } else {
      CK(cudaMemsetAsync(c->d_scalar, 0, sizeof(double), c->stream));
    }
  }
  if (c->comm) TRYC(c->comm->allreduce_sum_f64(c->d_scalar, 1, c->stream));
  CK(cudaMemcpyAsync(c->h_scalar, c->d_scalar, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const double normB = std::sqrt(std::max(0.0, *c->h_scalar));
  if (normB == 0.0) {  // B = 0: X = 0 exactly
    if (c->n > 0) CK(cudaMemsetAsync(X, 0, sizeof(double) * c->slot, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    info->outcome = LSBA_CONVERGED;
    info->true_relres = 0.0;
    info->m_final = m;
    finish();
    return LSBA_OK;
  }
  // explicit relative residual of Xv; R = B - A Xv written to out_R
  auto true_relres = [&](const double* Xv, double* out_R, double* rel) -> lsba_status {
    TRY(residual(c, B, Xv, out_R));
    double r2;
    TRY(read_scalar(c, &r2));
    *rel = std::sqrt(std::max(0.0, r2)) / normB;
    return LSBA_OK;
  };

  // U = B - A X0 (R13); U = B exactly when X0 = 0 (every rank must agree: one flag allreduce)
  {
    CK(cudaMemsetAsync(c->d_info, 0, sizeof(int), c->stream));
    if (c->n > 0) {
      LaunchScope Ls(c, LSBA_K_MISC, 8.0 * c->slot);
      k_any_nonzero<<<std::min(4 * c->n_sms, cdiv((long)c->slot, kThreads)), kThreads, 0, c->stream>>>(
          (long)c->slot, X, c->d_info);
      CKL();
    }
    if (c->comm) TRYC(c->comm->allreduce_max_i32(c->d_info, 1, c->stream));
    CK(cudaMemcpyAsync(c->h_info, c->d_info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->h_info[0]) {
      TRY(residual(c, B, X, slotp(c, 0)));
    } else if (c->n > 0 && !c->prec) {       // (preconditioned: slot 0 already holds M^{-1} B)
      CK(cudaMemcpyAsync(slotp(c, 0), B, sizeof(double) * c->slot, cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  TRY(set_identity(c));                   // C_acc = I
  int m_cur = m;
  bool sing_pending = false;   // a guarded combine was enqueued; its flag is read later
  int sing_slot = 1;           // ... in d_info[sing_slot]
  CycleCtl cc;
  info->outcome = LSBA_MAX_RESTARTS;
  bool finished = false;
  for (int cycle = 1; cycle <= max_restarts + 1 && !finished; ++cycle) {
    info->cycles = cycle;
    c->cur_cycle = cycle;
    // enqueue IO(U) and all m_cur steps of the cycle; the step kernels take the
    // continue/restart decision on the device and later launches no-op (one host sync)
    CycleParams prm;
    prm.m_cur = m_cur;
    prm.gmres = gmres;
    prm.force_k = c->force_flag_k;
    prm.reset_forced = (cycle == 1) ? 1 : 0;
    prm.tol_abs = tol * normB;                               // R5, R18
    prm.tau = tau;                                           // R8
    prm.need_kappa = std::isfinite(tau) ? 1 : 0;
    c->h_prog[0] = -1;                                       // (device idle: cycle boundary)
    TRY(io_begin_async(c, prm));                             // [V_1, beta] = IO(U)
    if (lagged(c->skel))
      TRY(cwy_iter1_async(c));                               // Alg 6 iteration 1
    for (int k = 1; k <= m_cur; ++k) {
      // keep at most kLookahead steps enqueued beyond the last decided one; stop enqueueing
      // once the device has ended the cycle (flag, convergence, kappa trigger)
      if (!throttle(c, k)) break;
      TRY(step_async(c, k, k == m_cur));
    }
    TRY(join_update(c));
    // speculative cycle end for the common case (the cycle runs to m): enqueued before the
    // status read, so the GPU solves the projected problem and combines while the host wakes
    // up; it no-ops on the device for any other ending, which the host then handles below
    const int par = cycle & 1;
    // (also on P > 1: the cycle end and the combine are row-local, no collective, and the
    // device guard is a replicated decision, so every rank runs or skips them alike)
    const bool spec = c->spec_end && m_cur >= 1;
    if (spec) {
      // the status is copied (and waited for) BEFORE the speculative kernels, so the host
      // decides while the GPU solves and combines, and enqueues the next cycle behind them
      CK(cudaMemcpyAsync(c->h_status, c->st.status, sizeof(StepStatus), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(c->h_ctl, c->d_ctl, sizeof(CycleCtl), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaMemcpyAsync(c->h_info + 1, c->d_info + 1, 7 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
      CK(cudaEventRecord(c->ev_status, c->stream));
      TRY(cycle_solve_spec(c, m_cur, gmres, par, sing_pending ? c->d_info + sing_slot : nullptr));
      const double comb0 = c->prof.bytes[LSBA_K_COMBINE];
      TRY(project(c, slotp(c, 0), c->slot_stride, m_cur, c->d_Y, X, X, m_cur + 1, c->d_Z, slotp(c, 0),
                  c->d_info + 4 + par, LSBA_K_COMBINE));
      CK(cudaEventSynchronize(c->ev_status));
      cc = *c->h_ctl;
      // the speculative combine moves its bytes only if it ran (k = m ending, no pending
      // singular guard); otherwise it no-op'd on the device: take its bytes back out
      if (!(cc.why == 4 && cc.k_used == m_cur && !(sing_pending && c->h_info[sing_slot])))
        c->prof.bytes[LSBA_K_COMBINE] = comb0;
    } else {
      TRY(read_status(c, nullptr, &cc));
    }
    if (sing_pending && c->h_info[sing_slot]) {             // last cycle end was singular:
      fail(c, LSBA_OK, "projected system singular at cycle end");   // its combine no-op'd,
      info->cycles = cycle - 1;                             // this cycle ran on stale data
      info->outcome = LSBA_DEAD;
      break;
    }
    sing_pending = false;
    if (cc.why == 5) { info->outcome = LSBA_DEAD; break; }   // IO flagged (R4)
    int k_used = cc.k_used;
    info->iterations += k_used;
    info->gram_blocks += (int64_t)k_used * (k_used + 3) / 2;    // sum_{k=1}^{k_used} (k+1)
    info->attempted_steps += k_used + (cc.why == 1 ? 1 : 0);
    if (k_used > 0) info->res_est = cc.res_est;
    if (cc.why == 1) {
      const int k = cc.k_flag;
      if (!cc.forced_here) {
        // R7: happy-breakdown candidate with H_{k+1,k} := 0 (M = 0), checked explicitly
        int sing = 1;
        TRY(cycle_solve(c, k, 0, 1, &sing));
        if (!sing) {
          TRY(project(c, slotp(c, 0), c->slot_stride, k, c->d_Y, X, c->d_Xc, 0, nullptr, nullptr,
                      nullptr, LSBA_K_COMBINE));
          double rel;
          TRY(true_relres(c->d_Xc, slotp(c, k), &rel));    // slot k (flagged W) is free
          if (rel <= tol) {
            CK(cudaMemcpyAsync(X, c->d_Xc, sizeof(double) * c->slot, cudaMemcpyDeviceToDevice, c->stream));
            info->iterations++;
            info->happy++;
            info->true_relres = rel;
            info->outcome = LSBA_CONVERGED;
            finished = true;
            break;
          }
        }
      }
      info->nan_flags++;
      m_cur = k - 1;                                        // R6
    } else if (cc.why == 3) {
      info->cond_restarts++;
    }
    if (k_used == 0) { info->outcome = LSBA_DEAD; break; }
    if (spec && cc.why == 4 && k_used == m_cur) {   // the speculative cycle end ran (its guard)
      sing_pending = true;
      sing_slot = 4 + par;
      continue;
    }
    if (cc.why != 2) {
      // X += V_k Xi C_acc ;  U = V_{k+1} [M; -H_{k+1,k}] -> slot 0,
      // enqueued behind the projected solve without a host round trip (guarded by its flag)
      TRY(cycle_solve_async(c, k_used, gmres));               // Xi, M, cos; C_acc <- cos C_acc
      TRY(project(c, slotp(c, 0), c->slot_stride, k_used, c->d_Y, X, X, k_used + 1, c->d_Z, slotp(c, 0),
                  c->d_info + 1, LSBA_K_COMBINE));
      sing_pending = true;
      sing_slot = 1;
      continue;
    }
    int sing = 0;
    TRY(cycle_solve(c, k_used, gmres, 0, &sing));            // Xi, M, cos; C_acc <- cos C_acc
    if (sing) {
      fail(c, LSBA_OK, "projected system singular at cycle end (k=%d)", k_used);
      info->outcome = LSBA_DEAD;
      break;
    }
    {
      // X += V_k Xi C_acc, then confirm with the explicit residual (R19)
      TRY(project(c, slotp(c, 0), c->slot_stride, k_used, c->d_Y, X, X, 0, nullptr, nullptr, nullptr,
                  LSBA_K_COMBINE));
      double rel;
      TRY(true_relres(X, slotp(c, 0), &rel));                // slot 0 <- B - A X
      if (rel <= tol) {
        info->true_relres = rel;
        info->outcome = LSBA_CONVERGED;
        finished = true;
        break;
      }
      info->false_convergences++;
      TRY(set_identity(c));                                  // restart from the true residual
      continue;
    }
  }
  if (sing_pending) {                                        // the last cycle's combine
    CK(cudaMemcpyAsync(c->h_info + sing_slot, c->d_info + sing_slot, sizeof(int), cudaMemcpyDeviceToHost,
                       c->stream));
    CK(cudaStreamSynchronize(c->stream));
    if (c->h_info[sing_slot]) {
      fail(c, LSBA_OK, "projected system singular at cycle end");
      info->outcome = LSBA_DEAD;
    }
  }
  info->m_final = m_cur;
  if (!(info->outcome == LSBA_CONVERGED)) {
    double rel;
    TRY(true_relres(X, slotp(c, 0), &rel));
    info->true_relres = rel;
  }
  CK(cudaStreamSynchronize(c->stream));
  c->k = -1;
  finish();
  return LSBA_OK;
}

// ------------------------------------------------------------------------------------------
// host-only helpers (exported)
// ------------------------------------------------------------------------------------------
extern "C" lsba_status lsba_csr_validate(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                                         const int32_t* col_idx, const char** msg) {
  static thread_local char buf[256];
  auto bad = [&](const char* m) {
    if (msg) *msg = m;
    return LSBA_E_ARG;
  };
  if (msg) *msg = "";
  if (n_rows < 0 || n_cols < 0) return bad("negative size");
  if (!row_ptr) return bad("row_ptr is NULL");
  if (row_ptr[0] != 0) return bad("row_ptr[0] != 0");
  for (int64_t i = 0; i < n_rows; ++i) {
    if (row_ptr[i + 1] < row_ptr[i]) {
      snprintf(buf, sizeof buf, "row_ptr not monotone at row %lld", (long long)i);
      return bad(buf);
    }
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
      const int64_t cidx = col_idx[p];
      if (cidx < 0 || cidx >= n_cols) {
        snprintf(buf, sizeof buf, "column %lld out of range in row %lld", (long long)cidx, (long long)i);
        return bad(buf);
      }
      if (p > row_ptr[i] && col_idx[p - 1] >= cidx) {
        snprintf(buf, sizeof buf, "columns not strictly increasing in row %lld", (long long)i);
        return bad(buf);
      }
    }
  }
  return LSBA_OK;
}

extern "C" lsba_status lsba_ghost_plan(int64_t row_begin, int64_t row_end, const int32_t* col_idx,
                                       int64_t nnz, const int64_t* part, int32_t nranks,
                                       int32_t* col_local, int64_t* ghost_global, int64_t* n_ghost,
                                       int64_t* recv_counts) {
  if (!col_idx && nnz > 0) return LSBA_E_ARG;
  if (!part || nranks < 1 || !n_ghost || !recv_counts) return LSBA_E_ARG;
  if (row_end < row_begin) return LSBA_E_ARG;
  for (int r = 0; r < nranks; ++r)
    if (part[r + 1] < part[r]) return LSBA_E_ARG;
  const int64_t n_local = row_end - row_begin;
  std::vector<int64_t> remote;
  remote.reserve(1024);
  for (int64_t p = 0; p < nnz; ++p) {
    const int64_t cidx = col_idx[p];
    if (cidx < row_begin || cidx >= row_end) remote.push_back(cidx);
  }
  std::sort(remote.begin(), remote.end());
  remote.erase(std::unique(remote.begin(), remote.end()), remote.end());
  for (int64_t p = 0; p < nnz; ++p) {
    const int64_t cidx = col_idx[p];
    int64_t loc;
    if (cidx >= row_begin && cidx < row_end) {
      loc = cidx - row_begin;
    } else {
      loc = n_local + (std::lower_bound(remote.begin(), remote.end(), cidx) - remote.begin());
    }
    if (loc > INT32_MAX) return LSBA_E_ARG;
    if (col_local) col_local[p] = (int32_t)loc;
  }
  for (int r = 0; r < nranks; ++r) recv_counts[r] = 0;
  for (size_t g = 0; g < remote.size(); ++g) {
    const int64_t cidx = remote[g];
    const int r = (int)(std::upper_bound(part, part + nranks + 1, cidx) - part) - 1;
    if (r < 0 || r >= nranks) return LSBA_E_ARG;
    recv_counts[r]++;
    if (ghost_global) ghost_global[g] = cidx;
  }
  *n_ghost = (int64_t)remote.size();
  return LSBA_OK;
}

// ------------------------------------------------------------------------------------------
// lifecycle
// ------------------------------------------------------------------------------------------
extern "C" const char* lsba_status_str(lsba_status st) {
  switch (st) {
    case LSBA_OK: return "LSBA_OK";
    case LSBA_E_ARG: return "LSBA_E_ARG";
    case LSBA_E_CUDA: return "LSBA_E_CUDA";
    case LSBA_E_NCCL: return "LSBA_E_NCCL";
    case LSBA_E_OOM: return "LSBA_E_OOM";
    case LSBA_E_STATE: return "LSBA_E_STATE";
    case LSBA_E_NUMERIC: return "LSBA_E_NUMERIC";
  }
  return "LSBA_E_UNKNOWN";
}

extern "C" const char* lsba_last_error(lsba_ctx c) { return c ? c->err.c_str() : ""; }

extern "C" lsba_status lsba_get_unique_id(uint8_t id[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!id) return LSBA_E_ARG;
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return LSBA_E_NCCL;
  std::memcpy(id, &u, 128);
  return LSBA_OK;
}

// Every long-lived device buffer of a context comes from here: cudaMalloc, or the caller's
// allocator (lsba_create_with_allocator, e.g. PyTorch's caching allocator).
static lsba_status dalloc_bytes(lsba_ctx c, void** p, size_t bytes) {
  if (c->has_alloc) {
    *p = c->alloc.alloc(bytes, c->device, (void*)c->stream, c->alloc.user);
    if (!*p) return fail(c, LSBA_E_OOM, "caller allocator returned NULL for %zu bytes", bytes);
    c->owned.push_back(*p);
    if ((uintptr_t)*p & 255) return fail(c, LSBA_E_ARG, "caller allocator: buffer not 256-byte aligned");
  } else {
    CK(cudaMalloc(p, bytes));
  }
  c->ws_bytes += (int64_t)bytes;
  return LSBA_OK;
}
template <typename T>
static lsba_status dalloc(lsba_ctx c, T** p, size_t count) {
  return dalloc_bytes(c, (void**)p, std::max<size_t>(count, 1) * sizeof(T));
}

// The persisting-L2 limit is device state shared by every context on the device: reference-
// count it per device, raise it to the largest set-aside any live context asked for, and
// restore the limit found by the first user when the last one releases it.
static std::mutex g_l2_mu;
static int g_l2_users[64];
static size_t g_l2_prev[64], g_l2_cur[64];
static cudaError_t l2_setaside_acquire(int dev, size_t aside) {
  std::lock_guard<std::mutex> lk(g_l2_mu);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (g_l2_users[dev] == 0) {
    cudaError_t e = cudaDeviceGetLimit(&g_l2_prev[dev], cudaLimitPersistingL2CacheSize);
    if (e != cudaSuccess) return e;
    g_l2_cur[dev] = g_l2_prev[dev];
  }
  if (aside > g_l2_cur[dev]) {
    cudaError_t e = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, aside);
    if (e != cudaSuccess) return e;
    g_l2_cur[dev] = aside;
  }
  ++g_l2_users[dev];
  return cudaSuccess;
}
static void l2_setaside_release(int dev) {
  std::lock_guard<std::mutex> lk(g_l2_mu);
  if (dev < 0 || dev >= 64 || g_l2_users[dev] == 0) return;
  if (--g_l2_users[dev] == 0) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, g_l2_prev[dev]);
    g_l2_cur[dev] = g_l2_prev[dev];
  }
}

static void release(lsba_ctx c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->l2win > 0) l2_setaside_release(c->device);   // give the L2 set-aside back
  void* ptrs[] = {c->d_rp, c->d_ci, c->d_V, c->d_ghost, c->d_send_idx, c->d_sendbuf,
                  c->d_part, c->d_Gbase, c->d_small, c->d_Y, c->d_Z, c->d_info, c->d_Xc,
                  c->d_sq, c->d_scalar, c->d_Bh, c->d_Xh, c->st.status, c->st.flag_dev,
                  c->d_gpart, c->d_tickets, c->d_ctl, c->d_zeros, c->st.rscr, c->st.iscr, c->st.upd_done,
                  c->st.Tm, c->st.TmT, c->st.gpip, c->st.Jb, c->d_lu, c->d_diag, c->d_ordL, c->d_lvlL, c->d_lvlU,
                  c->packL.row, c->packL.rest, c->packL.k, c->packL.v, c->packL.piv, c->packU.row,
                  c->packU.rest, c->packU.k, c->packU.v, c->packU.piv,
                  c->d_ordU, c->d_ticket, c->d_ilu_tmp, c->d_rpL, c->d_ciL, c->d_vaL, c->d_rowsG,
                  c->d_rpG, c->d_ciG, c->d_vaG};
  // (the caller's allocator may hand the memory to other work at once: drain our streams first)
  cudaStreamSynchronize(c->stream);
  if (c->stream2) cudaStreamSynchronize(c->stream2);
  if (c->cstream) cudaStreamSynchronize(c->cstream);
  if (c->has_alloc) {
    for (void* p : c->owned) c->alloc.free(p, c->device, (void*)c->stream, c->alloc.user);
  } else {
    for (void* p : ptrs)
      if (p) cudaFree(p);
  }
  if (c->h_status) cudaFreeHost(c->h_status);
  if (c->h_info) cudaFreeHost(c->h_info);
  if (c->h_scalar) cudaFreeHost(c->h_scalar);
  if (c->h_ctl) cudaFreeHost(c->h_ctl);
  if (c->h_prog) cudaFreeHost((void*)c->h_prog);
  if (c->ev_coef) cudaEventDestroy(c->ev_coef);
  if (c->ev_upd) cudaEventDestroy(c->ev_upd);
  if (c->stream2) cudaStreamDestroy(c->stream2);
  if (c->ev_status) cudaEventDestroy(c->ev_status);
  if (c->ev_pack) cudaEventDestroy(c->ev_pack);
  if (c->ev_halo) cudaEventDestroy(c->ev_halo);
  if (c->cstream) cudaStreamDestroy(c->cstream);
  for (int k = 0; k < LSBA_K_COUNT; ++k)
    for (auto& e : c->prof.ev[k]) { cudaEventDestroy(e.a); cudaEventDestroy(e.b); }
  delete c->comm;
}

static lsba_status create_impl(lsba_ctx c, int64_t n, int32_t s, int32_t m_max, const int64_t* row_ptr,
                               const int32_t* col_idx, const double* vals, const uint8_t* nccl_id,
                               LoopGroup* loop) {
  const int64_t n_local = c->row_end - c->row_begin;
  if (n_local > INT32_MAX / 16) return fail(c, LSBA_E_ARG, "n_local too large");
  const char* msg = nullptr;
  if (lsba_csr_validate(n_local, n, row_ptr, col_idx, &msg) != LSBA_OK)
    return fail(c, LSBA_E_ARG, "invalid CSR: %s", msg);
  c->nnz = row_ptr[n_local];
  if (c->nnz > INT32_MAX) return fail(c, LSBA_E_ARG, "local nnz exceeds int32");
  if (vals == nullptr && c->nnz > 0) return fail(c, LSBA_E_ARG, "vals is NULL");
  CK(cudaSetDevice(c->device));
  // ---- communicator (NCCL across processes, the loopback test group, or a one-rank NCCL
  // communicator when LSBA_FORCE_COMM=1 runs the distributed code path on one rank)
  if (loop) {
    auto* lc = new (std::nothrow) LoopComm(loop, c->rank);
    if (!lc) return fail(c, LSBA_E_OOM, "comm");
    c->comm = lc;
    TRYC(lc->init());
  } else if (c->nranks > 1 || c->force_comm) {
    auto* nc = new (std::nothrow) NcclComm();
    if (!nc) return fail(c, LSBA_E_OOM, "comm");
    c->comm = nc;
    c->nccl = nc;
    ncclUniqueId uid;
    if (nccl_id) std::memcpy(&uid, nccl_id, 128);
    else CKN(ncclGetUniqueId(&uid));
    TRYC(nc->init(uid, c->nranks, c->rank));
  }
  bool any_empty = (c->row_end == c->row_begin);
  // ---- ghost plan
  std::vector<int32_t> col_local(c->nnz);
  std::vector<int64_t> ghost_global;
  c->send_cnt.assign(c->nranks, 0);
  c->recv_cnt.assign(c->nranks, 0);
  c->send_off.assign(c->nranks, 0);
  c->recv_off.assign(c->nranks, 0);
  std::vector<int64_t> send_idx;
  if (c->nranks == 1) {
    for (int64_t p = 0; p < c->nnz; ++p) col_local[p] = col_idx[p];
  } else {
    // partition starts
    int64_t* d_tmp = nullptr;
    CK(cudaMalloc((void**)&d_tmp, sizeof(int64_t) * (2 * c->nranks + 2 * (size_t)c->nranks * c->nranks + 2)));
    int64_t mine[2] = {c->row_begin, c->row_end};
    CK(cudaMemcpy(d_tmp, mine, sizeof mine, cudaMemcpyHostToDevice));
    TRYC(c->comm->allgather_i64(d_tmp, d_tmp + 2, 2, c->stream));
    std::vector<int64_t> rr(2 * c->nranks);
    CK(cudaMemcpyAsync(rr.data(), d_tmp + 2, sizeof(int64_t) * 2 * c->nranks, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    std::vector<int64_t> part(c->nranks + 1);
    for (int r = 0; r < c->nranks; ++r) {
      part[r] = rr[2 * r];
      if (r > 0 && rr[2 * r] != rr[2 * r - 1]) { cudaFree(d_tmp); return fail(c, LSBA_E_ARG, "row ranges not contiguous"); }
    }
    part[c->nranks] = rr[2 * c->nranks - 1];
    for (int r = 0; r < c->nranks; ++r) any_empty = any_empty || rr[2 * r + 1] == rr[2 * r];
    if (part[0] != 0 || part[c->nranks] != n) { cudaFree(d_tmp); return fail(c, LSBA_E_ARG, "row ranges do not cover [0,n)"); }
    ghost_global.resize(std::max<int64_t>(c->nnz, 1));
    int64_t ng = 0;
    if (lsba_ghost_plan(c->row_begin, c->row_end, col_idx, c->nnz, part.data(), c->nranks,
                        col_local.data(), ghost_global.data(), &ng, c->recv_cnt.data()) != LSBA_OK) {
      cudaFree(d_tmp);
      return fail(c, LSBA_E_ARG, "ghost plan failed");
    }
    ghost_global.resize(ng);
    c->n_ghost = (int)ng;
    // everyone's recv counts -> my send counts
    int64_t* d_cnt = d_tmp + 2 * c->nranks + 2;
    CK(cudaMemcpy(d_cnt, c->recv_cnt.data(), sizeof(int64_t) * c->nranks, cudaMemcpyHostToDevice));
    TRYC(c->comm->allgather_i64(d_cnt, d_cnt + c->nranks, c->nranks, c->stream));
    std::vector<int64_t> allc((size_t)c->nranks * c->nranks);
    CK(cudaMemcpyAsync(allc.data(), d_cnt + c->nranks, sizeof(int64_t) * allc.size(), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    int64_t so = 0, ro = 0;
    for (int r = 0; r < c->nranks; ++r) {
      c->send_cnt[r] = (r == c->rank) ? 0 : allc[(size_t)r * c->nranks + c->rank];
      c->send_off[r] = so;
      so += c->send_cnt[r];
      c->recv_off[r] = ro;
      ro += c->recv_cnt[r];
    }
    c->n_send = so;
    CK(cudaFree(d_tmp));
    // exchange the requested global row lists
    int64_t *d_req = nullptr, *d_want = nullptr;
    CK(cudaMalloc((void**)&d_req, sizeof(int64_t) * std::max<int64_t>(ng, 1)));
    CK(cudaMalloc((void**)&d_want, sizeof(int64_t) * std::max<int64_t>(so, 1)));
    if (ng) CK(cudaMemcpy(d_req, ghost_global.data(), sizeof(int64_t) * ng, cudaMemcpyHostToDevice));
    std::vector<P2POp> ops;
    for (int r = 0; r < c->nranks; ++r) {
      if (r == c->rank || (c->recv_cnt[r] == 0 && c->send_cnt[r] == 0)) continue;
      ops.push_back({r, d_req + c->recv_off[r], sizeof(int64_t) * (size_t)c->recv_cnt[r],
                     d_want + c->send_off[r], sizeof(int64_t) * (size_t)c->send_cnt[r]});
    }
    TRYC(c->comm->exchange(ops, c->stream));
    send_idx.resize(std::max<int64_t>(so, 1));
    CK(cudaMemcpyAsync(send_idx.data(), d_want, sizeof(int64_t) * std::max<int64_t>(so, 1), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    cudaFree(d_req);
    cudaFree(d_want);
    for (int64_t i = 0; i < so; ++i) {
      send_idx[i] -= c->row_begin;
      if (send_idx[i] < 0 || send_idx[i] >= n_local) return fail(c, LSBA_E_ARG, "peer requested a row this rank does not own");
    }
    // the interior block: first and last row without ghost columns; used only if every row
    // between them is ghost-free too (z-slabs of a stencil: all but the boundary planes)
    auto ghost_row = [&](int64_t r) {
      for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p)
        if (col_local[p] >= n_local) return true;
      return false;
    };
    int64_t b0 = 0, b1 = n_local;
    while (b0 < n_local && ghost_row(b0)) ++b0;
    while (b1 > b0 && ghost_row(b1 - 1)) --b1;
    bool clean = b1 - b0 >= 256;
    for (int64_t r = b0; clean && r < b1; ++r) clean = !ghost_row(r);
    if (clean) { c->int0 = (int)b0; c->int1 = (int)b1; }
  }
  // f2: the device-API Gram allreduce (collective; every rank takes the same decision from the
  // replicated partition): two window slots of the largest fused Gram ((m_max+1) s^2 doubles).
  // A rank without rows would not run the Gram kernel, so then the plain allreduce stays.
  if (c->nccl && c->devar_req && !any_empty) {
    c->ar_slot = ((size_t)(m_max + 2) * s * s * sizeof(double) + 255) / 256 * 256;
    TRYC(c->nccl->init_devar(2 * c->ar_slot));
  }
  // ---- device CSR
  std::vector<int32_t> rp32(n_local + 1);
  for (int64_t i = 0; i <= n_local; ++i) rp32[i] = (int32_t)row_ptr[i];
  TRY(dalloc(c, &c->d_rp, n_local + 1));
  {  // column indices and values in one allocation: one L2 access-policy window covers both
    const size_t ci_bytes = ((std::max<int64_t>(c->nnz, 1) * sizeof(int32_t)) + 255) / 256 * 256;
    const size_t bytes = ci_bytes + std::max<int64_t>(c->nnz, 1) * sizeof(double);
    char* base = nullptr;
    TRY(dalloc_bytes(c, (void**)&base, bytes));
    c->d_ci = reinterpret_cast<int*>(base);
    c->d_va = reinterpret_cast<double*>(base + ci_bytes);
    c->csr_bytes = bytes;
  }
  CK(cudaMemcpy(c->d_rp, rp32.data(), sizeof(int32_t) * (n_local + 1), cudaMemcpyHostToDevice));
  if (c->nnz) {
    CK(cudaMemcpy(c->d_ci, col_local.data(), sizeof(int32_t) * c->nnz, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(c->d_va, vals, sizeof(double) * c->nnz, cudaMemcpyHostToDevice));
  }
  if (c->comm && c->halo_ovl && c->int1 <= c->int0 && c->n_ghost > 0) {
    // local / ghost split of the local rows (overlap config 4's ghost
    // exchange with the band part of the SpMM)
    std::vector<int32_t> rpL(n_local + 1, 0), ciL, rowsG, rpG(1, 0), ciG;
    std::vector<double> vaL, vaG;
    ciL.reserve(c->nnz);
    vaL.reserve(c->nnz);
    for (int64_t r = 0; r < n_local; ++r) {
      bool has_g = false;
      for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
        if (col_local[p] < n_local) {
          ciL.push_back(col_local[p]);
          vaL.push_back(vals[p]);
        } else {
          ciG.push_back((int32_t)(col_local[p] - n_local));
          vaG.push_back(vals[p]);
          has_g = true;
        }
      }
      rpL[r + 1] = (int32_t)ciL.size();
      if (has_g) {
        rowsG.push_back((int32_t)r);
        rpG.push_back((int32_t)ciG.size());
      }
    }
    c->ng_rows = (int)rowsG.size();
    TRY(dalloc(c, &c->d_rpL, n_local + 1));
    TRY(dalloc(c, &c->d_ciL, ciL.size()));
    TRY(dalloc(c, &c->d_vaL, vaL.size()));
    TRY(dalloc(c, &c->d_rowsG, rowsG.size()));
    TRY(dalloc(c, &c->d_rpG, rpG.size()));
    TRY(dalloc(c, &c->d_ciG, ciG.size()));
    TRY(dalloc(c, &c->d_vaG, vaG.size()));
    CK(cudaMemcpy(c->d_rpL, rpL.data(), sizeof(int32_t) * rpL.size(), cudaMemcpyHostToDevice));
    if (!ciL.empty()) {
      CK(cudaMemcpy(c->d_ciL, ciL.data(), sizeof(int32_t) * ciL.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->d_vaL, vaL.data(), sizeof(double) * vaL.size(), cudaMemcpyHostToDevice));
    }
    if (!rowsG.empty()) {
      CK(cudaMemcpy(c->d_rowsG, rowsG.data(), sizeof(int32_t) * rowsG.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->d_rpG, rpG.data(), sizeof(int32_t) * rpG.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->d_ciG, ciG.data(), sizeof(int32_t) * ciG.size(), cudaMemcpyHostToDevice));
      CK(cudaMemcpy(c->d_vaG, vaG.data(), sizeof(double) * vaG.size(), cudaMemcpyHostToDevice));
    }
    c->split = true;
  }
  if (c->l2persist != 0 && c->nnz > 0 && !c->comm) {
    // The SpMM's column indices and values (constant across the solve) are kept in an L2
    // set-aside when they fit: config 2 (63 MB) +4%; a CSR larger than the set-aside (config 3,
    // 175 MB) lost 3.5% (tools/l2persist_exp.sh), so "auto" requires it to fit in the set-aside
    // and in half of L2.
    int max_win = 0, max_persist = 0, l2 = 0;
    CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, c->device));
    CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, c->device));
    const bool fits = c->csr_bytes <= (size_t)max_win && c->csr_bytes <= (size_t)max_persist &&
                      c->csr_bytes <= (size_t)l2 / 2;
    if (c->l2persist < 0 && !fits) c->l2persist = 0;
  }
  if (c->l2persist != 0 && c->nnz > 0 && !c->comm) {
    int max_win = 0, max_persist = 0;
    CK(cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, c->device));
    CK(cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, c->device));
    // (LSBA_L2PERSIST=2: the column indices only)
    const size_t want = (c->l2persist == 2) ? (size_t)((char*)c->d_va - (char*)c->d_ci) : c->csr_bytes;
    c->l2win = std::min<size_t>(want, (size_t)max_win);
    const size_t aside = std::min<size_t>(c->l2win, (size_t)max_persist);
    if (aside > 0) {
      CK(l2_setaside_acquire(c->device, aside));
      c->l2hit = (float)std::min(1.0, (double)aside / (double)c->l2win);
    } else {
      c->l2win = 0;
    }
  }
  if (c->nranks > 1) {
    TRY(dalloc(c, &c->d_ghost, (size_t)c->n_ghost * s));
    TRY(dalloc(c, &c->d_sendbuf, (size_t)c->n_send * s));
    TRY(dalloc(c, &c->d_send_idx, c->n_send));
    std::vector<int32_t> si(std::max<int64_t>(c->n_send, 1));
    for (int64_t i = 0; i < c->n_send; ++i) si[i] = (int32_t)send_idx[i];
    if (c->n_send) CK(cudaMemcpy(c->d_send_idx, si.data(), sizeof(int32_t) * c->n_send, cudaMemcpyHostToDevice));
  }
  // ---- basis and work buffers
  c->slot = (size_t)n_local * s;
  c->slot_stride = (size_t)((n_local + kRowPad - 1) / kRowPad) * kRowPad * s;
  // m_max + 2 slots: V_1..V_{m+1} plus W of the last step of a BMGS-(I)CWY cycle (Alg 6 applies
  // A to the unnormalised V_{k+1} one slot ahead)
  TRY(dalloc(c, &c->d_V, (size_t)(m_max + 2) * c->slot_stride));
  CK(cudaMemset(c->d_V, 0, sizeof(double) * (size_t)(m_max + 2) * c->slot_stride));   // zero pad rows
  TRY(dalloc(c, &c->d_zeros, 64));
  CK(cudaMemset(c->d_zeros, 0, sizeof(double) * 64));
  TRY(dalloc(c, &c->d_Xc, c->slot));
  {
    int sms = 148;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device) == cudaSuccess && sms > 0)
      c->n_sms = sms;
  }
  if (c->spmm_pf < 0) {
    // the L2 bulk prefetch helps banded / stencil matrices (standalone: configs 2, 3 -8..-10%
    // time at 2 x #SMs CTAs ahead, config 5 neutral) and hurts matrices whose gathers reach far
    // (config 4's uniform-random columns: +7..12%): off when > 10% of the entries lie more than
    // 2^20 rows from the diagonal (profiles/r02_spmm_q256_raw.txt)
    int64_t far = 0;
    for (int64_t r = 0; r < n_local; ++r)
      for (int64_t p = row_ptr[r]; p < row_ptr[r + 1]; ++p) {
        const int64_t d = (int64_t)col_idx[p] - (c->row_begin + r);
        far += (d > (1 << 20) || d < -(1 << 20)) ? 1 : 0;
      }
    c->spmm_pf = (c->nnz > 0 && far * 10 > c->nnz) ? 0 : 2 * c->n_sms;
  }
  // DMMA Gram: persistent grid of 2 CTAs per SM; partials [cta][E] and [group][E]
  c->gram_grid = 4 * c->n_sms;
  const size_t Emax = 2 * (size_t)(m_max + 2) * s * s;      // (k+1)s x 2s for BMGS-(I)CWY
  c->part_cap = std::max((size_t)(kGramCtas + 16 * (m_max + 1)) * s * s + 2 * Emax,
                         (size_t)c->gram_grid * Emax);
  TRY(dalloc(c, &c->d_part, c->part_cap));
  {
    const int ngroups = (c->gram_grid + kGramGroup - 1) / kGramGroup;
    TRY(dalloc(c, &c->d_gpart, (size_t)ngroups * Emax));
    TRY(dalloc(c, &c->d_tickets, (size_t)(kMaxGramPasses + 1) * (ngroups + 1)));
    CK(cudaMemset(c->d_tickets, 0, sizeof(unsigned) * (kMaxGramPasses + 1) * (ngroups + 1)));
  }
  TRY(dalloc(c, &c->d_ctl, 1));
  CK(cudaMemset(c->d_ctl, 0, sizeof(CycleCtl)));
  CK(cudaMallocHost((void**)&c->h_ctl, sizeof(CycleCtl)));
  c->g_half = Emax;
  TRY(dalloc(c, &c->d_Gbase, 2 * c->g_half));
  c->d_G = c->d_Gbase;
  c->sq_cap = std::max(1, cdiv((long)n_local * 16, kThreads));
  TRY(dalloc(c, &c->d_sq, c->sq_cap));
  TRY(dalloc(c, &c->d_scalar, 4));
  // ---- small state (sized for b = s)
  const int ldH = (m_max + 1) * s;
  const size_t nH = (size_t)ldH * m_max * s, nBeta = (size_t)s * s, nCoef = 2 * (size_t)(m_max + 2) * s * s,
               nQv = (size_t)m_max * s * 2 * s, nQt = (size_t)m_max * s, nG = (size_t)ldH * s,
               nRf = (size_t)ldH * ldH, nHt = (size_t)m_max * s * s, nGh = (size_t)m_max * s * s,
               nRi = (size_t)ldH * ldH, nSc = 4, nCacc = (size_t)s * s;
  const size_t total = nH + nBeta + nCoef + nQv + nQt + nG + nRf + nHt + nGh + nRi + nSc + nCacc;
  TRY(dalloc(c, &c->d_small, total));
  CK(cudaMemset(c->d_small, 0, sizeof(double) * total));
  double* q = c->d_small;
  c->st.Hbar = q; q += nH;
  c->st.beta = q; q += nBeta;
  c->st.coef = q; q += nCoef;
  c->st.qr_v = q; q += nQv;
  c->st.qr_tau = q; q += nQt;
  c->st.g = q; q += nG;
  c->st.Rfac = q; q += nRf;
  c->st.htil = q; q += nHt;
  c->st.ghat = q; q += nGh;
  c->st.Rinv = q; q += nRi;
  c->st.sc = q; q += nSc;
  c->st.Cacc = q; q += nCacc;
  c->st.ldH = ldH;
  c->st.m = m_max;
  c->st.bmax = s;
  TRY(dalloc(c, &c->st.Tm, (size_t)ldH * ldH));
  TRY(dalloc(c, &c->st.TmT, (size_t)ldH * ldH));
  TRY(dalloc(c, &c->st.gpip, (size_t)ldH * s));
  TRY(dalloc(c, &c->st.Jb, (size_t)ldH * s));
  c->st.ctl = c->d_ctl;
  {  // progress word in mapped pinned host memory (written by the device, polled by the host)
    CK(cudaHostAlloc((void**)&c->h_prog, 2 * sizeof(int), cudaHostAllocMapped));
    c->h_prog[0] = -1;
    int* dp = nullptr;
    CK(cudaHostGetDevicePointer((void**)&dp, (void*)c->h_prog, 0));
    c->st.prog = dp;
  }
  TRY(dalloc(c, &c->st.rscr, 2 * (size_t)s * s));
  TRY(dalloc(c, &c->st.iscr, 4));
  TRY(dalloc(c, &c->st.upd_done, 1));
  CK(cudaMemset(c->st.upd_done, 0, sizeof(unsigned)));
  c->st.upd_seq = 0;
  {  // the update kernel's single CTA should get an SM as soon as one frees up
    int lo = 0, hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CK(cudaStreamCreateWithPriority(&c->stream2, cudaStreamNonBlocking, hi));
  }
  CK(cudaEventCreateWithFlags(&c->ev_coef, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_upd, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_status, cudaEventDisableTiming));
  if (c->comm) {
    CK(cudaStreamCreateWithFlags(&c->cstream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&c->ev_pack, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
  }
  TRY(dalloc(c, &c->st.status, 1));
  TRY(dalloc(c, &c->st.flag_dev, 1));
  CK(cudaMemset(c->st.flag_dev, 0, sizeof(int)));
  TRY(dalloc(c, &c->d_Y, (size_t)(m_max + 1) * s * s));
  TRY(dalloc(c, &c->d_Z, (size_t)(m_max + 1) * s * s));
  TRY(dalloc(c, &c->d_info, 8));
  CK(cudaMallocHost((void**)&c->h_status, sizeof(StepStatus)));
  CK(cudaMallocHost((void**)&c->h_info, sizeof(int) * 8));
  CK(cudaMallocHost((void**)&c->h_scalar, sizeof(double) * 4));
  set_ip(c, LSBA_IP_CLASSICAL);
  return LSBA_OK;
}

static lsba_status create_any(lsba_ctx* out, int64_t n, int32_t s, int32_t m_max,
                              const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                              int64_t row_begin, int64_t row_end, int32_t rank, int32_t nranks,
                              const uint8_t* nccl_id, LoopGroup* loop, int32_t device, void* cuda_stream,
                              const lsba_allocator* allocator = nullptr) {
  if (!out) return LSBA_E_ARG;
  *out = nullptr;
  lsba_ctx c = new (std::nothrow) lsba_ctx_();
  if (!c) return LSBA_E_OOM;
  *out = c;  // returned even on failure so that lsba_last_error works; destroy it
  if (const char* e = std::getenv("LSBA_NO_FUSE")) c->no_fuse = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_PDL")) c->pdl = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_G7")) c->g7force = std::atoi(e);
  if (const char* e = std::getenv("LSBA_UPD_MAIN")) c->upd_main = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_DEVJOIN")) c->devjoin = std::atoi(e);
  if (const char* e = std::getenv("LSBA_PDL_PROJ")) c->pdl_proj = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_L2PERSIST")) c->l2persist = std::atoi(e);
  if (const char* e = std::getenv("LSBA_SPEC_END")) c->spec_end = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_SPMM_PF")) c->spmm_pf = std::atoi(e);
  if (const char* e = std::getenv("LSBA_SPMM_PFV")) c->spmm_pfv = std::atoi(e);
  if (const char* e = std::getenv("LSBA_SPMM_LANES16")) c->spmm_lanes16 = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_PROJ_DFMA")) c->proj_dfma = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_PROJ_PF_MB")) c->proj_pf = std::atol(e) << 20;
  if (const char* e = std::getenv("LSBA_GRAM_PF_MB")) c->gram_pf = std::atol(e) << 20;
  if (const char* e = std::getenv("LSBA_ILU_CTAS")) c->ilu_ctas = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("LSBA_ILU_BACKOFF")) c->ilu_backoff = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("LSBA_ILU_SOLVE")) c->ilu_solve = std::atoi(e);
  if (const char* e = std::getenv("LSBA_FORCE_COMM")) c->force_comm = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_HALO_OVERLAP")) c->halo_ovl = (e[0] == '1');
  if (const char* e = std::getenv("LSBA_DEVAR")) c->devar_req = (e[0] == '1');
  if (n < 1 || s < 1 || s > 16 || m_max < 1) return fail(c, LSBA_E_ARG, "need n >= 1, 1 <= s <= 16, m_max >= 1");
  if (n < s) return fail(c, LSBA_E_ARG, "n < s");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(c, LSBA_E_ARG, "bad rank/nranks");
  if (row_begin < 0 || row_end < row_begin || row_end > n) return fail(c, LSBA_E_ARG, "bad row range");
  if (nranks == 1 && (row_begin != 0 || row_end != n)) return fail(c, LSBA_E_ARG, "nranks == 1 needs rows [0, n)");
  if (nranks > 1 && !nccl_id && !loop) return fail(c, LSBA_E_ARG, "nccl_id required when nranks > 1");
  if (loop && loop->P != nranks) return fail(c, LSBA_E_ARG, "loopback group size != nranks");
  if (!row_ptr || (!col_idx && row_end > row_begin)) return fail(c, LSBA_E_ARG, "CSR arrays NULL");
  c->device = device;
  c->stream = (cudaStream_t)cuda_stream;
  if (allocator) {
    if (!allocator->alloc || !allocator->free) return fail(c, LSBA_E_ARG, "allocator without alloc/free");
    c->alloc = *allocator;
    c->has_alloc = true;
  }
  c->n_global = n;
  c->row_begin = row_begin;
  c->row_end = row_end;
  c->n = (int)(row_end - row_begin);
  c->s = s;
  c->m_max = m_max;
  c->rank = rank;
  c->nranks = nranks;
  return create_impl(c, n, s, m_max, row_ptr, col_idx, vals, nccl_id, loop);
}

extern "C" lsba_status lsba_create(lsba_ctx* out, int64_t n, int32_t s, int32_t m_max,
                                   const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                                   int64_t row_begin, int64_t row_end, int32_t rank, int32_t nranks,
                                   const uint8_t* nccl_id, int32_t device, void* cuda_stream) {
  return create_any(out, n, s, m_max, row_ptr, col_idx, vals, row_begin, row_end, rank, nranks, nccl_id,
                    nullptr, device, cuda_stream);
}

extern "C" lsba_status lsba_create_with_allocator(lsba_ctx* out, int64_t n, int32_t s, int32_t m_max,
                                                  const int64_t* row_ptr, const int32_t* col_idx,
                                                  const double* vals, int64_t row_begin, int64_t row_end,
                                                  int32_t rank, int32_t nranks, const uint8_t* nccl_id,
                                                  int32_t device, void* cuda_stream,
                                                  const lsba_allocator* allocator) {
  if (!allocator) return LSBA_E_ARG;
  return create_any(out, n, s, m_max, row_ptr, col_idx, vals, row_begin, row_end, rank, nranks, nccl_id,
                    nullptr, device, cuda_stream, allocator);
}

struct lsba_loopback_ {
  LoopGroup g;
  explicit lsba_loopback_(int P) : g(P) {}
};

extern "C" lsba_status lsba_loopback_create(int32_t nranks, lsba_loopback* out) {
  if (!out || nranks < 1 || nranks > kLoopMaxRanks) return LSBA_E_ARG;
  *out = new (std::nothrow) lsba_loopback_(nranks);
  return *out ? LSBA_OK : LSBA_E_OOM;
}

extern "C" lsba_status lsba_loopback_destroy(lsba_loopback g) {
  delete g;
  return LSBA_OK;
}

extern "C" lsba_status lsba_create_loopback(lsba_ctx* out, int64_t n, int32_t s, int32_t m_max,
                                            const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                                            int64_t row_begin, int64_t row_end, int32_t rank, int32_t nranks,
                                            lsba_loopback group, int32_t device, void* cuda_stream) {
  if (!group) return LSBA_E_ARG;
  return create_any(out, n, s, m_max, row_ptr, col_idx, vals, row_begin, row_end, rank, nranks, nullptr,
                    &group->g, device, cuda_stream);
}

extern "C" lsba_status lsba_destroy(lsba_ctx c) {
  if (!c) return LSBA_OK;
  release(c);
  delete c;
  return LSBA_OK;
}

// ------------------------------------------------------------------------------------------
// step API
// ------------------------------------------------------------------------------------------
extern "C" lsba_status lsba_arnoldi_begin(lsba_ctx c, const double* B_dev, lsba_ip ip, int32_t* io_flag) {
  if (!c) return LSBA_E_ARG;
  if (ip != LSBA_IP_CLASSICAL && ip != LSBA_IP_GLOBAL) return fail(c, LSBA_E_ARG, "bad inner product");
  if (c->n > 0 && !B_dev) return fail(c, LSBA_E_ARG, "B is NULL");
  if ((uintptr_t)B_dev & 15) return fail(c, LSBA_E_ARG, "B not 16-byte aligned");
  CK(cudaSetDevice(c->device));
  set_ip(c, ip);
  if (c->n > 0)
    CK(cudaMemcpyAsync(slotp(c, 0), B_dev, sizeof(double) * c->slot, cudaMemcpyDeviceToDevice, c->stream));
  TRY(set_identity(c));
  CycleParams prm;
  prm.m_cur = c->m_max;
  prm.gmres = 1;
  prm.force_k = c->force_flag_k;
  prm.reset_forced = 1;
  prm.tol_abs = -1.0;            // the step API never declares convergence
  prm.tau = INFINITY;
  prm.need_kappa = 1;
  c->skel = c->skel_default;
  TRY(io_begin_async(c, prm));
  if (lagged(c->skel))
    TRY(cwy_iter1_async(c));                                       // Alg 6 loop iteration 1
  StepStatus stt;
  TRY(read_status(c, &stt, nullptr));
  if (io_flag) *io_flag = stt.flag;
  c->k = stt.flag ? -1 : 0;
  c->flagged = false;
  return LSBA_OK;
}

extern "C" lsba_status lsba_block_arnoldi_step(lsba_ctx c, lsba_step_info* info) {
  if (!c) return LSBA_E_ARG;
  if (c->k < 0 || c->flagged) return fail(c, LSBA_E_STATE, "no active Arnoldi process (begin first; a flag ends it)");
  if (c->k >= c->m_max) return fail(c, LSBA_E_STATE, "basis full (k == m_max)");
  CK(cudaSetDevice(c->device));
  const int k = c->k + 1;
  TRY(step_async(c, k, k == c->m_max));
  TRY(join_update(c));
  StepStatus stt;
  CycleCtl cc;
  TRY(read_status(c, &stt, &cc));
  const bool flagged = (cc.why == 1 && cc.k_flag == k);
  if (flagged) c->flagged = true;
  else c->k = k;
  if (info) {
    info->k = k;
    info->chol_flag = stt.flag;
    info->cond_est = stt.kappa_F;
    info->res_est = stt.res_gmres;
    info->res_est_fom = stt.res_fom;
    info->proj_singular = stt.proj_singular;
  }
  return LSBA_OK;
}

extern "C" lsba_status lsba_projected_solve(lsba_ctx c, int32_t fom, double* Xi_host, double* Z_host) {
  if (!c || !Xi_host || !Z_host) return LSBA_E_ARG;
  if (c->k < 1 || c->flagged) return fail(c, LSBA_E_STATE, "needs k >= 1 accepted steps and no flag");
  CK(cudaSetDevice(c->device));
  int sing = 0;
  TRY(cycle_solve(c, c->k, fom ? 0 : 1, 0, &sing, 0));
  const int kb = c->k * c->b;
  CK(cudaMemcpyAsync(Xi_host, c->d_Y, sizeof(double) * kb * c->b, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(Z_host, c->d_Z, sizeof(double) * (kb + c->b) * c->b, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return sing ? fail(c, LSBA_OK, "singular projected system") : LSBA_OK;
}

extern "C" lsba_status lsba_copy_hessenberg(lsba_ctx c, double* H_host, int32_t ld) {
  if (!c || !H_host) return LSBA_E_ARG;
  if (c->k < 0) return fail(c, LSBA_E_STATE, "no Arnoldi process");
  const int ncol = (c->k + (c->flagged ? 1 : 0)) * c->b;
  const int nrow = ncol + c->b;
  if (ld < nrow) return fail(c, LSBA_E_ARG, "ld < (k+1)b");
  if (ncol == 0) return LSBA_OK;
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpy2DAsync(H_host, sizeof(double) * ld, c->st.Hbar, sizeof(double) * c->st.ldH,
                       sizeof(double) * nrow, ncol, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

extern "C" lsba_status lsba_copy_beta(lsba_ctx c, double* beta_host) {
  if (!c || !beta_host) return LSBA_E_ARG;
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(beta_host, c->st.beta, sizeof(double) * c->b * c->b, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

extern "C" lsba_status lsba_copy_basis_block(lsba_ctx c, int32_t j, double* dst_dev) {
  if (!c) return LSBA_E_ARG;
  if (c->k < 0) return fail(c, LSBA_E_STATE, "no Arnoldi process");
  if (j < 1 || j > c->k + 1) return fail(c, LSBA_E_ARG, "j outside [1, k+1]");
  if (c->n == 0) return LSBA_OK;
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(dst_dev, slotp(c, j - 1), sizeof(double) * c->slot, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

// ------------------------------------------------------------------------------------------
// solvers
// ------------------------------------------------------------------------------------------
extern "C" lsba_status lsba_bgmres_solve(lsba_ctx c, const double* B, double* X, int32_t m, double tol,
                                         int32_t max_restarts, lsba_skel skel, lsba_ip ip,
                                         double cond_threshold, lsba_solve_info* info) {
  if (!c) return LSBA_E_ARG;
  return solve_impl(c, B, X, m, tol, max_restarts, 1, ip, cond_threshold, info, skel);
}

extern "C" lsba_status lsba_bfom_solve(lsba_ctx c, const double* B, double* X, int32_t m, double tol,
                                       int32_t max_restarts, lsba_skel skel, lsba_ip ip,
                                       double cond_threshold, lsba_solve_info* info) {
  if (!c) return LSBA_E_ARG;
  return solve_impl(c, B, X, m, tol, max_restarts, 0, ip, cond_threshold, info, skel);
}

extern "C" lsba_status lsba_solve_host(lsba_ctx c, const double* B_host, double* X_host, int32_t m,
                                       double tol, int32_t max_restarts, int32_t fom, lsba_ip ip,
                                       double cond_threshold, lsba_solve_info* info) {
  if (!c) return LSBA_E_ARG;
  if (c->n > 0 && (!B_host || !X_host)) return fail(c, LSBA_E_ARG, "B/X NULL");
  CK(cudaSetDevice(c->device));
  if (!c->d_Bh) {
    TRY(dalloc(c, &c->d_Bh, c->slot));
    TRY(dalloc(c, &c->d_Xh, c->slot));
  }
  const auto t0 = std::chrono::steady_clock::now();
  if (c->n > 0) {
    CK(cudaMemcpyAsync(c->d_Bh, B_host, sizeof(double) * c->slot, cudaMemcpyHostToDevice, c->stream));
    CK(cudaMemcpyAsync(c->d_Xh, X_host, sizeof(double) * c->slot, cudaMemcpyHostToDevice, c->stream));
  }
  TRY(solve_impl(c, c->d_Bh, c->d_Xh, m, tol, max_restarts, fom ? 0 : 1, ip, cond_threshold, info,
                 c->skel_default));
  if (c->n > 0)
    CK(cudaMemcpyAsync(X_host, c->d_Xh, sizeof(double) * c->slot, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  info->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return LSBA_OK;
}

// ------------------------------------------------------------------------------------------
// single kernels, debug and measurement
// ------------------------------------------------------------------------------------------
extern "C" lsba_status lsba_spmm(lsba_ctx c, const double* V_dev, double* W_dev) {
  if (!c) return LSBA_E_ARG;
  if (c->n > 0 && (!V_dev || !W_dev || V_dev == W_dev)) return fail(c, LSBA_E_ARG, "V/W NULL or aliased");
  if (((uintptr_t)V_dev | (uintptr_t)W_dev) & 15) return fail(c, LSBA_E_ARG, "V/W not 16-byte aligned");
  CK(cudaSetDevice(c->device));
  const bool prec = c->prec;   // lsba_spmm is the plain operator A V (a1), never M^{-1} A V
  c->prec = false;
  const lsba_status st = (c->n > 0) ? spmm(c, V_dev, W_dev) : LSBA_OK;
  c->prec = prec;
  TRY(st);
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

// ---------------------------------------------------------------- f4: ILU(0) setup / apply
static lsba_status ilu0_factor(lsba_ctx c) {
  const int n = c->n;
  std::vector<int32_t> rp(n + 1), ci(std::max<int64_t>(c->nnz, 1));
  CK(cudaMemcpy(rp.data(), c->d_rp, sizeof(int32_t) * (n + 1), cudaMemcpyDeviceToHost));
  if (c->nnz) CK(cudaMemcpy(ci.data(), c->d_ci, sizeof(int32_t) * c->nnz, cudaMemcpyDeviceToHost));
  std::vector<int32_t> diag(std::max(n, 1), -1), levL(std::max(n, 1), 0), levU(std::max(n, 1), 0);
  for (int i = 0; i < n; ++i)
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] == i) diag[i] = p;
  for (int i = 0; i < n; ++i)
    if (diag[i] < 0) return fail(c, LSBA_E_NUMERIC, "ILU(0): structurally missing diagonal in local row %d", i);
  // level sets (host graph analysis): L row i after every k < i of its row, U row i after j > i
  int nlL = 0, nlU = 0;
  for (int i = 0; i < n; ++i) {
    int l = 0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] < i) l = std::max(l, levL[ci[p]] + 1);
    levL[i] = l;
    nlL = std::max(nlL, l + 1);
  }
  for (int i = n - 1; i >= 0; --i) {
    int l = 0;
    for (int p = rp[i]; p < rp[i + 1]; ++p)
      if (ci[p] > i && ci[p] < n) l = std::max(l, levU[ci[p]] + 1);
    levU[i] = l;
    nlU = std::max(nlU, l + 1);
  }
  auto order_by = [&](const std::vector<int32_t>& lev, int nl, std::vector<int32_t>& ord, std::vector<int32_t>& ptr) {
    ptr.assign(nl + 1, 0);
    for (int i = 0; i < n; ++i) ptr[lev[i] + 1]++;
    for (int l = 0; l < nl; ++l) ptr[l + 1] += ptr[l];
    std::vector<int32_t> pos(ptr.begin(), ptr.end() - 1);
    ord.assign(std::max(n, 1), 0);
    for (int i = 0; i < n; ++i) ord[pos[lev[i]]++] = i;     // ascending rows within a level
  };
  std::vector<int32_t> ordL, ptrL, ordU, ptrU;
  order_by(levL, nlL, ordL, ptrL);
  order_by(levU, nlU, ordU, ptrU);
  if (!c->d_lu) {
    TRY(dalloc(c, &c->d_lu, c->nnz));
    TRY(dalloc(c, &c->d_diag, n));
    TRY(dalloc(c, &c->d_ordL, n));
    TRY(dalloc(c, &c->d_ordU, n));
    TRY(dalloc(c, &c->d_lvlL, (size_t)nlL + 1));
    TRY(dalloc(c, &c->d_lvlU, (size_t)nlU + 1));
    for (IluPack* pk : {&c->packL, &c->packU}) {
      TRY(dalloc(c, &pk->row, n));
      TRY(dalloc(c, &pk->rest, n));
      TRY(dalloc(c, &pk->k, (size_t)kIluW * n));
      TRY(dalloc(c, &pk->v, (size_t)kIluW * n));
      TRY(dalloc(c, &pk->piv, n));
    }
    TRY(dalloc(c, &c->d_ticket, 8));
    TRY(dalloc(c, &c->d_ilu_tmp, (size_t)n * c->s));
  }
  CK(cudaMemcpy(c->d_diag, diag.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_ordL, ordL.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_ordU, ordU.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_lvlL, ptrL.data(), sizeof(int32_t) * (nlL + 1), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(c->d_lvlU, ptrU.data(), sizeof(int32_t) * (nlU + 1), cudaMemcpyHostToDevice));
  CK(cudaMemset(c->d_ticket, 0, sizeof(unsigned) * 8));
  if (c->nnz) CK(cudaMemcpy(c->d_lu, c->d_va, sizeof(double) * c->nnz, cudaMemcpyDeviceToDevice));
  CK(cudaMemsetAsync(c->d_info, 0, sizeof(int), c->stream));
  for (int l = 0; l < nlL; ++l) {          // one launch per level of L (setup only)
    const int cnt = ptrL[l + 1] - ptrL[l];
    LaunchScope Ls(c, LSBA_K_MISC, 0.0);
    k_ilu0_level<<<cdiv((long)cnt * 32, kThreads), kThreads, 0, c->stream>>>(
        cnt, c->d_ordL + ptrL[l], c->d_rp, c->d_ci, c->d_diag, n, c->d_lu, c->d_info);
    CKL();
  }
  CK(cudaMemcpyAsync(c->h_info, c->d_info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->h_info[0]) return fail(c, LSBA_E_NUMERIC, "ILU(0): zero pivot");
  // level-ordered packs for the level-synchronous solve (factor values final now)
  k_ilu_pack<true><<<cdiv(n, kThreads), kThreads, 0, c->stream>>>(n, c->d_ordL, c->d_rp, c->d_ci, c->d_lu,
                                                                   c->d_diag, n, c->packL);
  k_ilu_pack<false><<<cdiv(n, kThreads), kThreads, 0, c->stream>>>(n, c->d_ordU, c->d_rp, c->d_ci, c->d_lu,
                                                                    c->d_diag, n, c->packU);
  CKL();
  CK(cudaStreamSynchronize(c->stream));
  c->ilu_levels[0] = nlL;
  c->ilu_levels[1] = nlU;
  c->ilu_ready = true;
  return LSBA_OK;
}

extern "C" lsba_status lsba_ilu0_setup(lsba_ctx c, int32_t enable) {
  if (!c) return LSBA_E_ARG;
  CK(cudaSetDevice(c->device));
  if (!enable) {
    c->prec = false;
    return LSBA_OK;
  }
  if (!c->ilu_ready && c->n > 0) TRY(ilu0_factor(c));
  if (c->n == 0) c->ilu_ready = true;
  c->prec = true;
  return LSBA_OK;
}

extern "C" lsba_status lsba_ilu0_apply(lsba_ctx c, const double* X_dev, double* Y_dev) {
  if (!c) return LSBA_E_ARG;
  if (!c->ilu_ready) return fail(c, LSBA_E_STATE, "ILU(0) not set up (lsba_ilu0_setup)");
  if (c->n > 0 && (!X_dev || !Y_dev)) return fail(c, LSBA_E_ARG, "X/Y NULL");
  CK(cudaSetDevice(c->device));
  if (c->n == 0) return LSBA_OK;
  if (X_dev != Y_dev)
    CK(cudaMemcpyAsync(Y_dev, X_dev, sizeof(double) * c->slot, cudaMemcpyDeviceToDevice, c->stream));
  TRY(ilu_apply(c, Y_dev));
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

extern "C" lsba_status lsba_copy_ilu0_factors(lsba_ctx c, double* lu_host, int64_t capacity,
                                              int32_t* levels_host) {
  if (!c) return LSBA_E_ARG;
  if (!c->ilu_ready) return fail(c, LSBA_E_STATE, "ILU(0) not set up (lsba_ilu0_setup)");
  if (lu_host && capacity < c->nnz) return fail(c, LSBA_E_ARG, "capacity %lld < nnz %lld",
                                                (long long)capacity, (long long)c->nnz);
  CK(cudaSetDevice(c->device));
  if (lu_host && c->nnz)
    CK(cudaMemcpy(lu_host, c->d_lu, sizeof(double) * c->nnz, cudaMemcpyDeviceToHost));
  if (levels_host) {
    levels_host[0] = c->ilu_levels[0];
    levels_host[1] = c->ilu_levels[1];
  }
  return LSBA_OK;
}

extern "C" lsba_status lsba_block_inner_product(lsba_ctx c, const double* V_dev, int32_t nblocks,
                                                const double* Y_dev, lsba_ip ip, double* G_host) {
  if (!c || !G_host) return LSBA_E_ARG;
  if (nblocks < 1 || nblocks > c->m_max + 1) return fail(c, LSBA_E_ARG, "nblocks outside [1, m_max+1]");
  if (ip != LSBA_IP_CLASSICAL && ip != LSBA_IP_GLOBAL) return fail(c, LSBA_E_ARG, "bad inner product");
  if (((uintptr_t)V_dev | (uintptr_t)Y_dev) & 15) return fail(c, LSBA_E_ARG, "not 16-byte aligned");
  CK(cudaSetDevice(c->device));
  TRY(gram(c, V_dev, c->slot, nblocks, const_cast<double*>(Y_dev), ip));
  const size_t E = (ip == LSBA_IP_GLOBAL) ? (size_t)nblocks : (size_t)nblocks * c->s * c->s;
  CK(cudaMemcpyAsync(G_host, c->d_G, sizeof(double) * E, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

extern "C" lsba_status lsba_set_basis_block(lsba_ctx c, int32_t j, const double* src_dev) {
  if (!c) return LSBA_E_ARG;
  if (j < 1 || j > c->m_max + 2) return fail(c, LSBA_E_ARG, "j outside [1, m_max+2]");
  if ((uintptr_t)src_dev & 15) return fail(c, LSBA_E_ARG, "not 16-byte aligned");
  c->k = -1;                          // the step API's Arnoldi process is no longer valid
  if (c->n == 0) return LSBA_OK;
  CK(cudaSetDevice(c->device));
  CK(cudaMemcpyAsync(slotp(c, j - 1), src_dev, sizeof(double) * c->slot, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

extern "C" lsba_status lsba_basis_inner_product(lsba_ctx c, int32_t j0, int32_t nblocks, int32_t y,
                                                int32_t y2, lsba_ip ip, double* G_host) {
  if (!c || !G_host) return LSBA_E_ARG;
  const int top = c->m_max + 2;
  if (nblocks < 1 || j0 < 1 || j0 + nblocks - 1 > top || y < 1 || y > top || y2 < 0 || y2 > top)
    return fail(c, LSBA_E_ARG, "basis slots outside [1, m_max+2]");
  if (ip != LSBA_IP_CLASSICAL && ip != LSBA_IP_GLOBAL) return fail(c, LSBA_E_ARG, "bad inner product");
  CK(cudaSetDevice(c->device));
  set_ip(c, ip);
  c->k = -1;
  c->d_G = c->d_Gbase;
  const double* X = slotp(c, j0 - 1);
  if (y2 > 0) TRY(gram2(c, X, c->slot_stride, nblocks, slotp(c, y - 1), slotp(c, y2 - 1), ip, nullptr));
  else TRY(gram(c, X, c->slot_stride, nblocks, slotp(c, y - 1), ip));
  const size_t E = ((ip == LSBA_IP_GLOBAL) ? (size_t)nblocks : (size_t)nblocks * c->s * c->s) * (y2 > 0 ? 2 : 1);
  CK(cudaMemcpyAsync(G_host, c->d_G, sizeof(double) * E, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  return LSBA_OK;
}

extern "C" lsba_status lsba_set_force_flag(lsba_ctx c, int32_t k_flag) {
  if (!c) return LSBA_E_ARG;
  if (k_flag < 0) return fail(c, LSBA_E_ARG, "k_flag < 0");
  c->force_flag_k = k_flag;
  c->forced_done = false;
  return LSBA_OK;
}

extern "C" lsba_status lsba_set_force_singular(lsba_ctx c, int32_t cycle) {
  if (!c) return LSBA_E_ARG;
  if (cycle < 0) return fail(c, LSBA_E_ARG, "cycle < 0");
  c->force_sing_cycle = cycle;
  return LSBA_OK;
}

extern "C" lsba_status lsba_set_skeleton(lsba_ctx c, lsba_skel skel) {
  if (!c) return LSBA_E_ARG;
  if (skel < LSBA_SKEL_BCGS_PIP || skel > LSBA_SKEL_BCGS_IROLS) return fail(c, LSBA_E_ARG, "bad skeleton");
  c->skel_default = skel;
  return LSBA_OK;
}

extern "C" lsba_status lsba_set_kernel_variant(lsba_ctx c, int32_t variant) {
  if (!c) return LSBA_E_ARG;
  if (variant < 0 || variant > 1) return fail(c, LSBA_E_ARG, "variant must be 0 or 1");
  c->variant = variant;
  return LSBA_OK;
}

extern "C" lsba_status lsba_profile_enable(lsba_ctx c, int32_t enable) {
  if (!c) return LSBA_E_ARG;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  for (int k = 0; k < LSBA_K_COUNT; ++k) {
    c->prof.used[k] = 0;
    c->prof.bytes[k] = 0.0;
    c->prof.launches[k] = 0;
  }
  c->prof.order.clear();
  c->prof.on = enable != 0;
  return LSBA_OK;
}

extern "C" lsba_status lsba_profile_timeline(lsba_ctx c, int32_t* kids, double* t_start_ms, double* t_end_ms,
                                             int64_t cap, int64_t* count) {
  if (!c || !count) return LSBA_E_ARG;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaStreamSynchronize(c->stream2));
  const auto& ord = c->prof.order;
  *count = (int64_t)ord.size();
  if (ord.empty()) return LSBA_OK;
  const cudaEvent_t origin = c->prof.ev[ord[0].first][ord[0].second].a;
  for (size_t i = 0; i < ord.size() && (int64_t)i < cap; ++i) {
    const EvPair& e = c->prof.ev[ord[i].first][ord[i].second];
    float a = 0.f, b = 0.f;
    CK(cudaEventElapsedTime(&a, origin, e.a));
    CK(cudaEventElapsedTime(&b, origin, e.b));
    if (kids) kids[i] = ord[i].first;
    if (t_start_ms) t_start_ms[i] = a;
    if (t_end_ms) t_end_ms[i] = b;
  }
  return LSBA_OK;
}

extern "C" lsba_status lsba_profile_read(lsba_ctx c, int32_t kid, int64_t* launches, double* ms, double* bytes) {
  if (!c || kid < 0 || kid >= LSBA_K_COUNT) return LSBA_E_ARG;
  CK(cudaSetDevice(c->device));
  CK(cudaStreamSynchronize(c->stream));
  double tot = 0.0;
  for (size_t i = 0; i < c->prof.used[kid]; ++i) {
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, c->prof.ev[kid][i].a, c->prof.ev[kid][i].b));
    tot += t;
  }
  if (launches) *launches = c->prof.launches[kid];
  if (ms) *ms = tot;
  if (bytes) *bytes = c->prof.bytes[kid];
  return LSBA_OK;
}

extern "C" lsba_status lsba_launch_count(lsba_ctx c, int64_t* launches) {
  if (!c || !launches) return LSBA_E_ARG;
  *launches = c->launches;
  return LSBA_OK;
}

extern "C" lsba_status lsba_workspace_bytes(lsba_ctx c, int64_t* bytes) {
  if (!c || !bytes) return LSBA_E_ARG;
  *bytes = c->ws_bytes;
  return LSBA_OK;
}

#ifdef LSBA_TAIL_TRACE
// Diagnostics build only: copy the trace records (kernels.cuh trace_rec) to `out` (2 words per
// record), reset the buffer, return the number of words copied.  Not declared in lsba.h.
extern "C" int lsba_trace_dump(unsigned long long* out, int max_words) {
  unsigned n = 0;
  if (cudaDeviceSynchronize() != cudaSuccess) return -1;
  cudaMemcpyFromSymbol(&n, lsba::g_trace_n, sizeof(unsigned));
  if (n > lsba::kTraceWords) n = lsba::kTraceWords;
  if ((int)n > max_words) n = (unsigned)max_words & ~1u;
  if (out && n) cudaMemcpyFromSymbol(out, lsba::g_trace, sizeof(unsigned long long) * n);
  const unsigned z = 0;
  cudaMemcpyToSymbol(lsba::g_trace_n, &z, sizeof(unsigned));
  return (int)n;
}
#endif
