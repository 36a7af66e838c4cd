/*
 * lsba.h — C ABI of the B200-native low-synchronization block Arnoldi hot path.
 *
 * Problem statement: solve A X = B with A (n x n) large and sparse and
 * B (n x s) tall and skinny, by restarted modified BFOM / BGMRES (Eq (Xm))
 * whose Krylov basis is built by BCGS-PIP block Arnoldi (Alg 3) in the
 * classical or global block inner product (Table 1), with the adaptive
 * restart of Sec 4 and a basis-condition trigger (reading R8).
 *
 * Conventions (all calls):
 *   - Return an lsba_status; none aborts or exits.  Numerical breakdown (a Cholesky
 *     "NaN-flag") is NOT an error: it is reported through the info structs.
 *   - Arithmetic is IEEE fp64 throughout.
 *   - Block vectors (B, X, basis blocks) are ROW-MAJOR n_local x s fp64 arrays (row i's s
 *     values contiguous), contiguous, 16-byte aligned, in device memory unless the name says
 *     _host.  They are caller-owned; the library never frees them.
 *   - The library owns its workspace (basis of m_max+1 blocks, Gram partials, small state);
 *     it is allocated by lsba_create and freed by lsba_destroy.
 *   - All device work is enqueued on the CUDA stream given to lsba_create.  *_solve and
 *     lsba_block_arnoldi_step return after completion (they synchronise that stream).
 *   - Multi-GPU: one context per rank (process); rows are partitioned into contiguous
 *     ranges [row_begin, row_end).  Every block step performs exactly one ncclAllReduce of
 *     the Gram block (the step's single sync point); halos move with
 *     grouped ncclSend/ncclRecv.  Small (s x s, ks x ks) state is replicated on every rank.
 *   - One context per host thread; a context is not thread-safe.
 */
#ifndef LSBA_H
#define LSBA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct lsba_ctx_* lsba_ctx;

typedef enum {
  LSBA_OK = 0,
  LSBA_E_ARG = 1,    /* invalid argument (message in lsba_last_error)           */
  LSBA_E_CUDA = 2,   /* a CUDA runtime call or kernel launch failed              */
  LSBA_E_NCCL = 3,   /* an NCCL call failed                                      */
  LSBA_E_OOM = 4,    /* device or pinned-host allocation failed                  */
  LSBA_E_STATE = 5,  /* call out of order (e.g. step before arnoldi_begin)       */
  LSBA_E_NUMERIC = 6 /* ILU(0) zero pivot: the problem is unpreconditionable     */
} lsba_status;

/* Table 1. */
typedef enum { LSBA_IP_CLASSICAL = 0, LSBA_IP_GLOBAL = 1 } lsba_ip;

/* Gram-Schmidt skeleton (Table 2): BCGS-PIP (Alg 3) and
 * BMGS-CWY / BMGS-ICWY (Alg 6; one block inner product per iteration with the
 * normalisation lagged by one iteration: m+1 A-applications and m+2 syncs per cycle), and the
 * comparison skeletons BMGS (Alg 2) and BCGS-PIO (Alg 4),
 * and BCGS-IRO-LS (Alg 7). */
typedef enum {
  LSBA_SKEL_BCGS_PIP = 0,    /* Alg 3: one sync per step (the north star's skeleton)          */
  LSBA_SKEL_BMGS_CWY = 1,    /* Alg 6 (red): one sync per step, normalisation lagged           */
  LSBA_SKEL_BMGS_ICWY = 2,   /* Alg 6 (blue)                                                   */
  LSBA_SKEL_BMGS = 3,        /* Alg 2: k+1 syncs per step (comparison baseline)                */
  LSBA_SKEL_BCGS_PIO = 4,    /* Alg 4: two syncs per step (comparison baseline)                */
  LSBA_SKEL_BCGS_IROLS = 5   /* Alg 7: BCGS-IRO-LS (block DCGS2), one sync per step, lagged    */
} lsba_skel;

/* SPEC.md:327 outcome of a solve. */
typedef enum { LSBA_CONVERGED = 0, LSBA_MAX_RESTARTS = 1, LSBA_DEAD = 2 } lsba_outcome;

/* Result of one block Arnoldi step (lsba_block_arnoldi_step). */
typedef struct {
  int32_t k;          /* index of the step just attempted (1-based, Alg 3 line 2)           */
  int32_t chol_flag;  /* 1 iff chol(Omega - H^T H) flagged (reading R2)  */
  double cond_est;    /* kappa_F of R_{k+1} = [E_1 beta, Hbar_k] (reading R8)               */
  double res_est;     /* BGMRES residual-norm estimate ||g_{k+1}||_F for C_acc = I (Eq normF_Rm) */
  double res_est_fom; /* BFOM residual-norm estimate ||H_{k+1,k} E_k^T Xi_FOM||_F (Eq normF_Rm, M = 0) */
  int32_t proj_singular; /* 1 iff the BFOM projected matrix H_k is singular (reading R22)   */
  int32_t pad_;
} lsba_step_info;

/* Result of a solve.  Counters follow the paper's accounting (PAPER.md:650 tables): BCGS-PIP
 * syncs = iterations + cycles, matvecs (A-ct) = iterations, basis_evals (V-ct) = 3 iterations;
 * BMGS-(I)CWY one more of each per cycle; BMGS sum over steps of (k+1)
 * syncs plus one per cycle and V-ct = 2 iterations; BCGS-PIO 2 iterations
 * + cycles syncs. */
typedef struct {
  int32_t outcome;            /* lsba_outcome                                             */
  int32_t cycles;             /* restart cycles run                                       */
  int32_t restarts;           /* cycles - 1                                               */
  int32_t iterations;         /* accepted block Arnoldi steps                             */
  int32_t attempted_steps;    /* accepted + NaN-flagged steps                             */
  int32_t nan_flags;          /* Cholesky NaN-flags (each shrinks m, reading R6)          */
  int32_t cond_restarts;      /* cycles ended by kappa_F > cond_threshold (reading R8)    */
  int32_t happy;              /* flags recognised as happy breakdown (reading R7)         */
  int32_t false_convergences; /* estimate <= tol but true residual > tol (reading R19)    */
  int32_t m_final;            /* maximum basis size after adaptive reductions             */
  int64_t syncs, matvecs, basis_evals;
  int64_t kernel_launches;    /* this library's kernel launches during the call            */
  double res_est;             /* last residual estimate, ||.||_F (absolute)               */
  double true_relres;         /* ||B - A X||_F / ||B||_F at exit (explicit)               */
  double seconds;             /* wall time of the call                                    */
  int64_t gram_blocks;        /* sum over accepted steps k of (k+1): n x s blocks read by the
                                 single-sync Gram passes (algorithmic-bytes accounting)     */
} lsba_solve_info;

/* ---------------------------------------------------------------- lifecycle */

/* Rank 0 creates an NCCL unique id (128 bytes) to broadcast (e.g. torch.distributed). */
lsba_status lsba_get_unique_id(uint8_t id[128]);

/* Create a context on `device` for the local rows [row_begin, row_end) of an n x n sparse A.
 *   row_ptr : host, int64, length (row_end-row_begin)+1, row_ptr[0] = 0, monotone
 *   col_idx : host, int32 GLOBAL column indices, sorted strictly increasing per row
 *   vals    : host, fp64
 * The CSR is validated and copied; the caller keeps its arrays.
 * s in [1,16]; m_max >= 1 (basis of m_max+1 blocks is allocated: 8 n_local s (m_max+1) bytes).
 * nccl_id may be NULL iff nranks == 1.  cuda_stream is a cudaStream_t (NULL = legacy stream).
 * Device-wide side effect: on one rank, when the column indices and values fit in the device's
 * persisting-L2 set-aside (and in half of L2), the context sets cudaLimitPersistingL2CacheSize
 * to (at least) their size and marks them persisting on its SpMM launches; the limit is
 * reference-counted per device and restored when the last such context is destroyed
 * (LSBA_L2PERSIST=0 in the environment disables this).
 * Errors: LSBA_E_ARG on invalid sizes or CSR; LSBA_E_OOM; LSBA_E_CUDA; LSBA_E_NCCL. */
lsba_status lsba_create(lsba_ctx* out, int64_t n, int32_t s, int32_t m_max,
                        const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                        int64_t row_begin, int64_t row_end, int32_t rank, int32_t nranks,
                        const uint8_t* nccl_id, int32_t device, void* cuda_stream);
lsba_status lsba_destroy(lsba_ctx ctx);

/* Caller-owned workspace: the same as lsba_create, but every long-lived device
 * buffer of the context (CSR, basis slots, Gram partials, small state; lsba_workspace_bytes
 * reports the total afterwards) is obtained from the caller's allocator — e.g. PyTorch's
 * caching allocator (the Python binding's Context(..., allocator="torch")).
 *   alloc(bytes, device, stream, user): device memory, >= 256-byte aligned, NULL on failure
 *     (-> LSBA_E_OOM); stream is the context's stream;
 *   free(ptr, device, stream, user): called once per buffer by lsba_destroy, after the
 *     context's streams have drained.
 * Transient create-time buffers, pinned host words and NCCL's own memory stay with CUDA/NCCL. */
typedef struct {
  void* (*alloc)(size_t bytes, int32_t device, void* stream, void* user);
  void (*free)(void* ptr, int32_t device, void* stream, void* user);
  void* user;
} lsba_allocator;
lsba_status lsba_create_with_allocator(lsba_ctx* out, int64_t n, int32_t s, int32_t m_max,
                                       const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                                       int64_t row_begin, int64_t row_end, int32_t rank, int32_t nranks,
                                       const uint8_t* nccl_id, int32_t device, void* cuda_stream,
                                       const lsba_allocator* allocator);

/* Distributed code path on ONE rank: with LSBA_FORCE_COMM=1 in the environment, lsba_create on
 * nranks == 1 builds a one-rank NCCL communicator and runs exactly the P > 1 code path (every
 * Gram through ncclAllReduce, the small step as its own launch);
 * results match the default path to rounding. */

/* Loopback group (testing the multi-rank path on one device): P contexts, each driven by its
 * own host thread, whose collectives (the Gram / norm allreduces, the halo send/recv and the
 * create-time ghost-plan exchange) rendezvous on the host and move data with stream-ordered
 * device copies and one rank-ordered reduction kernel — no kernel waits on another rank's
 * kernel.  Not a performance path.  lsba_create_loopback is lsba_create with the group in place
 * of the NCCL id; the group must outlive its contexts; every rank must make the same sequence
 * of calls (as with NCCL).  nranks in [1, 16]. */
typedef struct lsba_loopback_* lsba_loopback;
lsba_status lsba_loopback_create(int32_t nranks, lsba_loopback* out);
lsba_status lsba_loopback_destroy(lsba_loopback group);
lsba_status lsba_create_loopback(lsba_ctx* out, int64_t n, int32_t s, int32_t m_max,
                                 const int64_t* row_ptr, const int32_t* col_idx, const double* vals,
                                 int64_t row_begin, int64_t row_end, int32_t rank, int32_t nranks,
                                 lsba_loopback group, int32_t device, void* cuda_stream);

const char* lsba_status_str(lsba_status st);
const char* lsba_last_error(lsba_ctx ctx);   /* never NULL; "" if no error */

/* ---------------------------------------------------------------- one cycle, step by step */

/* Alg 3 line 1: [V_1, beta] = IO(B) (CholQR for classical, (1/sqrt s)||B||_F for global;
 * PAPER.md:114, 265, 416).  B_dev: n_local x s.  *io_flag = 1 if IO's Cholesky flagged. */
lsba_status lsba_arnoldi_begin(lsba_ctx ctx, const double* B_dev, lsba_ip ip, int32_t* io_flag);

/* Alg 3 lines 3-6 for the next k: W = A V_k; ONE fused Gram <[V_k W], W> (+ one allreduce);
 * H_{k+1,k} = chol(Omega - H^T H) with NaN-flag; V_{k+1} = (W - V_k H_{1:k,k}) H_{k+1,k}^{-1}.
 * On a flag the step is not accepted (k does not advance; V_{k+1} is not formed).
 * LSBA_E_STATE if called before arnoldi_begin, after a flag, or when k == m_max. */
lsba_status lsba_block_arnoldi_step(lsba_ctx ctx, lsba_step_info* info);

/* The projected problem of the current Arnoldi state (after k >= 1 accepted steps, C_acc = I):
 * Xi = (H_k + M E_k^T)^{-1} E_1 beta (Eq Xm) with M = 0 (fom != 0) or the BGMRES
 * M of PAPER.md:191, written row-major (k b) x b to Xi_host, and Z = [M; -H_{k+1,k}]
 * ((k+1) b x b, row-major; Thm 2.4's restart generator coefficients) to Z_host. */
lsba_status lsba_projected_solve(lsba_ctx ctx, int32_t fom, double* Xi_host, double* Z_host);

/* Copy the block Hessenberg Hbar_k ((k+1)b x kb, b = s classical / 1 global) to host,
 * column-major with leading dimension ld >= (k+1)b.  Also valid after a flag (the flagged
 * step's column H_{1:k,k} is stored, its subdiagonal block is not). */
lsba_status lsba_copy_hessenberg(lsba_ctx ctx, double* H_host, int32_t ld);
/* beta (b x b, column-major) from the last IO. */
lsba_status lsba_copy_beta(lsba_ctx ctx, double* beta_host);
/* Copy basis block V_{j} (1-based, j <= k+1) to a caller device buffer (n_local x s). */
lsba_status lsba_copy_basis_block(lsba_ctx ctx, int32_t j, double* dst_dev);

/* ---------------------------------------------------------------- solvers */

/* Restarted BGMRES / BFOM (modification M of PAPER.md:191 / M = 0) with the skeleton `skel`
 * and the adaptive restart of Sec 4 (NaN-flag -> restart from the last safe block, m <- k-1;
 * PAPER.md:405) plus cond_threshold (kappa_F trigger, +inf = off; reading R8).
 *   B_dev : n_local x s (device);  X_dev : in X0, out X (device)
 *   m <= m_max; tol > 0 relative to ||B||_F; at most max_restarts+1 cycles.
 * Convergence: res_est <= tol ||B||_F after any accepted step, confirmed by the explicit
 * residual (reading R19).  Returns LSBA_OK also for MAX_RESTARTS and DEAD outcomes. */
lsba_status lsba_bgmres_solve(lsba_ctx ctx, const double* B_dev, double* X_dev, int32_t m,
                              double tol, int32_t max_restarts, lsba_skel skel, lsba_ip ip,
                              double cond_threshold, lsba_solve_info* info);
lsba_status lsba_bfom_solve(lsba_ctx ctx, const double* B_dev, double* X_dev, int32_t m,
                            double tol, int32_t max_restarts, lsba_skel skel, lsba_ip ip,
                            double cond_threshold, lsba_solve_info* info);
/* Same as lsba_bgmres_solve / lsba_bfom_solve (fom != 0) but B and X live in HOST memory
 * (pinned or pageable); the host<->device copies are part of the call. */
lsba_status lsba_solve_host(lsba_ctx ctx, const double* B_host, double* X_host, int32_t m,
                            double tol, int32_t max_restarts, int32_t fom, lsba_ip ip,
                            double cond_threshold, lsba_solve_info* info);

/* ---------------------------------------------------------------- single kernels (parity) */

/* W = A V over the local rows (halo exchange included when nranks > 1).  V_dev, W_dev:
 * n_local x s device buffers (distinct). */
lsba_status lsba_spmm(lsba_ctx ctx, const double* V_dev, double* W_dev);
/* G = [V_1..V_p]^T Y (classical, (p s) x s, row-major) or the p scalars (1/s) tr(V_j^T Y)
 * (global) for p = nblocks consecutive n_local x s blocks at V_dev; Y_dev n_local x s;
 * includes the allreduce.  G_host receives the result. */
lsba_status lsba_block_inner_product(lsba_ctx ctx, const double* V_dev, int32_t nblocks,
                                     const double* Y_dev, lsba_ip ip, double* G_host);
/* Basis-slot access for kernel-level parity of the shipped streaming Gram (Alg 3 line 4,
 * PAPER.md:268-269; Alg 6 line 10).  The basis owns m_max + 2 slots V_1..V_{m_max+2}
 * (1-based as in lsba_copy_basis_block).
 * lsba_set_basis_block: copy a caller device block (n_local x s, row-major) into slot V_j; it
 *   invalidates the step API's Arnoldi state (the next step needs lsba_arnoldi_begin).
 * lsba_basis_inner_product: G = <[V_{j0} .. V_{j0+nblocks-1}], Y> over slots with the kernels
 *   the solver runs (k_gram_v7 / k_gram_gl2; no small step fused), including the allreduce.
 *   Y = V_{y}; if y2 > 0, Y = [V_y V_{y2}] (the two-block Gram of BMGS-(I)CWY).  Classical:
 *   (nblocks s) x (s or 2s) row-major; global: nblocks scalars (1/s) tr(V^T Y) (or nblocks
 *   pairs).  LSBA_E_ARG for slots outside [1, m_max + 2] or j0 + nblocks - 1 > m_max + 2. */
lsba_status lsba_set_basis_block(lsba_ctx ctx, int32_t j, const double* src_dev);
lsba_status lsba_basis_inner_product(lsba_ctx ctx, int32_t j0, int32_t nblocks, int32_t y, int32_t y2,
                                     lsba_ip ip, double* G_host);

/* ---------------------------------------------------------------- debug / measurement */

/* Fault injection: make the Cholesky of step k_flag report a NaN-flag once (0 = off). */
lsba_status lsba_set_force_flag(lsba_ctx ctx, int32_t k_flag);
/* Fault injection: make the cycle-end projected solve of solve cycle `cycle` report singular
 * (its combine then no-ops and the solve ends DEAD with the previous cycle's X; 0 = off).
 * Covers the guard chain between a singular cycle end and the next cycle's speculative end. */
lsba_status lsba_set_force_singular(lsba_ctx ctx, int32_t cycle);
/* Skeleton of the step API (lsba_arnoldi_begin / lsba_block_arnoldi_step) and of
 * lsba_solve_host (default BCGS-PIP); the *_solve calls take theirs as an argument.
 * With BMGS-(I)CWY, lsba_arnoldi_begin also runs Alg 6's first loop iteration, and step k
 * (its iteration k+1) completes Hessenberg column k and forms V_{k+1}. */
lsba_status lsba_set_skeleton(lsba_ctx ctx, lsba_skel skel);
/* ---------------------------------------------------------------- ILU(0) left preconditioning
 * SURVEY.md 8(f) f4; PAPER.md:485 ("an incomplete LU (ILU) preconditioner with no fill");
 * SPEC.md:512-528 (IKJ ILU(0) restricted to pattern(A); LEFT preconditioning, every residual
 * and tolerance in the preconditioned norm — DESIGN.md reading R28).
 *
 * lsba_ilu0_setup(ctx, 1): on first use factors the context's matrix on the device (host level
 * analysis, one launch per level of L); from then on every operator application of the
 * Arnoldi process and the solvers is M^{-1} A (SpMM followed by two sync-free triangular
 * solves), the solvers target M^{-1} A X = M^{-1} B and report true_relres =
 * ||M^{-1}(B - A X)||_F / ||M^{-1} B||_F.  enable = 0 restores the plain operator (factors kept).
 * With P > 1 each rank factors its local diagonal block (block-Jacobi ILU(0); ghost columns
 * dropped) — identical to ILU(0) of A on one rank.  lsba_spmm stays the plain A V.
 * Errors: LSBA_E_NUMERIC on a zero or structurally missing pivot (message names the row). */
lsba_status lsba_ilu0_setup(lsba_ctx ctx, int32_t enable);
/* Y = M^{-1} X = U^{-1} L^{-1} X for device n_local x s row-major blocks (X == Y allowed).
 * LSBA_E_STATE before lsba_ilu0_setup. */
lsba_status lsba_ilu0_apply(lsba_ctx ctx, const double* X_dev, double* Y_dev);
/* Copy the factor values (nnz_local doubles in the CSR order of the matrix: strictly-lower
 * entries are L with unit diagonal implied, the rest U) to lu_host (capacity doubles;
 * LSBA_E_ARG if capacity < nnz_local), and the level counts of L and U to levels_host[2]
 * (either pointer may be NULL). */
lsba_status lsba_copy_ilu0_factors(lsba_ctx ctx, double* lu_host, int64_t capacity, int32_t* levels_host);

/* Kernel implementation choice: 0 = default (streaming tensor-core v7 Gram / streaming global
 * Gram, DMMA projection for s in {8, 16}, DFMA otherwise, small step fused into the Gram on one
 * rank), 1 = plain DFMA Gram and projection kernels (for parity tests of both paths). */
lsba_status lsba_set_kernel_variant(lsba_ctx ctx, int32_t variant);

/* Per-kernel timing with CUDA events on the context stream.  Kernel ids: */
enum {
  LSBA_K_SPMM = 0, LSBA_K_GRAM = 1, LSBA_K_GRAM_FINALIZE = 2, LSBA_K_SMALL_STEP = 3,
  LSBA_K_PROJECT = 4, LSBA_K_CYCLE_SOLVE = 5, LSBA_K_COMBINE = 6, LSBA_K_RESIDUAL = 7,
  LSBA_K_HALO_PACK = 8, LSBA_K_MISC = 9, LSBA_K_STEP_UPDATE = 10, LSBA_K_ILU_SOLVE = 11,
  LSBA_K_COUNT = 12
};
/* enable != 0 starts recording events around every launch (resets the records). */
lsba_status lsba_profile_enable(lsba_ctx ctx, int32_t enable);
/* For kernel id `kid`: launches, summed event time (ms) and summed ALGORITHMIC bytes
 * over the recorded launches.  Synchronises the stream. */
lsba_status lsba_profile_read(lsba_ctx ctx, int32_t kid, int64_t* launches, double* ms,
                              double* bytes);
/* The recorded launches in issue order (both streams): kernel id and start / end times in ms
 * relative to the first recorded launch's start event.  Writes min(count, cap) entries;
 * *count receives the number recorded.  Synchronises the context's streams. */
lsba_status lsba_profile_timeline(lsba_ctx ctx, int32_t* kids, double* t_start_ms, double* t_end_ms,
                                  int64_t cap, int64_t* count);
/* Total kernel launches of this context since creation. */
lsba_status lsba_launch_count(lsba_ctx ctx, int64_t* launches);
/* Device workspace bytes held by the context. */
lsba_status lsba_workspace_bytes(lsba_ctx ctx, int64_t* bytes);

/* ---------------------------------------------------------------- host-only (no GPU needed) */

/* Ghost plan for a row-partitioned CSR (SPEC 8(e)): given this rank's rows [row_begin,
 * row_end) with GLOBAL col_idx (nnz entries) and the partition starts part[0..nranks]
 * (part[0] = 0, part[nranks] = n), write col_local[nnz] (local index if owned, else
 * n_local + ghost slot), ghost_global[] (sorted unique remote columns, capacity nnz) and
 * recv_counts[nranks] (ghost rows owned by each rank).  *n_ghost receives the count.
 * Pure host code; used by lsba_create and unit-tested on CPU. */
lsba_status lsba_ghost_plan(int64_t row_begin, int64_t row_end, const int32_t* col_idx,
                            int64_t nnz, const int64_t* part, int32_t nranks,
                            int32_t* col_local, int64_t* ghost_global, int64_t* n_ghost,
                            int64_t* recv_counts);
/* Validate a CSR block; returns LSBA_E_ARG with a message in *msg
 * (static storage) on violation. */
lsba_status lsba_csr_validate(int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                              const int32_t* col_idx, const char** msg);

#ifdef __cplusplus
}
#endif
#endif /* LSBA_H */
