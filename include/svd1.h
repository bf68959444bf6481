/*
 * svd1.h — C ABI of the B200-native rank-1 SVD update (libsvd1.so).
 *
 * Method: Gandhi & Rajgor, "Updating Singular Value Decomposition for Rank One
 * Matrix Perturbation", arXiv 1707.08369 (/root/reference/PAPER.md, cited "P:n").
 *   Alg 6.1: A_hat = A + a b^T, A = U Sigma V^T, m <= n.
 *   Alg 6.2: RankOneUpdate, called twice per side.
 *   Secular equation w(mu) = 1 + rho sum z_i^2 / (d_i - mu).
 *   Eigenvector factor C~ = diag(z) C diag(1/||c_j||), C_ij = 1/(d_i - mu_j)
 *     (P:194-208), applied to every row of U — the hot path.
 *   1-D Chebyshev FMM for that product, re-derived per
 *     DESIGN.md §4 (the printed M2M/M2L operators are corrected).
 *
 * Conventions (all entry points):
 *   - Matrix/vector pointers are DEVICE pointers (cudaMalloc / torch CUDA
 *     tensors), caller-owned; the library never frees them.  Matrices are
 *     fp64, row-major, leading dimension in elements (ld >= number of columns).
 *     A row of U is one right-hand side of the Cauchy apply.
 *   - sigma is descending; eigenvalues are handled ascending inside.
 *   - Work is ordered on the plan's stream (svd1_config.stream, a cudaStream_t;
 *     NULL = legacy default stream).  svd1_update blocks the host until its
 *     result is on the device (it reads small vectors back several times).
 *   - Errors: every function returns svd1_status; on SVD1_E_NOCONV,
 *     SVD1_E_NONFINITE, SVD1_E_POLE, SVD1_E_ZEROCOL or SVD1_E_UNSUPPORTED from svd1_update the
 *     matrices are left UNMODIFIED (all checks happen in the spectral phase,
 *     before any write to U, Sigma or V).  SVD1_E_CUDA leaves them undefined.
 *   - Determinism: fixed reduction orders, no floating-point atomics: identical
 *     inputs give bitwise-identical outputs on the same GPU model.
 *   - A plan is not thread-safe; use one plan per stream.
 */
#ifndef SVD1_H
#define SVD1_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct svd1_plan_s* svd1_plan_t;

typedef enum {
  SVD1_OK = 0,
  SVD1_E_INVALID = 1,   /* DimensionMismatch, m > n, eps not in (0,1), NULL pointer */
  SVD1_E_NONFINITE = 2, /* NaN/Inf in an input vector or projection */
  SVD1_E_NOCONV = 3,    /* secular iteration did not converge */
  SVD1_E_POLE = 4,      /* a root coincides with a pole: tau == 0 */
  SVD1_E_ZEROCOL = 5,   /* ||c_j|| underflow/overflow */
  SVD1_E_CUDA = 6,      /* CUDA runtime error */
  SVD1_E_NOMEM = 7,     /* device or host allocation failed */
  SVD1_E_NCCL = 8,      /* NCCL unavailable or a collective failed (world > 1) */
  SVD1_E_UNSUPPORTED = 9 /* a singular value repeated beyond what the pairing of U_hat and V_hat
                            tracks (DESIGN.md §3.2 D5: more than 256 bitwise-equal positive
                            sigma in one update) -- refused, not paired wrongly */
} svd1_status;

/* flags */
#define SVD1_FORCE_DIRECT 0x1u /* always use the direct Cauchy-on-the-fly apply */
#define SVD1_FORCE_FMM 0x2u    /* use the FMM apply whenever n_active >= 2 leaves */
#define SVD1_SECULAR_FMM 0x4u  /* secular solve with the FMM far field for
                                  every size above 64 (default: from 6144 roots, or the
                                  environment variable SVD1_SEC_FMM_MIN) */
#define SVD1_SECULAR_DIRECT 0x8u /* secular solve with the direct O(n) sums only */
#define SVD1_THIN_V 0x10u        /* thin right factor (m < n):
                                    V is n x (m+1), ldv >= m+1; columns 0..m-1 hold V[:, :m],
                                    column m is workspace (the direction of b outside span(V),
                                    overwritten by every update).  The null space of A^T is
                                    never stored. */
#define SVD1_EMULATE_RANKS 0x20u /* world > 1 without NCCL (test mode): this
                                    process computes EVERY rank's slice of the spectral phase,
                                    so the all-gathers are concatenations in place; the rows
                                    are this process's as usual (normally all of them) */
#define SVD1_FUSED_SIDE 0x80u    /* fused per-side pass: each
                                    side's two applies (X1 then X2) run row chunk by
                                    row chunk with the chunk's rows, intermediate and FMM
                                    expansions L2-resident, so U and V are read and written once
                                    per update; apply_ms[0] / [2] then hold the whole side */
#define SVD1_FORCE_NCCL 0x40u    /* use the NCCL all-gathers even with world == 1 (test mode:
                                    exercises the communicator path on one GPU; nccl_id needed) */

typedef struct {
  int64_t m, n;      /* global sizes, 1 <= m <= n */
  int64_t u_rows;    /* rows of U held by this process (== m on one GPU) */
  int64_t v_rows;    /* rows of V held by this process (== n on one GPU) */
  int64_t u_row0;    /* global index of the first local row of U (probe rows) */
  int64_t v_row0;    /* global index of the first local row of V */
  double eps;        /* FMM precision: p = max(4, ceil(log5(1/eps))) rounded up to a
                        multiple of 4 (P:701 STEP 1; DESIGN.md §3.2 D6) */
  void* stream;      /* cudaStream_t */
  uint32_t flags;    /* SVD1_FORCE_* */
  int32_t fmm_min_n; /* active size from which the FMM apply is used (0 = 384) */
  /* Ranks (one process per GPU).  Rows of U and V are split by
   * the caller (u_row0/u_rows, v_row0/v_rows above).  With world > 1 the O(n^2) spectral phase
   * of every eigen-update (P:363 STEP 2 and the Loewner / column-norm sums) is SLICED: rank r
   * solves roots, Loewner weights and column norms of the index range [r c, r c + c),
   * c = ceil(n_active / world), and the plan all-gathers them over NCCL (NVLink); decisions
   * made on the host (deflation, merge, trees) see bitwise-identical data on every rank.
   * Slices are computed by the same code as the whole range, so results are bitwise those of
   * world == 1 (given the same all-reduced projections). */
  int32_t rank;        /* 0 <= rank < world */
  int32_t world;       /* number of ranks; 0 or 1 = one process */
  const void* nccl_id; /* world > 1 (or SVD1_FORCE_NCCL): 128-byte ncclUniqueId from
                          svd1_nccl_unique_id on rank 0, given to every rank by the caller;
                          svd1_plan_create is then collective (all ranks call it).  NULL with
                          SVD1_EMULATE_RANKS. */
} svd1_config;

typedef struct {
  double t_ms[8];        /* host wall times (ms): [0] projection read-back, [1] spectral
                            rounds, [2] apply planning + launch, [3] from the end of the
                            spectral phase to the final sync, [4] total; [5] device time
                            of the whole apply phase (U side and V side run concurrently) */
  int32_t n_active[4];   /* active sizes of the four eigen-updates */
  int32_t n_deflated[4]; /* deflated counts */
  int32_t max_iter[4];   /* max secular iterations per eigen-update */
  int32_t fmm_used[4];   /* 1 if that apply ran the FMM, 0 if direct */
  int32_t p;             /* Chebyshev order used */
  int32_t neg_clamped;   /* eigenvalues < 0 clamped before sqrt (STEP 8) */
  int32_t sign_flips;    /* columns of V_hat flipped by the sign alignment */
  int32_t noop;          /* 1 if a == 0 or b == 0 (A_hat = A) */
  int64_t kernel_launches; /* CUDA kernels launched by this call */
  double apply_ms[4];    /* device time of each Cauchy apply (CUDA events on the plan
                            stream; Householder + apply + passthrough) */
  double apply_flops[4]; /* algorithmic flops of each apply: FMM 2*rows*
                            sum(K*N) over level-by-level P2M/M2M/M2L/L2L/L2P/P2P terms;
                            direct 2*rows*n_a^2 */
  double spectral_ms[4]; /* device time of secular + Loewner + norms per eigen-update */
  int32_t fmm_levels[4]; /* tree depth L of each FMM apply (0 if direct) */
  int32_t fmm_max_near[4]; /* largest near-field list (leaves) of each FMM apply */
  double mean_iter[4];   /* mean secular evaluations per root (incl. the midpoint one) */
  int32_t pair_rotations; /* repeated-sigma clusters paired by a k x k rotation (D5) */
  double apply_flops_exec[4]; /* flops each apply executes: as apply_flops, except that the
                            coarse M2M / L2L levels run in bands, which
                            trade a few flops for fewer launches */
  double gemm_ms[4];     /* device time of each apply's FMM GEMM passes (CUDA events around
                            every pass launch on its stream) when the environment variable
                            SVD1_GEMM_EVENTS is set (diagnostics), else 0 */
  int64_t allocations;   /* device / pinned-host allocations the library made during this
                            update (0 in steady state: every workspace is sized by
                            svd1_plan_create; a buffer that depends on the FMM tree and
                            outgrows its create-time estimate grows once, stream-ordered) */
  int32_t unpaired_clusters; /* clusters of more than 4 final singular values equal to within
                            64 eps of their own size (so their columns are not determined one
                            by one) that are neither paired by the probes nor made of tracked
                            repeated columns (D5): near-equal but distinct sigma, whose U_hat /
                            V_hat columns inside the cluster may be mismatched by a rotation
                            (see DESIGN.md §10); 0 otherwise */
} svd1_report;

/* Plan: owns every workspace, allocated HERE (FMM STEPS 1-2 fix p, s and
 * the tree depth up front): W (u_rows x m, v_rows x n), the FMM expansions
 * Phi/Psi of both sides for the deepest tree the planner can choose at this eps
 * (rows x cells x p), the batch mode's carried rows and projections, the step records'
 * spectral buffers, pinned read-back and upload staging.  Updates allocate nothing
 * (svd1_report.allocations; stream-ordered growth only if a call's eps is smaller than
 * the plan's or a tree-dependent estimate is exceeded).  Returns SVD1_E_INVALID for bad
 * sizes, SVD1_E_NOMEM if the workspaces do not fit. */
svd1_status svd1_plan_create(const svd1_config* cfg, svd1_plan_t* out);
svd1_status svd1_plan_destroy(svd1_plan_t plan);

/* Full rank-1 SVD update on one GPU: Alg 6.1 STEPS 1-8.
 * U (m x m, ldu), sigma (m, descending), V (n x n, ldv) are updated IN PLACE so
 * that on return A + a b^T = U diag(sigma) V[:, :m]^T.  a (m), b (n) device.
 * eps <= 0 uses the plan's eps.  rep (host pointer) may be NULL.
 * Equivalent to svd1_project + svd1_update_projected with world size 1. */
svd1_status svd1_update(svd1_plan_t plan, double* U, int64_t ldu, double* sigma,
                        double* V, int64_t ldv, const double* a, const double* b,
                        double eps, svd1_report* rep);

/* A stream of K rank-1 updates A_t = A_{t-1} + a_t b_t^T, t = 0..K-1, applied in order
 * on one GPU (single process: u_rows = m, v_rows = n).  Results are those of K calls
 * of svd1_update (same algorithm, same tolerances), but the updates are pipelined
 * (DESIGN.md §4.9): every update's projections U_t^T a_t, U_t^T g, V_t^T b_t are
 * carried as a few extra rows through the previous updates' transforms (the rows of U
 * and of a projection transform alike, U_{t+1}^T a = X^T U_t^T a), so the spectral phase
 * of update t+1 runs while the applies of update t are still on the GPU.
 * A (device): a_t at A + t*lda (m doubles, lda >= m); B (device): b_t at B + t*ldb
 * (n doubles, ldb >= n).  U, sigma, V as for svd1_update (in place).  reps: K host
 * reports or NULL; in this mode apply_ms is 0, t_ms[5] is the update's apply window
 * (first apply start -> last apply end; windows of consecutive updates may overlap),
 * reps[K-1].t_ms[6] the whole batch's apply span (first apply start of update 0 ->
 * last apply end of update K-1), and gemm_ms is filled under SVD1_GEMM_EVENTS.  On an error at update t the factors hold the result of updates 0..t-1 and
 * the error is returned.  K <= 28 per call (longer streams: call repeatedly). */
svd1_status svd1_update_batch(svd1_plan_t plan, double* U, int64_t ldu, double* sigma,
                              double* V, int64_t ldv, const double* A, int64_t lda,
                              const double* B, int64_t ldb, int64_t K, double eps,
                              svd1_report* reps);

/* Row-sharded stream: svd1_update_batch after the projections.  proj (device): K
 * consecutive all-reduced svd1_project outputs (5*m + n + 6 doubles each, update t at
 * proj + t*(5*m + n + 6)), every one computed against the factors at the START of the
 * stream; sigma full, replicated; U_loc, V_loc this rank's row blocks.  B (device, the
 * FULL b_t at B + t*ldb, ldb >= n) is needed with SVD1_THIN_V only (else NULL).  Every
 * rank runs the same spectral phases and carried-row transforms (deterministic) on its
 * own GPU; no collective inside.  K <= 28. */
svd1_status svd1_update_batch_projected(svd1_plan_t plan, double* U_loc, int64_t ldu,
                                        double* sigma, double* V_loc, int64_t ldv,
                                        const double* proj, const double* B, int64_t ldb,
                                        int64_t K, double eps, svd1_report* reps);

/* Row-sharded update, phase 1 (STEP 1 projections over the LOCAL rows):
 * proj (device, 5*m + n + 6 doubles) receives the partial sums
 *   proj[0:m]        = U_loc^T a_loc          (x_a = U^T a)
 *   proj[(1+k)m:...] = U_loc^T g_k,loc, k=0..3 (sign probes)
 *   proj[5m:5m+n]    = V_loc^T b_loc          (y_b = V^T b)
 *   proj[5m+n+k]     = a_loc . g_k,loc (k<4), proj[5m+n+4] = a_loc.a_loc,
 *   proj[5m+n+5]     = b_loc . b_loc          (alpha, beta of STEP 1)
 * with a_loc = a[u_row0 : u_row0+u_rows], b_loc = b[v_row0 : v_row0+v_rows]
 * (a, b are the FULL vectors).  Sum proj over ranks (e.g. NCCL all-reduce)
 * before phase 2. */
svd1_status svd1_project(svd1_plan_t plan, const double* U_loc, int64_t ldu,
                         const double* V_loc, int64_t ldv, const double* a,
                         const double* b, double* proj);

/* Phase 2: everything after the projections (STEPS 2-8) on the local rows.
 * proj = all-reduced phase-1 output; a (m), b (n), sigma (m) full, replicated. */
svd1_status svd1_update_projected(svd1_plan_t plan, double* U_loc, int64_t ldu,
                                  double* sigma, double* V_loc, int64_t ldv,
                                  const double* proj, const double* a,
                                  const double* b, double eps, svd1_report* rep);

/* Standalone Cauchy apply (Alg 6.2 STEPS 3-7; Trummer's problem
 * for every row):
 *   U_out[r, j] = colscale[j] * sum_i U_in[r, i] * zhat[i] / ((d[i] - d[k[j]]) - tau[j])
 * for r < rows, i, j < n.  d ascending and distinct; roots mu_j = d[k_j] + tau_j
 * strictly interlace d (tau_j != 0).  All pointers device.  Uses the FMM when
 * n >= fmm_min_n (or FORCE_FMM) with precision eps (<= 0: plan eps), else the
 * direct DMMA kernel.  U_out must not alias U_in.  rows <= plan u_rows or v_rows
 * (the larger).  fmm_used (host, nullable) reports the path taken. */
svd1_status svd1_cauchy_apply(svd1_plan_t plan, int64_t rows, int64_t n,
                              const double* d, const int32_t* k, const double* tau,
                              const double* zhat, const double* colscale,
                              const double* U_in, int64_t ld_in, double* U_out,
                              int64_t ld_out, double eps, int32_t* fmm_used);

/* Test hooks on device arrays (same kernels as svd1_update):
 * secular roots of D + rho z z^T, d ascending distinct, z != 0:
 *   mu_j = d[k_out[j]] + tau_out[j]; iters (host, nullable) = max iterations. */
svd1_status svd1_secular_solve(svd1_plan_t plan, int64_t n, const double* d,
                               const double* z, double rho, int32_t* k_out,
                               double* tau_out, int32_t* iters);
/* Loewner weights zhat (device out) from the roots (north star item (2)). */
svd1_status svd1_loewner(svd1_plan_t plan, int64_t n, const double* d,
                         const int32_t* k, const double* tau, double rho,
                         const double* z, double* zhat_out);
/* Column norms ||c_j|| of diag(zhat) C into colnorm_out (device). */
svd1_status svd1_colnorms(svd1_plan_t plan, int64_t n, const double* d,
                          const int32_t* k, const double* tau, const double* zhat,
                          double* colnorm_out);

/* Host-only introspection of the FMM plan the apply would build for the sorted
 * sources d and roots mu_j = d[k_j] + tau_j (HOST pointers; no GPU needed).
 * stats_out (9 int64): [0] tree depth L, [1] non-empty cells, [2] largest leaf,
 * [3] largest near list (leaves), [4] near pairs, [5] M2L pairs,
 * [6] algorithmic flops per row of U (2 * sum K*N, level by level), [7] GEMM tasks,
 * [8] flops per row the plan executes (coarse levels in bands). */
svd1_status svd1_fmm_tree_stats(int64_t n, const double* d, const int32_t* k,
                                const double* tau, double eps, int64_t* stats_out);

/* Host-only planning diagnostics of the secular FMM (DESIGN.md §4.2 K2'): builds the
 * plan for the ascending sources d (host, n) and fills stats_out (8 int64): depth L,
 * cells, leaves, M2L partners, near ranges, max near terms per root, direct roots,
 * planning time in ns.  No GPU needed. */
svd1_status svd1_secfmm_plan_stats(int64_t n, const double* d, int64_t* stats_out);

/* A fresh 128-byte ncclUniqueId (out: host buffer of 128 bytes) for svd1_config.nccl_id:
 * call on rank 0 and broadcast (e.g. torch.distributed.broadcast_object_list).
 * SVD1_E_NCCL if libnccl.so.2 cannot be opened. */
svd1_status svd1_nccl_unique_id(void* out);

const char* svd1_status_string(svd1_status s);
/* Library build identifier (for the bench/smoke evidence). */
const char* svd1_version(void);

#ifdef __cplusplus
}
#endif
#endif /* SVD1_H */
