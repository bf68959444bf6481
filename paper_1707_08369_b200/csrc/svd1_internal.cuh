// Internal declarations of libsvd1 (kernels + host runtime).  Not part of the ABI.
#pragma once
#include <cuda.h>  // CUtensorMap (TMA descriptors; encoded through the runtime entry point)
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <vector>

#include "../../include/svd1.h"

namespace svd1 {

constexpr double kEps = 2.220446049250313e-16;  // 2^-52
constexpr int kMaxCarry = 6;                    // small vectors carried through X^T
constexpr int kNumProbes = 4;                   // sign probes g_k
constexpr int kMaxP = 32;                       // Chebyshev order cap
constexpr int kMaxLeaf = 32;                    // leaf capacity cap (s = 2p <= 32 at p = 16)

#define SVD1_CUDA_TRY(expr)                                  \
  do {                                                       \
    cudaError_t _e = (expr);                                 \
    if (_e != cudaSuccess) return ::svd1::cuda_fail(_e, #expr, __FILE__, __LINE__); \
  } while (0)

svd1_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

// ---------------------------------------------------------------- probes
// Counter-based Gaussian: g_k[r] for global row r (splitmix64 + Box-Muller).
__host__ __device__ inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// ---------------------------------------------------------------- kernels
// K1: partial projections over row chunks.  out layout (length 5m + n + 6):
// [x_a (m)][x_g0..3 (4m)][y_b (n)][a.g0..3 (4)][a.a][b.b]
// the projections of K updates (a_t at A + t*lda, b_t at B + t*ldb) against the same
// factors into proj + t*nproj (svd1_project's layout; the probe block is NOT written):
// one pass over U (and V) per 8 updates
// dst row (base - s) <- src row s, s = 1 .. count, cols doubles each (batch carried rows)
svd1_status copy_rows_rev(double* dst, int64_t ldd, int64_t base, const double* src, int64_t lds, int64_t cols,
                          int count, cudaStream_t st, int64_t* launches);
svd1_status project_many(const double* U, int64_t ldu, int64_t u_rows, int64_t m, int64_t u_row0,
                         const double* V, int64_t ldv, int64_t v_rows, int64_t n, int64_t v_row0, int64_t vcols,
                         const double* A, int64_t lda, const double* B, int64_t ldb, int K, const double* probes,
                         double* part, int64_t partial_cap, double* proj, int64_t nproj, cudaStream_t st,
                         int64_t* launches);
svd1_status project(const double* U, int64_t ldu, int64_t u_rows, int64_t m, int64_t u_row0,
                    const double* V, int64_t ldv, int64_t v_rows, int64_t n, int64_t v_row0,
                    const double* a, const double* b, double* partial_ws, int64_t partial_cap,
                    double* proj, const double* probes, cudaStream_t st, int64_t* launches,
                    int64_t vcols = -1);
// probes g_k(row0 + r), k < 4, r < rows, into g[k * rows + r] (splitmix64 + Box-Muller)
svd1_status fill_probes(uint64_t seed, int64_t row0, int64_t rows, double* g, cudaStream_t st,
                        int64_t* launches);
int64_t project_partial_elems(int64_t u_rows, int64_t m, int64_t v_rows, int64_t n);

// K2: secular roots (warp per root).  status bit 1 = no convergence, 2 = pole.
// d, z2: the rho > 0 view of the problem (for rho < 0: -d reversed, z^2 reversed);
// outputs (k, tau) are in the original orientation.
// roots j0 <= j < j1 of the rho > 0 view (a rank's slice; 0, n: all)
svd1_status secular(const double* d, const double* z2, double rho, int n, int j0, int j1, int32_t* k_out,
                    double* tau_out, int32_t* iters_out, int32_t* status, cudaStream_t st,
                    int64_t* launches);
svd1_status secular_orient(const double* d, const double* z, double rho, int n, double* dr,
                           double* z2r, cudaStream_t st, int64_t* launches);
// scratch (doubles) needed by loewner / colnorm_carry for size n and ncarry vectors
int64_t spectral_scratch_elems(int n, int ncarry);
// K2': FMM-accelerated secular evaluation.  Tree over
// the (oriented) sources; each target cell Y carries local expansions of the far field of
// the sources left (psiL) and right (psiR) of its target interval [d_lo, d_next]; a root
// in leaf Y sums its near-leaf sources directly (exact left/right split) and evaluates
// the two polynomials, so an evaluation costs O(near + p) instead of O(n).
#ifndef SVD1_SECP
#define SVD1_SECP 20
#endif
constexpr int kSecP = SVD1_SECP;  // Chebyshev order of the secular far field
struct SecFmmCell {        // heap-ordered; empty cells have lo == hi
  int32_t lo, hi;          // source index range
  int32_t m2l_off;         // partners m2l[m2l_off .. next cell's m2l_off)
  int32_t pad;             // leaf: 1 = its last root (outlier-gap bracket) sums directly
  double c, r;             // source hull
  double ct, rt;           // target interval (centre, radius); see secfmm_plan
};
struct SecFmmPart {        // M2L partner of a target cell
  int32_t cell, flags;     // flags bit 0: right of the target (phi), bit 1: P2L (few sources)
};
struct SecFmmDev {         // device view of one plan
  int L, ncells, nleaf, ndirect;
  const int32_t* direct;    // ndirect roots solved with the direct sum (one block each)
  const SecFmmCell* cells;
  const SecFmmPart* parts;  // size cells[ncells].m2l_off (sentinel entry)
  const int32_t* leaf_lo;   // nleaf + 1: source ranges of the leaves (non-empty, in order)
  const int32_t* leaf_cell; // heap index of leaf q
  const int32_t* near_off;  // nleaf + 1 into near_lo / near_hi
  const int32_t* near_lo;   // near source index ranges [near_lo, near_hi) of leaf q
  const int32_t* near_hi;
  double* phi;              // ncells * kSecP far-field coefficients (scaled, as the apply's)
  double* psiL;             // ncells * kSecP local expansions: sources left of the interval
  double* psiR;             //                                 and right of it
};
svd1_status secular_fmm(const double* d, const double* z2, double rho, int n, int j0, int j1,
                        const SecFmmDev& F, int32_t* k_out, double* tau_out, int32_t* iters_out,
                        int32_t* status, cudaStream_t st, int64_t* launches);

// K3a: Loewner zhat (thread per i, split-j partial products + ordered combine)
// (zhat_i for i0 <= i < i1: a rank's slice)
svd1_status loewner(const double* d, const int32_t* k, const double* tau, double rho,
                    const double* z, int n, int i0, int i1, double* zhat, double* scratch, int* ctr,
                    cudaStream_t st, int64_t* launches);
// K3b + K12: colscale_j = 1/||c_j|| and carry_out[q][j] = (X^T carry_q)_j
// (thread per j, split-i partial sums + ordered combine).
// (columns j0 <= j < j1: a rank's slice; carry_out[q] at carry_out + q * ldc)
svd1_status colnorm_carry(const double* d, const int32_t* k, const double* tau,
                          const double* zhat, int n, int j0, int j1, const double* carry, int ncarry,
                          double* colscale, double* carry_out, int64_t ldc, int32_t* status, double* scratch,
                          int* ctr, cudaStream_t st, int64_t* launches);

// K11: direct apply  U_out[r, dst[j]] = cs[j] * sum_i U_in[r, src[i]] zhat[i] / ((d_i - d_kj) - tau_j)
svd1_status apply_direct(int64_t rows, int n, const double* d, const int32_t* k,
                         const double* tau, const double* zhat, const double* cs,
                         const double* U_in, int64_t ld_in, const int32_t* src,
                         double* U_out, int64_t ld_out, const int32_t* dst,
                         cudaStream_t st, int64_t* launches);

// thin right factor: q[r] = (b[row0 + r] - sum_{c<m} V[r, c] y[c]) * inv_beta written into
// column m of V (the direction of b outside span(V); SVD1_THIN_V)
svd1_status null_direction(int64_t rows, double* V, int64_t ldv, int64_t m, const double* b, int64_t row0,
                           const double* y, double inv_beta, cudaStream_t st, int64_t* launches);

// thin V in a batch: the carried rows of later updates s get their coordinate along this
// update's q: rv[j][m] = (b_t . b_s - yt[:m] . rv[j][:m]) * inv_beta for j < rows, row j
// holding update s = K-1-j, b_t . b_s = gram[t K + s]; rv row-major with ld; yt = V_t^T b_t
svd1_status thin_carry(int rows, double* rv, int64_t ld, int64_t m, const double* yt, const double* gram, int t,
                       int K, double inv_beta, cudaStream_t st, int64_t* launches);
// gram[t * K + s] = b_t . b_s for t, s < K (rows of B, ld)
svd1_status gram_rows(int K, const double* B, int64_t ldb, int64_t n, double* gram, cudaStream_t st,
                      int64_t* launches);

// K11': the same product for a few rows (rows <= 32: the carried projection rows of a
// batch): thread per target j, sources split over blocks (partials in
// `scratch`, at least few_rows_scratch_elems doubles), ordered combine (deterministic).
int64_t few_rows_scratch_elems(int rows, int n);
svd1_status apply_few_rows(int rows, int n, const double* d, const int32_t* k, const double* tau,
                           const double* zhat, const double* cs, const double* U_in, int64_t ld_in,
                           const int32_t* src, double* U_out, int64_t ld_out, const int32_t* dst,
                           double* scratch, cudaStream_t st, int64_t* launches);

// K4: Householder column groups, in place: for each group g, cols idx[off_g..off_g+len_g)
// U[:, idx] <- U[:, idx] (I - 2 v v^T / v^T v), v = hv[off_g..].
// maxlen: the longest group (<= 16: a warp per row over all groups, else a block per group)
svd1_status householder_cols(int64_t rows, double* U, int64_t ld, int ngroups,
                             const int32_t* goff, const int32_t* cols, const double* hv, int maxlen,
                             cudaStream_t st, int64_t* launches);
// pairing rotations: for group g with columns c_0..c_{k-1} (k <= 8) and row-major k x k R,
// U[r, c_b] <- sum_a U[r, c_a] R[a][b]  (in place)
svd1_status col_rotate(int64_t rows, double* U, int64_t ld, int ngroups, const int32_t* goff,
                       const int32_t* cols, const double* mats, cudaStream_t st, int64_t* launches, int max_k = 8);
// passthrough: U_out[r, dst[q]] = scale[q] * U_in[r, src[q]]
svd1_status passthrough(int64_t rows, int nq, const double* U_in, int64_t ld_in,
                        const int32_t* src, double* U_out, int64_t ld_out,
                        const int32_t* dst, const double* scale, cudaStream_t st,
                        int64_t* launches);

// ---------------------------------------------------------------- FMM
struct FmmCell {      // one tree cell: a contiguous range [lo, hi) of the merged sorted
                      // sequence of sources d_i and targets mu_j (2 n points)
  double c, r;        // centre and radius of the hull of its points
  int32_t lo, hi;     // merged range
  int32_t slo, shi;   // its sources  d_slo .. d_{shi-1}
  int32_t tlo, thi;   // its targets mu_tlo .. mu_{thi-1}
};
enum FmmOpKind : int32_t {
  OP_P2M = 0, OP_M2M = 1, OP_M2L = 2, OP_L2L = 3, OP_L2P = 4, OP_P2P = 5,
  OP_P2L = 6,       // sources of a cell with fewer than p points straight into a local expansion
  OP_ID = 7,        // p x p identity (in-place accumulation of the L2L chain)
  OP_L2P_FROM = 8,  // local expansion of cell a evaluated at the targets of leaf b
  OP_M2P = 9        // far field of leaf a evaluated at the targets of leaf b (adaptive W list)
};
struct FmmOpDesc {    // one operator block: rows x cols, written into its term's op
  int32_t kind, a, b; // a = source cell (expansion kinds) or first source index (source
                      // kinds P2M/P2L/P2P); b = target-side cell
  int32_t rows, cols;
  int32_t kb;         // first k (row) of this block inside the term's op
  int32_t npad;       // the term's op: chunks of [npad][16] doubles (see FmmTerm)
  int32_t nb;         // first n (column) of this block inside the term's op (a task over
                      // two sibling targets holds each target's block in its own columns)
  int64_t op_row;     // the term's first 16-double row in the ops buffer
  int32_t c0, s_hi;   // source kinds: row q <-> input column c0 + q, holding active source
                      // s = col2src[c0 + q]; rows with s outside [a, s_hi) are zero
};
enum FmmIoKind : int32_t { IO_U = 0, IO_PHI = 1, IO_PSI = 2 };
// Expansions are stored as row-major matrices Phi, Psi (rows x ldE, ldE = ncells * p):
// cell c's p coefficients of row r at [r * ldE + c * p].  Adjacent cells are adjacent
// columns, so consecutive interaction partners merge into one long-K term.
struct FmmTerm {      // in[:, col0 : col0 + K] * op (K x N)
  int32_t in_kind;    // IO_U (physical columns of U_in) or IO_PHI / IO_PSI
  int32_t col0;
  int32_t K;
  int32_t npad;       // op stored chunk-transposed: chunk c (k = 16c .. 16c+15) is an
                      // [npad][16] block at ops row op_row + c*npad (zero past K and N)
  int64_t op_row;
};
struct FmmTask {      // out[:, col0 : col0 + N] = sum of terms
  int32_t out_kind;   // IO_U (columns mapped through dst[]) or IO_PHI / IO_PSI
  int32_t col0;
  int32_t N;
  int32_t t_begin, t_end;
  int32_t op_col0;    // column offset into every term's op (tasks split along N)
};
svd1_status fmm_build_ops(int n_ops, const FmmOpDesc* descs, const FmmCell* cells, int p,
                          const double* d, const int32_t* k, const double* tau,
                          const double* zhat, const double* cs, const int32_t* col2src,
                          double* ops, int64_t ops_elems, cudaStream_t st, int64_t* launches);
// One pass: every task's output block for all rows.  bn = 16 or 32 (>= every task N).
// Terms read physical column windows of U_in (col0 even) or of Phi/Psi; op rows are
// 16-byte aligned with even op_ld; the ops buffer has kOpsPad doubles of slack.
// TMA descriptors of one apply (per tile width: [0] BN = 16, [1] BN = 32)
struct FmmMaps {
  CUtensorMap u[2], phi[2], psi[2];
};
// U_in must be 16-byte aligned with even ld (the host pads otherwise)
svd1_status fmm_make_maps(FmmMaps* m, int64_t rows, const double* U_in, int64_t ncols_in, int64_t ld_in,
                          const double* phi, const double* psi, int64_t ldE);
// tile_ctr (device int, zero on entry; nullptr: static striding): the pass's tiles are
// claimed with an atomic counter in the host's longest-first order; rb_major: tile order
// row-block-major instead of task-major (kernels_apply.cu, tile_task)
svd1_status fmm_run_tasks(int n_tasks, const FmmTask* tasks, const FmmTerm* terms, int bn,
                          int64_t rows, const FmmMaps* maps /* device */, double* U_out, int64_t ld_out,
                          const int32_t* dst, double* phi, double* psi, int64_t ldE, int64_t out_cols,
                          int64_t exp_elems, const double* ops_raw, int64_t ops_rows, int* tile_ctr,
                          int rb_major, cudaStream_t st, int64_t* launches);


}  // namespace svd1
