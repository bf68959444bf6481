// Cauchy-apply kernels of the rank-1 SVD update (sm_100a, fp64 tensor cores):
//   K11 direct Cauchy-on-the-fly apply: U_out = U_in diag(zhat) C diag(colscale),
//       C_ij = 1/((d_i - d_kj) - tau_j)   (Alg 6.2 STEPS 3-7 P:365-377)
//   K5  FMM operator construction (re-derived: DESIGN.md §4.4)
//   K6-K10 FMM passes as row-batched small GEMMs (P2M, M2M, M2L, L2L, L2P, P2P;
//       P:727-796) — all rows of U are right-hand sides sharing one tree.
//   K4  Householder deflation transforms on column groups
// FP64 tensor work uses mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4): tcgen05 has no fp64 kind.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "svd1_internal.cuh"

namespace svd1 {
namespace {

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// ------------------------------------------------------------------- K11
constexpr int DBM = 128, DBN = 64, DBK = 16;
constexpr int DLDA = DBK + 4;  // 20 doubles: conflict-free A fragment loads
constexpr int DLDB = DBN + 4;  // 68 doubles: conflict-free B fragment loads

__global__ void __launch_bounds__(256) apply_direct_kernel(
    int64_t rows, int n, const double* __restrict__ d, const int32_t* __restrict__ k,
    const double* __restrict__ tau, const double* __restrict__ zhat, const double* __restrict__ cs,
    const double* __restrict__ U_in, int64_t ld_in, const int32_t* __restrict__ src,
    double* __restrict__ U_out, int64_t ld_out, const int32_t* __restrict__ dst) {
  __shared__ double As[DBM * DLDA];
  __shared__ double Bs[DBK * DLDB];
  __shared__ double s_dk[DBN], s_tau[DBN], s_cs[DBN];
  __shared__ double s_di[DBK], s_zi[DBK];
  __shared__ int32_t s_src[DBK];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp & 3, wn = warp >> 2;  // 4 x 2 warps, warp tile 32 x 32
  const int64_t row0 = int64_t(blockIdx.y) * DBM;
  const int j0 = blockIdx.x * DBN;
  if (tid < DBN) {
    const int j = j0 + tid;
    if (j < n) {
      s_dk[tid] = d[k[j]];
      s_tau[tid] = tau[j];
      s_cs[tid] = cs[j];
    } else {
      s_dk[tid] = 0.0;
      s_tau[tid] = 1.0;
      s_cs[tid] = 0.0;
    }
  }
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  for (int i0 = 0; i0 < n; i0 += DBK) {
    __syncthreads();
    if (tid < DBK) {
      const int i = i0 + tid;
      s_di[tid] = (i < n) ? d[i] : 0.0;
      s_zi[tid] = (i < n) ? zhat[i] : 0.0;
      s_src[tid] = (i < n) ? (src ? src[i] : i) : 0;
    }
    __syncthreads();
    // A: 128 rows x 16 sources, 8 per thread; consecutive threads -> consecutive sources
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int idx = tid + e * 256;
      const int rr = idx >> 4, kk = idx & 15;
      const int64_t r = row0 + rr;
      double v = 0.0;
      if (r < rows && i0 + kk < n) v = __ldg(U_in + r * ld_in + s_src[kk]);
      As[rr * DLDA + kk] = v;
    }
    // B generated on the fly: zhat_i cs_j / ((d_i - d_kj) - tau_j), 4 per thread
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int idx = tid + e * 256;
      const int kk = idx >> 6, jj = idx & 63;
      // padded sources (i >= n) and targets (j >= n) get exact zeros: a padding d_i = 0
      // meets a root mu_j = 0 (the null-space root of a rank-deficient side) as 0 / 0
      const double del = (s_di[kk] - s_dk[jj]) - s_tau[jj];
      Bs[kk * DLDB + jj] = (i0 + kk < n && j0 + jj < n) ? (s_zi[kk] * s_cs[jj]) / del : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < DBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = As[(wm * 32 + mt * 8 + (lane >> 2)) * DLDA + kk + (lane & 3)];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = Bs[(kk + (lane & 3)) * DLDB + wn * 32 + nt * 8 + (lane >> 2)];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma_8x8x4(acc[mt][nt], af[mt], bf[nt]);
    }
  }
  // epilogue: C fragment (row = lane/4, cols 2*(lane%4) + {0,1})
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int64_t r = row0 + wm * 32 + mt * 8 + (lane >> 2);
    if (r >= rows) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = j0 + wn * 32 + nt * 8 + (lane & 3) * 2 + h;
        if (j < n) U_out[r * ld_out + (dst ? dst[j] : j)] = acc[mt][nt][h];
      }
    }
  }
}

// ------------------------------------------------------------------- K4
__global__ void __launch_bounds__(256) householder_kernel(int64_t rows, double* __restrict__ U,
                                                         int64_t ld, const int32_t* __restrict__ goff,
                                                         const int32_t* __restrict__ cols,
                                                         const double* __restrict__ hv) {
  const int g = blockIdx.y;
  const int o0 = goff[g], o1 = goff[g + 1], len = o1 - o0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ double s_vv;
  if (warp == 0) {
    double s = 0.0;
    for (int t = lane; t < len; t += 32) s = fma(hv[o0 + t], hv[o0 + t], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) s_vv = s;
  }
  __syncthreads();
  const double coef = 2.0 / s_vv;
  const int64_t rbase = int64_t(blockIdx.x) * 32;
  for (int rr = warp; rr < 32; rr += 8) {
    const int64_t r = rbase + rr;
    if (r >= rows) break;
    double* row = U + r * ld;
    double s = 0.0;
    for (int t = lane; t < len; t += 32) s = fma(row[cols[o0 + t]], hv[o0 + t], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const double f = coef * s;
    for (int t = lane; t < len; t += 32) {
      const int c = cols[o0 + t];
      row[c] = fma(-f, hv[o0 + t], row[c]);
    }
  }
}

// K4 for many small groups (C5: ~800 pairs of bitwise-equal sigma^2): a warp per row,
// lanes over the groups (a group's few columns are read once, transformed in registers,
// written once); the block-per-(rows, group) kernel above keeps the long groups (C4's
// null space: one group of n - m columns).
__global__ void __launch_bounds__(256) householder_rows_kernel(int64_t rows, double* __restrict__ U, int64_t ld,
                                                              int ngroups, const int32_t* __restrict__ goff,
                                                              const int32_t* __restrict__ cols,
                                                              const double* __restrict__ hv) {
  constexpr int kMaxSmall = 16;
  const int lane = threadIdx.x & 31;
  const int64_t r = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (r >= rows) return;
  double* row = U + r * ld;
  for (int g = lane; g < ngroups; g += 32) {
    const int o0 = goff[g], len = min(goff[g + 1] - o0, kMaxSmall);
    double x[kMaxSmall], v[kMaxSmall];
    double vv = 0.0, dot = 0.0;
#pragma unroll
    for (int t = 0; t < kMaxSmall; ++t)
      if (t < len) {
        v[t] = hv[o0 + t];
        x[t] = row[cols[o0 + t]];
        vv = fma(v[t], v[t], vv);
        dot = fma(x[t], v[t], dot);
      }
    const double f = (2.0 / vv) * dot;
#pragma unroll
    for (int t = 0; t < kMaxSmall; ++t)
      if (t < len) row[cols[o0 + t]] = fma(-f, v[t], x[t]);
  }
}

__global__ void col_rotate_kernel(int64_t rows, double* __restrict__ U, int64_t ld,
                                  const int32_t* __restrict__ goff, const int32_t* __restrict__ cols,
                                  const double* __restrict__ mats) {
  const int g = blockIdx.y;
  const int o0 = goff[g], k = goff[g + 1] - o0;
  int64_t moff = 0;  // groups' matrices are stored back to back
  for (int h = 0; h < g; ++h) {
    const int kh = goff[h + 1] - goff[h];
    moff += int64_t(kh) * kh;
  }
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows || k > 8) return;
  double v[8], o[8];
  for (int a = 0; a < k; ++a) v[a] = U[r * ld + cols[o0 + a]];
  for (int b = 0; b < k; ++b) {
    double acc = 0.0;
    for (int a = 0; a < k; ++a) acc = fma(v[a], mats[moff + a * k + b], acc);
    o[b] = acc;
  }
  for (int b = 0; b < k; ++b) U[r * ld + cols[o0 + b]] = o[b];
}

// The same rotation for groups of more than 8 columns (D5 clusters paired from the tracked
// coordinates, up to 256 columns): a block per 8 rows and group, the rows' k values staged in
// shared memory before any is overwritten.
constexpr int kRotRows = 8;
__global__ void __launch_bounds__(256) col_rotate_big_kernel(int64_t rows, double* __restrict__ U, int64_t ld,
                                                             const int32_t* __restrict__ goff,
                                                             const int32_t* __restrict__ cols,
                                                             const double* __restrict__ mats) {
  extern __shared__ double s_v[];  // [kRotRows][k]
  const int g = blockIdx.y;
  const int o0 = goff[g], k = goff[g + 1] - o0;
  if (k <= 8) return;
  int64_t moff = 0;
  for (int h = 0; h < g; ++h) {
    const int kh = goff[h + 1] - goff[h];
    moff += int64_t(kh) * kh;
  }
  const int64_t r0 = int64_t(blockIdx.x) * kRotRows;
  for (int e = threadIdx.x; e < kRotRows * k; e += blockDim.x) {
    const int rr = e / k, a = e % k;
    s_v[e] = r0 + rr < rows ? U[(r0 + rr) * ld + cols[o0 + a]] : 0.0;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kRotRows * k; e += blockDim.x) {
    const int rr = e / k, b = e % k;
    if (r0 + rr >= rows) continue;
    double acc = 0.0;
    for (int a = 0; a < k; ++a) acc = fma(s_v[rr * k + a], mats[moff + int64_t(a) * k + b], acc);
    U[(r0 + rr) * ld + cols[o0 + b]] = acc;
  }
}

__global__ void passthrough_kernel(int64_t rows, int nq, const double* __restrict__ U_in,
                                   int64_t ld_in, const int32_t* __restrict__ src,
                                   double* __restrict__ U_out, int64_t ld_out,
                                   const int32_t* __restrict__ dst, const double* __restrict__ scale) {
  const int q = blockIdx.x * 32 + (threadIdx.x & 31);
  const int64_t r = int64_t(blockIdx.y) * 8 + (threadIdx.x >> 5);
  if (q >= nq || r >= rows) return;
  U_out[r * ld_out + dst[q]] = scale[q] * U_in[r * ld_in + src[q]];
}

// ------------------------------------------------------------------- K5
// Chebyshev nodes t_k = cos((2k+1) pi / 2p) (k 0-based) and barycentric weights
// w_k = (-1)^k sin((2k+1) pi / 2p); u_k(t) = [w_k/(t - t_k)] / sum_m w_m/(t - t_m).

// blockIdx.y = 1: expansion kinds (M2M, M2L, L2L, L2P, L2P_FROM, M2P), a warp per
// operator block: they are Lagrange bases evaluated at a point that depends only on the
// column j, so lane j forms the barycentric denominator once and then the p rows (2p
// reciprocals and one division per column).  blockIdx.y = 0: source kinds (P2M, P2L, P2P)
// and ID, a block per operator, one reciprocal per element (MUFU seed + 2 Newton steps).
__device__ __forceinline__ bool is_lagrange(int kind) {
  return kind == OP_M2M || kind == OP_M2L || kind == OP_L2L || kind == OP_L2P || kind == OP_L2P_FROM ||
         kind == OP_M2P;
}

__device__ __forceinline__ double ops_rcp(double x) {  // 1/x to ~1 ulp: MUFU seed + 2 Newton steps
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__global__ void __launch_bounds__(256) fmm_ops_kernel(int n_ops, const FmmOpDesc* __restrict__ descs,
                                                     const FmmCell* __restrict__ cells, int p,
                                                     const double* __restrict__ d,
                                                     const int32_t* __restrict__ k,
                                                     const double* __restrict__ tau,
                                                     const double* __restrict__ zhat,
                                                     const double* __restrict__ cs,
                                                     const int32_t* __restrict__ col2src,
                                                     double* __restrict__ ops, int64_t ops_elems) {
  __shared__ double t[kMaxP], w[kMaxP];
  if (threadIdx.x < p) {
    const double th = (2.0 * threadIdx.x + 1.0) / (2.0 * p);  // in units of pi
    t[threadIdx.x] = cospi(th);
    w[threadIdx.x] = ((threadIdx.x & 1) ? -1.0 : 1.0) * sinpi(th);
  }
  __syncthreads();
  const bool lag_mode = blockIdx.y == 1;
  const int lane = threadIdx.x & 31;
  const int nunits = lag_mode ? gridDim.x * (blockDim.x >> 5) : gridDim.x;  // warps | blocks
  const int unit = lag_mode ? blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5) : blockIdx.x;
  const int ustride = lag_mode ? 32 : blockDim.x, uid = lag_mode ? lane : threadIdx.x;
  for (int o = unit; o < n_ops; o += nunits) {
    const FmmOpDesc D = descs[o];
    if (is_lagrange(D.kind) != lag_mode) continue;
    // chunk-transposed layout of the term's op: chunk (kb + i) / 16 is an [npad][16]
    // block (n-major, 16 k contiguous), the GEMM's B tile
    auto store = [&](int i, int j, double v) {
      const int kk = D.kb + i;
      j += D.nb;
#ifdef SVD1_BOUNDS
      if ((D.op_row + int64_t(kk >> 4) * D.npad + j) * 16 + (kk & 15) >= ops_elems || j >= D.npad) {
        printf("[svd1 bounds] ops desc %d kind %d row %lld kb %d rows %d cols %d npad %d\n", o, D.kind,
               (long long)D.op_row, D.kb, D.rows, D.cols, D.npad);
        __trap();
      }
#endif
      ops[(D.op_row + int64_t(kk >> 4) * D.npad + j) * 16 + (kk & 15)] = v;
    };
    if (is_lagrange(D.kind)) {
      for (int j = lane; j < D.cols; j += 32) {
        double x, f = 1.0;  // u_i(x) * f for rows i < p
        switch (D.kind) {
          case OP_M2M: {  // child (a) -> ancestor (b): i = child node, j = parent node
            const FmmCell C = cells[D.a], P = cells[D.b];
            const double den = 3.0 * P.r + t[j] * (P.c - C.c);
            x = 3.0 * C.r * t[j] / den;
            f = 3.0 * C.r / den;
            break;
          }
          case OP_M2L: {  // source X (a) -> target Y (b): i = X node, j = Y node
            const FmmCell X = cells[D.a], Y = cells[D.b];
            x = 3.0 * X.r / ((Y.c - X.c) + Y.r * t[j]);
            f = x;
            break;
          }
          case OP_L2L: {  // ancestor (a) -> cell (b): i = ancestor node, j = cell node
            const FmmCell P = cells[D.a], C = cells[D.b];
            x = ((C.c - P.c) + C.r * t[j]) / P.r;
            break;
          }
          case OP_L2P: {  // leaf Y (b): i = node, j = target
            const FmmCell Y = cells[D.b];
            const int jt = Y.tlo + j;
            x = ((d[k[jt]] - Y.c) + tau[jt]) / Y.r;
            f = cs[jt];
            break;
          }
          case OP_M2P: {  // far field of leaf a at the targets of leaf b: t_X = 3 r_X / (mu_j - c_X)
            const FmmCell X = cells[D.a], Y = cells[D.b];
            const int jt = Y.tlo + j;
            x = 3.0 * X.r / ((d[k[jt]] - X.c) + tau[jt]);
            f = x * cs[jt];
            break;
          }
          default: {  // OP_L2P_FROM: expansion of cell a (an ancestor) at the targets of leaf b
            const FmmCell A = cells[D.a], Y = cells[D.b];
            const int jt = Y.tlo + j;
            x = ((d[k[jt]] - A.c) + tau[jt]) / A.r;
            f = cs[jt];
            break;
          }
        }
        // barycentric form u_i(x) = (w_i / (x - t_i)) / sum_m w_m / (x - t_m), with
        // reciprocals by MUFU + Newton (<= 1 ulp) and one division for the column's scale
        // (instead of 3p IEEE divisions per column)
        double den = 0.0;
        int hit = -1;
        for (int m = 0; m < p; ++m) {
          const double dx = x - t[m];
          if (dx == 0.0) hit = m;
          else den = fma(w[m], ops_rcp(dx), den);
        }
        const double sc = f / den;
        for (int i = 0; i < D.rows; ++i) {
          const double dx = x - t[i];
          store(i, j, hit >= 0 ? (i == hit ? f : 0.0) : (w[i] * ops_rcp(dx)) * sc);
        }
      }
      continue;
    }
    const int total = D.rows * D.cols;
    for (int e = uid; e < total; e += ustride) {
      const int i = e / D.cols, j = e % D.cols;
      double v = 0.0;
      switch (D.kind) {
        case OP_ID: {
          v = (i == j) ? 1.0 : 0.0;
          break;
        }
        default: {  // source kinds: row i holds input column c0 + i (zero unless an active
                    // source of the term's range [a, s_hi) sits there)
          int s = col2src ? col2src[D.c0 + i] : D.c0 + i;
          if (s < D.a || s >= D.s_hi) break;
          if (D.kind == OP_P2M) {  // Phi~_X[j] += zhat_s U_s / (t_j (x_s - c_X) - 3 r_X), X = b
            const FmmCell X = cells[D.b];
            v = zhat[s] * ops_rcp(t[j] * (d[s] - X.c) - 3.0 * X.r);
          } else if (D.kind == OP_P2L) {  // source s -> local expansion of Y (b) at c_Y + r_Y t_j
            const FmmCell Y = cells[D.b];
            v = zhat[s] * ops_rcp((d[s] - Y.c) - Y.r * t[j]);
          } else {  // OP_P2P: source s, target leaf Y (b)
            const FmmCell Y = cells[D.b];
            const int jt = Y.tlo + j;
            v = (zhat[s] * cs[jt]) * ops_rcp((d[s] - d[k[jt]]) - tau[jt]);
          }
          break;
        }
      }
      store(i, j, v);
    }
  }
}

// ------------------------------------------------------------------- K6-K10
// One FMM pass = a batch of "gathered small GEMMs": for task T and every row,
//   out[r, T.col0 : T.col0 + N] = sum_t in_t[r, col0_t : col0_t + K_t] * op_t (K_t x N).
// in = U (physical column windows resolved on the host) or the expansion matrices
// Phi/Psi; out = U (through dst[]) or Phi/Psi.
//
// Warp-specialised persistent kernel.  One producer warp walks the CTA's tiles (task,
// block of BM rows; stride gridDim.x; tasks ordered longest first by the host) and, per
// 16-wide K chunk, fills one slot of a STAGES-deep ring: the A tile (BM rows x 16
// columns of U / Phi / Psi) by one TMA load (rows past `rows` and columns past the
// matrix arrive as zeros), the B tile (the op chunk, stored transposed as [n][16 k]) by
// cp.async from the warp's 32 lanes; both land 128B-swizzled.  CW consumer warps (32 rows each) wait on the stage's full mbarrier,
// read their fragments with conflict-free 16-byte loads, run the DMMAs and release the
// stage on its empty mbarrier -- no CTA barrier and no address arithmetic in the math
// loop.  Within a chunk, lane t4 carries k = 4 t4 + q in k-step q (the same permutation
// for A and B, so the sum over k is unchanged), which makes each lane's four A (and
// B) values for the chunk one contiguous 32-byte run.  Op chunks are zero past K, so
// the A columns of a chunk that fall outside the term only ever meet zeros.
constexpr int KC = 16;  // chunk (k) width: one 128-byte swizzle row of doubles
#ifndef SVD1_STAGES16
#define SVD1_STAGES16 4   // ring depth of the 16-wide passes (3 CTAs / SM; measured best)
#endif
#ifndef SVD1_STAGES32
#define SVD1_STAGES32 3   // ring depth of the 32-wide passes (3 CTAs / SM; measured best)
#endif

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ double2 lds128(const unsigned char* p) {
  return *reinterpret_cast<const double2*>(p);
}

#ifndef SVD1_CW16
#define SVD1_CW16 4  // consumer warps of the 16-wide passes (experiments)
#endif
#ifndef SVD1_CW32
#define SVD1_CW32 4  // consumer warps of the 32-wide passes (experiments)
#endif
#ifndef SVD1_MT16
#define SVD1_MT16 4  // 8-row m-tiles per consumer warp of the 16-wide passes (experiments)
#endif
#ifndef SVD1_MT32
#define SVD1_MT32 4  // the same for the 32-wide passes
#endif
#ifndef SVD1_CPS16
#define SVD1_CPS16 1  // KC-column chunks per ring stage of the 16-wide passes (experiments)
#endif
#ifndef SVD1_CPS32
#define SVD1_CPS32 1  // the same for the 32-wide passes
#endif
template <int BN>
struct GemmCfg {
  static constexpr int CPS = BN <= 16 ? SVD1_CPS16 : SVD1_CPS32;  // chunks per stage
  static constexpr int CW = BN <= 16 ? SVD1_CW16 : SVD1_CW32;  // consumer warps (RW rows each)
  static constexpr int MT = BN <= 16 ? SVD1_MT16 : SVD1_MT32;  // 8-row m-tiles per consumer warp
  static constexpr int RW = 8 * MT;
  static constexpr int NTHR = 32 * (CW + 1); // + one producer warp
  static constexpr int NT = BN / 8;
  static constexpr int BM = RW * CW;
  static constexpr int STAGES = BN <= 16 ? SVD1_STAGES16 : SVD1_STAGES32;
  static constexpr int A_BYTES = BM * KC * 8;
  static constexpr int B_BYTES = BN * KC * 8;
  static constexpr int STAGE_A = CPS * A_BYTES, STAGE_B = CPS * B_BYTES;
  static constexpr int STAGE_BYTES = STAGE_A + STAGE_B;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + STAGES * (16 + 16);
};

// Tile -> (task, row block).  Task-major (default): consecutive CTAs take the same task's
// row blocks (its operator chunks stay hot, the A windows stream down the rows).
// Row-block-major (per pass, chosen by the host): the CTAs in flight cover a few row
// blocks and every task, so shared input rows are re-read from L2 -- measured at C3 for
// every pass: DRAM per apply 1.26 -> 1.10 GB, but 481 -> 505 us (the final pass loses);
// the host uses it for the 16-wide passes (svd1_host.cu, rb_kinds).
__device__ __forceinline__ int tile_task(int tile, int nrb, int ntask, int rb_major) {
  return rb_major ? tile % ntask : tile / nrb;
}
__device__ __forceinline__ int tile_rb(int tile, int nrb, int ntask, int rb_major) {
  return rb_major ? tile / ntask : tile % nrb;
}

struct StageInfo {
  int32_t tile;   // tile the chunk belongs to; -1: no more chunks
  int32_t last;   // bit 0: last chunk of the tile (epilogue after it); CPS > 1: the stage's
                  // KC-column chunks (1 .. CPS) in bits 8..; -1: end of the ring
  int32_t kindN;  // the tile's task: out_kind << 8 | N (read by the epilogue from shared
  int32_t col0;   //   memory, not from global memory)
};

#ifndef SVD1_MINB32
#define SVD1_MINB32 3  // resident CTAs per SM the 32-wide kernel is compiled for: <= 128 registers
                       // (153 unconstrained: 2 CTAs / SM); C3 stream 430 -> 436-440 updates/s
#endif
#ifndef SVD1_MINB16
#define SVD1_MINB16 1  // the same for the 16-wide kernel (101 registers: 3 CTAs / SM; experiments)
#endif
template <int BN>
__global__ void __launch_bounds__(GemmCfg<BN>::NTHR, BN == 32 ? SVD1_MINB32 : SVD1_MINB16) fmm_gemm_kernel(
    const FmmMaps* __restrict__ maps, const FmmTask* __restrict__ tasks, const FmmTerm* __restrict__ terms, int ntiles, int nrb,
    int ntask, int rb_major, int* __restrict__ tile_ctr,
    int64_t rows, double* __restrict__ U_out, int64_t ld_out, const int32_t* __restrict__ dst,
    double* __restrict__ phi, double* __restrict__ psi, int64_t ldE, int64_t out_cols, int64_t exp_elems,
    const double* __restrict__ ops_raw, int64_t ops_rows) {
  using G = GemmCfg<BN>;
  constexpr int NT = G::NT, S = G::STAGES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // SWIZZLE_128B tiles need 1024-byte aligned shared addresses
  unsigned char* sbase = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char* sA = sbase;                   // [S][CPS][BM][16] doubles, swizzled
  unsigned char* sB = sbase + S * G::STAGE_A;  // [S][CPS][BN][16] doubles, swizzled
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + S * G::STAGE_B);
  uint64_t* empty = full + S;
  StageInfo* info = reinterpret_cast<StageInfo*>(empty + S);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int q = 0; q < S; ++q) {
      mbar_init(&full[q], 33);
      mbar_init(&empty[q], G::CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp == G::CW) {  // ---------------- producer warp
    // A tiles by TMA (lane 0); B tiles (the op chunk, [BN][16] doubles, 2-4 KB) by
    // cp.async from all 32 lanes into the same 128B-swizzled layout, their completion
    // tracked by the stage's full barrier (32 noinc arrivals + lane 0's expect_tx).
    // (A TMA load of the op chunk, written by the operator kernel just before, was
    // measured to return stale data when another stream's kernels ran concurrently.)
    // Descriptors: the next tile's task is loaded while this tile's chunks are issued, and
    // a task's terms are loaded once, one per lane (no global round trip per term).  (A
    // pipeline two tiles deep -- the next tile's terms in flight too -- measured the same.)
    const int w = BN == 32 ? 1 : 0;
    const CUtensorMap* tm_u = &maps->u[w];
    const CUtensorMap* tm_phi = &maps->phi[w];
    const CUtensorMap* tm_psi = &maps->psi[w];
    if (lane == 0)
      for (const CUtensorMap* m : {tm_u, tm_phi, tm_psi})
        asm volatile("fence.proxy.tensormap::generic.acquire.gpu [%0], 128;\n" ::"l"(m) : "memory");
    int stage = 0;
    uint32_t phase = 0;
    // tiles are claimed dynamically (an atomic counter per pass, in the host's longest-first
    // order) when tile_ctr is given, else strided by the grid
    auto claim = [&]() -> int {
      int tl = 0;
      if (lane == 0) tl = atomicAdd(tile_ctr, 1);
      return __shfl_sync(0xffffffffu, tl, 0);
    };
    int tile = tile_ctr ? claim() : int(blockIdx.x);
    FmmTask T{};
    if (tile < ntiles) T = tasks[tile_task(tile, nrb, ntask, rb_major)];
    while (tile < ntiles) {
      const int next = tile_ctr ? claim() : tile + int(gridDim.x);
      FmmTask Tn{};
      if (next < ntiles) Tn = tasks[tile_task(next, nrb, ntask, rb_major)];  // in flight while this tile is issued
      const int row0 = tile_rb(tile, nrb, ntask, rb_major) * G::BM;
      const int32_t kindN = (T.out_kind << 8) | T.N;
      for (int tb = T.t_begin; tb < T.t_end; tb += 32) {
        FmmTerm mine{};
        if (tb + lane < T.t_end) mine = terms[tb + lane];
        const int nterm = min(32, T.t_end - tb);
        for (int q = 0; q < nterm; ++q) {
          const int in_kind = __shfl_sync(0xffffffffu, mine.in_kind, q);
          const int col0 = __shfl_sync(0xffffffffu, mine.col0, q);
          const int K = __shfl_sync(0xffffffffu, mine.K, q);
          const int npad = __shfl_sync(0xffffffffu, mine.npad, q);
          const int64_t op_row = __shfl_sync(0xffffffffu, mine.op_row, q);
          const CUtensorMap* ma = in_kind == IO_U ? tm_u : (in_kind == IO_PHI ? tm_phi : tm_psi);
          const bool last_term = tb + q == T.t_end - 1;
          for (int k0 = 0; k0 < K; k0 += KC * G::CPS) {
            const int nch = G::CPS == 1 ? 1 : min(G::CPS, (K - k0 + KC - 1) / KC);
            mbar_wait(&empty[stage], phase ^ 1);
            for (int c = 0; c < nch; ++c) {
              const int64_t brow = op_row + int64_t((k0 + c * KC) / KC) * npad + T.op_col0;
              const double* bsrc = ops_raw + brow * 16;
              unsigned char* bdst = sB + stage * G::STAGE_B + c * G::B_BYTES;
              for (int e = lane; e < BN * 8; e += 32) {
                const int n = e >> 3, j = e & 7;
                const int64_t row = brow + n;
                const bool ok = row < ops_rows;
                const unsigned sa = smem_u32(bdst + n * 128 + ((j ^ (n & 7)) << 4));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa),
                             "l"(bsrc + (ok ? n * 16 + 2 * j : 0)), "r"(ok ? 16 : 0));
              }
            }
            if (lane == 0) {
              info[stage] = StageInfo{tile, ((last_term && k0 + KC * G::CPS >= K) ? 1 : 0) | (G::CPS > 1 ? nch << 8 : 0),
                                      kindN, T.col0};
              mbar_arrive_tx(&full[stage], uint32_t(nch * G::A_BYTES));
              for (int c = 0; c < nch; ++c)
                tma_load_2d(sA + stage * G::STAGE_A + c * G::A_BYTES, ma, col0 + k0 + c * KC, row0, &full[stage]);
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full[stage])) : "memory");
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
      tile = next;
      T = Tn;
    }
    mbar_wait(&empty[stage], phase ^ 1);
    if (lane == 0) info[stage] = StageInfo{-1, -1, 0, 0};
    __syncwarp();
    mbar_arrive(&full[stage]);
    if (lane == 0) mbar_arrive(&full[stage]);  // 33 arrivals per phase
    return;
  }
  // ------------------------------------ consumers: warp owns rows warp*RW .. +RW-1
  const int g = lane >> 2, t4 = lane & 3;
  // byte offsets (within a stage) of this lane's 16-byte fragment runs: row r, k pair j
  // sits at r*128 + ((j ^ (r & 7)) << 4) (TMA SWIZZLE_128B); r & 7 == g for every row
  // this lane reads (fragment rows are 8-aligned)
  const int sw0 = ((2 * t4) ^ g) << 4, sw1 = ((2 * t4 + 1) ^ g) << 4;
  constexpr int MT = G::MT, RW = G::RW;
  const int a_row = (warp * RW + g) * 128;
  const int b_row = g * 128;
  double acc[MT][NT][2];
#pragma unroll
  for (int x = 0; x < MT; ++x)
#pragma unroll
    for (int y = 0; y < NT; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
  int stage = 0;
  uint32_t phase = 0;
  int cur_tile = -1;
  int dcol[NT][2];  // output columns of this lane's accumulators (IO_U: through dst[]),
                    // loaded at the tile's first chunk, used by its epilogue
  for (;;) {
    mbar_wait(&full[stage], phase);
    const StageInfo I = info[stage];
    if (I.last < 0) break;
    if (I.tile != cur_tile) {
      cur_tile = I.tile;
      const int N = I.kindN & 255;
      if ((I.kindN >> 8) == IO_U) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int jj = nt * 8 + 2 * t4;
          const int col = I.col0 + jj;
          dcol[nt][0] = jj < N ? (dst ? __ldg(dst + col) : col) : -1;
          dcol[nt][1] = jj + 1 < N ? (dst ? __ldg(dst + col + 1) : col + 1) : -1;
        }
      }
    }
#pragma unroll 1
    for (int c = 0; c < (G::CPS == 1 ? 1 : (I.last >> 8)); ++c) {
    const unsigned char* a = sA + stage * G::STAGE_A + c * G::A_BYTES + a_row;
    const unsigned char* b = sB + stage * G::STAGE_B + c * G::B_BYTES + b_row;
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // k-steps q = 2h, 2h + 1
      const int sw = h ? sw1 : sw0;
      double2 af[MT], bf[NT];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) af[mt] = lds128(a + mt * 8 * 128 + sw);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[nt] = lds128(b + nt * 8 * 128 + sw);
      // every accumulator's first k-step, then every accumulator's second: 4 NT
      // independent DMMAs between two that share an accumulator
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], af[mt].x, bf[nt].x);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], af[mt].y, bf[nt].y);
    }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == S) {
      stage = 0;
      phase ^= 1;
    }
    if (G::CPS == 1 ? I.last : (I.last & 1)) {  // epilogue of tile I.tile (registers -> global)
      const int task = tile_task(I.tile, nrb, ntask, rb_major);
      const int64_t row0 = int64_t(tile_rb(I.tile, nrb, ntask, rb_major)) * G::BM;
      (void)task;
      const int out_kind = I.kindN >> 8, N = I.kindN & 255;
      double* E = out_kind == IO_PHI ? phi : psi;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int jj = nt * 8 + 2 * t4;
        if (jj >= N) continue;
        const int col = I.col0 + jj;
        if (out_kind == IO_U) {
          const int c0 = dcol[nt][0], c1 = dcol[nt][1];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int64_t r = row0 + warp * RW + mt * 8 + g;
            if (r >= rows) continue;
#ifdef SVD1_BOUNDS
            if (c0 < 0 || c0 >= out_cols || c1 >= out_cols) {
              printf("[svd1 bounds] U_out col %d/%d of %lld (task %d N %d col %d)\n", c0, c1, (long long)out_cols,
                     task, N, col);
              __trap();
            }
#endif
            U_out[r * ld_out + c0] = acc[mt][nt][0];
            if (c1 >= 0) U_out[r * ld_out + c1] = acc[mt][nt][1];
          }
        } else {  // expansions: N is a multiple of 4, col0 even -> 16-byte stores
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            const int64_t r = row0 + warp * RW + mt * 8 + g;
            if (r >= rows) continue;
#ifdef SVD1_BOUNDS
            if (col + 1 >= ldE || r * ldE + col + 1 >= exp_elems) {
              printf("[svd1 bounds] expansion col %d ldE %lld r %lld elems %lld\n", col, (long long)ldE,
                     (long long)r, (long long)exp_elems);
              __trap();
            }
#endif
            *reinterpret_cast<double2*>(E + r * ldE + col) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
          }
        }
      }
#pragma unroll
      for (int x = 0; x < MT; ++x)
#pragma unroll
        for (int y = 0; y < NT; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;
    }
  }
}

}  // namespace

// ------------------------------------------------------------------ wrappers
svd1_status apply_direct(int64_t rows, int n, const double* d, const int32_t* k,
                         const double* tau, const double* zhat, const double* cs,
                         const double* U_in, int64_t ld_in, const int32_t* src,
                         double* U_out, int64_t ld_out, const int32_t* dst,
                         cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || n <= 0) return SVD1_OK;
  dim3 grid(unsigned((n + DBN - 1) / DBN), unsigned((rows + DBM - 1) / DBM));
  apply_direct_kernel<<<grid, 256, 0, st>>>(rows, n, d, k, tau, zhat, cs, U_in, ld_in, src, U_out,
                                            ld_out, dst);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

// ------------------------------------------------------------------ K11' few rows
// part[s][r][j] = sum_{i in split s} U_in[r, src_i] zhat_i / ((d_i - d_kj) - tau_j): thread
// per target j (128 per block), the split's sources staged 32 at a time with their rows;
// RB = rows rounded up (registers).  Then U_out[r, dst_j] = cs_j sum_s part[s][r][j].
#ifndef SVD1_FEW_CHUNK
#define SVD1_FEW_CHUNK 256
#endif
constexpr int kFewSplitChunk = SVD1_FEW_CHUNK;  // sources per split (many blocks: latency-bound work)

__device__ __forceinline__ double few_rcp(double x) {  // 1/x to ~1 ulp: MUFU seed + 2 Newton steps
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
template <int RB>
__global__ void __launch_bounds__(128) few_rows_partial_kernel(
    int rows, int n, const double* __restrict__ d, const int32_t* __restrict__ k,
    const double* __restrict__ tau, const double* __restrict__ zhat, const double* __restrict__ U_in,
    int64_t ld_in, const int32_t* __restrict__ src, double* __restrict__ part) {
  __shared__ double s_u[RB][32];
  __shared__ double s_d[32], s_z[32];
  const int j = blockIdx.x * 128 + threadIdx.x;
  const int i_lo = blockIdx.y * kFewSplitChunk, i_hi = min(n, i_lo + kFewSplitChunk);
  const double dk = j < n ? d[k[j]] : 0.0, tj = j < n ? tau[j] : 1.0;
  double acc[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) acc[r] = 0.0;
  for (int i0 = i_lo; i0 < i_hi; i0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < RB * 32; e += 128) {
      const int r = e >> 5, ii = e & 31, i = i0 + ii;
      s_u[r][ii] = (r < rows && i < i_hi) ? U_in[int64_t(r) * ld_in + (src ? src[i] : i)] : 0.0;
    }
    if (threadIdx.x < 32) {
      const int i = i0 + threadIdx.x;
      s_d[threadIdx.x] = i < i_hi ? d[i] : 0.0;
      s_z[threadIdx.x] = i < i_hi ? zhat[i] : 0.0;
    }
    __syncthreads();
    // padded sources (ii >= cnt) are skipped, not weighted by zero: d = 0 meets a root
    // mu_j = 0 as 0 / 0 (see apply_direct_kernel)
    const int cnt = min(32, i_hi - i0);
#pragma unroll 4
    for (int ii = 0; ii < 32; ++ii) {
      const double c = ii < cnt ? s_z[ii] * few_rcp((s_d[ii] - dk) - tj) : 0.0;
#pragma unroll
      for (int r = 0; r < RB; ++r) acc[r] = fma(c, s_u[r][ii], acc[r]);
    }
  }
  if (j < n) {
    const int64_t base = int64_t(blockIdx.y) * rows * n;
#pragma unroll
    for (int r = 0; r < RB; ++r)
      if (r < rows) part[base + int64_t(r) * n + j] = acc[r];
  }
}

// The same partial sums with TWO targets per thread (j and j + 128): every broadcast
// shared-memory read of a carried row's source value feeds two FMAs (the rows x n^2 products
// of the carried rows are FP64-ALU work whose shared-memory reads were the other half)
template <int RB>
__global__ void __launch_bounds__(128) few_rows_partial2_kernel(
    int rows, int n, const double* __restrict__ d, const int32_t* __restrict__ k,
    const double* __restrict__ tau, const double* __restrict__ zhat, const double* __restrict__ U_in,
    int64_t ld_in, const int32_t* __restrict__ src, double* __restrict__ part) {
  __shared__ double s_u[RB][32];
  __shared__ double s_d[32], s_z[32];
  const int j0 = blockIdx.x * 256 + threadIdx.x, j1 = j0 + 128;
  const int i_lo = blockIdx.y * kFewSplitChunk, i_hi = min(n, i_lo + kFewSplitChunk);
  const double dk0 = j0 < n ? d[k[j0]] : 0.0, t0 = j0 < n ? tau[j0] : 1.0;
  const double dk1 = j1 < n ? d[k[j1]] : 0.0, t1 = j1 < n ? tau[j1] : 1.0;
  double a0[RB], a1[RB];
#pragma unroll
  for (int r = 0; r < RB; ++r) a0[r] = a1[r] = 0.0;
  for (int i0 = i_lo; i0 < i_hi; i0 += 32) {
    __syncthreads();
    for (int e = threadIdx.x; e < RB * 32; e += 128) {
      const int r = e >> 5, ii = e & 31, i = i0 + ii;
      s_u[r][ii] = (r < rows && i < i_hi) ? U_in[int64_t(r) * ld_in + (src ? src[i] : i)] : 0.0;
    }
    if (threadIdx.x < 32) {
      const int i = i0 + threadIdx.x;
      s_d[threadIdx.x] = i < i_hi ? d[i] : 0.0;
      s_z[threadIdx.x] = i < i_hi ? zhat[i] : 0.0;
    }
    __syncthreads();
    const int cnt = min(32, i_hi - i0);
#pragma unroll 2
    for (int ii = 0; ii < 32; ++ii) {
      const double z = s_z[ii], di = s_d[ii];
      const double c0 = ii < cnt ? z * few_rcp((di - dk0) - t0) : 0.0;
      const double c1 = ii < cnt ? z * few_rcp((di - dk1) - t1) : 0.0;
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        const double u = s_u[r][ii];
        a0[r] = fma(c0, u, a0[r]);
        a1[r] = fma(c1, u, a1[r]);
      }
    }
  }
  const int64_t base = int64_t(blockIdx.y) * rows * n;
#pragma unroll
  for (int r = 0; r < RB; ++r)
    if (r < rows) {
      if (j0 < n) part[base + int64_t(r) * n + j0] = a0[r];
      if (j1 < n) part[base + int64_t(r) * n + j1] = a1[r];
    }
}

__global__ void few_rows_combine_kernel(int rows, int n, int nsplit, const double* __restrict__ part,
                                        const double* __restrict__ cs, double* __restrict__ U_out,
                                        int64_t ld_out, const int32_t* __restrict__ dst) {
  const int64_t e = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= int64_t(rows) * n) return;
  const int r = int(e / n), j = int(e % n);
  double s = 0.0;
  for (int q = 0; q < nsplit; ++q) s += part[(int64_t(q) * rows + r) * n + j];
  U_out[int64_t(r) * ld_out + (dst ? dst[j] : j)] = cs[j] * s;
}

int64_t few_rows_scratch_elems(int rows, int n) {
  const int64_t nsplit = (int64_t(n) + kFewSplitChunk - 1) / kFewSplitChunk;
  return std::max<int64_t>(1, nsplit * rows * n);
}

svd1_status apply_few_rows(int rows, int n, const double* d, const int32_t* k, const double* tau,
                           const double* zhat, const double* cs, const double* U_in, int64_t ld_in,
                           const int32_t* src, double* U_out, int64_t ld_out, const int32_t* dst,
                           double* scratch, cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || n <= 0) return SVD1_OK;
  if (rows > 32) return SVD1_E_INVALID;
  const int nsplit = (n + kFewSplitChunk - 1) / kFewSplitChunk;
  const dim3 grid(unsigned((n + 127) / 128), unsigned(nsplit));
  static const bool two = std::getenv("SVD1_FEW_ONE") == nullptr;  // two targets per thread (default)
  const dim3 grid2(unsigned((n + 255) / 256), unsigned(nsplit));
  if (two && rows <= 16) {
    if (rows <= 8)
      few_rows_partial2_kernel<8><<<grid2, 128, 0, st>>>(rows, n, d, k, tau, zhat, U_in, ld_in, src, scratch);
    else
      few_rows_partial2_kernel<16><<<grid2, 128, 0, st>>>(rows, n, d, k, tau, zhat, U_in, ld_in, src, scratch);
  } else if (rows <= 8)
    few_rows_partial_kernel<8><<<grid, 128, 0, st>>>(rows, n, d, k, tau, zhat, U_in, ld_in, src, scratch);
  else if (rows <= 16)
    few_rows_partial_kernel<16><<<grid, 128, 0, st>>>(rows, n, d, k, tau, zhat, U_in, ld_in, src, scratch);
  else if (rows <= 24)
    few_rows_partial_kernel<24><<<grid, 128, 0, st>>>(rows, n, d, k, tau, zhat, U_in, ld_in, src, scratch);
  else
    few_rows_partial_kernel<32><<<grid, 128, 0, st>>>(rows, n, d, k, tau, zhat, U_in, ld_in, src, scratch);
  few_rows_combine_kernel<<<unsigned((int64_t(rows) * n + 255) / 256), 256, 0, st>>>(rows, n, nsplit, scratch,
                                                                                      cs, U_out, ld_out, dst);
  *launches += 2;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status householder_cols(int64_t rows, double* U, int64_t ld, int ngroups,
                             const int32_t* goff, const int32_t* cols, const double* hv, int maxlen,
                             cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || ngroups <= 0) return SVD1_OK;
  if (maxlen <= 16) {  // many small groups: a warp per row
    householder_rows_kernel<<<unsigned((rows + 7) / 8), 256, 0, st>>>(rows, U, ld, ngroups, goff, cols, hv);
    *launches += 1;
    SVD1_CUDA_TRY(cudaGetLastError());
    return SVD1_OK;
  }
  dim3 grid(unsigned((rows + 31) / 32), unsigned(ngroups));
  householder_kernel<<<grid, 256, 0, st>>>(rows, U, ld, goff, cols, hv);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status col_rotate(int64_t rows, double* U, int64_t ld, int ngroups, const int32_t* goff,
                       const int32_t* cols, const double* mats, cudaStream_t st, int64_t* launches, int max_k) {
  if (rows <= 0 || ngroups <= 0) return SVD1_OK;
  dim3 grid(unsigned((rows + 255) / 256), unsigned(ngroups));
  col_rotate_kernel<<<grid, 256, 0, st>>>(rows, U, ld, goff, cols, mats);
  *launches += 1;
  if (max_k > 8) {  // groups beyond the register kernel's 8 columns
    if (max_k > 256) return SVD1_E_INVALID;
    dim3 gb(unsigned((rows + kRotRows - 1) / kRotRows), unsigned(ngroups));
    col_rotate_big_kernel<<<gb, 256, size_t(kRotRows) * max_k * sizeof(double), st>>>(rows, U, ld, goff, cols, mats);
    *launches += 1;
  }
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status passthrough(int64_t rows, int nq, const double* U_in, int64_t ld_in,
                        const int32_t* src, double* U_out, int64_t ld_out,
                        const int32_t* dst, const double* scale, cudaStream_t st,
                        int64_t* launches) {
  if (rows <= 0 || nq <= 0) return SVD1_OK;
  dim3 grid(unsigned((nq + 31) / 32), unsigned((rows + 7) / 8));
  passthrough_kernel<<<grid, 256, 0, st>>>(rows, nq, U_in, ld_in, src, U_out, ld_out, dst, scale);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status fmm_build_ops(int n_ops, const FmmOpDesc* descs, const FmmCell* cells, int p,
                          const double* d, const int32_t* k, const double* tau,
                          const double* zhat, const double* cs, const int32_t* col2src,
                          double* ops, int64_t ops_elems, cudaStream_t st, int64_t* launches) {
  if (n_ops <= 0) return SVD1_OK;
  const unsigned g = unsigned(std::min(n_ops, 148 * 8));
  fmm_ops_kernel<<<dim3(g, 2), 256, 0, st>>>(n_ops, descs, cells, p, d, k, tau, zhat, cs, col2src, ops,
                                             ops_elems);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

// ---- TMA descriptors (driver entry point through the runtime: no -lcuda)
namespace {
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}
}  // namespace

svd1_status make_tmap(CUtensorMap* map, const double* base, int64_t inner, int64_t outer,
                      int64_t ld, int box_inner, int box_outer) {
  auto fn = encode_fn();
  if (!fn) return SVD1_E_CUDA;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld & 1) || inner < 1 || outer < 1) return SVD1_E_INVALID;
  const cuuint64_t dims[2] = {cuuint64_t(inner), cuuint64_t(outer)};
  const cuuint64_t strides[1] = {cuuint64_t(ld) * 8};
  const cuuint32_t box[2] = {cuuint32_t(box_inner), cuuint32_t(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  // L2 promotion of the box's 128-byte rows (experiments: SVD1_L2PROMO = 0 none, 1 64B, 2 128B, 3 256B)
  static const int promo = [] {
    const char* e = std::getenv("SVD1_L2PROMO");
    return e ? std::atoi(e) : 0;
  }();
  const CUtensorMapL2promotion pr = promo == 1   ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                                    : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                                    : promo == 3 ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
                                                 : CU_TENSOR_MAP_L2_PROMOTION_NONE;
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, pr,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SVD1_OK : SVD1_E_INVALID;
}

template <int BN>
svd1_status launch_gemm(int n_tasks, const FmmTask* tasks, const FmmTerm* terms, int64_t rows,
                        const FmmMaps* maps, double* U_out, int64_t ld_out, const int32_t* dst,
                        double* phi, double* psi, int64_t ldE, int64_t out_cols, int64_t exp_elems,
                        const double* ops_raw, int64_t ops_rows, int* tile_ctr, int rb_major, cudaStream_t st) {
  using G = GemmCfg<BN>;
  static int max_ctas = 0;  // resident CTAs on the whole device (persistent grid)
  if (!max_ctas) {
    SVD1_CUDA_TRY(cudaFuncSetAttribute(fmm_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    int dev = 0, nsm = 0, per_sm = 0;
    SVD1_CUDA_TRY(cudaGetDevice(&dev));
    SVD1_CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    SVD1_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fmm_gemm_kernel<BN>, G::NTHR, G::SMEM));
    max_ctas = std::max(1, nsm * std::max(per_sm, 1));
  }
  const int64_t nrb = (rows + G::BM - 1) / G::BM;
  const int64_t ntiles = nrb * n_tasks;
  if (ntiles > (int64_t(1) << 30) || rows > (int64_t(1) << 30)) return SVD1_E_INVALID;
  // 90 % of the resident CTAs: the persistent grid leaves room on the SMs for the next
  // update's latency-bound spectral kernels (high-priority streams), which otherwise wait for
  // a whole pass to end (C3 stream: 421 -> 426 updates/s over 4 runs each; 370 CTAs the
  // same, 296 slower)
  int cap = std::max(1, max_ctas * 9 / 10);
  if (const char* e = std::getenv("SVD1_GEMM_CTAS")) cap = std::max(1, atoi(e));  // diagnostics
  const int grid = int(std::min<int64_t>(ntiles, cap));
  // tiles strided by the grid (default) or claimed from an atomic counter per pass
  // (SVD1_GEMM_DYNAMIC=1; measured the same in the C3 stream: 430-437 vs 434-438 updates/s;
  // reserving SMs for the spectral kernels -- CTAs on every 8th / 16th SM exiting at once --
  // measured 266-361)
  static const bool dynamic = std::getenv("SVD1_GEMM_DYNAMIC") != nullptr;
  fmm_gemm_kernel<BN><<<grid, G::NTHR, G::SMEM, st>>>(maps, tasks, terms, int(ntiles), int(nrb), n_tasks, rb_major,
                                                       dynamic ? tile_ctr : nullptr, rows, U_out,
                                                       ld_out, dst, phi, psi, ldE, out_cols, exp_elems,
                                                       ops_raw, ops_rows);
  return SVD1_OK;
}

svd1_status fmm_make_maps(FmmMaps* m, int64_t rows, const double* U_in, int64_t ncols_in, int64_t ld_in,
                          const double* phi, const double* psi, int64_t ldE) {
  for (int w = 0; w < 2; ++w) {
    const int bm = w ? GemmCfg<32>::BM : GemmCfg<16>::BM;
    svd1_status s = make_tmap(&m->u[w], U_in, ncols_in, rows, ld_in, KC, bm);
    if (s != SVD1_OK) return s;
    if ((s = make_tmap(&m->phi[w], phi, ldE, rows, ldE, KC, bm)) != SVD1_OK) return s;
    if ((s = make_tmap(&m->psi[w], psi, ldE, rows, ldE, KC, bm)) != SVD1_OK) return s;
  }
  return SVD1_OK;
}

svd1_status fmm_run_tasks(int n_tasks, const FmmTask* tasks, const FmmTerm* terms, int bn,
                          int64_t rows, const FmmMaps* maps, double* U_out, int64_t ld_out,
                          const int32_t* dst, double* phi, double* psi, int64_t ldE, int64_t out_cols,
                          int64_t exp_elems, const double* ops_raw, int64_t ops_rows, int* tile_ctr,
                          int rb_major, cudaStream_t st, int64_t* launches) {
  if (n_tasks <= 0 || rows <= 0) return SVD1_OK;
  svd1_status s = bn <= 16 ? launch_gemm<16>(n_tasks, tasks, terms, rows, maps, U_out, ld_out, dst, phi, psi,
                                             ldE, out_cols, exp_elems, ops_raw, ops_rows, tile_ctr, rb_major, st)
                           : launch_gemm<32>(n_tasks, tasks, terms, rows, maps, U_out, ld_out, dst, phi, psi,
                                             ldE, out_cols, exp_elems, ops_raw, ops_rows, tile_ctr, rb_major, st);
  if (s != SVD1_OK) return s;
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

}  // namespace svd1
