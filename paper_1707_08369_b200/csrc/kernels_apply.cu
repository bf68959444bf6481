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
      const double del = (s_di[kk] - s_dk[jj]) - s_tau[jj];
      Bs[kk * DLDB + jj] = (s_zi[kk] * s_cs[jj]) / del;
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
__device__ double lagrange(const double* __restrict__ t, const double* __restrict__ w, int p,
                           int kk, double x) {
  double den = 0.0, num = 0.0;
  for (int m = 0; m < p; ++m) {
    const double dx = x - t[m];
    if (dx == 0.0) return (m == kk) ? 1.0 : 0.0;
    const double q = w[m] / dx;
    den += q;
    if (m == kk) num = q;
  }
  return num / den;
}

__global__ void __launch_bounds__(256) fmm_ops_kernel(int n_ops, const FmmOpDesc* __restrict__ descs,
                                                     const FmmCell* __restrict__ cells, int p,
                                                     const double* __restrict__ d,
                                                     const int32_t* __restrict__ k,
                                                     const double* __restrict__ tau,
                                                     const double* __restrict__ zhat,
                                                     const double* __restrict__ cs,
                                                     const int32_t* __restrict__ col2src,
                                                     double* __restrict__ ops) {
  __shared__ double t[kMaxP], w[kMaxP];
  if (threadIdx.x < p) {
    const double th = (2.0 * threadIdx.x + 1.0) / (2.0 * p);  // in units of pi
    t[threadIdx.x] = cospi(th);
    w[threadIdx.x] = ((threadIdx.x & 1) ? -1.0 : 1.0) * sinpi(th);
  }
  __syncthreads();
  for (int o = blockIdx.x; o < n_ops; o += gridDim.x) {
    const FmmOpDesc D = descs[o];
    double* out = ops + D.off;
    const int total = D.rows * D.cols;
    for (int e = threadIdx.x; e < total; e += blockDim.x) {
      const int i = e / D.cols, j = e % D.cols;
      double v = 0.0;
      // source kinds: row i holds input column c0 + i (zero unless an active source of
      // the term's range [a, s_hi) sits there)
      int s = -1;
      if (D.kind == OP_P2M || D.kind == OP_P2L || D.kind == OP_P2P) {
        s = col2src ? col2src[D.c0 + i] : D.c0 + i;
        if (s < D.a || s >= D.s_hi) s = -1;
      }
      switch (D.kind) {
        case OP_P2M: {  // Phi~_X[j] += zhat_s U_s / (t_j (x_s - c_X) - 3 r_X), X = b
          const FmmCell X = cells[D.b];
          if (s >= 0) v = zhat[s] / (t[j] * (d[s] - X.c) - 3.0 * X.r);
          break;
        }
        case OP_M2M: {  // child (a) -> parent (b): i = child node, j = parent node
          const FmmCell C = cells[D.a], P = cells[D.b];
          const double den = 3.0 * P.r + t[j] * (P.c - C.c);
          const double tc = 3.0 * C.r * t[j] / den;
          v = (3.0 * C.r / den) * lagrange(t, w, p, i, tc);
          break;
        }
        case OP_M2L: {  // source X (a) -> target Y (b): i = X node, j = Y node
          const FmmCell X = cells[D.a], Y = cells[D.b];
          const double tx = 3.0 * X.r / ((Y.c - X.c) + Y.r * t[j]);
          v = tx * lagrange(t, w, p, i, tx);
          break;
        }
        case OP_L2L: {  // parent (a) -> child (b): i = parent node, j = child node
          const FmmCell P = cells[D.a], C = cells[D.b];
          v = lagrange(t, w, p, i, ((C.c - P.c) + C.r * t[j]) / P.r);
          break;
        }
        case OP_L2P: {  // leaf Y (b): i = node, j = target
          const FmmCell Y = cells[D.b];
          const int jt = Y.tlo + j;
          v = lagrange(t, w, p, i, ((d[k[jt]] - Y.c) + tau[jt]) / Y.r) * cs[jt];
          break;
        }
        case OP_ID: {
          v = (i == j) ? 1.0 : 0.0;
          break;
        }
        case OP_L2P_FROM: {  // Psi of cell a (an ancestor) at the targets of leaf b
          const FmmCell A = cells[D.a], Y = cells[D.b];
          const int jt = Y.tlo + j;
          v = lagrange(t, w, p, i, ((d[k[jt]] - A.c) + tau[jt]) / A.r) * cs[jt];
          break;
        }
        case OP_P2L: {  // source s -> local expansion of Y (b) at y_j = c_Y + r_Y t_j
          const FmmCell Y = cells[D.b];
          if (s >= 0) v = zhat[s] / ((d[s] - Y.c) - Y.r * t[j]);
          break;
        }
        default: {  // OP_P2P: source s, target leaf Y (b)
          const FmmCell Y = cells[D.b];
          const int jt = Y.tlo + j;
          if (s >= 0) v = (zhat[s] * cs[jt]) / ((d[s] - d[k[jt]]) - tau[jt]);
          break;
        }
      }
      out[int64_t(i) * D.ld + j] = v;
    }
  }
}

// ------------------------------------------------------------------- K6-K10
// One FMM pass = a batch of "gathered small GEMMs": for task T and every row,
//   out[r, T.col0 : T.col0 + N] = sum_t in_t[r, col0_t : col0_t + K_t] * op_t (K_t x N).
// in = U (physical column windows resolved on the host, so no column map is read here)
// or the expansion matrices Phi/Psi; out = U (through dst[]) or Phi/Psi.
// Persistent CTAs walk the pass's tiles (task, block of BM rows) with stride gridDim.x;
// the host orders tasks by decreasing K, so the longest tiles start first.  One
// continuous STAGES-deep cp.async ring runs across term, chunk and tile boundaries, so
// a tile's first loads are in flight while the previous tile finishes.  K tails (terms
// are not multiples of KC) are masked per 4-wide k-step; A reads past the term stay
// inside the row (columns clamped to ld - 2) and B reads past the op inside the padded
// ops buffer, and both only ever meet masked k-steps.  Each warp owns a 32 x BN tile
// (4 x BN/8 DMMA m8n8k4 fragments); 4 warps -> BM = 128 rows per tile.
constexpr int KC = 16;
constexpr int ALD = KC + 4;  // 20 doubles: conflict-free A fragment loads

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BN>
struct GemmCfg {
  static constexpr int NWARP = 4;
  static constexpr int NTHR = 32 * NWARP;
  static constexpr int NT = BN / 8;
  static constexpr int BM = 32 * NWARP;   // rows per tile
  static constexpr int BLD = BN + 4;      // B row stride (doubles): conflict-free fragments
  static constexpr int STAGES = 3;        // cp.async ring depth
  static constexpr int A_ELEMS = BM * ALD;
  static constexpr int B_ELEMS = KC * BLD;
  static constexpr int SMEM = STAGES * (A_ELEMS + B_ELEMS) * 8 + STAGES * 16;
};

struct StageInfo {   // written by the loader, read by the compute side of the same stage
  int32_t rem;       // K - k0 of the chunk's term (k-steps beyond it are masked)
  int32_t tile;      // tile the chunk belongs to
  int32_t last;      // 1: last chunk of the tile (epilogue after it), -1: no chunk
  int32_t pad;
};

template <int BN>
__global__ void __launch_bounds__(GemmCfg<BN>::NTHR) fmm_gemm_kernel(
    const FmmTask* __restrict__ tasks, const FmmTerm* __restrict__ terms, int ntiles, int nrb,
    int64_t rows, const double* __restrict__ ops, const double* __restrict__ U_in, int64_t ld_in,
    double* __restrict__ U_out, int64_t ld_out, const int32_t* __restrict__ dst,
    double* __restrict__ phi, double* __restrict__ psi, int64_t ldE) {
  using G = GemmCfg<BN>;
  constexpr int NT = G::NT;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                            // [STAGES][BM][ALD]
  double* Bs = smem + G::STAGES * G::A_ELEMS;   // [STAGES][KC][BLD]
  StageInfo* info = reinterpret_cast<StageInfo*>(Bs + G::STAGES * G::B_ELEMS);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- loader iterator (uniform across the CTA)
  int l_tile = blockIdx.x, l_term = 0, l_tend = 0, l_k0 = 0, l_opc0 = 0;
  int64_t l_row0 = 0;   // first row of the tile
  bool l_full = true;   // the tile's rows are all < rows (no clamping)
  FmmTerm R{};
  auto l_start_tile = [&]() {
    if (l_tile < ntiles) {
      const int task = l_tile / nrb;
      const FmmTask T = tasks[task];
      l_row0 = int64_t(l_tile - task * nrb) * G::BM;
      l_full = l_row0 + G::BM <= rows;
      l_term = T.t_begin;
      l_tend = T.t_end;
      l_k0 = 0;
      l_opc0 = T.op_col0;
      R = terms[l_term];
    }
  };
  l_start_tile();
  // A: thread -> column pair kp (of KC/2), rows rr0 + 16 i (BM / 16 of them)
  const int kp = (tid & (KC / 2 - 1)) * 2, rr0 = tid >> 3;
  auto issue = [&](int buf) {
    if (tid == 0) info[buf].last = -1;
    if (l_tile >= ntiles) return;
    const bool inU = R.in_kind == IO_U;
    const double* base = inU ? U_in : (R.in_kind == IO_PHI ? phi : psi);
    const int64_t ld = inU ? ld_in : ldE;
    double* a = As + buf * G::A_ELEMS + rr0 * ALD + kp;
    const int cu = R.col0 + l_k0 + kp;
    if (!(ld & 1)) {  // pairs (c, c+1), c even: in the row whenever c <= ld - 2
      const int c = min(cu, int(ld - 2));
      if (l_full) {
        const double* g = base + (l_row0 + rr0) * ld + c;
        const int64_t step = 16 * ld;
#pragma unroll
        for (int i = 0; i < G::BM / 16; ++i) {
          cp_async16(a + 16 * i * ALD, g);
          g += step;
        }
      } else {
#pragma unroll
        for (int i = 0; i < G::BM / 16; ++i) {
          const int64_t r = min(l_row0 + rr0 + 16 * i, rows - 1);
          cp_async16(a + 16 * i * ALD, base + r * ld + c);
        }
      }
    } else {  // odd leading dimension: rows are not 16-byte aligned; clamp per column
      const int c0 = min(cu, int(ld - 1)), c1 = min(cu + 1, int(ld - 1));
#pragma unroll
      for (int i = 0; i < G::BM / 16; ++i) {
        const int64_t r = min(l_row0 + rr0 + 16 * i, rows - 1);
        cp_async8(a + 16 * i * ALD, base + r * ld + c0);
        cp_async8(a + 16 * i * ALD + 1, base + r * ld + c1);
      }
    }
    // B: KC x BN block of the op (row stride op_ld even, 16-byte aligned rows)
    double* b = Bs + buf * G::B_ELEMS;
    const double* bsrc = ops + R.op_off + int64_t(l_k0) * R.op_ld + l_opc0;
#pragma unroll
    for (int e = tid; e < KC * BN / 2; e += G::NTHR) {
      const int kk = e / (BN / 2), jj = (e % (BN / 2)) * 2;
      cp_async16(b + kk * G::BLD + jj, bsrc + kk * R.op_ld + jj);
    }
    const int rem = R.K - l_k0;
    // advance
    l_k0 += KC;
    int last = 0;
    const int tile = l_tile;
    if (l_k0 >= R.K) {
      l_k0 = 0;
      if (++l_term == l_tend) {
        last = 1;
        l_tile += gridDim.x;
        l_start_tile();
      } else {
        R = terms[l_term];
      }
    }
    if (tid == 0) info[buf] = StageInfo{rem, tile, last, 0};
  };

  double acc[4][NT][2];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < NT; ++y) acc[x][y][0] = acc[x][y][1] = 0.0;

#pragma unroll
  for (int q = 0; q < G::STAGES - 1; ++q) {
    issue(q);
    cp_async_commit();
  }
  const int a_off = (warp * 32 + (lane >> 2)) * ALD + (lane & 3);
  const int b_off = (lane & 3) * G::BLD + (lane >> 2);
  for (int it = 0;; ++it) {
    const int buf = it % G::STAGES;
    issue((it + G::STAGES - 1) % G::STAGES);
    cp_async_commit();
    cp_async_wait<G::STAGES - 1>();
    __syncthreads();
    const StageInfo I = info[buf];
    if (I.last < 0) break;
    const double* a = As + buf * G::A_ELEMS + a_off;
    const double* b = Bs + buf * G::B_ELEMS + b_off;
    // fragments double-buffered in registers: k-step kk+1 loads while kk multiplies
    double af[2][4], bf[2][NT];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) af[0][mt] = a[mt * 8 * ALD];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) bf[0][nt] = b[nt * 8];
#pragma unroll
    for (int q = 0; q < KC / 4; ++q) {
      const int kk = 4 * q, cur = q & 1;
      if (kk >= I.rem) break;
      if (q + 1 < KC / 4) {
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) af[cur ^ 1][mt] = a[mt * 8 * ALD + kk + 4];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bf[cur ^ 1][nt] = b[(kk + 4) * G::BLD + nt * 8];
      }
      if (kk + 4 > I.rem) {  // ragged K tail: zero both operands of the missing k
        const bool ok = kk + (lane & 3) < I.rem;
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) af[cur][mt] = ok ? af[cur][mt] : 0.0;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) bf[cur][nt] = ok ? bf[cur][nt] : 0.0;
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], af[cur][mt], bf[cur][nt]);
    }
    __syncthreads();  // buffer `buf` is refilled by a later prefetch
    if (I.last) {     // epilogue of tile I.tile (registers -> global only)
      const FmmTask T = tasks[I.tile / nrb];
      const int64_t row0 = int64_t(I.tile % nrb) * G::BM;
      double* E = T.out_kind == IO_PHI ? phi : psi;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int jj = nt * 8 + (lane & 3) * 2;
        if (jj >= T.N) continue;
        const int col = T.col0 + jj;
        if (T.out_kind == IO_U) {
          const int c0 = dst ? dst[col] : col;
          const int c1 = (jj + 1 < T.N) ? (dst ? dst[col + 1] : col + 1) : -1;
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const int64_t r = row0 + warp * 32 + mt * 8 + (lane >> 2);
            if (r >= rows) continue;
            U_out[r * ld_out + c0] = acc[mt][nt][0];
            if (c1 >= 0) U_out[r * ld_out + c1] = acc[mt][nt][1];
          }
        } else {  // expansions: N is a multiple of 4, col0 even -> 16-byte stores
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) {
            const int64_t r = row0 + warp * 32 + mt * 8 + (lane >> 2);
            if (r >= rows) continue;
            *reinterpret_cast<double2*>(E + r * ldE + col) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
          }
        }
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
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

svd1_status householder_cols(int64_t rows, double* U, int64_t ld, int ngroups,
                             const int32_t* goff, const int32_t* cols, const double* hv,
                             cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || ngroups <= 0) return SVD1_OK;
  dim3 grid(unsigned((rows + 31) / 32), unsigned(ngroups));
  householder_kernel<<<grid, 256, 0, st>>>(rows, U, ld, goff, cols, hv);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status col_rotate(int64_t rows, double* U, int64_t ld, int ngroups, const int32_t* goff,
                       const int32_t* cols, const double* mats, cudaStream_t st, int64_t* launches) {
  if (rows <= 0 || ngroups <= 0) return SVD1_OK;
  dim3 grid(unsigned((rows + 255) / 256), unsigned(ngroups));
  col_rotate_kernel<<<grid, 256, 0, st>>>(rows, U, ld, goff, cols, mats);
  *launches += 1;
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
                          double* ops, cudaStream_t st, int64_t* launches) {
  if (n_ops <= 0) return SVD1_OK;
  const unsigned g = unsigned(std::min(n_ops, 148 * 16));
  fmm_ops_kernel<<<g, 256, 0, st>>>(n_ops, descs, cells, p, d, k, tau, zhat, cs, col2src, ops);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

template <int BN>
svd1_status launch_gemm(int n_tasks, const FmmTask* tasks, const FmmTerm* terms, int64_t rows,
                        const double* ops, const double* U_in, int64_t ld_in, double* U_out,
                        int64_t ld_out, const int32_t* dst, double* phi, double* psi, int64_t ldE,
                        cudaStream_t st) {
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
  if (ntiles > (int64_t(1) << 30)) return SVD1_E_INVALID;
  const int grid = int(std::min<int64_t>(ntiles, max_ctas));
  fmm_gemm_kernel<BN><<<grid, G::NTHR, G::SMEM, st>>>(tasks, terms, int(ntiles), int(nrb), rows, ops, U_in,
                                                       ld_in, U_out, ld_out, dst, phi, psi, ldE);
  return SVD1_OK;
}

svd1_status fmm_run_tasks(int n_tasks, const FmmTask* tasks, const FmmTerm* terms, int bn,
                          int64_t rows, const double* ops, const double* U_in, int64_t ld_in,
                          double* U_out, int64_t ld_out, const int32_t* dst, double* phi,
                          double* psi, int64_t ldE, cudaStream_t st, int64_t* launches) {
  if (n_tasks <= 0 || rows <= 0) return SVD1_OK;
  svd1_status s = bn <= 16 ? launch_gemm<16>(n_tasks, tasks, terms, rows, ops, U_in, ld_in, U_out, ld_out,
                                             dst, phi, psi, ldE, st)
                           : launch_gemm<32>(n_tasks, tasks, terms, rows, ops, U_in, ld_in, U_out, ld_out,
                                             dst, phi, psi, ldE, st);
  if (s != SVD1_OK) return s;
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

}  // namespace svd1
