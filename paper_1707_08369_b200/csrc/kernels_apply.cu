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
      switch (D.kind) {
        case OP_P2M: {  // Phi~_X[j] += zhat_i U_i / (t_j (x_i - c_X) - 3 r_X)
          const FmmCell X = cells[D.a];
          const int s = X.slo + i;
          v = zhat[s] / (t[j] * (d[s] - X.c) - 3.0 * X.r);
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
        case OP_P2L: {  // sources of X (a) -> local expansion of Y (b) at y_j = c_Y + r_Y t_j
          const FmmCell X = cells[D.a], Y = cells[D.b];
          const int s = X.slo + i;
          v = zhat[s] / ((d[s] - Y.c) - Y.r * t[j]);
          break;
        }
        default: {  // OP_P2P: source leaf X (a), target leaf Y (b)
          const FmmCell X = cells[D.a], Y = cells[D.b];
          const int s = X.slo + i, jt = Y.tlo + j;
          v = (zhat[s] * cs[jt]) / ((d[s] - d[k[jt]]) - tau[jt]);
          break;
        }
      }
      out[e] = v;
    }
  }
}

// ------------------------------------------------------------------- K6-K10
// One FMM pass = a batch of "gathered small GEMMs": for task T and a tile of BM rows,
//   out[:, T.col0 : T.col0 + N] = sum_t in_t[:, col0_t : col0_t + K_t] * op_t (K_t x N).
// in/out are U (columns through src/dst maps) or the expansion matrices Phi/Psi.
// K is streamed in chunks of KC through a 2-stage cp.async pipeline; each warp owns a
// 32 x 16 output tile (4 x 2 DMMA m8n8k4 fragments).  BN = 16: 8 warps down the rows
// (BM = 256); BN = 32: 4 x 2 warps (BM = 128).
constexpr int KC = 16;
constexpr int ALD = KC + 4;  // 20 doubles: conflict-free A fragment loads

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 8 : 0;  // src-size 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

template <int BN>
struct GemmCfg {
  // every warp owns 32 rows x BN columns (4 x BN/8 DMMA m8n8k4 fragments)
  static constexpr int NWARP = BN <= 16 ? 8 : 4;
  static constexpr int NTHR = 32 * NWARP;
  static constexpr int NT = BN / 8;
  static constexpr int BM = 32 * NWARP;   // rows per CTA
  static constexpr int BLD = BN + 4;      // B row stride (doubles)
  static constexpr int STAGES = 2;        // cp.async pipeline depth
  static constexpr int A_ELEMS = BM * ALD;
  static constexpr int B_ELEMS = KC * BLD;
  static constexpr int SMEM = STAGES * (A_ELEMS + B_ELEMS) * 8;
};
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BN>
__global__ void __launch_bounds__(GemmCfg<BN>::NTHR) fmm_gemm_kernel(
    const FmmTask* __restrict__ tasks, const FmmTerm* __restrict__ terms, int64_t rows,
    const double* __restrict__ ops, const double* __restrict__ U_in, int64_t ld_in,
    const int32_t* __restrict__ src, double* __restrict__ U_out, int64_t ld_out,
    const int32_t* __restrict__ dst, double* __restrict__ phi, double* __restrict__ psi, int64_t ldE) {
  using G = GemmCfg<BN>;
  constexpr int NT = G::NT;
  extern __shared__ __align__(16) double smem[];
  double* As = smem;                            // [STAGES][BM][ALD]
  double* Bs = smem + G::STAGES * G::A_ELEMS;   // [STAGES][KC][BLD]
  const FmmTask T = tasks[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t row0 = int64_t(blockIdx.y) * G::BM;
  const int nrow = int(rows - row0 < G::BM ? rows - row0 : G::BM);

  auto load_stage = [&](int buf, int term, int kk0) {
    const FmmTerm R = terms[term];
    double* a = As + buf * G::A_ELEMS;
    double* b = Bs + buf * G::B_ELEMS;
    const double* base = R.in_kind == IO_U ? U_in : (R.in_kind == IO_PHI ? phi : psi);
    const int64_t ld = R.in_kind == IO_U ? ld_in : ldE;
    // Every thread owns one fixed column pair (kp, kp+1) of the chunk for rows rr0,
    // rr0 + 2*NTHR/KC, ...: the column map is read once per stage, and a pair of
    // adjacent, 16-byte aligned source columns moves as one 16-byte cp.async.
    {
      const int kp = (tid % (KC / 2)) * 2, rr0 = tid / (KC / 2);
      const int k = kk0 + kp;
      const bool ok0 = k < R.K, ok1 = k + 1 < R.K;
      int c0 = R.col0 + (ok0 ? k : 0), c1 = R.col0 + (ok1 ? k + 1 : 0);
      if (R.in_kind == IO_U && src) {
        c0 = src[c0];
        c1 = src[c1];
      }
      const bool vec = ok1 && c1 == c0 + 1 && !(c0 & 1) && !(ld & 1);
      const double* p0 = base + row0 * ld + c0;
      const double* p1 = base + row0 * ld + c1;
#pragma unroll 4
      for (int rr = rr0; rr < G::BM; rr += 2 * G::NTHR / KC) {
        const bool rok = rr < nrow;
        const int64_t ro = rok ? int64_t(rr) * ld : 0;
        if (vec) {
          cp_async16(a + rr * ALD + kp, p0 + ro, rok);
        } else {
          cp_async8(a + rr * ALD + kp, p0 + (ok0 ? ro : 0), ok0 && rok);
          cp_async8(a + rr * ALD + kp + 1, p1 + (ok1 ? ro : 0), ok1 && rok);
        }
      }
    }
    for (int e = tid; e < KC * BN; e += G::NTHR) {
      const int kk = e / BN, jj = e % BN;
      const int k = kk0 + kk;
      const bool ok = k < R.K && jj < T.N;
      cp_async8(b + kk * G::BLD + jj, ops + R.op_off + (ok ? int64_t(k) * R.op_ld + T.op_col0 + jj : 0), ok);
    }
  };
  double acc[4][NT][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // stage list = (term, K-chunk) pairs; a STAGES-deep cp.async ring
  int nst = 0;
  for (int t = T.t_begin; t < T.t_end; ++t) nst += (terms[t].K + KC - 1) / KC;
  int lti = T.t_begin, lk0 = 0;
  auto load_next = [&](int buf) {
    load_stage(buf, lti, lk0);
    lk0 += KC;
    if (lk0 >= terms[lti].K) {
      ++lti;
      lk0 = 0;
    }
  };
#pragma unroll
  for (int q = 0; q < G::STAGES - 1; ++q) {
    if (q < nst) load_next(q);
    cp_async_commit();
  }
  for (int it = 0; it < nst; ++it) {
    const int buf = it % G::STAGES;
    if (it + G::STAGES - 1 < nst) load_next((it + G::STAGES - 1) % G::STAGES);
    cp_async_commit();
    cp_async_wait<G::STAGES - 1>();
    __syncthreads();
    const double* a = As + buf * G::A_ELEMS;
    const double* b = Bs + buf * G::B_ELEMS;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double af[4], bf[NT];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) af[mt] = a[(warp * 32 + mt * 8 + (lane >> 2)) * ALD + kk + (lane & 3)];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) bf[nt] = b[(kk + (lane & 3)) * G::BLD + nt * 8 + (lane >> 2)];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) dmma_8x8x4(acc[mt][nt], af[mt], bf[nt]);
    }
    __syncthreads();  // buffer `buf` is refilled by a later prefetch
  }
  // epilogue
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int rr = warp * 32 + mt * 8 + (lane >> 2);
    if (rr >= nrow) continue;
    const int64_t r = row0 + rr;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int jj = nt * 8 + (lane & 3) * 2 + h;
        if (jj >= T.N) continue;
        const int col = T.col0 + jj;
        if (T.out_kind == IO_U) {
          U_out[r * ld_out + (dst ? dst[col] : col)] = acc[mt][nt][h];
        } else {
          (T.out_kind == IO_PHI ? phi : psi)[r * ldE + col] = acc[mt][nt][h];
        }
      }
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
                          const double* zhat, const double* cs, double* ops, cudaStream_t st,
                          int64_t* launches) {
  if (n_ops <= 0) return SVD1_OK;
  const unsigned g = unsigned(std::min(n_ops, 148 * 16));
  fmm_ops_kernel<<<g, 256, 0, st>>>(n_ops, descs, cells, p, d, k, tau, zhat, cs, ops);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

template <int BN>
svd1_status launch_gemm(int n_tasks, const FmmTask* tasks, const FmmTerm* terms, int64_t rows,
                        const double* ops, const double* U_in, int64_t ld_in, const int32_t* src,
                        double* U_out, int64_t ld_out, const int32_t* dst, double* phi, double* psi,
                        int64_t ldE, cudaStream_t st) {
  using G = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    SVD1_CUDA_TRY(cudaFuncSetAttribute(fmm_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM));
    attr = true;
  }
  dim3 grid(unsigned(n_tasks), unsigned((rows + G::BM - 1) / G::BM));
  fmm_gemm_kernel<BN><<<grid, G::NTHR, G::SMEM, st>>>(tasks, terms, rows, ops, U_in, ld_in, src, U_out,
                                                  ld_out, dst, phi, psi, ldE);
  return SVD1_OK;
}

svd1_status fmm_run_tasks(int n_tasks, const FmmTask* tasks, const FmmTerm* terms, int bn,
                          int64_t rows, const double* ops, const double* U_in, int64_t ld_in,
                          const int32_t* src, double* U_out, int64_t ld_out, const int32_t* dst,
                          double* phi, double* psi, int64_t ldE, cudaStream_t st, int64_t* launches) {
  if (n_tasks <= 0 || rows <= 0) return SVD1_OK;
  svd1_status s = bn <= 16 ? launch_gemm<16>(n_tasks, tasks, terms, rows, ops, U_in, ld_in, src, U_out,
                                             ld_out, dst, phi, psi, ldE, st)
                           : launch_gemm<32>(n_tasks, tasks, terms, rows, ops, U_in, ld_in, src, U_out,
                                             ld_out, dst, phi, psi, ldE, st);
  if (s != SVD1_OK) return s;
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

}  // namespace svd1
