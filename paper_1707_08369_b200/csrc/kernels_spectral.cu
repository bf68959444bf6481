// Spectral-phase kernels of the rank-1 SVD update (sm_100a, fp64):
//   K1  projections U^T [a, g_0..g_3], V^T b and the scalars a.g, a.a, b.b
//       (Alg 6.1 STEP 1, via the small-vector identities of DESIGN.md §4.1)
//   K2  secular roots of w(mu) = 1 + rho sum z_i^2/(d_i - mu)
//   K3a Loewner recomputation of z from the roots               (north star item 2)
//   K3b column norms ||c_j|| of diag(zhat) C
//   K12 small transposed Cauchy products X^T v
// All are FP64-ALU or HBM bound; none is a dense contraction, so no tensor cores.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "svd1_internal.cuh"

namespace svd1 {

svd1_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  fprintf(stderr, "[svd1] CUDA error %s (%s) at %s:%d\n", cudaGetErrorString(e), what, file, line);
  return SVD1_E_CUDA;
}

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;  // bitwise identical in every lane (fp add is commutative)
}

// fp64 reciprocal: MUFU.RCP64H seed + two Newton steps (<= 1 ulp off the IEEE result;
// the hot loop of K2 does one per term).  Arguments are normal, finite, nonzero.
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}

__device__ __forceinline__ double probe_value(uint64_t seed, int kq, int64_t row) {
  uint64_t h1 = splitmix64(seed ^ (uint64_t(kq) << 56) ^ uint64_t(row) * 2ull);
  uint64_t h2 = splitmix64(h1 ^ 0x5851F42D4C957F2Dull);
  double u1 = 1.0 - double(h1 >> 11) * 0x1.0p-53;  // (0, 1]
  double u2 = double(h2 >> 11) * 0x1.0p-53;
  return sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
}

// ------------------------------------------------------------------- K1
// partial[chunk][v][c] = sum_{r in chunk} M[r, c] * vec_v(r); vec_0 = x[row0 + r],
// vec_{1..4} = probe g_{v-1}(row0 + r) when nv == 5.
template <int NV>
__global__ void __launch_bounds__(256) proj_partial_kernel(const double* __restrict__ M, int64_t ld,
                                                          int64_t rows, int64_t cols,
                                                          const double* __restrict__ x,
                                                          int64_t row0, int rows_per_chunk,
                                                          const double* __restrict__ probes,
                                                          double* __restrict__ part) {
  __shared__ double vec[NV][64];
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r_begin = int64_t(blockIdx.y) * rows_per_chunk;
  const int64_t r_end = min(rows, r_begin + rows_per_chunk);
  double acc[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) acc[v] = 0.0;
  for (int64_t rb = r_begin; rb < r_end; rb += 64) {
    const int nr = int((r_end - rb < 64) ? (r_end - rb) : 64);
    __syncthreads();
    for (int t = threadIdx.x; t < nr * NV; t += blockDim.x) {
      const int rr = t % nr, v = t / nr;
      vec[v][rr] = (v == 0) ? x[row0 + rb + rr] : probes[(v - 1) * rows + rb + rr];
    }
    __syncthreads();
    if (c < cols) {
      const double* p = M + rb * ld + c;
      int rr = 0;
      for (; rr + 8 <= nr; rr += 8) {  // 8 rows of loads in flight per thread (HBM-bound)
        double mm[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) mm[q] = __ldg(p + q * ld);
        p += 8 * ld;
#pragma unroll
        for (int q = 0; q < 8; ++q)
#pragma unroll
          for (int v = 0; v < NV; ++v) acc[v] = fma(mm[q], vec[v][rr + q], acc[v]);
      }
      for (; rr < nr; ++rr, p += ld) {
        const double m0 = __ldg(p);
#pragma unroll
        for (int v = 0; v < NV; ++v) acc[v] = fma(m0, vec[v][rr], acc[v]);
      }
    }
  }
  if (c < cols) {
#pragma unroll
    for (int v = 0; v < NV; ++v) part[(int64_t(blockIdx.y) * NV + v) * cols + c] = acc[v];
  }
}

// out[v*cols + c] = sum over chunks in order (deterministic)
// M^T x_v for up to MV vectors x_v = X[v * ldx + row0 + r] (a stream's a's or b's): the
// same row-chunked partial sums as proj_partial_kernel, one pass over M for all of them
constexpr int kMV = 8;
__global__ void __launch_bounds__(256) proj_multi_kernel(const double* __restrict__ M, int64_t ld,
                                                        int64_t rows, int64_t cols,
                                                        const double* __restrict__ X, int64_t ldx, int nv,
                                                        int64_t row0, int rows_per_chunk,
                                                        double* __restrict__ part) {
  __shared__ double vec[kMV][64];
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t r_begin = int64_t(blockIdx.y) * rows_per_chunk;
  const int64_t r_end = min(rows, r_begin + rows_per_chunk);
  double acc[kMV];
#pragma unroll
  for (int v = 0; v < kMV; ++v) acc[v] = 0.0;
  for (int64_t rb = r_begin; rb < r_end; rb += 64) {
    const int nr = int((r_end - rb < 64) ? (r_end - rb) : 64);
    __syncthreads();
    for (int t = threadIdx.x; t < nr * kMV; t += blockDim.x) {
      const int rr = t % nr, v = t / nr;
      vec[v][rr] = v < nv ? X[int64_t(v) * ldx + row0 + rb + rr] : 0.0;
    }
    __syncthreads();
    if (c < cols) {
      const double* p = M + rb * ld + c;
      for (int rr = 0; rr < nr; ++rr, p += ld) {
        const double m0 = __ldg(p);
#pragma unroll
        for (int v = 0; v < kMV; ++v) acc[v] = fma(m0, vec[v][rr], acc[v]);
      }
    }
  }
  if (c < cols)
    for (int v = 0; v < nv; ++v) part[(int64_t(blockIdx.y) * nv + v) * cols + c] = acc[v];
}

// out[v * ostride + c] = sum over chunks (fixed order)
__global__ void proj_reduce_strided_kernel(const double* __restrict__ part, int nchunks, int nv, int64_t cols,
                                           double* __restrict__ out, int64_t ostride) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nv * cols) return;
  double s = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) s += part[int64_t(ch) * nv * cols + t];
  out[(t / cols) * ostride + t % cols] = s;
}

__global__ void proj_reduce_kernel(const double* __restrict__ part, int nchunks, int nv,
                                   int64_t cols, double* __restrict__ out) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nv * cols) return;
  double s = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) s += part[int64_t(ch) * nv * cols + t];
  out[t] = s;
}

// probes g_k(row) for this process's rows, row-major [4][u_rows] (computed once per plan)
__global__ void probe_fill_kernel(uint64_t seed, int64_t row0, int64_t rows, double* __restrict__ g) {
  const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= 4 * rows) return;
  const int kq = int(t / rows);
  const int64_t r = t % rows;
  g[t] = probe_value(seed, kq, row0 + r);
}

// scalars: out[0..3] = a_loc . g_k,loc ; out[4] = a_loc . a_loc ; out[5] = b_loc . b_loc
// block partials [gridDim.x][6], then proj_dots_final sums them in block order.
__global__ void __launch_bounds__(256) proj_dots_kernel(const double* __restrict__ a, int64_t u_rows,
                                                       int64_t u_row0, const double* __restrict__ b,
                                                       int64_t v_rows, int64_t v_row0,
                                                       const double* __restrict__ probes,
                                                       double* __restrict__ part, int64_t lda = 0,
                                                       int64_t ldb = 0) {
  // blockIdx.y: the update (project_many: a_t = a + t lda, b_t = b + t ldb, its own partials)
  a += int64_t(blockIdx.y) * lda;
  b += int64_t(blockIdx.y) * ldb;
  part += int64_t(blockIdx.y) * gridDim.x * 6;
  __shared__ double red[6][8];
  double acc[6] = {0, 0, 0, 0, 0, 0};
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < u_rows; r += stride) {
    const double av = a[u_row0 + r];
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[q] = fma(av, probes[q * u_rows + r], acc[q]);
    acc[4] = fma(av, av, acc[4]);
  }
  for (int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; r < v_rows; r += stride) {
    const double bv = b[v_row0 + r];
    acc[5] = fma(bv, bv, acc[5]);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const double s = warp_sum(acc[q]);
    if (lane == 0) red[q][w] = s;
  }
  __syncthreads();
  if (threadIdx.x < 6) {
    double s = 0.0;
    for (int i = 0; i < 8; ++i) s += red[threadIdx.x][i];
    part[blockIdx.x * 6 + threadIdx.x] = s;
  }
}

__global__ void proj_dots_final(const double* __restrict__ part, int nblocks, double* __restrict__ out,
                                int64_t ldo = 0) {
  // blockIdx.x: the update (its partials, its output at out + t ldo)
  part += int64_t(blockIdx.x) * nblocks * 6;
  out += int64_t(blockIdx.x) * ldo;
  if (threadIdx.x < 6) {
    double s = 0.0;
    for (int i = 0; i < nblocks; ++i) s += part[i * 6 + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// ------------------------------------------------------------------- K2
struct SecAcc {
  double psi, phi, dpsi, dphi, eabs;
};

// Sums of w in the gap form: delta_i = (d_i - d_k) - tau.
// d, z2 are the rho > 0 view (reflected by the host when rho < 0; z2 = z^2).  Left set
// i <= sp (psi, all terms negative), right set i > sp (phi, one sign), so
// sum |z_i^2/delta_i| = |psi| + |phi|.
// Reduction groups: one warp per root, or one block per root (the FMM path's few
// direct roots, so they do not set the kernel's tail).
struct WarpGrp {
  int tid;
  static constexpr int size = 32;
  __device__ double sum(double v) const { return warp_sum(v); }
  __device__ void sum4(double& a, double& b, double& c, double& d) const {
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    d = warp_sum(d);
  }
};
struct BlockGrp {  // all threads of the block call sum() together (uniform control flow)
  int tid, size;
  double* sm;      // 4 * 8 doubles (blockDim.x <= 256)
  __device__ double sum(double v) const {
    v = warp_sum(v);
    __syncthreads();
    if ((tid & 31) == 0) sm[tid >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int q = 0; q < (size >> 5); ++q) s += sm[q];
    return s;
  }
  __device__ void sum4(double& a, double& b, double& c, double& d) const {  // sm: 4 * 8 doubles
    a = warp_sum(a);
    b = warp_sum(b);
    c = warp_sum(c);
    d = warp_sum(d);
    __syncthreads();
    if ((tid & 31) == 0) {
      sm[tid >> 5] = a;
      sm[8 + (tid >> 5)] = b;
      sm[16 + (tid >> 5)] = c;
      sm[24 + (tid >> 5)] = d;
    }
    __syncthreads();
    a = b = c = d = 0.0;
    for (int q = 0; q < (size >> 5); ++q) {
      a += sm[q];
      b += sm[8 + q];
      c += sm[16 + q];
      d += sm[24 + q];
    }
  }
};

template <class G>
__device__ SecAcc sec_eval(const double* __restrict__ d, const double* __restrict__ z2, int n,
                           double dk, double tau, int sp, const G& g) {
  SecAcc a = {0, 0, 0, 0, 0};
#pragma unroll 4
  for (int i = g.tid; i <= sp; i += g.size) {
    const double rr = fast_rcp((__ldg(d + i) - dk) - tau);
    const double t = __ldg(z2 + i) * rr;
    a.psi += t;
    a.dpsi = fma(t, rr, a.dpsi);
  }
#pragma unroll 4
  for (int i = sp + 1 + g.tid; i < n; i += g.size) {
    const double rr = fast_rcp((__ldg(d + i) - dk) - tau);
    const double t = __ldg(z2 + i) * rr;
    a.phi += t;
    a.dphi = fma(t, rr, a.dphi);
  }
  g.sum4(a.psi, a.phi, a.dpsi, a.dphi);
  a.eabs = fabs(a.psi) + fabs(a.phi);
  return a;
}

// One safeguarded step from tau inside the open bracket (lo, hi).
// Two-pole rational model (poles at the bracketing d's, offsets p1, p2 from the
// origin): w(tau + eta) ~ C + r dpsi del1^2/(del1 - eta) + r dphi del2^2/(del2 - eta),
// del_i = p_i - tau, C = w - r (dpsi del1 + dphi del2)  =>
// C eta^2 - [(del1 + del2) w - del1 del2 w'] eta + del1 del2 w = 0.
// Falls back to Newton, then to bisection, if the root leaves the bracket.
__device__ __forceinline__ double sec_step(double w, const SecAcc& a, double r, double p1,
                                           double p2, double tau, double lo, double hi) {
  const double del1 = p1 - tau, del2 = p2 - tau;
  const double wp = r * (a.dpsi + a.dphi);
  const double C = w - r * (a.dpsi * del1 + a.dphi * del2);
  const double B = -((del1 + del2) * w - del1 * del2 * wp);
  const double Dc = del1 * del2 * w;
  const double elo = lo - tau, ehi = hi - tau;
  double eta = NAN;
  if (C != 0.0) {
    const double disc = fma(B, B, -4.0 * C * Dc);
    const double sq = sqrt(fmax(disc, 0.0));
    const double q = -0.5 * (B + copysign(sq, B));
    const double e1 = q / C;
    const double e2 = (q != 0.0) ? Dc / q : e1;
    const bool ok1 = e1 > elo && e1 < ehi, ok2 = e2 > elo && e2 < ehi;
    if (ok1 && ok2) eta = fabs(e1) < fabs(e2) ? e1 : e2;
    else if (ok1) eta = e1;
    else if (ok2) eta = e2;
  } else if (B != 0.0) {
    const double e = -Dc / B;
    if (e > elo && e < ehi) eta = e;
  }
  if (!(eta == eta)) {
    const double e = -w / wp;
    if (e > elo && e < ehi) eta = e;
  }
  if (eta == eta) {
    const double tn = tau + eta;
    if (tn == tau) return tau;               // step below the resolution of tau: converged
    if (tn > lo && tn < hi) return tn;
  }
  // bisection safeguard (geometric across a bracket spanning many binades)
  return (lo > 0.0 && hi > 64.0 * lo) ? sqrt(lo) * sqrt(hi) : 0.5 * (lo + hi);
}

constexpr int kSecMaxIt = 100;

// rho > 0 view of (d, z): reflected (-d reversed, z reversed) when rho < 0; z squared.
__global__ void secular_orient_kernel(const double* __restrict__ d, const double* __restrict__ z,
                                      double rho, int n, double* __restrict__ dr,
                                      double* __restrict__ z2r) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int src = rho < 0.0 ? n - 1 - i : i;
  dr[i] = rho < 0.0 ? -d[src] : d[src];
  z2r[i] = z[src] * z[src];
}

// far-field evaluation of the secular sums for a root of leaf q (FMM path): near-leaf
// sources directly (exact left/right split at sp), far field from the leaf's two local
// expansions at t = ((d_k - c_t) + tau) / r_t (barycentric value and t-derivative).
// What does not depend on tau (the lane's node values of the two expansions, the leaf's
// interval) is loaded once per root (init); an evaluation takes six warp sums: the
// barycentric denominator and its derivative first, then every lane's far terms divided
// by it join the four near sums.  (Round 2: C3 37.5 -> 34.4 us, C5 84 -> 78 us.  Keeping
// the lane's near sources in registers as well cost occupancy: slower.)
struct FarEval {
  const SecFmmDev* F;
  int q;          // leaf of the root
  double tk, wk;  // this lane's Chebyshev node and barycentric weight (lane < kSecP)
  double pl, pr;  // the leaf's two local expansions at this lane's node
  double ct, irt; // the leaf's target interval: centre, 1 / radius
  __device__ void init(int lane) {
    const int cell = F->leaf_cell[q];
    const SecFmmCell C = F->cells[cell];
    irt = fast_rcp(C.rt);  // (MUFU + Newton: no IEEE division in the loop)
    ct = C.ct;
    pl = pr = 0.0;
    if (lane < kSecP) {
      pl = F->psiL[cell * kSecP + lane];
      pr = F->psiR[cell * kSecP + lane];
    }
  }
  __device__ SecAcc operator()(const double* __restrict__ d, const double* __restrict__ z2,
                               double dk, double tau, int sp, int lane) const {
    const double t = ((dk - ct) + tau) * irt;
    double qk = 0.0, idx = 0.0;
    if (lane < kSecP) {
      double dx = t - tk;
      if (dx == 0.0) dx = 0x1.0p-50 * (1.0 + fabs(t));  // exact node: an ulp-scale nudge
      idx = fast_rcp(dx);
      qk = wk * idx;
    }
    const double den = warp_sum(qk), dden = warp_sum(-qk * idx);
    SecAcc a = {0, 0, 0, 0, 0};
    for (int g = F->near_off[q]; g < F->near_off[q + 1]; ++g) {
      const int lo = F->near_lo[g], hi = F->near_hi[g];
      for (int i = lo + lane; i < hi; i += 32) {
        const double rr = fast_rcp((__ldg(d + i) - dk) - tau);
        const double v = __ldg(z2 + i) * rr;
        if (i <= sp) {
          a.psi += v;
          a.dpsi = fma(v, rr, a.dpsi);
        } else {
          a.phi += v;
          a.dphi = fma(v, rr, a.dphi);
        }
      }
    }
    // far: value N/D and t-derivative (N' - (N/D) D')/D, split over the nodes
    const double id = fast_rcp(den);
    if (lane < kSecP) {
      const double nl = pl * qk * id, nr = pr * qk * id;
      a.psi += nl;
      a.phi += nr;
      a.dpsi += (-(pl * qk) * idx - nl * dden) * id * irt;
      a.dphi += (-(pr * qk) * idx - nr * dden) * id * irt;
    }
    a.psi = warp_sum(a.psi);
    a.phi = warp_sum(a.phi);
    a.dpsi = warp_sum(a.dpsi);
    a.dphi = warp_sum(a.dphi);
    a.eabs = fabs(a.psi) + fabs(a.phi);
    return a;
  }
};

// Solve root j (0-based, rho > 0 view) with the group g; eval(dk, tau, sp) returns the
// group-reduced sums.  All threads of g run the same control flow.
template <class G, class E>
__device__ void solve_root(int j, const double* __restrict__ d, const double* __restrict__ z2,
                           double rho, int n, const G& g, const E& eval, int32_t* __restrict__ k_out,
                           double* __restrict__ tau_out, int32_t* __restrict__ iters_out,
                           int32_t* __restrict__ status) {
#ifdef SVD1_SECPROF
  const long long clk0 = clock64();
#endif
  const bool refl = rho < 0.0;  // d, z2 hold (-d reversed, z^2 reversed); map the roots back
  const double r = fabs(rho);
  int k = j, it = 0, stat = 0;
  double tau;
  if (n == 1) {
    tau = r * z2[0];  // mu = d + rho z^2
  } else {
    const int sp = (j < n - 1) ? j : n - 2;
    const double dsp = d[sp], dsp1 = d[sp + 1];
    double lo, hi;
    bool solved = false;
    if (j < n - 1) {
      // interlacing bracket (d_j, d_{j+1}); origin = nearer pole by the sign of w(mid)
      const double gap = dsp1 - dsp, mid = 0.5 * gap;
      const SecAcc a = eval(dsp, mid, sp);
      const double w = 1.0 + r * (a.psi + a.phi);
      it = 1;
      if (w == 0.0) {  // the midpoint is the root
        k = j;
        tau = mid;
        lo = hi = 0.0;
        solved = true;
      } else if (w > 0.0) {
        k = j;  // root in (d_j, d_j + mid]
        lo = 0.0;
        hi = mid;
        tau = sec_step(w, a, r, 0.0, gap, mid, 0.0, mid);
      } else {
        k = j + 1;  // root in [d_{j+1} - mid, d_{j+1})
        lo = -mid;
        hi = 0.0;
        tau = sec_step(w, a, r, 0.0, gap, mid, mid, gap) - gap;  // offset from d_j -> from d_{j+1}
        if (!(tau > lo && tau < hi)) tau = -0.5 * mid;
      }
    } else {
      // last root in (d_{n-1}, d_{n-1} + rho ||z||^2]
      double s = 0.0;
      for (int i = g.tid; i < n; i += g.size) s += z2[i];
      s = g.sum(s);
      k = n - 1;
      lo = 0.0;
      hi = r * s;
      tau = hi;
      hi = hi * (1.0 + 4.0 * kEps);  // keep tau = r||z||^2 strictly inside
      // probe at the scale of the last gap: a root near d_{n-1} (the reflected view of a
      // rank-one downdate of a nearly singular Gram matrix) gets a bracket of its own
      // scale instead of (0, rho ||z||^2], where bisection would need ~50 halvings
      const double t0 = fmin(dsp1 - dsp, 0.5 * tau);
      if (t0 > 0.0) {
        const SecAcc a = eval(dsp1, t0, sp);
        ++it;
        const double w = 1.0 + r * (a.psi + a.phi);
        if (w >= 0.0) {
          hi = t0;
          tau = t0;
        } else {
          lo = t0;
        }
      }
    }
    if (!solved) {
      const double dk = d[k];
      const double p1 = dsp - dk, p2 = dsp1 - dk;  // pole offsets (one of them is 0)
      bool fin = false;
      for (;;) {
        if (++it > kSecMaxIt) {
          stat |= 1;
          break;
        }
        const SecAcc a = eval(dk, tau, sp);
        const double w = 1.0 + r * (a.psi + a.phi);
        if (w == 0.0) break;
        if (w < 0.0) lo = tau; else hi = tau;
        const double tolw = 8.0 * n * kEps * (1.0 + r * a.eabs);
        if (fabs(w) <= tolw) fin = true;
        const double tn = sec_step(w, a, r, p1, p2, tau, lo, hi);
        const bool tiny = fabs(tn - tau) <= 2.0 * kEps * fabs(tau);
        tau = tn;
        if (fin || tiny) break;
        if (hi - lo <= 4.0 * kEps * fmax(fabs(lo), fabs(hi))) break;
      }
    }
  }
  if (tau == 0.0) stat |= 2;
  if (g.tid == 0) {
    const int jo = refl ? n - 1 - j : j;
    k_out[jo] = refl ? n - 1 - k : k;
    tau_out[jo] = refl ? -tau : tau;
#ifdef SVD1_SECPROF
    if (iters_out) iters_out[jo] = int(((clock64() - clk0) >> 10) << 8) | min(it, 255);
#else
    if (iters_out) iters_out[jo] = it;
#endif
    if (stat) atomicOr(status, stat);
  }
}

// One warp per root.  FMM = false: every evaluation sums all n terms (sec_eval), the
// last root (widest bracket) on a block of its own.  FMM = true: roots 0..n-2 use
// FarEval (their leaf's near sources + two local expansions); the last root and the
// roots bracketed by outlier gaps (outside every target interval, listed in F.direct)
// take one block each, ahead of the nfar warp blocks, with the direct sum.
template <bool FMM>
// 4 blocks of 8 warps per SM (<= 64 registers, a few bytes spilled): a C3 solve's 4096
// warps fit in one wave (3 blocks: 80 registers, two waves; 34.7 -> 29.5 us)
#ifndef SVD1_SEC_MINB
#define SVD1_SEC_MINB 4
#endif
__global__ void __launch_bounds__(256, SVD1_SEC_MINB) secular_kernel(const double* __restrict__ d,
                                                     const double* __restrict__ z2, double rho, int n,
                                                     int32_t* __restrict__ k_out,
                                                     double* __restrict__ tau_out,
                                                     int32_t* __restrict__ iters_out,
                                                     int32_t* __restrict__ status, SecFmmDev F,
                                                     int j0, int j1) {
  const int lane = threadIdx.x & 31;
  // Roots j0 <= j < j1 of the rho > 0 view (a rank's slice; every root is
  // solved by the same code whatever the slice, so slices concatenate bitwise).
  // direct blocks first (they are the longest-running), then the warp blocks
  // (the direct solver's one such root is the last, with the widest bracket)
  const int ndir = FMM ? F.ndirect : 1;
  if (int(blockIdx.x) < ndir) {
    __shared__ double red[32];
    const BlockGrp g{int(threadIdx.x), int(blockDim.x), red};
    const int j = FMM ? F.direct[blockIdx.x] : n - 1;
    if (j < j0 || j >= j1) return;  // another rank's root
    solve_root(j, d, z2, rho, n, g,
               [&](double dk, double tau, int sp) { return sec_eval(d, z2, n, dk, tau, sp, g); },
               k_out, tau_out, iters_out, status);
    return;
  }
  const int j = j0 + int((int64_t(blockIdx.x - ndir) * blockDim.x + threadIdx.x) >> 5);
  if (j >= j1) return;
  const WarpGrp g{lane};
  if (j == n - 1) return;   // a direct block's
  if (!FMM) {
    solve_root(j, d, z2, rho, n, g,
               [&](double dk, double tau, int sp) { return sec_eval(d, z2, n, dk, tau, sp, g); },
               k_out, tau_out, iters_out, status);
    return;
  }
  FarEval fe;
  fe.F = &F;
  fe.tk = fe.wk = 0.0;
  int lo = 0, hi = F.nleaf;  // leaf q with leaf_lo[q] <= j < leaf_lo[q + 1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (F.leaf_lo[mid] <= j) lo = mid;
    else hi = mid;
  }
  fe.q = lo;
  // the root bracketed by an outlier gap lies outside its leaf's target interval
  if (F.cells[F.leaf_cell[lo]].pad && j == F.leaf_lo[lo + 1] - 1) return;  // a direct block's
  if (lane < kSecP) {
    const double th = (2.0 * lane + 1.0) / (2.0 * kSecP);
    fe.tk = cospi(th);
    fe.wk = ((lane & 1) ? -1.0 : 1.0) * sinpi(th);
  }
  fe.init(lane);
  solve_root(j, d, z2, rho, n, g,
             [&](double dk, double tau, int sp) { return fe(d, z2, dk, tau, sp, lane); }, k_out,
             tau_out, iters_out, status);
}

// ------------------------------------------------------------------ K2' build
// Far field of the secular sums on the source tree (one right-hand side, the charges
// z_i^2).  Operators as the apply's (scaled far field), each target
// cell's interval [d_lo, d_next] as its local-expansion box, evaluated on the fly.
__device__ __forceinline__ double bary(const double* __restrict__ t, const double* __restrict__ w,
                                       const double* __restrict__ f, double x) {
  // sum_i f_i u_i(x), barycentric Lagrange on the kSecP Chebyshev nodes
  // (unrolled: kSecP independent loads and reciprocals in flight; an exact node is
  // nudged by an ulp-scale step, whose interpolation error is below rounding)
  double num = 0.0, den = 0.0;
#pragma unroll
  for (int i = 0; i < kSecP; ++i) {
    double dx = x - t[i];
    if (dx == 0.0) dx = 0x1.0p-50;
    const double q = w[i] * fast_rcp(dx);
    num = fma(q, f[i], num);
    den += q;
  }
  return num * fast_rcp(den);
}

// Four launches, no level-by-level chain: phase 0 P2M (leaves); phase 1 M2M of every
// non-leaf cell directly from its leaf descendants (the M2M operator of any descendant
// has the same closed form, and is better conditioned than a chain); phase 2 M2L / P2L
// into the left / right expansions of every cell; phase 3 L2L into every leaf directly
// from all its ancestors (a local expansion is a polynomial: re-interpolation is
// exact), accumulated in place (leaves are nobody's ancestors).  Items are (cell, node).
__global__ void __launch_bounds__(256) secfmm_phase_kernel(SecFmmDev F, const double* __restrict__ d,
                                                          const double* __restrict__ z2, int phase) {
  __shared__ double t[kSecP], w[kSecP];
  if (threadIdx.x < kSecP) {
    const double th = (2.0 * threadIdx.x + 1.0) / (2.0 * kSecP);
    t[threadIdx.x] = cospi(th);
    w[threadIdx.x] = ((threadIdx.x & 1) ? -1.0 : 1.0) * sinpi(th);
  }
  __syncthreads();
  const int L = F.L, first_leaf = (1 << L) - 1;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (phase == 0) {  // P2M: Phi~_X[i] = sum_s z_s^2 / (t_i (d_s - c_X) - 3 r_X)
    if (e >= (1 << L) * kSecP) return;
    const int c = first_leaf + e / kSecP, i = e % kSecP;
    const SecFmmCell C = F.cells[c];
    double v = 0.0;
    for (int s = C.lo; s < C.hi; ++s) v += z2[s] * fast_rcp(t[i] * (d[s] - C.c) - 3.0 * C.r);
    F.phi[c * kSecP + i] = v;
  } else if (phase == 1) {  // M2M: Phi_P[i] = sum_leaves D (3 r_D / den) Phi_D(tc); warp per item
    const int e32 = e >> 5, lane = threadIdx.x & 31;
    if (e32 >= first_leaf * kSecP) return;
    const int c = e32 / kSecP, i = e32 % kSecP;
    const SecFmmCell P = F.cells[c];
    double v = 0.0;
    if (P.hi > P.lo) {
      int l = 0;
      while ((2 << l) - 1 <= c) ++l;                 // level of c
      const int dep = L - l, d0 = ((c + 1) << dep) - 1;
      for (int q = lane; q < (1 << dep); q += 32) {
        const int dc = d0 + q;
        const SecFmmCell D = F.cells[dc];
        if (D.hi <= D.lo) continue;
        const double rden = fast_rcp(3.0 * P.r + t[i] * (P.c - D.c));
        v += (3.0 * D.r * rden) * bary(t, w, F.phi + dc * kSecP, 3.0 * D.r * t[i] * rden);
      }
    }
    v = warp_sum(v);
    if (lane == 0) F.phi[c * kSecP + i] = v;
  } else if (phase == 2) {  // M2L / P2L into the left / right local expansions; warp per item
    const int e32 = e >> 5, lane = threadIdx.x & 31;
    if (e32 >= F.ncells * kSecP) return;
    const int c = e32 / kSecP, i = e32 % kSecP;
    const SecFmmCell Y = F.cells[c];
    const double y = Y.rt * t[i];  // node offset from c_t
    double vl = 0.0, vr = 0.0;
    for (int g = Y.m2l_off + lane; g < F.cells[c + 1].m2l_off; g += 32) {  // lane per partner
      const SecFmmPart X = F.parts[g];
      const SecFmmCell C = F.cells[X.cell];
      double v = 0.0;
      if (X.flags & 2) {  // P2L: sources of X at the node c_t + r_t t_i
        for (int s = C.lo; s < C.hi; ++s) v += z2[s] * fast_rcp((d[s] - Y.ct) - y);
      } else {  // M2L: t_X = 3 r_X / ((c_t - c_X) + r_t t_i), value t_X Phi_X(t_X)
        const double tx = 3.0 * C.r * fast_rcp((Y.ct - C.c) + y);
        v = tx * bary(t, w, F.phi + X.cell * kSecP, tx);
      }
      if (X.flags & 1) vr += v;
      else vl += v;
    }
    vl = warp_sum(vl);
    vr = warp_sum(vr);
    if (lane == 0) {
      F.psiL[c * kSecP + i] = vl;
      F.psiR[c * kSecP + i] = vr;
    }
  } else if (phase == 4) {  // direct P2M of EVERY cell from its own sources (replaces 0 + 1)
    const int e32 = e >> 5, lane = threadIdx.x & 31;
    if (e32 >= F.ncells * kSecP) return;
    const int c = e32 / kSecP, i = e32 % kSecP;
    const SecFmmCell C = F.cells[c];
    double v = 0.0;
    for (int s = C.lo + lane; s < C.hi; s += 32) v += z2[s] * fast_rcp(t[i] * (d[s] - C.c) - 3.0 * C.r);
    v = warp_sum(v);
    if (lane == 0) F.phi[c * kSecP + i] = v;
  } else if (phase == 5) {  // every leaf's local expansions directly from the M2L / P2L partners of
    // the leaf and of all its ancestors, evaluated at the leaf's nodes (replaces 2 + 3: the
    // ancestors' expansions interpolate the same far field the leaf's nodes see, and the
    // partners of an ancestor are admissible for every point of the leaf's interval)
    const int e32 = e >> 5, lane = threadIdx.x & 31;
    if (e32 >= (1 << L) * kSecP) return;
    const int c = first_leaf + e32 / kSecP, i = e32 % kSecP;
    const SecFmmCell Y = F.cells[c];
    if (Y.hi <= Y.lo) return;
    const double x = Y.ct + Y.rt * t[i];  // the node
    double vl = 0.0, vr = 0.0;
    // the (ancestor, partner) pairs of the chain, spread over the lanes: ancestor q's
    // partners are parts[off_q, off_q + cnt_q) (a few per cell, ~L cells)
    int offs[24], cnts[24], na = 0, total = 0;
    for (int a = c;; a = (a - 1) / 2) {
      if (na < 24) {
        offs[na] = F.cells[a].m2l_off;
        cnts[na] = F.cells[a + 1].m2l_off - offs[na];
        total += cnts[na];
        ++na;
      }
      if (a == 0) break;
    }
    for (int q = lane; q < total; q += 32) {
      int qa = 0, r = q;
      while (r >= cnts[qa]) r -= cnts[qa++];
      {
        const int g = offs[qa] + r;
        const SecFmmPart X = F.parts[g];
        const SecFmmCell C = F.cells[X.cell];
        double v = 0.0;
        if (X.flags & 2) {
          for (int s2 = C.lo; s2 < C.hi; ++s2) v += z2[s2] * fast_rcp(d[s2] - x);
        } else {
          const double tx = 3.0 * C.r * fast_rcp(x - C.c);
          v = tx * bary(t, w, F.phi + X.cell * kSecP, tx);
        }
        if (X.flags & 1) vr += v;
        else vl += v;
      }
    }
    vl = warp_sum(vl);
    vr = warp_sum(vr);
    if (lane == 0) {
      F.psiL[c * kSecP + i] = vl;
      F.psiR[c * kSecP + i] = vr;
    }
  } else {  // L2L: Psi_Y[i] += sum_{ancestors A} Psi_A(((c_Yt - c_At) + r_Yt t_i) / r_At); warp
    // per item, lane 2 a' + s evaluates side s of the a'-th ancestor
    const int e32 = e >> 5, lane = threadIdx.x & 31;
    if (e32 >= (1 << L) * kSecP) return;
    const int c = first_leaf + e32 / kSecP, i = e32 % kSecP;
    const SecFmmCell Y = F.cells[c];
    if (Y.hi <= Y.lo) return;
    double v = 0.0;
    if (lane < 2 * L) {
      int a = c;
      for (int q = 0; q <= (lane >> 1); ++q) a = (a - 1) / 2;
      const SecFmmCell A = F.cells[a];
      const double x = ((Y.ct - A.ct) + Y.rt * t[i]) * fast_rcp(A.rt);
      v = bary(t, w, ((lane & 1) ? F.psiR : F.psiL) + a * kSecP, x);
    }
    const double vl = warp_sum((lane & 1) ? 0.0 : v), vr = warp_sum((lane & 1) ? v : 0.0);
    if (lane == 0) {
      F.psiL[c * kSecP + i] += vl;
      F.psiR[c * kSecP + i] += vr;
    }
  }
}

// ------------------------------------------------------------------ K3a
// zhat_i^2 = |prod_j (mu_j - d_i)| / (|rho| prod_{j != i} |d_j - d_i|).  Thread per i,
// the j range split over gridDim.y chunks staged in shared memory (broadcast reads);
// numerator and denominator are separate running products (no division per term)
// renormalised with frexp every 8 factors.  Partials (mantissa, exponent) per chunk are
// combined in a fixed order by loewner_combine_kernel (deterministic).
constexpr int kLT = 128;   // threads (i) per block
constexpr int kLJ = 256;   // j per shared-memory tile

// The last block of each column of the grid (counted on ctr[blockIdx.x], which it
// resets) combines the chunks' partials in chunk order: deterministic, one launch.
__device__ __forceinline__ bool last_block_of_column(int* ctr) {
  __shared__ bool last;
  __threadfence();  // this block's partials are visible before it is counted
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ctr + blockIdx.x, 1) == int(gridDim.y) - 1;
  __syncthreads();
  if (last) __threadfence();
  return last;
}

// frexp by the exponent bits (the same mantissa in [0.5, 1) and exponent as frexp for a
// positive normal x; a zero, denormal, inf or NaN sets `bad`, and the caller redoes the
// index with frexp): a quarter of frexp's instructions, which dominated the kernel
__device__ __forceinline__ double frexp_bits(double x, int& e, bool& bad) {
  const int hi = __double2hiint(x), ex = (hi >> 20) & 0x7ff;
  bad |= (ex == 0) | (ex == 0x7ff);
  e = ex - 1022;
  return __hiloint2double((hi & 0x800fffff) | (1022 << 20), __double2loint(x));
}
__device__ __forceinline__ void renorm4_bits(double& Pn, double& Pd, double& Qn, double& Qd, int& E,
                                             bool& bad) {
  int e1, e2, e3, e4;
  Pn = frexp_bits(Pn, e1, bad);
  Pd = frexp_bits(Pd, e2, bad);
  Qn = frexp_bits(Qn, e3, bad);
  Qd = frexp_bits(Qd, e4, bad);
  E += (e1 - e2) + (e3 - e4);
}

__global__ void __launch_bounds__(kLT) loewner_partial_kernel(
    const double* __restrict__ d, const int32_t* __restrict__ k, const double* __restrict__ tau, int n,
    int chunk, double* __restrict__ pm, int32_t* __restrict__ pe, int* __restrict__ ctr, double rho,
    const double* __restrict__ z, double* __restrict__ zhat, int i_lo, int i_hi) {
  __shared__ double s_d[kLJ], s_mu[kLJ], s_t[kLJ];
  // i_lo <= i < i_hi: a rank's slice; the j chunks depend on n only (bitwise slices)
  const int i = i_lo + blockIdx.x * kLT + threadIdx.x;
  const int j0 = blockIdx.y * chunk, j1 = min(n, j0 + chunk);
  const double di = i < i_hi ? d[i] : 0.0;
  double Pn = 1.0, Pd = 1.0;
  int E = 0;
  bool bad = false;  // a product left the normal range between two renormalisations
  for (int jb = j0; jb < j1; jb += kLJ) {
    const int nj = min(kLJ, j1 - jb);
    __syncthreads();
    for (int t = threadIdx.x; t < nj; t += kLT) {
      s_d[t] = d[jb + t];
      s_mu[t] = d[k[jb + t]];
      s_t[t] = tau[jb + t];
    }
    __syncthreads();
    // two independent product chains (even / odd t) for ILP, renormalised every 8
    // factors each; merged below
    double Qn = 1.0, Qd = 1.0;
    int cnt = 0, t = 0;
    for (; t + 1 < nj; t += 2) {
      const int j = jb + t;
      Pn *= fabs((s_mu[t] - di) + s_t[t]);
      Pd *= (j == i) ? 1.0 : fabs(s_d[t] - di);
      Qn *= fabs((s_mu[t + 1] - di) + s_t[t + 1]);
      Qd *= (j + 1 == i) ? 1.0 : fabs(s_d[t + 1] - di);
      if (++cnt == 8) {
        renorm4_bits(Pn, Pd, Qn, Qd, E, bad);
        cnt = 0;
      }
    }
    if (t < nj) {
      Pn *= fabs((s_mu[t] - di) + s_t[t]);
      Pd *= (jb + t == i) ? 1.0 : fabs(s_d[t] - di);
    }
    renorm4_bits(Pn, Pd, Qn, Qd, E, bad);
    Pn *= Qn;
    Pd *= Qd;
  }
  if (bad && i < i_hi) {
    // a product left the normal range between two renormalisations (extreme spectra):
    // this chunk again from global memory, renormalised after every factor
    Pn = Pd = 1.0;
    E = 0;
    for (int j = j0; j < j1; ++j) {
      int e1, e2;
      Pn = frexp(Pn * fabs((d[k[j]] - di) + tau[j]), &e1);
      Pd = frexp(Pd * (j == i ? 1.0 : fabs(d[j] - di)), &e2);
      E += e1 - e2;
    }
  }
  if (i < i_hi) {
    int e;
    const double m = frexp(Pn / Pd, &e);
    pm[int64_t(blockIdx.y) * n + i] = m;
    pe[int64_t(blockIdx.y) * n + i] = E + e;
  }
  if (!last_block_of_column(ctr)) return;
  if (i < i_hi) {  // combine (the partials of other blocks: L2, not this SM's L1)
    double P = 1.0;
    int Et = 0;
    for (int c = 0; c < int(gridDim.y); ++c) {
      int e;
      P = frexp(P * __ldcg(pm + int64_t(c) * n + i), &e);
      Et += e + __ldcg(pe + int64_t(c) * n + i);
    }
    const double zh2 = ldexp(P, Et) / fabs(rho);
    zhat[i] = copysign(sqrt(zh2), z[i]);
  }
  if (threadIdx.x == 0) ctr[blockIdx.x] = 0;
}


// ------------------------------------------------------------------ K3b/K12
// For column j: y_i = zhat_i |tau_j| / ((d_i - d_kj) - tau_j)  (|y_i| <~ |zhat_i|: the
// origin pole is the nearest), s = sum y^2, colscale_j = |tau_j| / sqrt(s) = 1/||c_j||,
// carry_out[q][j] = (sum_i y_i carry_q[i]) / sqrt(s) = (X^T carry_q)_j.
// Thread per column j; the i range is split over gridDim.y chunks staged in shared
// memory; partial sums are reduced in chunk order by colnorm_combine_kernel.
constexpr int kCT = 128;
constexpr int kCI = 256;

template <int NC>
__global__ void __launch_bounds__(kCT) colnorm_partial_kernel(
    const double* __restrict__ d, const int32_t* __restrict__ k, const double* __restrict__ tau,
    const double* __restrict__ zhat, int n, int chunk, const double* __restrict__ carry,
    double* __restrict__ part, int* __restrict__ ctr, double* __restrict__ colscale,
    double* __restrict__ carry_out, int32_t* __restrict__ status, int j_lo, int j_hi, int64_t ldc) {
  __shared__ double s_d[kCI], s_z[kCI], s_c[NC > 0 ? NC : 1][kCI];
  // j_lo <= j < j_hi: a rank's slice; the i chunks depend on n only (bitwise slices);
  // carry_out[q] at carry_out + q * ldc
  const int j = j_lo + blockIdx.x * kCT + threadIdx.x;
  const int i0 = blockIdx.y * chunk, i1 = min(n, i0 + chunk);
  const bool ok = j < j_hi;
  const double dk = ok ? d[k[j]] : 0.0, tj = ok ? tau[j] : 1.0, at = fabs(tj);
  double s = 0.0, t[NC > 0 ? NC : 1];
#pragma unroll
  for (int q = 0; q < NC; ++q) t[q] = 0.0;
  for (int ib = i0; ib < i1; ib += kCI) {
    const int ni = min(kCI, i1 - ib);
    __syncthreads();
    for (int u = threadIdx.x; u < ni; u += kCT) {
      s_d[u] = d[ib + u];
      s_z[u] = zhat[ib + u] * 1.0;
#pragma unroll
      for (int q = 0; q < NC; ++q) s_c[q][u] = carry[int64_t(q) * n + ib + u];
    }
    __syncthreads();
#pragma unroll 4
    for (int u = 0; u < ni; ++u) {
      const double y = s_z[u] * at * fast_rcp((s_d[u] - dk) - tj);
      s = fma(y, y, s);
#pragma unroll
      for (int q = 0; q < NC; ++q) t[q] = fma(y, s_c[q][u], t[q]);
    }
  }
  if (ok) {
    const int64_t base = int64_t(blockIdx.y) * (NC + 1) * n;
    part[base + j] = s;
#pragma unroll
    for (int q = 0; q < NC; ++q) part[base + int64_t(q + 1) * n + j] = t[q];
  }
  if (!last_block_of_column(ctr)) return;
  if (ok) {  // combine in chunk order
    const int64_t cstride = int64_t(NC + 1) * n;
    double ss = 0.0;
    for (int c = 0; c < int(gridDim.y); ++c) ss += __ldcg(part + int64_t(c) * cstride + j);
    const double rs = sqrt(ss);
    const double cs = fabs(tj) / rs;
    if (!(cs > 0.0) || !isfinite(cs)) atomicOr(status, 4);
    colscale[j] = cs;
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      double tt = 0.0;
      for (int c = 0; c < int(gridDim.y); ++c) tt += __ldcg(part + int64_t(c) * cstride + int64_t(q + 1) * n + j);
      carry_out[int64_t(q) * ldc + j] = tt / rs;
    }
  }
  if (threadIdx.x == 0) ctr[blockIdx.x] = 0;
}

// ------------------------------------------------------- K3a/K3b, warp per index
// The same sums with a WARP per index (i for Loewner, j for the norms) and the lanes
// striding the inner index: n warps of n/32 terms each (instead of blocks of short
// chunks combined by a last block), so the kernels have enough resident warps to hide
// the FP64 / MUFU latency.  The block's 8 warps share the inner index's tiles in shared
// memory.  Every index's result depends on n only (lane partials combined by a fixed xor
// tree), so a rank's slice of indices is bitwise the same as in the full range.
constexpr int kWW = 8;     // warps (indices) per block
constexpr int kWT = 256;   // inner-index tile

__device__ __forceinline__ void mant_exp_mul(double& m, int& e, double m2, int e2) {
  int ee;
  m = frexp(m * m2, &ee);
  e += e2 + ee;
}

// j tiles of 1024 (24 KB of shared memory), the next tile's values prefetched into
// registers while the current one is multiplied (its k two tiles ahead: d[k[j]] is a
// dependent load), so the global-memory latency is not exposed once per tile
constexpr int kLWT = 1024;
constexpr int kLWQ = kLWT / (32 * kWW);  // tile elements per thread

__global__ void __launch_bounds__(32 * kWW) loewner_warp_kernel(
    const double* __restrict__ d, const int32_t* __restrict__ k, const double* __restrict__ tau, int n,
    double rho, const double* __restrict__ z, double* __restrict__ zhat, int i_lo, int i_hi) {
  __shared__ double s_d[kLWT], s_mu[kLWT], s_t[kLWT];
  const int lane = threadIdx.x & 31;
  const int i = i_lo + blockIdx.x * kWW + (threadIdx.x >> 5);
  const bool ok = i < i_hi;
  const double di = ok ? d[i] : 0.0;
  // two product chains per lane (even / odd 32-strides), numerator and denominator apart
  // (no division per term), renormalised with frexp (exact) every 4 factors per chain
  double Pn = 1.0, Pd = 1.0, Qn = 1.0, Qd = 1.0;
  int E = 0, cnt = 0;
  bool bad = false;  // a product left the normal range between two exponent-bit renorms
  double rd[kLWQ], rm[kLWQ], rt[kLWQ];
  int rk[kLWQ];
  auto fetch_k = [&](int jb) {
#pragma unroll
    for (int q = 0; q < kLWQ; ++q) {
      const int j = jb + int(threadIdx.x) + 32 * kWW * q;
      rk[q] = j < n ? __ldg(k + j) : 0;
    }
  };
  auto fetch = [&](int jb) {  // (rk holds tile jb's k)
#pragma unroll
    for (int q = 0; q < kLWQ; ++q) {
      const int j = jb + int(threadIdx.x) + 32 * kWW * q;
      if (j < n) {
        rd[q] = __ldg(d + j);
        rm[q] = __ldg(d + rk[q]);
        rt[q] = __ldg(tau + j);
      }
    }
  };
  fetch_k(0);
  fetch(0);
  fetch_k(kLWT);
  for (int jb = 0; jb < n; jb += kLWT) {
    const int nj = min(kLWT, n - jb);
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kLWQ; ++q) {
      const int t = int(threadIdx.x) + 32 * kWW * q;
      if (t < nj) {
        s_d[t] = rd[q];
        s_mu[t] = rm[q];
        s_t[t] = rt[q];
      }
    }
    __syncthreads();
    if (jb + kLWT < n) {  // next tile in flight during this one
      fetch(jb + kLWT);
      fetch_k(jb + 2 * kLWT);
    }
    if (nj == kLWT && (i < jb || i >= jb + kLWT)) {
      // a full tile without the diagonal (warp-uniform): unrolled, no j == i select
#pragma unroll
      for (int u = 0; u < kLWT / 64; ++u) {
        const int t = lane + 64 * u;
        Pn *= fabs((s_mu[t] - di) + s_t[t]);
        Pd *= fabs(s_d[t] - di);
        Qn *= fabs((s_mu[t + 32] - di) + s_t[t + 32]);
        Qd *= fabs(s_d[t + 32] - di);
        if ((u & 3) == 3) renorm4_bits(Pn, Pd, Qn, Qd, E, bad);
      }
      continue;
    }
    for (int t = lane; t < nj; t += 64) {
      Pn *= fabs((s_mu[t] - di) + s_t[t]);
      Pd *= (jb + t == i) ? 1.0 : fabs(s_d[t] - di);
      if (t + 32 < nj) {
        Qn *= fabs((s_mu[t + 32] - di) + s_t[t + 32]);
        Qd *= (jb + t + 32 == i) ? 1.0 : fabs(s_d[t + 32] - di);
      }
      if (++cnt == 4) {
        renorm4_bits(Pn, Pd, Qn, Qd, E, bad);
        cnt = 0;
      }
    }
  }
  renorm4_bits(Pn, Pd, Qn, Qd, E, bad);
  if (__any_sync(0xffffffffu, bad)) {
    // out of range between renorms (extreme spectra): this index again, from global
    // memory, renormalised after every factor (the same products, the same order)
    Pn = Pd = Qn = Qd = 1.0;
    E = 0;
    for (int jb = 0; jb < n; jb += 64)
      for (int h = 0; h < 2; ++h) {
        const int j = jb + lane + 32 * h;
        if (j >= n) continue;
        double& N = h ? Qn : Pn;
        double& D = h ? Qd : Pd;
        int e1, e2;
        N = frexp(N * fabs((d[k[j]] - di) + tau[j]), &e1);
        D = frexp(D * (j == i ? 1.0 : fabs(d[j] - di)), &e2);
        E += e1 - e2;
      }
  }
  int e;
  double m = frexp((Pn * Qn) / (Pd * Qd), &e);
  E += e;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
    mant_exp_mul(m, E, __shfl_xor_sync(0xffffffffu, m, o), __shfl_xor_sync(0xffffffffu, E, o));
  if (ok && lane == 0) zhat[i] = copysign(sqrt(ldexp(m, E) / fabs(rho)), z[i]);
}

template <int NC>
__global__ void __launch_bounds__(32 * kWW) colnorm_warp_kernel(
    const double* __restrict__ d, const int32_t* __restrict__ k, const double* __restrict__ tau,
    const double* __restrict__ zhat, int n, const double* __restrict__ carry, double* __restrict__ colscale,
    double* __restrict__ carry_out, int32_t* __restrict__ status, int j_lo, int j_hi, int64_t ldc) {
  __shared__ double s_d[kWT], s_z[kWT], s_c[NC > 0 ? NC : 1][kWT];
  const int lane = threadIdx.x & 31;
  const int j = j_lo + blockIdx.x * kWW + (threadIdx.x >> 5);
  const bool ok = j < j_hi;
  const double dk = ok ? d[k[j]] : 0.0, tj = ok ? tau[j] : 1.0, at = fabs(tj);
  double s = 0.0, t[NC > 0 ? NC : 1];
#pragma unroll
  for (int q = 0; q < NC; ++q) t[q] = 0.0;
  for (int ib = 0; ib < n; ib += kWT) {
    const int ni = min(kWT, n - ib);
    __syncthreads();
    for (int u = threadIdx.x; u < ni; u += 32 * kWW) {
      s_d[u] = d[ib + u];
      s_z[u] = zhat[ib + u];
#pragma unroll
      for (int q = 0; q < NC; ++q) s_c[q][u] = carry[int64_t(q) * n + ib + u];
    }
    __syncthreads();
#pragma unroll 2
    for (int u = lane; u < ni; u += 32) {
      // y_i = zhat_i |tau_j| / ((d_i - d_kj) - tau_j): bounded by |zhat_i| (nearest pole)
      const double y = s_z[u] * at * fast_rcp((s_d[u] - dk) - tj);
      s = fma(y, y, s);
#pragma unroll
      for (int q = 0; q < NC; ++q) t[q] = fma(y, s_c[q][u], t[q]);
    }
  }
  s = warp_sum(s);
#pragma unroll
  for (int q = 0; q < NC; ++q) t[q] = warp_sum(t[q]);
  if (ok && lane == 0) {
    const double rs = sqrt(s);
    const double cs = at / rs;
    if (!(cs > 0.0) || !isfinite(cs)) atomicOr(status, 4);
    colscale[j] = cs;
#pragma unroll
    for (int q = 0; q < NC; ++q) carry_out[int64_t(q) * ldc + j] = t[q] / rs;
  }
}

// The chunked norm kernel with J columns per thread (columns j and j + kCT, ...): every
// broadcast shared-memory read of a source feeds J terms.  Same partials / combine as
// colnorm_partial_kernel (J = 1 is that kernel's arithmetic).
template <int NC, int J>
__global__ void __launch_bounds__(kCT) colnorm_multi_kernel(
    const double* __restrict__ d, const int32_t* __restrict__ k, const double* __restrict__ tau,
    const double* __restrict__ zhat, int n, int chunk, const double* __restrict__ carry,
    double* __restrict__ part, int* __restrict__ ctr, double* __restrict__ colscale,
    double* __restrict__ carry_out, int32_t* __restrict__ status, int j_lo, int j_hi, int64_t ldc) {
  __shared__ double s_d[kCI], s_z[kCI], s_c[NC > 0 ? NC : 1][kCI];
  const int i0 = blockIdx.y * chunk, i1 = min(n, i0 + chunk);
  int jj[J];
  bool ok[J];
  double dk[J], tj[J], at[J], s[J], t[J][NC > 0 ? NC : 1];
#pragma unroll
  for (int c = 0; c < J; ++c) {
    jj[c] = j_lo + blockIdx.x * (kCT * J) + c * kCT + threadIdx.x;
    ok[c] = jj[c] < j_hi;
    dk[c] = ok[c] ? d[k[jj[c]]] : 0.0;
    tj[c] = ok[c] ? tau[jj[c]] : 1.0;
    at[c] = fabs(tj[c]);
    s[c] = 0.0;
#pragma unroll
    for (int q = 0; q < NC; ++q) t[c][q] = 0.0;
  }
  for (int ib = i0; ib < i1; ib += kCI) {
    const int ni = min(kCI, i1 - ib);
    __syncthreads();
    for (int u = threadIdx.x; u < ni; u += kCT) {
      s_d[u] = d[ib + u];
      s_z[u] = zhat[ib + u];
#pragma unroll
      for (int q = 0; q < NC; ++q) s_c[q][u] = carry[int64_t(q) * n + ib + u];
    }
    __syncthreads();
#pragma unroll 2
    for (int u = 0; u < ni; ++u) {
      const double du = s_d[u], zu = s_z[u];
      double cq[NC > 0 ? NC : 1];
#pragma unroll
      for (int q = 0; q < NC; ++q) cq[q] = s_c[q][u];
#pragma unroll
      for (int c = 0; c < J; ++c) {
        const double y = zu * at[c] * fast_rcp((du - dk[c]) - tj[c]);
        s[c] = fma(y, y, s[c]);
#pragma unroll
        for (int q = 0; q < NC; ++q) t[c][q] = fma(y, cq[q], t[c][q]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < J; ++c)
    if (ok[c]) {
      const int64_t base = int64_t(blockIdx.y) * (NC + 1) * n;
      part[base + jj[c]] = s[c];
#pragma unroll
      for (int q = 0; q < NC; ++q) part[base + int64_t(q + 1) * n + jj[c]] = t[c][q];
    }
  if (!last_block_of_column(ctr)) return;
  const int64_t cstride = int64_t(NC + 1) * n;
#pragma unroll
  for (int c = 0; c < J; ++c)
    if (ok[c]) {  // combine in chunk order
      const int j = jj[c];
      double ss = 0.0;
      for (int b = 0; b < int(gridDim.y); ++b) ss += __ldcg(part + int64_t(b) * cstride + j);
      const double rs = sqrt(ss);
      const double cs = fabs(tj[c]) / rs;
      if (!(cs > 0.0) || !isfinite(cs)) atomicOr(status, 4);
      colscale[j] = cs;
#pragma unroll
      for (int q = 0; q < NC; ++q) {
        double tt = 0.0;
        for (int b = 0; b < int(gridDim.y); ++b) tt += __ldcg(part + int64_t(b) * cstride + int64_t(q + 1) * n + j);
        carry_out[int64_t(q) * ldc + j] = tt / rs;
      }
    }
  if (threadIdx.x == 0) ctr[blockIdx.x] = 0;
}

// thread per (j, q): q = 0 -> colscale_j (and the status check), q >= 1 -> carried
// vector q-1 (which also needs ||y||: recomputed, the partials are L2-resident)

inline unsigned blocks_for_warps(int64_t nwarps, int threads = 256) {
  return unsigned((nwarps * 32 + threads - 1) / threads);
}

}  // namespace

// ------------------------------------------------------------------ wrappers
constexpr int kDotBlocks = 64;
constexpr int kMaxDotVecs = 32;  // project_many: the dots of up to this many updates in one launch

int64_t project_partial_elems(int64_t u_rows, int64_t m, int64_t v_rows, int64_t n) {
  const int64_t cu = std::min<int64_t>(64, std::max<int64_t>(1, (u_rows + 31) / 32));
  const int64_t cv = std::min<int64_t>(64, std::max<int64_t>(1, (v_rows + 31) / 32));
  // (also enough for project_many's 8-vector passes)
  return std::max(cu * 5 * m + cv * n, std::max(cu * 8 * m, cv * 8 * n)) + 6 * kDotBlocks * kMaxDotVecs;
}

svd1_status fill_probes(uint64_t seed, int64_t row0, int64_t rows, double* g, cudaStream_t st,
                        int64_t* launches) {
  if (rows <= 0) return SVD1_OK;
  probe_fill_kernel<<<unsigned((4 * rows + 255) / 256), 256, 0, st>>>(seed, row0, rows, g);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status project(const double* U, int64_t ldu, int64_t u_rows, int64_t m, int64_t u_row0,
                    const double* V, int64_t ldv, int64_t v_rows, int64_t n, int64_t v_row0,
                    const double* a, const double* b, double* part, int64_t partial_cap,
                    double* proj, const double* probes, cudaStream_t st, int64_t* launches,
                    int64_t vcols) {
  // vcols < n (thin V): only the first vcols entries of V^T b are formed, the rest of the
  // n-wide block is zero (the layout stays 5m + n + 6)
  if (vcols < 0) vcols = n;
  const int64_t cu = std::min<int64_t>(64, std::max<int64_t>(1, (u_rows + 31) / 32));
  const int64_t cv = std::min<int64_t>(64, std::max<int64_t>(1, (v_rows + 31) / 32));
  if (cu * 5 * m + cv * n + 6 * kDotBlocks > partial_cap) return SVD1_E_NOMEM;
  const int rpc_u = int((u_rows + cu - 1) / cu), rpc_v = int((v_rows + cv - 1) / cv);
  double* part_u = part;
  double* part_v = part + cu * 5 * m;
  if (u_rows > 0) {
    proj_partial_kernel<5><<<dim3(unsigned((m + 255) / 256), unsigned(cu)), 256, 0, st>>>(
        U, ldu, u_rows, m, a, u_row0, rpc_u, probes, part_u);
    proj_reduce_kernel<<<unsigned((5 * m + 255) / 256), 256, 0, st>>>(part_u, int(cu), 5, m, proj);
    *launches += 2;
  } else {
    SVD1_CUDA_TRY(cudaMemsetAsync(proj, 0, sizeof(double) * 5 * m, st));
  }
  if (v_rows > 0) {
    proj_partial_kernel<1><<<dim3(unsigned((vcols + 255) / 256), unsigned(cv)), 256, 0, st>>>(
        V, ldv, v_rows, vcols, b, v_row0, rpc_v, nullptr, part_v);
    proj_reduce_kernel<<<unsigned((vcols + 255) / 256), 256, 0, st>>>(part_v, int(cv), 1, vcols, proj + 5 * m);
    if (vcols < n) SVD1_CUDA_TRY(cudaMemsetAsync(proj + 5 * m + vcols, 0, sizeof(double) * (n - vcols), st));
    *launches += 2;
  } else {
    SVD1_CUDA_TRY(cudaMemsetAsync(proj + 5 * m, 0, sizeof(double) * n, st));
  }
  double* part_d = part + cu * 5 * m + cv * n;
  proj_dots_kernel<<<kDotBlocks, 256, 0, st>>>(a, u_rows, u_row0, b, v_rows, v_row0, probes, part_d);
  proj_dots_final<<<1, 32, 0, st>>>(part_d, kDotBlocks, proj + 5 * m + n);
  *launches += 2;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

// dst row (base - s) <- src row s for s = 1 .. count (the batch's carried rows are stored
// newest-last: row 4 + (K - 1 - s) of the U side holds update s's x_a)
__global__ void copy_rows_rev_kernel(double* __restrict__ dst, int64_t ldd, int64_t base,
                                     const double* __restrict__ src, int64_t lds, int64_t cols, int count) {
  const int s = 1 + int(blockIdx.y);
  if (s > count) return;
  const double* in = src + int64_t(s) * lds;
  double* out = dst + (base - s) * ldd;
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < cols; c += int64_t(gridDim.x) * blockDim.x)
    out[c] = in[c];
}

svd1_status copy_rows_rev(double* dst, int64_t ldd, int64_t base, const double* src, int64_t lds, int64_t cols,
                          int count, cudaStream_t st, int64_t* launches) {
  if (count <= 0 || cols <= 0) return SVD1_OK;
  copy_rows_rev_kernel<<<dim3(unsigned(std::min<int64_t>(16, (cols + 255) / 256)), unsigned(count)), 256, 0, st>>>(
      dst, ldd, base, src, lds, cols, count);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

// warp per row: q = (b_r - V_r . y) / beta into column m
__global__ void null_direction_kernel(int64_t rows, double* __restrict__ V, int64_t ldv, int64_t m,
                                      const double* __restrict__ b, const double* __restrict__ y,
                                      double inv_beta) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const double* row = V + r * ldv;
  double s = 0.0;
  for (int64_t c = lane; c < m; c += 32) s = fma(row[c], y[c], s);
  s = warp_sum(s);
  if (lane == 0) V[r * ldv + m] = (b[r] - s) * inv_beta;
}

svd1_status null_direction(int64_t rows, double* V, int64_t ldv, int64_t m, const double* b, int64_t row0,
                           const double* y, double inv_beta, cudaStream_t st, int64_t* launches) {
  if (rows <= 0) return SVD1_OK;
  null_direction_kernel<<<unsigned((rows * 32 + 255) / 256), 256, 0, st>>>(rows, V, ldv, m, b + row0, y,
                                                                           inv_beta);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

__global__ void thin_carry_kernel(int rows, double* __restrict__ rv, int64_t ld, int64_t m,
                                  const double* __restrict__ yt, const double* __restrict__ gram, int t,
                                  int K, double inv_beta) {
  const int j = blockIdx.x;  // block per carried row
  if (j >= rows) return;
  const double* ys = rv + int64_t(j) * ld;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < m; c += blockDim.x) s = fma(yt[c], ys[c], s);
  __shared__ double red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (int q = 0; q < int(blockDim.x >> 5); ++q) acc += red[q];
    rv[int64_t(j) * ld + m] = (gram[int64_t(t) * K + (K - 1 - j)] - acc) * inv_beta;
  }
}

svd1_status thin_carry(int rows, double* rv, int64_t ld, int64_t m, const double* yt, const double* gram, int t,
                       int K, double inv_beta, cudaStream_t st, int64_t* launches) {
  if (rows <= 0) return SVD1_OK;
  thin_carry_kernel<<<rows, 256, 0, st>>>(rows, rv, ld, m, yt, gram, t, K, inv_beta);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

__global__ void gram_rows_kernel(int K, const double* __restrict__ B, int64_t ldb, int64_t n,
                                 double* __restrict__ gram) {
  const int t = blockIdx.x / K, s2 = blockIdx.x % K;
  double s = 0.0;
  for (int64_t c = threadIdx.x; c < n; c += blockDim.x) s = fma(B[int64_t(t) * ldb + c], B[int64_t(s2) * ldb + c], s);
  __shared__ double red[8];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int q = 0; q < int(blockDim.x >> 5); ++q) u += red[q];
    gram[int64_t(t) * K + s2] = u;
  }
}

svd1_status gram_rows(int K, const double* B, int64_t ldb, int64_t n, double* gram, cudaStream_t st,
                      int64_t* launches) {
  if (K <= 0) return SVD1_OK;
  gram_rows_kernel<<<K * K, 256, 0, st>>>(K, B, ldb, n, gram);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status project_many(const double* U, int64_t ldu, int64_t u_rows, int64_t m, int64_t u_row0,
                         const double* V, int64_t ldv, int64_t v_rows, int64_t n, int64_t v_row0, int64_t vcols,
                         const double* A, int64_t lda, const double* B, int64_t ldb, int K, const double* probes,
                         double* part, int64_t partial_cap, double* proj, int64_t nproj, cudaStream_t st,
                         int64_t* launches) {
  if (K <= 0) return SVD1_OK;
  const int64_t cu = std::min<int64_t>(64, std::max<int64_t>(1, (u_rows + 31) / 32));
  const int64_t cv = std::min<int64_t>(64, std::max<int64_t>(1, (v_rows + 31) / 32));
  if (K > kMaxDotVecs || std::max(cu * kMV * m, cv * kMV * n) + 6 * kDotBlocks * K > partial_cap)
    return SVD1_E_NOMEM;
  const int rpc_u = int((u_rows + cu - 1) / cu), rpc_v = int((v_rows + cv - 1) / cv);
  for (int t0 = 0; t0 < K; t0 += kMV) {
    const int nv = std::min(kMV, K - t0);
    if (u_rows > 0) {
      proj_multi_kernel<<<dim3(unsigned((m + 255) / 256), unsigned(cu)), 256, 0, st>>>(
          U, ldu, u_rows, m, A + int64_t(t0) * lda, lda, nv, u_row0, rpc_u, part);
      proj_reduce_strided_kernel<<<unsigned((nv * m + 255) / 256), 256, 0, st>>>(part, int(cu), nv, m,
                                                                                 proj + int64_t(t0) * nproj, nproj);
    }
    if (v_rows > 0) {
      proj_multi_kernel<<<dim3(unsigned((vcols + 255) / 256), unsigned(cv)), 256, 0, st>>>(
          V, ldv, v_rows, vcols, B + int64_t(t0) * ldb, ldb, nv, v_row0, rpc_v, part);
      proj_reduce_strided_kernel<<<unsigned((nv * vcols + 255) / 256), 256, 0, st>>>(
          part, int(cv), nv, vcols, proj + int64_t(t0) * nproj + 5 * m, nproj);
    }
    *launches += 4;
  }
  double* part_d = part + std::max(cu * kMV * m, cv * kMV * n);
  for (int t = 0; t < K; ++t) {  // zeros where nothing is projected
    double* pt = proj + int64_t(t) * nproj;
    if (u_rows <= 0) SVD1_CUDA_TRY(cudaMemsetAsync(pt, 0, sizeof(double) * m, st));
    if (v_rows <= 0 || vcols < n)
      SVD1_CUDA_TRY(cudaMemsetAsync(pt + 5 * m + (v_rows > 0 ? vcols : 0), 0,
                                    sizeof(double) * (n - (v_rows > 0 ? vcols : 0)), st));
  }
  // the dots of every update: one launch each for the block partials and their sums (the
  // same blocks and order as one update's, so bitwise the per-update values)
  proj_dots_kernel<<<dim3(kDotBlocks, unsigned(K)), 256, 0, st>>>(A, u_rows, u_row0, B, v_rows, v_row0, probes,
                                                                  part_d, lda, ldb);
  proj_dots_final<<<unsigned(K), 32, 0, st>>>(part_d, kDotBlocks, proj + 5 * m + n, nproj);
  *launches += 2;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status secular(const double* d, const double* z2, double rho, int n, int j0, int j1, int32_t* k_out,
                    double* tau_out, int32_t* iters_out, int32_t* status, cudaStream_t st,
                    int64_t* launches) {
  if (n <= 0 || j1 <= j0) return SVD1_OK;
  secular_kernel<false><<<1 + blocks_for_warps(j1 - j0), 256, 0, st>>>(d, z2, rho, n, k_out, tau_out, iters_out,
                                                                         status, SecFmmDev{}, j0, j1);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status secular_fmm(const double* d, const double* z2, double rho, int n, int j0, int j1,
                        const SecFmmDev& F, int32_t* k_out, double* tau_out, int32_t* iters_out,
                        int32_t* status, cudaStream_t st, int64_t* launches) {
  if (n <= 0 || j1 <= j0) return SVD1_OK;
  auto grid = [](int items) { return unsigned(std::max(1, (items + 255) / 256)); };
  const int L = F.L;
  static const bool chain = std::getenv("SVD1_SECFMM_CHAIN") != nullptr;  // the round-1 four phases
  if (chain) {
    secfmm_phase_kernel<<<grid((1 << L) * kSecP), 256, 0, st>>>(F, d, z2, 0);
    secfmm_phase_kernel<<<grid(((1 << L) - 1) * kSecP * 32), 256, 0, st>>>(F, d, z2, 1);
    secfmm_phase_kernel<<<grid(F.ncells * kSecP * 32), 256, 0, st>>>(F, d, z2, 2);
    secfmm_phase_kernel<<<grid((1 << L) * kSecP * 32), 256, 0, st>>>(F, d, z2, 3);
    *launches += 2;
  } else {  // two launches: every cell's far field from its sources, every leaf's local
            // expansions from the partners of its ancestor chain
    secfmm_phase_kernel<<<grid(F.ncells * kSecP * 32), 256, 0, st>>>(F, d, z2, 4);
    secfmm_phase_kernel<<<grid((1 << L) * kSecP * 32), 256, 0, st>>>(F, d, z2, 5);
  }
  const int nfar = blocks_for_warps(j1 - j0);
  secular_kernel<true><<<nfar + F.ndirect, 256, 0, st>>>(d, z2, rho, n, k_out, tau_out, iters_out, status, F,
                                                          j0, j1);
  *launches += 3;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

// Loewner: warp per index below n = 8192 (C3: 30 vs 37 us), the chunked kernel above it
// (C5, n = 16384: 222 vs 312 us -- the warp kernel's strided shared-memory reads become the
// bound); SVD1_LOEWNER_CHUNKED=0/1 forces one.  Norms: the chunked kernel (its per-source
// values are broadcast shared-memory reads; the warp-per-column variant, selected by
// SVD1_COLNORM_WARP=1, reads twice the shared-memory wavefronts and measured 48 vs 36 us)
static bool loewner_chunked(int n) {
  static const int v = [] {
    const char* e = std::getenv("SVD1_LOEWNER_CHUNKED");
    return e ? atoi(e) : -1;
  }();
  return v >= 0 ? v != 0 : n >= 8192;
}
static bool colnorm_chunked() {
  static const bool v = std::getenv("SVD1_COLNORM_WARP") == nullptr;
  return v;
}

static int colnorm_J() {  // columns per thread of the norm kernel (SVD1_COLNORM_J, tuning)
  static const int v = [] {
    const char* e = std::getenv("SVD1_COLNORM_J");
    return e ? std::max(1, std::min(2, atoi(e))) : 1;
  }();
  return v;
}
static int chunk_blocks() {  // target blocks (x 148) of the chunked kernels (SVD1_CHUNK_BLOCKS, tuning)
  static const int v = [] {
    const char* e = std::getenv("SVD1_CHUNK_BLOCKS");
    return e ? std::max(1, atoi(e)) : 8;  // measured: 8 (C5 norms 229 -> 200 us), C3 unchanged
  }();
  return v;
}

// chunks over the inner index: enough blocks to fill 148 SMs a few times over (a function
// of n only: rank slices of the outer index see the same chunks)
static int inner_chunks(int n, int threads, int per_thread = 1) {
  const int outer = (n + threads * per_thread - 1) / (threads * per_thread);
  static const int min_chunk = [] {  // smallest inner chunk (SVD1_CHUNK_MIN, tuning)
    const char* e = std::getenv("SVD1_CHUNK_MIN");
    return e ? std::max(32, atoi(e)) : 256;
  }();
  int ch = (chunk_blocks() * 148 + outer - 1) / outer;
  ch = std::max(1, std::min(ch, (n + min_chunk - 1) / min_chunk));
  return ch;
}

// the Loewner kernel is latency-bound (a running product with renormalisation): more
// j chunks, so more warps per SM, than the norm kernel
static int loewner_chunks(int n) {
  const int outer = (n + kLT - 1) / kLT;
  int ch = (16 * 148 + outer - 1) / outer;
  return std::max(1, std::min(ch, (n + 63) / 64));
}




int64_t spectral_scratch_elems(int n, int ncarry) {
  const int ch = std::max(loewner_chunks(n), std::max(inner_chunks(n, kCT), inner_chunks(n, kCT, 2)));
  return int64_t(ch) * n * (ncarry + 2) + 16;
}

svd1_status secular_orient(const double* d, const double* z, double rho, int n, double* dr,
                           double* z2r, cudaStream_t st, int64_t* launches) {
  if (n <= 0) return SVD1_OK;
  secular_orient_kernel<<<unsigned((n + 255) / 256), 256, 0, st>>>(d, z, rho, n, dr, z2r);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status loewner(const double* d, const int32_t* k, const double* tau, double rho,
                    const double* z, int n, int i0, int i1, double* zhat, double* scratch, int* ctr,
                    cudaStream_t st, int64_t* launches) {
  if (n <= 0 || i1 <= i0) return SVD1_OK;
  if (!loewner_chunked(n)) {
    loewner_warp_kernel<<<unsigned((i1 - i0 + kWW - 1) / kWW), 32 * kWW, 0, st>>>(d, k, tau, n, rho, z, zhat,
                                                                                  i0, i1);
    *launches += 1;
    SVD1_CUDA_TRY(cudaGetLastError());
    return SVD1_OK;
  }
  const int ch = loewner_chunks(n);
  const int chunk = (n + ch - 1) / ch;
  double* pm = scratch;
  int32_t* pe = reinterpret_cast<int32_t*>(scratch + int64_t(ch) * n);
  loewner_partial_kernel<<<dim3(unsigned((i1 - i0 + kLT - 1) / kLT), unsigned(ch)), kLT, 0, st>>>(
      d, k, tau, n, chunk, pm, pe, ctr, rho, z, zhat, i0, i1);
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status colnorm_carry(const double* d, const int32_t* k, const double* tau,
                          const double* zhat, int n, int j0, int j1, const double* carry, int ncarry,
                          double* colscale, double* carry_out, int64_t ldc, int32_t* status, double* scratch,
                          int* ctr, cudaStream_t st, int64_t* launches) {
  if (n <= 0 || j1 <= j0) return SVD1_OK;
  if (!colnorm_chunked()) {
    const unsigned gw = unsigned((j1 - j0 + kWW - 1) / kWW);
    switch (ncarry) {
#define SVD1_CW(NC) case NC: colnorm_warp_kernel<NC><<<gw, 32 * kWW, 0, st>>>(d, k, tau, zhat, n, carry, colscale, \
                                                                     carry_out, status, j0, j1, ldc); break;
      SVD1_CW(0) SVD1_CW(1) SVD1_CW(2) SVD1_CW(3) SVD1_CW(4) SVD1_CW(5) SVD1_CW(6)
#undef SVD1_CW
      default: return SVD1_E_INVALID;
    }
    *launches += 1;
    SVD1_CUDA_TRY(cudaGetLastError());
    return SVD1_OK;
  }
  if (colnorm_J() == 2) {  // two columns per thread (chunks as for one: they depend on n only)
    const int ch = inner_chunks(n, kCT, 2);
    const int chunk = (n + ch - 1) / ch;
    const dim3 g(unsigned((j1 - j0 + 2 * kCT - 1) / (2 * kCT)), unsigned(ch));
    switch (ncarry) {
#define SVD1_CM(NC) case NC: colnorm_multi_kernel<NC, 2><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, \
                                                                 ctr, colscale, carry_out, status, j0, j1, ldc); break;
      SVD1_CM(0) SVD1_CM(1) SVD1_CM(2) SVD1_CM(3) SVD1_CM(4) SVD1_CM(5) SVD1_CM(6)
#undef SVD1_CM
      default: return SVD1_E_INVALID;
    }
    *launches += 1;
    SVD1_CUDA_TRY(cudaGetLastError());
    return SVD1_OK;
  }
  const int ch = inner_chunks(n, kCT);
  const int chunk = (n + ch - 1) / ch;
  const dim3 g(unsigned((j1 - j0 + kCT - 1) / kCT), unsigned(ch));
  switch (ncarry) {
    case 0: colnorm_partial_kernel<0><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, ctr, colscale, carry_out, status, j0, j1, ldc); break;
    case 1: colnorm_partial_kernel<1><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, ctr, colscale, carry_out, status, j0, j1, ldc); break;
    case 2: colnorm_partial_kernel<2><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, ctr, colscale, carry_out, status, j0, j1, ldc); break;
    case 3: colnorm_partial_kernel<3><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, ctr, colscale, carry_out, status, j0, j1, ldc); break;
    case 4: colnorm_partial_kernel<4><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, ctr, colscale, carry_out, status, j0, j1, ldc); break;
    case 5: colnorm_partial_kernel<5><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, ctr, colscale, carry_out, status, j0, j1, ldc); break;
    case 6: colnorm_partial_kernel<6><<<g, kCT, 0, st>>>(d, k, tau, zhat, n, chunk, carry, scratch, ctr, colscale, carry_out, status, j0, j1, ldc); break;
    default: return SVD1_E_INVALID;
  }
  *launches += 1;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

}  // namespace svd1
