// TMA streaming bandwidth into shared memory on this GPU: the feed ceiling of the FMM GEMM's
// 16-wide passes.  The same structure as fmm_gemm_kernel's producer /
// consumer ring -- one producer warp issuing 128-row x 16-double boxes (SWIZZLE_128B, 16 KB)
// into an S-stage ring, CW consumer warps that read every stage with 128-bit shared loads and
// release it -- but no DMMA, so the rate is what TMA + L2 (or HBM) deliver.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_bw tools/tma_bw.cu  (on the GPU box)
//   /tmp/tma_bw            (prints one line per working-set size and CTAs/SM)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int CW = 4, S = 4, BM = 128, A_BYTES = BM * 16 * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n"
               ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

__global__ void __launch_bounds__(32 * (CW + 1)) tma_stream(const __grid_constant__ CUtensorMap tm, int ncb, long ntiles, long tiles_once,
                                                           double* sink) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* base = raw + ((1024 - (smem_u32(raw) & 1023)) & 1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(base + S * A_BYTES);
  uint64_t* empty = full + S;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int q = 0; q < S; ++q) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&full[q])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&empty[q])), "r"(CW));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  int stage = 0;
  uint32_t phase = 0;
  if (warp == CW) {
    if (lane == 0) {
      for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        mbar_wait(&empty[stage], phase ^ 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&full[stage])),
                     "r"(A_BYTES) : "memory");
        const long u = t % tiles_once;  // passes over the working set
        const int c0 = int(u % ncb) * 16, r0 = int(u / ncb) * BM;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n"
            ::"r"(smem_u32(base + stage * A_BYTES)), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(c0), "r"(r0),
            "r"(smem_u32(&full[stage])) : "memory");
        if (++stage == S) stage = 0, phase ^= 1;
      }
    }
    return;
  }
  double acc = 0.0;
  for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
    mbar_wait(&full[stage], phase);
    const unsigned char* a = base + stage * A_BYTES + (warp * 32 + (lane >> 2)) * 128;
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {  // the consumer's fragment reads of one stage (8 x 16 B per lane)
      const int g = lane >> 2, t4 = lane & 3;  // 128B-swizzled 16-byte chunks, as the GEMM reads them
      const double2 v0 = *reinterpret_cast<const double2*>(a + mt * 1024 + (((2 * t4) ^ g) << 4));
      const double2 v1 = *reinterpret_cast<const double2*>(a + mt * 1024 + (((2 * t4 + 1) ^ g) << 4));
      acc += v0.x + v0.y + v1.x + v1.y;
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&empty[stage])) : "memory");
    if (++stage == S) stage = 0, phase ^= 1;
  }
  if (acc == 12345.678) sink[0] = acc;  // keep the reads
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int smem = 1024 + S * A_BYTES + 2 * S * 8;
  CK(cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  double* sink;
  CK(cudaMalloc(&sink, 8));
  // working sets: L2-resident (8, 32, 64 MB) and HBM (2 GB); rows of 4096 doubles (C3's U)
  const long cols = 4096;
  for (long mb : {8L, 32L, 64L, 2048L}) {
    const long rows = mb * (1L << 20) / (cols * 8);
    double* buf;
    CK(cudaMalloc(&buf, rows * cols * 8));
    CK(cudaMemset(buf, 0, rows * cols * 8));
    CUtensorMap tm;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols * 8)};
    const cuuint32_t box[2] = {16, BM}, estr[2] = {1, 1};
    if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, buf, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
        CUDA_SUCCESS) {
      printf("encode failed\n");
      return 1;
    }
    const int ncb = int(cols / 16);
    const long tiles_once = long(ncb) * (rows / BM);
    const long reps = mb >= 1024 ? 1 : (2048 / mb);  // ~2 GB of traffic per measurement
    const long ntiles = tiles_once * reps;  // reps passes over the set in one launch
    for (int per_sm : {1, 2, 3, 4}) {
      const int grid = sms * per_sm;
      cudaEvent_t e0, e1;
      CK(cudaEventCreate(&e0));
      CK(cudaEventCreate(&e1));
      tma_stream<<<grid, 32 * (CW + 1), smem>>>(tm, ncb, tiles_once, tiles_once, sink);  // warm
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      tma_stream<<<grid, 32 * (CW + 1), smem>>>(tm, ncb, ntiles, tiles_once, sink);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      const double bytes = double(ntiles) * A_BYTES;
      printf("working set %5ld MB  CTAs/SM %d  grid %4d  %7.3f ms  %7.2f TB/s  (%ld passes)\n", mb, per_sm, grid,
             ms, bytes / (ms * 1e-3) / 1e12, reps);
      CK(cudaEventDestroy(e0));
      CK(cudaEventDestroy(e1));
    }
    CK(cudaFree(buf));
  }
  return 0;
}
