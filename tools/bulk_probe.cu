// Probe: mbarrier expect_tx and the 1-D bulk copy (no tensor map), one mode per process.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const double* src, double* out, int mode) {
  __shared__ __align__(128) double buf[256];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
    } else if (mode == 1) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(2048) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_u32(buf)), "l"(src), "r"(2048), "r"(smem_u32(&bar)) : "memory");
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;\n" ::"r"(smem_u32(&bar)), "r"(2048) : "memory");
      asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                   ::"r"(smem_u32(buf)), "l"(src), "r"(2048), "r"(smem_u32(&bar)) : "memory");
    }
  }
  asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < 256; i += blockDim.x) out[i] = buf[i];
}
int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  double *s, *o; cudaMalloc(&s, 2048); cudaMalloc(&o, 2048);
  double h[256]; for (int i = 0; i < 256; ++i) h[i] = i;
  cudaMemcpy(s, h, 2048, cudaMemcpyHostToDevice);
  k<<<1, 64>>>(s, o, mode);
  cudaError_t e = cudaDeviceSynchronize();
  double ho[256]; int bad = 0;
  if (e == cudaSuccess) { cudaMemcpy(ho, o, 2048, cudaMemcpyDeviceToHost); for (int i = 0; i < 256; ++i) bad += ho[i] != h[i]; }
  printf("mode %d: %s bad=%d\n", mode, cudaGetErrorString(e), bad);
  return 0;
}
