// FP64 peak microbenchmark for B200 (sm_100a): DMMA (mma.sync f64) and DFMA.
// Used once to fill the FP64 roofline denominator (MEASURED_PEAKS.json has only
// HBM and bf16). Sustained loop ~2 s per mode, CUDA-event timed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

template <int NACC>
__global__ void dmma_m8n8k4(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dmma_m16n8k8(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-9, a1 = a0 * 0.5, a2 = a0 * 0.25, a3 = a0 * 0.125;
  double b0 = 1.0 - threadIdx.x * 1e-9, b1 = b0 * 0.5;
  double c[NACC][4];
#pragma unroll
  for (int i = 0; i < NACC; ++i) { c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
__global__ void dfma_loop(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i) c[i] = fma(a, c[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

// reciprocal throughput of a full IEEE fp64 divide vs rcp.approx + 2 Newton
__global__ void ddiv_loop(double* out, int iters, int mode) {
  double x = 1.0 + threadIdx.x * 1e-7;
  double acc[4] = {0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      double den = x + (double)(i + it);
      double r;
      if (mode == 0) {
        r = 1.0 / den;
      } else {
        double y;
        asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(den));
        double e = fma(-den, y, 1.0);
        y = fma(y, e, y);
        e = fma(-den, y, 1.0);
        r = fma(y, e, y);
      }
      acc[i] += r;
    }
  }
  double s = acc[0] + acc[1] + acc[2] + acc[3];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
double time_kernel(F launch, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  launch();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) launch();
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  CK(cudaGetLastError());
  return ms / reps;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev));
  double* out; CK(cudaMalloc(&out, 8));
  const int iters = 20000;
  for (int bpsm : {1, 2, 4}) {
    int blocks = sms * bpsm, threads = 256;
    double ms = time_kernel([&] { dmma_m8n8k4<8><<<blocks, threads>>>(out, iters); }, 20);
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * (threads / 32);
    printf("{\"mode\": \"dmma_m8n8k4\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", bpsm, ms, flops / ms / 1e9);
    ms = time_kernel([&] { dmma_m16n8k8<4><<<blocks, threads>>>(out, iters / 2); }, 20);
    flops = 2.0 * 1024 * 4 * (double)(iters / 2) * blocks * (threads / 32);
    printf("{\"mode\": \"dmma_m16n8k8\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", bpsm, ms, flops / ms / 1e9);
    ms = time_kernel([&] { dfma_loop<8><<<blocks, threads>>>(out, iters * 4); }, 20);
    flops = 2.0 * 8 * (double)iters * 4 * blocks * threads;
    printf("{\"mode\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.2f}\n", bpsm, ms, flops / ms / 1e9);
  }
  for (int mode : {0, 1}) {
    int blocks = sms * 4, threads = 256;
    double ms = time_kernel([&] { ddiv_loop<<<blocks, threads>>>(out, iters, mode); }, 10);
    double divs = 4.0 * iters * blocks * threads;
    printf("{\"mode\": \"%s\", \"gdiv_per_s\": %.1f}\n", mode ? "rcp_newton" : "ieee_div", divs / ms / 1e6);
  }
  // sustained ~2 s DMMA loop for the sustained peak
  {
    int blocks = sms * 2, threads = 256;
    double ms = time_kernel([&] { dmma_m8n8k4<8><<<blocks, threads>>>(out, iters * 5); }, 20);
    double flops = 2.0 * 256 * 8 * (double)iters * 5 * blocks * (threads / 32);
    printf("{\"mode\": \"dmma_m8n8k4_sustained\", \"ms\": %.3f, \"tflops\": %.2f}\n", ms, flops / ms / 1e9);
  }
  printf("{\"sms\": %d, \"clock_khz_attr\": %d}\n", sms, clk);
  return 0;
}
