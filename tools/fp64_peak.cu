// FP64 peak micro-benchmark for B200 (sm_100a): DMMA (mma.sync m8n8k4 f64)
// and DFMA issue rates.  The measured number is the roofline denominator for
// the HSC contraction kernels (MEASURED_PEAKS.json carries no FP64 figure).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0.0; c[i][1] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  CK(cudaMalloc(&out, 8));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps = 4; warps <= 32; warps *= 2) {
    for (int blocks_per_sm = 1; blocks_per_sm <= 2; ++blocks_per_sm) {
      dim3 grid(sms * blocks_per_sm), block(32 * warps);
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(e0);
        dmma_kernel<8><<<grid, block>>>(out, iters);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * warps;
      printf("DMMA m8n8k4 warps/blk=%d blk/sm=%d: %.2f TFLOP/s (%.3f ms)\n", warps,
             blocks_per_sm, flops / best / 1e9, best);
    }
  }
  for (int warps = 4; warps <= 32; warps *= 2) {
    dim3 grid(sms * 2), block(32 * warps);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<8><<<grid, block>>>(out, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    double flops = 2.0 * 8.0 * iters * (double)grid.x * block.x;
    printf("DFMA warps/blk=%d blk/sm=2: %.2f TFLOP/s (%.3f ms)\n", warps, flops / best / 1e9, best);
  }
  CK(cudaGetLastError());
  return 0;
}
