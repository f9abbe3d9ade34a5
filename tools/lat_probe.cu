// Latency probe: dependent DFMA chain, double division, __syncthreads (8 warps),
// REDUX + ballot argmax step, smem round trip.  One CTA, clock64 deltas.
#include <cstdio>
__global__ void probe(double* out, long long* t, double seed) {
  __shared__ double sm[256];
  const int tid = threadIdx.x;
  double x = seed + tid, y = 1.0000001;
  long long c0, c1;
  __syncthreads();
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, y, 1e-9);
  c1 = clock64();
  if (tid == 0) t[0] = (c1 - c0);  // 1000 dependent DFMA
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 100; ++i) x = 1.0 / (x + 1.0);
  c1 = clock64();
  if (tid == 0) t[1] = (c1 - c0);  // 100 dependent divisions (+add)
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) __syncthreads();
  c1 = clock64();
  if (tid == 0) t[2] = (c1 - c0);  // 1000 barriers
  c0 = clock64();
  unsigned k = tid;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) k = __reduce_max_sync(0xffffffffu, k + i) & 0xffff;
  c1 = clock64();
  if (tid == 0) t[3] = (c1 - c0);  // 1000 dependent REDUX
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffffu, x, (tid + 1) & 31);
  c1 = clock64();
  if (tid == 0) t[4] = (c1 - c0);  // 1000 dependent SHFL
  c0 = clock64();
  sm[tid] = x;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    const double v = sm[(tid + i) & 255];
    sm[tid] = v + 1.0;
  }
  c1 = clock64();
  if (tid == 0) t[5] = (c1 - c0);  // 1000 dependent LDS->DADD->STS
  c0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) {
    if (tid == (i & 255)) sm[0] = x + i;
    __syncthreads();
    x += sm[0];
  }
  c1 = clock64();
  if (tid == 0) t[6] = (c1 - c0);  // 1000 x (STS by one thread, barrier, LDS, DADD)
  out[tid] = x + k;
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 8 * 256); cudaMallocManaged(&t, 8 * 8);
  for (int nt : {32, 256}) {
    probe<<<1, nt>>>(o, t, 1.0); cudaDeviceSynchronize();
    probe<<<1, nt>>>(o, t, 1.0); cudaDeviceSynchronize();
    printf("threads %d: DFMA dep %.1f  div dep %.1f  bar %.1f  redux %.1f  shfl %.1f  lds-sts %.1f  sts-bar-lds %.1f (cycles each)\n",
           nt, t[0] / 1000.0, t[1] / 100.0, t[2] / 1000.0, t[3] / 1000.0, t[4] / 1000.0, t[5] / 1000.0, t[6] / 1000.0);
  }
  return 0;
}
