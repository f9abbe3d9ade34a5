// Micro-benchmark of the batched inverse kernels:
//   inv_bench m blocks energies [dominant=1]
// dominant=0: random complex entries (row interchanges at most steps).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1305_1070_b200/csrc/kernels.cu"

using namespace negfb;

int main(int argc, char** argv) {
  const int m = atoi(argv[1]), nb = atoi(argv[2]), nE = atoi(argv[3]);
  const double dom = argc > 4 ? atof(argv[4]) : 1.0;
  const int64_t stride = int64_t(m) * m * nb;
  std::vector<double2> h(stride);
  for (int b = 0; b < nb; ++b)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < m; ++j)
        h[int64_t(b) * m * m + i * m + j] = make_double2(drand48() - 0.5 + (i == j ? 2.0 * m * dom : 0.0), getenv("INV_REAL") ? 0.0 * drand48() : drand48() - 0.5);
  double2* arena;
  cudaMalloc(&arena, sizeof(double2) * stride * nE);
  for (int e = 0; e < nE; ++e) cudaMemcpy(arena + e * stride, h.data(), sizeof(double2) * stride, cudaMemcpyHostToDevice);
  if (m > kSmemInvMax) {
    printf("m > %d uses the multi-CTA path (see plan.cpp); not benchmarked here\n", kSmemInvMax);
    return 0;
  }
  std::vector<InvTask> t(nb);
  for (int b = 0; b < nb; ++b) t[b] = InvTask{m, b, b, getenv("INV_REAL") && !getenv("INV_REAL_COMPLEX_KERNEL") ? 1 : 0, int64_t(b) * m * m};
  InvTask* dt;
  cudaMalloc(&dt, sizeof(InvTask) * nb);
  cudaMemcpy(dt, t.data(), sizeof(InvTask) * nb, cudaMemcpyHostToDevice);
  DevStatus* st;
  cudaMalloc(&st, sizeof(DevStatus));
  cudaMemset(st, 0xff, sizeof(DevStatus));
  BatchArgs b{arena, stride, nE, 0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int64_t L = 0;
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    for (int e = 0; e < nE; ++e) cudaMemcpy(arena + e * stride, h.data(), sizeof(double2) * stride, cudaMemcpyHostToDevice);
    cudaEventRecord(e0);
    const char* shape = getenv("RG_SHAPE");  // force one register-inverse shape
    dim3 grid(nb, nE);
    if (!shape) launch_inverse(b, dt, t.data(), nb, st, 0, L);
    else if (!strcmp(shape, "32x1")) k_inverse_rg<32, 1, 32><<<grid, 32>>>(arena, stride, dt, 0, st);
    else if (!strcmp(shape, "32x2")) k_inverse_rg<32, 2, 16><<<grid, 64>>>(arena, stride, dt, 0, st);
    else if (!strcmp(shape, "64x2")) k_inverse_rg<64, 2, 32><<<grid, 128>>>(arena, stride, dt, 0, st);
    else if (!strcmp(shape, "64x4")) k_inverse_rg<64, 4, 16><<<grid, 256>>>(arena, stride, dt, 0, st);
    else if (!strcmp(shape, "48x2")) k_inverse_rg<48, 2, 24><<<grid, 96>>>(arena, stride, dt, 0, st);
    // shifting-window kernel: sw:ROWSxHxS
#define SWV(R, HH, SS, MB) else if (!strcmp(shape, "sw:" #R "x" #HH "x" #SS "x" #MB)) \
      { if (getenv("SW_REAL")) k_inverse_sw<R, HH, SS, MB, true><<<grid, R * HH>>>(arena, stride, dt, 0, st); \
        else k_inverse_sw<R, HH, SS, MB, false><<<grid, R * HH>>>(arena, stride, dt, 0, st); }
    SWV(32, 1, 8, 16) SWV(32, 1, 12, 16) SWV(32, 1, 16, 16) SWV(32, 1, 16, 12) SWV(32, 1, 28, 8) SWV(32, 1, 32, 8) SWV(32, 1, 32, 10) SWV(32, 2, 14, 8) SWV(32, 2, 16, 8) SWV(32, 2, 16, 10)
    SWV(32, 4, 8, 8) SWV(32, 4, 8, 12)
    SWV(48, 2, 20, 4) SWV(48, 2, 24, 4) SWV(48, 2, 24, 5) SWV(48, 4, 12, 4) SWV(48, 4, 12, 5) SWV(64, 1, 48, 2) SWV(64, 1, 48, 3) SWV(64, 1, 64, 3) SWV(64, 1, 64, 4) SWV(64, 1, 64, 5) SWV(64, 1, 64, 6) SWV(64, 1, 64, 7) SWV(64, 1, 56, 5) SWV(64, 1, 52, 5) SWV(64, 1, 52, 6) SWV(64, 1, 60, 5) SWV(64, 1, 60, 6) SWV(64, 1, 48, 6) SWV(64, 1, 40, 6) SWV(64, 1, 40, 8)
    SWV(64, 2, 28, 2) SWV(64, 2, 32, 2) SWV(64, 2, 32, 3) SWV(64, 4, 16, 2) SWV(64, 4, 16, 3) SWV(64, 4, 16, 4)
    SWV(96, 4, 24, 1) SWV(112, 4, 28, 1) SWV(104, 4, 25, 1) SWV(128, 4, 28, 1) SWV(80, 4, 20, 1) SWV(80, 4, 19, 1) SWV(80, 4, 20, 2) SWV(104, 4, 26, 1) SWV(104, 8, 13, 1) SWV(80, 2, 38, 1) SWV(112, 8, 14, 1) SWV(128, 8, 15, 1)
    else { printf("unknown RG_SHAPE %s\n", shape); return 1; }
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0 && ms < best) best = ms;
  }
  std::vector<double2> out(m * m);
  cudaMemcpy(out.data(), arena, sizeof(double2) * m * m, cudaMemcpyDeviceToHost);
  // every energy holds the same blocks: the last block of energies 1 and nE - 1 must equal energy 0's bit for bit
  {
    std::vector<double2> o0(m * m), o1(m * m);
    const int64_t lastb = int64_t(nb - 1) * m * m;
    cudaMemcpy(o0.data(), arena + lastb, sizeof(double2) * m * m, cudaMemcpyDeviceToHost);
    for (int e : {1, nE - 1}) {
      if (e <= 0 || e >= nE) continue;
      cudaMemcpy(o1.data(), arena + int64_t(e) * stride + lastb, sizeof(double2) * m * m, cudaMemcpyDeviceToHost);
      if (memcmp(o0.data(), o1.data(), sizeof(double2) * m * m)) printf("  MISMATCH between energies 0 and %d\n", e);
    }
  }
  // residual of block 0: max |A * X - I|
  double res = 0;
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      double re = (i == j) ? -1.0 : 0.0, im = 0.0;
      for (int k = 0; k < m; ++k) {
        const double2 a = h[i * m + k], x = out[k * m + j];
        re += a.x * x.x - a.y * x.y;
        im += a.x * x.y + a.y * x.x;
      }
      res = std::max(res, std::hypot(re, im));
    }
  const double fl = 8.0 * m * double(m) * m * nb * nE;
  DevStatus hs;
  cudaMemcpy(&hs, st, sizeof hs, cudaMemcpyDeviceToHost);
  printf("m=%d blocks=%dx%d dom=%g: %.3f ms  %.2f TF/s  residual %.2e singular_key %llx (%s)\n", m, nb, nE, dom, best,
         fl / best / 1e9, res, hs.singular_key, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
