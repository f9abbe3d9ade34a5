// Micro-benchmark of the grouped complex GEMM kernel on uniform tasks:
//   gemm_bench M N K tasks energies [opa opb kterm arr]   (arr 3: the plan's mixed tiling)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/gemm_bench.cu \
//        paper_1305_1070_b200/csrc/plan.cpp paper_1305_1070_b200/csrc/tree.cpp -o tools/gemm_bench
// Every task: C (M x N) = A (M x K) * B (K x N), one term, per energy arena.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <cmath>

#include "../paper_1305_1070_b200/csrc/kernels.cu"
#include "../paper_1305_1070_b200/csrc/plan.hpp"

using namespace negfb;

int main(int argc, char** argv) {
  const int M = atoi(argv[1]), N = atoi(argv[2]), K = atoi(argv[3]), T = atoi(argv[4]), nE = atoi(argv[5]);
  const int opa = argc > 6 ? atoi(argv[6]) : OP_N, opb = argc > 7 ? atoi(argv[7]) : OP_N;
  const int kterm = argc > 8 ? atoi(argv[8]) : K;  // split K into terms of this size
  const int ARR = argc > 9 ? atoi(argv[9]) : 0;
  const int64_t per_task = int64_t(M) * K + int64_t(K) * N + int64_t(M) * N;
  const int64_t stride = per_task * T;
  std::vector<GemmTask> tasks;
  std::vector<GemmTerm> terms;
  std::vector<GemmTile> tiles[1];
  for (int t = 0; t < T; ++t) {
    const int64_t base = per_task * t;
    const int tb = static_cast<int>(terms.size());
    for (int k0 = 0; k0 < K; k0 += kterm) {
      GemmTerm g{};
      g.k = std::min(kterm, K - k0);
      g.a_op = opa;
      g.b_op = opb;
      g.sign = 1;
      g.lda = opa == OP_N ? K : M;
      g.ldb = (opb == OP_N || opb == OP_C) ? N : K;
      g.a_off = base + (opa == OP_N ? k0 : int64_t(k0) * M);
      g.b_off = base + int64_t(M) * K + ((opb == OP_N || opb == OP_C) ? int64_t(k0) * N : k0);
      terms.push_back(g);
    }
    GemmTask tk{};
    tk.c2_off = -1;
    tk.m = M;
    tk.n = N;
    tk.ldc = N;
    tk.mode = MODE_SET;
    tk.c_off = base + int64_t(M) * K + int64_t(K) * N;
    tk.term_begin = tb;
    tk.term_count = static_cast<int>(terms.size()) - tb;
    tasks.push_back(tk);
    if (ARR == 3) {
      tile_task(t, M, N, 1 << 30, tiles[0]);  // the plan's mixed tiling (never warp tiles)
    } else {
      for (int m0 = 0; m0 < M; m0 += kArrTM[ARR])
        for (int n0 = 0; n0 < N; n0 += kArrTN[ARR]) tiles[0].push_back(GemmTile{t, m0, n0, ARR});
    }
  }
  double2* arena;
  cudaMalloc(&arena, sizeof(double2) * stride * nE);
  {
    std::vector<double2> h(stride);
    for (auto& v : h) v = make_double2(drand48() - 0.5, drand48() - 0.5);
    for (int e = 0; e < nE; ++e) cudaMemcpy(arena + e * stride, h.data(), sizeof(double2) * stride, cudaMemcpyHostToDevice);
  }
  GemmTask* dt;
  GemmTerm* dm;
  GemmTile* dl[1];
  cudaMalloc(&dt, sizeof(GemmTask) * tasks.size());
  cudaMalloc(&dm, sizeof(GemmTerm) * terms.size());
  cudaMemcpy(dt, tasks.data(), sizeof(GemmTask) * tasks.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dm, terms.data(), sizeof(GemmTerm) * terms.size(), cudaMemcpyHostToDevice);
  for (int sh = 0; sh < 1; ++sh) {
    cudaMalloc(&dl[sh], sizeof(GemmTile) * tiles[sh].size());
    cudaMemcpy(dl[sh], tiles[sh].data(), sizeof(GemmTile) * tiles[sh].size(), cudaMemcpyHostToDevice);
  }
  BatchArgs b{arena, stride, nE, 0};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double flops = 8.0 * M * N * K * double(T) * nE;
  for (int sh = 0; sh < 1; ++sh) {
    int64_t L = 0;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      launch_gemm(b, dt, dm, dl[0], tiles[0].data(), 0, static_cast<int>(tiles[0].size()), 0, L);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 0 && ms < best) best = ms;
    }
    printf("M=%d N=%d K=%d T=%d nE=%d ops=%d/%d arr=%d: %.3f ms  %.2f TF/s  (%s)\n", M, N, K, T, nE, opa, opb,
           ARR, best, flops / best / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  // Correctness: task 0..3 of the last energy against a host product.
  {
    std::vector<double2> h(stride);
    cudaMemcpy(h.data(), arena + int64_t(nE - 1) * stride, sizeof(double2) * stride, cudaMemcpyDeviceToHost);
    double err = 0, mx = 0;
    for (int t = 0; t < std::min(T, 4); ++t) {
      const int64_t base = per_task * t;
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          double cr = 0, ci = 0;
          for (int k = 0; k < K; ++k) {
            const double2 a = opa == OP_N ? h[base + int64_t(i) * K + k] : h[base + int64_t(k) * M + i];
            double2 b = (opb == OP_N || opb == OP_C) ? h[base + int64_t(M) * K + int64_t(k) * N + j]
                                                     : h[base + int64_t(M) * K + int64_t(j) * K + k];
            if (opb == OP_C || opb == OP_H) b.y = -b.y;
            cr += a.x * b.x - a.y * b.y;
            ci += a.x * b.y + a.y * b.x;
          }
          const double2 c = h[base + int64_t(M) * K + int64_t(K) * N + int64_t(i) * N + j];
          err = std::max(err, std::max(std::abs(c.x - cr), std::abs(c.y - ci)));
          mx = std::max(mx, std::max(std::abs(cr), std::abs(ci)));
        }
    }
    printf("  check: max abs err %.3e (max |C| %.3e) %s\n", err, mx, err <= 1e-12 * std::max(1.0, mx) ? "OK" : "FAIL");
  }
  return 0;
}
