// Per-pivot cost of the warp-level Gauss-Jordan panel step (panel_regs in
// kernels.cu): one warp, a 64 x 8 complex panel in registers (2 rows per lane),
// 8 pivot steps; variants isolate the argmax, the reciprocal and the shuffles.
#include <cstdio>
__device__ __forceinline__ double cnorm(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <int V>
__global__ void probe(double2* data, long long* out) {
  const int lane = threadIdx.x & 31;
  constexpr int RPL = 2, NB = 8;
  double2 v[RPL][NB];
  int pos[RPL];
  for (int i = 0; i < RPL; ++i) {
    pos[i] = lane + 32 * i;
    for (int c = 0; c < NB; ++c) v[i][c] = data[(lane + 32 * i) * NB + c];
  }
  long long t0 = clock64();
  for (int rep = 0; rep < 16; ++rep) {
#pragma unroll
    for (int kk = 0; kk < NB; ++kk) {
      const int k = kk;
      double best = -1.0;
      int bpos = 0x7fffffff, bslot = 0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        if (pos[i] >= k) {
          const double x = cnorm(v[i][kk]);
          if (x > best || (x == best && pos[i] < bpos)) { best = x; bpos = pos[i]; bslot = i; }
        }
      }
      int wl;
      if (V == 1) {  // shuffle argmax (double)
        double cb = best; int cp = bpos, cl = lane;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, cb, o);
          const int op = __shfl_xor_sync(0xffffffffu, cp, o);
          const int ol = __shfl_xor_sync(0xffffffffu, cl, o);
          if (ob > cb || (ob == cb && op < cp)) { cb = ob; cp = op; cl = ol; }
        }
        wl = cl;
      } else {  // float-key REDUX + ballot (kernels.cu)
        const unsigned key = best >= 0.0 ? __float_as_uint(__double2float_ru(best)) : 0u;
        const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
        const unsigned tied = __ballot_sync(0xffffffffu, best >= 0.0 && key == kmax);
        wl = tied ? __ffs(tied) - 1 : 0;
      }
      const int p = __shfl_sync(0xffffffffu, bpos, wl);
      const int ws = __shfl_sync(0xffffffffu, bslot, wl);
      double2 pr[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        double2 x = v[0][c];
        if (ws == 1) x = v[1][c];
        pr[c].x = __shfl_sync(0xffffffffu, x.x, wl);
        pr[c].y = __shfl_sync(0xffffffffu, x.y, wl);
      }
      const double2 piv = pr[kk];
      double2 ip;
      if (V == 2) {  // no division
        ip = make_double2(piv.x, -piv.y);
      } else {
        const double rd = 1.0 / fma(piv.x, piv.x, piv.y * piv.y);
        ip = make_double2(piv.x * rd, -piv.y * rd);
      }
#pragma unroll
      for (int c = 0; c < NB; ++c) pr[c] = (c == kk) ? ip : cmul(pr[c], ip);
      const double2 nip = make_double2(-ip.x, -ip.y);
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        if (lane == wl && i == ws) {
#pragma unroll
          for (int c = 0; c < NB; ++c) v[i][c] = pr[c];
        } else {
          const double2 f = v[i][kk];
#pragma unroll
          for (int c = 0; c < NB; ++c) v[i][c] = (c == kk) ? cmul(f, nip) : make_double2(v[i][c].x - (f.x * pr[c].x - f.y * pr[c].y), v[i][c].y - (f.x * pr[c].y + f.y * pr[c].x));
        }
        if (pos[i] == k) pos[i] = p;
        else if (pos[i] == p) pos[i] = k;
      }
    }
    for (int i = 0; i < RPL; ++i) pos[i] = lane + 32 * i;
  }
  long long t1 = clock64();
  if (lane == 0) out[blockIdx.x] = (t1 - t0) / (16 * NB);
  for (int i = 0; i < RPL; ++i)
    for (int c = 0; c < NB; ++c) data[(lane + 32 * i) * NB + c] = v[i][c];
}
int main() {
  double2* d; long long* o;
  cudaMalloc(&d, 64 * 8 * 16 * 1000);
  cudaMallocManaged(&o, 8 * 1000);
  double2 h[512];
  for (int i = 0; i < 512; ++i) h[i] = make_double2(1.0 + (i * 7919 % 113) / 113.0, (i * 104729 % 97) / 97.0);
  for (int b = 0; b < 1000; ++b) cudaMemcpy(d + b * 512, h, sizeof h, cudaMemcpyHostToDevice);
  const char* names[3] = {"redux argmax + div", "shuffle argmax + div", "redux argmax, no div"};
  for (int V = 0; V < 3; ++V)
    for (int nb : {1, 148, 148 * 8}) {
      for (int it = 0; it < 2; ++it) {
        if (V == 0) probe<0><<<nb, 32>>>(d, o);
        if (V == 1) probe<1><<<nb, 32>>>(d, o);
        if (V == 2) probe<2><<<nb, 32>>>(d, o);
        cudaDeviceSynchronize();
      }
      printf("%-24s warps %5d: %lld cycles per pivot step\n", names[V], nb, o[0]);
    }
  return 0;
}
