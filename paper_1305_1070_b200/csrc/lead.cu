// Contact self-energies on the GPU, C ABI in
// include/negf_gpu.h:
//   * negf_lead_*: the reference's energy-doubling decimation
//     (surface_self_energy, proj/src/device.cpp:195-251) batched over
//     energies.  One arena per energy holds the lead's w x w blocks
//     (plan.hpp LeadBlock); each sweep is the same grouped program -- batched
//     inverses of z-es and z-e, grouped DMMA GEMMs, the fixed-point test --
//     replayed for every energy of the batch at once.  Energies that pass
//     the test freeze their `refined` block (the reference returns there);
//     the batch sweeps until every energy converged or failed.
//   * negf_lead_modes_sigma_device: analytic transverse-mode Sigma of a
//     uniform 2-D lead.
//   * negf_contacts_fill_device: lesser_self_energy (device.cpp:322-366) and
//     the pattern placement of the contact and phonon values.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "kernels.hpp"
#include "plan.hpp"

using namespace negfb;

namespace {

struct LeadOffs {
  int64_t o[LB_COUNT];
};

__device__ __forceinline__ double2 zsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// Per-energy constants and the decimation's initial state (device.cpp:208-214).
__global__ void k_lead_init(double2* arena, int64_t stride, int w, LeadOffs off, const double2* __restrict__ h00,
                            const double2* __restrict__ h01, const double* __restrict__ energies, double eta,
                            int criterion) {
  double2* a = arena + blockIdx.x * stride;
  const double2 z = make_double2(energies[blockIdx.x], eta);
  const int w2 = w * w;
  for (int idx = threadIdx.x; idx < w2; idx += blockDim.x) {
    const int i = idx / w, j = idx - (idx / w) * w;
    const double2 v00 = h00[idx], v01 = h01[idx];
    const double2 t = h01[j * w + i];
    // criterion 0 (device.cpp:208-214): alpha = h01^H, beta = h01, sigma = h01^H g h01
    // criterion 1 (decay): alpha = h01, beta = h01^T, sigma = h01^T g_s h01
    const double2 ct = criterion == 0 ? make_double2(t.x, -t.y) : t;
    a[off.o[LB_H00] + idx] = v00;
    a[off.o[LB_H01] + idx] = v01;
    a[off.o[LB_H01CT] + idx] = ct;
    a[off.o[LB_ZH] + idx] = zsub(i == j ? z : make_double2(0.0, 0.0), v00);  // z_minus (device.cpp:45-51)
    a[off.o[LB_ES] + idx] = v00;
    a[off.o[LB_E] + idx] = v00;
    a[off.o[LB_ALPHA0] + idx] = criterion == 0 ? ct : v01;
    a[off.o[LB_BETA0] + idx] = criterion == 0 ? v01 : t;
  }
}

// g <- z - es, m <- z - e (inverted in place by the next op).
__global__ void k_lead_prep(double2* arena, int64_t stride, int w, LeadOffs off, const double* __restrict__ energies,
                            double eta) {
  double2* a = arena + blockIdx.y * stride;
  const double2 z = make_double2(energies[blockIdx.y], eta);
  const int w2 = w * w;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < w2; idx += gridDim.x * blockDim.x) {
    const int i = idx / w, j = idx - (idx / w) * w;
    const double2 zd = i == j ? z : make_double2(0.0, 0.0);
    a[off.o[LB_G] + idx] = zsub(zd, a[off.o[LB_ES] + idx]);
    a[off.o[LB_M] + idx] = zsub(zd, a[off.o[LB_E] + idx]);
  }
}

// Fixed-point test ||refined - g||_F <= 1e-10 (device.cpp:223-225); the first
// passing sweep freezes `refined` into FIN.  Counts energies still open and
// the lowest open energy index.
__global__ void k_lead_check(double2* arena, int64_t stride, int w, LeadOffs off, int sweep, int* conv,
                             int* pending, int* lowest_open, int e_base) {
  double2* a = arena + blockIdx.x * stride;
  __shared__ double red[32];
  __shared__ int now;
  const int w2 = w * w;
  if (conv[blockIdx.x] >= 0) return;  // block-uniform
  double s = 0.0;
  for (int idx = threadIdx.x; idx < w2; idx += blockDim.x) {
    const double2 d = zsub(a[off.o[LB_RHS] + idx], a[off.o[LB_G] + idx]);
    s += d.x * d.x + d.y * d.y;
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) t += red[k];
    now = std::sqrt(t) <= 1e-10;
    if (now) conv[blockIdx.x] = sweep;
    else {
      atomicAdd(pending, 1);
      atomicMin(lowest_open, e_base + static_cast<int>(blockIdx.x));
    }
  }
  __syncthreads();
  if (!now) return;
  for (int idx = threadIdx.x; idx < w2; idx += blockDim.x) a[off.o[LB_FIN] + idx] = a[off.o[LB_RHS] + idx];
}

// Decay test max|alpha|, max|beta| < tol after the update (the criterion of
// devices.sancho_rubio); the first passing sweep freezes es into FIN.
__global__ void k_lead_check_decay(double2* arena, int64_t stride, int w, int64_t off_al, int64_t off_be,
                                   int64_t off_es, int64_t off_fin, double tol, int sweep, int* conv, int* pending,
                                   int* lowest_open, int e_base) {
  double2* a = arena + blockIdx.x * stride;
  __shared__ double red[32];
  __shared__ int now;
  const int w2 = w * w;
  if (conv[blockIdx.x] >= 0) return;  // block-uniform
  double mx = 0.0;
  for (int idx = threadIdx.x; idx < w2; idx += blockDim.x) {
    const double2 u = a[off_al + idx], v = a[off_be + idx];
    mx = fmax(mx, fmax(hypot(u.x, u.y), hypot(v.x, v.y)));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < static_cast<int>(blockDim.x >> 5); ++k) t = fmax(t, red[k]);
    now = t < tol;
    if (now) conv[blockIdx.x] = sweep;
    else {
      atomicAdd(pending, 1);
      atomicMin(lowest_open, e_base + static_cast<int>(blockIdx.x));
    }
  }
  __syncthreads();
  if (!now) return;
  for (int idx = threadIdx.x; idx < w2; idx += blockDim.x) a[off_fin + idx] = a[off_es + idx];
}

// FIN <- z - FIN (the frozen surface block, inverted next).
__global__ void k_lead_zfin(double2* arena, int64_t stride, int w, int64_t off_fin, const double* __restrict__ energies,
                            double eta) {
  double2* a = arena + blockIdx.y * stride + off_fin;
  const double2 z = make_double2(energies[blockIdx.y], eta);
  const int w2 = w * w;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < w2; idx += gridDim.x * blockDim.x) {
    const int i = idx / w, j = idx - (idx / w) * w;
    a[idx] = zsub(i == j ? z : make_double2(0.0, 0.0), a[idx]);
  }
}

// Exact complex symmetry of the lead Sigma (device.cpp:228-235).
__global__ void k_lead_sym(const double2* arena, int64_t stride, int w, int64_t off_sig, double2* out, int64_t ld) {
  const double2* s = arena + blockIdx.y * stride + off_sig;
  double2* o = out + blockIdx.y * ld;
  const int w2 = w * w;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < w2; idx += gridDim.x * blockDim.x) {
    const int i = idx / w, j = idx - (idx / w) * w;
    if (i == j) {
      o[idx] = s[idx];
    } else {
      const int lo = i < j ? idx : j * w + i, hi = i < j ? j * w + i : idx;  // (i<j) entry first
      const double2 a = s[lo], b = s[hi];
      o[idx] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y + b.y));
    }
  }
}

// ---- analytic transverse-mode lead ---------------------------------------
// Principal complex square root (C99 csqrt / numpy semantics).
__device__ double2 zsqrt(double2 z) {
  if (z.x == 0.0 && z.y == 0.0) return make_double2(0.0, z.y);
  const double r = hypot(z.x, z.y);
  if (z.x >= 0.0) {
    const double t = sqrt(0.5 * (r + z.x));
    return make_double2(t, z.y / (2.0 * t));
  }
  const double t = sqrt(0.5 * (r - z.x));
  return make_double2(fabs(z.y) / (2.0 * t), copysign(t, z.y));
}

__global__ void k_modes_lambda(int w, double t, double eta, const double* __restrict__ energies, double2* sig_m) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;  // mode index 0..w-1 (m+1 in the formula)
  const int e = blockIdx.y;
  if (m >= w) return;
  const double eps = 4.0 * t - 2.0 * t * cos((m + 1) * M_PI / (w + 1));
  const double2 z = make_double2((eps - energies[e]) / (2.0 * t), -eta / (2.0 * t));
  const double2 z2 = make_double2(z.x * z.x - z.y * z.y - 1.0, 2.0 * z.x * z.y);
  const double2 s = zsqrt(z2);
  double2 lam = make_double2(z.x - s.x, z.y - s.y);
  if (hypot(lam.x, lam.y) > 1.0) lam = make_double2(z.x + s.x, z.y + s.y);
  sig_m[static_cast<int64_t>(e) * w + m] = make_double2(-t * lam.x, -t * lam.y);
}

__global__ void k_modes_phi(int w, double* phi) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= w * w) return;
  const int y = idx / w, m = idx - (idx / w) * w;
  phi[idx] = sqrt(2.0 / (w + 1)) * sin(double(y + 1) * double(m + 1) * M_PI / (w + 1));
}

// Sigma_ab = sum_m phi_am sigma_m phi_bm, then symmetrised: one CTA row of
// 32x32 output tile per block, phi and sigma staged in shared memory.
__global__ void k_modes_sigma(int w, const double* __restrict__ phi, const double2* __restrict__ sig_m,
                              double2* out, int64_t ld) {
  const int e = blockIdx.z;
  const int a = blockIdx.y * 32 + threadIdx.y, b = blockIdx.x * 32 + threadIdx.x;
  __shared__ double pa[32][33], pb[32][33];
  __shared__ double2 sm[32];
  double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
  for (int m0 = 0; m0 < w; m0 += 32) {
    const int mm = m0 + threadIdx.x;
    const int ra = blockIdx.y * 32 + threadIdx.y, rb = blockIdx.x * 32 + threadIdx.y;
    pa[threadIdx.y][threadIdx.x] = (ra < w && mm < w) ? phi[ra * w + mm] : 0.0;
    pb[threadIdx.y][threadIdx.x] = (rb < w && mm < w) ? phi[rb * w + mm] : 0.0;
    if (threadIdx.y == 0) sm[threadIdx.x] = mm < w ? sig_m[static_cast<int64_t>(e) * w + mm] : make_double2(0.0, 0.0);
    __syncthreads();
    for (int k = 0; k < 32; ++k) {
      // (phi_am sigma_m) phi_bm, the association of (phi * sigma) @ phi.T
      const double2 l1 = make_double2(pa[threadIdx.y][k] * sm[k].x, pa[threadIdx.y][k] * sm[k].y);
      acc.x += l1.x * pb[threadIdx.x][k];
      acc.y += l1.y * pb[threadIdx.x][k];
      const double2 l2 = make_double2(pb[threadIdx.y][k] * sm[k].x, pb[threadIdx.y][k] * sm[k].y);
      acc2.x += l2.x * pa[threadIdx.x][k];
      acc2.y += l2.y * pa[threadIdx.x][k];
    }
    __syncthreads();
  }
  // acc = S[a][b]; acc2 = S[b'][a'] with b' = blockIdx.x*32+ty, a' = blockIdx.y*32+tx.
  // Exchange through shared memory to pair S[a][b] with S[b][a].
  __shared__ double2 mirror[32][33];
  mirror[threadIdx.y][threadIdx.x] = acc2;  // S[bx*32+ty][by*32+tx]
  __syncthreads();
  if (a < w && b < w) {
    const double2 sba = mirror[threadIdx.x][threadIdx.y];  // S[bx*32+tx][by*32+ty] = S[b][a]
    double2 v;
    if (a == b) v = acc;
    else if (a < b) v = make_double2(0.5 * (acc.x + sba.x), 0.5 * (acc.y + sba.y));
    else v = make_double2(0.5 * (sba.x + acc.x), 0.5 * (sba.y + acc.y));
    out[static_cast<int64_t>(e) * ld + static_cast<int64_t>(a) * w + b] = v;
  }
}

// ---- pattern fill (lesser_self_energy) -------------------------------------
__device__ double fermi_dev(double e, double mu, double kT) {
  const double x = (e - mu) / kT;
  if (x > 700.0) return 0.0;
  if (x < -700.0) return 1.0;
  return 1.0 / (1.0 + exp(x));
}

__global__ void k_fill_contact(int w, const double2* __restrict__ sig, int64_t ld, int64_t sr_off, int64_t sl_off,
                               double mu, double kT, const double* __restrict__ energies, double2* sr,
                               int64_t sr_stride, double2* sl, int64_t sl_stride) {
  const int e = blockIdx.y;
  const double2* s = sig + static_cast<int64_t>(e) * ld;
  const double f = fermi_dev(energies[e], mu, kT);
  const int w2 = w * w;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < w2; idx += gridDim.x * blockDim.x) {
    const int i = idx / w, j = idx - (idx / w) * w;
    const double2 v = s[idx];
    if (sr_off >= 0) sr[static_cast<int64_t>(e) * sr_stride + sr_off + idx] = v;
    if (sl_off >= 0) {
      const double2 u = s[j * w + i];
      const double2 d = make_double2(v.x - u.x, v.y + u.y);  // S_ij - conj(S_ji)
      sl[static_cast<int64_t>(e) * sl_stride + sl_off + idx] = make_double2(-f * d.x, -f * d.y);
    }
  }
}

__global__ void k_fill_phonon(int n, const double* __restrict__ gamma, int64_t sr_off, int64_t sl_off, double mu,
                              double kT, const double* __restrict__ energies, double2* sr, int64_t sr_stride,
                              double2* sl, int64_t sl_stride) {
  const int e = blockIdx.y;
  const double f = fermi_dev(energies[e], mu, kT);
  for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < n; d += gridDim.x * blockDim.x) {
    const double2 s = make_double2(0.0, -gamma[d]);
    if (sr_off >= 0) sr[static_cast<int64_t>(e) * sr_stride + sr_off + d] = s;
    if (sl_off >= 0) {
      const double2 diff = make_double2(s.x - s.x, s.y + s.y);  // s - conj(s)
      sl[static_cast<int64_t>(e) * sl_stride + sl_off + d] = make_double2(-f * diff.x, -f * diff.y);
    }
  }
}

}  // namespace

struct negf_lead {
  LeadPlan L;
  int device = 0;
  double eta = 0.0;
  int criterion = 0;
  double tol = 1e-12;
  cudaStream_t stream = nullptr;
  std::vector<void*> owned;
  int capacity = 1;
  double2* arena = nullptr;
  double2 *d_h00 = nullptr, *d_h01 = nullptr;
  GemmTask* d_tasks = nullptr;
  GemmTerm* d_terms = nullptr;
  GemmTile* d_tiles = nullptr;
  InvTask* d_inv = nullptr;
  BigTask* d_big = nullptr;
  int* d_conv = nullptr;
  int* d_counters = nullptr;  // [pending, lowest_open]
  DevStatus* d_status = nullptr;
  unsigned long long* d_gemm_ctr = nullptr;  // BatchArgs::gemm_ctr
  double* d_energies = nullptr;
  double2* d_out = nullptr;
  int64_t launches = 0;
  std::vector<int> sweeps;
};

namespace {

void replay(negf_lead* l, const BatchArgs& b, const int* range) {
  const Plan& P = l->L.P;
  for (int oi = range[0]; oi < range[1]; ++oi) {
    const Op& op = P.ops[oi];
    switch (op.kind) {
      case K_INVERSE:
        launch_inverse(b, l->d_inv + op.begin, P.inv_tasks.data() + op.begin, op.count, l->d_status, l->stream,
                       l->launches);
        break;
      case K_GEMM:
        launch_gemm(b, l->d_tasks, l->d_terms, l->d_tiles, P.gemm_tiles.data(), op.begin, op.count, l->stream,
                    l->launches);
        break;
      case K_PANEL:
        launch_bigpanel(b, l->d_big + op.begin, P.big_tasks.data() + op.begin, op.count, op.k0, op.k1, l->d_status,
                        l->stream, l->launches);
        break;
      case K_PERM:
        launch_bigperm(b, l->d_big + op.begin, P.big_tasks.data() + op.begin, op.count, l->stream, l->launches);
        break;
      case K_BIGSWAP:
        launch_bigswap(b, l->d_big + op.begin, op.count, op.k1, l->stream, l->launches);
        break;
      default:
        throw Failure(kInternal, "lead: unexpected op kind");
    }
  }
}

// One batch of energies through the decimation; results into d_out + k*ld.
int lead_batch(negf_lead* l, int nE, int e_base, const double* d_E, double2* d_out, int64_t ld, negf_status* st) {
  const LeadPlan& L = l->L;
  const int w = L.w;
  cudaStream_t s = l->stream;
  LeadOffs off;
  for (int k = 0; k < LB_COUNT; ++k) off.o[k] = L.off[k];
  BatchArgs b{l->arena, L.P.arena, nE, e_base, l->d_gemm_ctr};
  const DevStatus clean{~0ull, ~0ull, ~0ull, 0ull};
  ck(cudaMemcpyAsync(l->d_status, &clean, sizeof clean, cudaMemcpyHostToDevice, s), "status reset");
  ck(cudaMemsetAsync(l->d_conv, 0xFF, sizeof(int) * nE, s), "conv reset");
  k_lead_init<<<nE, 256, 0, s>>>(l->arena, L.P.arena, w, off, l->d_h00, l->d_h01, d_E, l->eta, l->criterion);
  ++l->launches;
  const int w2 = w * w;
  const dim3 eg(std::max(1, std::min(64, (w2 + 255) / 256)), nE);
  const bool fixed_point = l->criterion == 0;
  int par = 0;
  int fail_e = -1, fail_tag = 0, fail_pivot = 0, fail_sweep = -1;
  int pending = nE, lowest_open = e_base;
  for (int sweep = 0; sweep < 200; ++sweep) {
    k_lead_prep<<<eg, 256, 0, s>>>(l->arena, L.P.arena, w, off, d_E, l->eta);
    ++l->launches;
    const int init[2] = {0, 0x7fffffff};
    if (fixed_point) {
      replay(l, b, L.inv_gm);
      replay(l, b, L.gemm_a[par]);
      replay(l, b, L.gemm_b);
      replay(l, b, L.inv_rhs);
      ck(cudaMemcpyAsync(l->d_counters, init, sizeof init, cudaMemcpyHostToDevice, s), "counter reset");
      k_lead_check<<<nE, 256, 0, s>>>(l->arena, L.P.arena, w, off, sweep, l->d_conv, l->d_counters,
                                      l->d_counters + 1, e_base);
      ++l->launches;
    } else {  // devices.sancho_rubio: m, update, then the decay test
      replay(l, b, L.inv_m);
      replay(l, b, L.gemm_a2[par]);
      replay(l, b, L.gemm_c[par]);
      par ^= 1;
      ck(cudaMemcpyAsync(l->d_counters, init, sizeof init, cudaMemcpyHostToDevice, s), "counter reset");
      k_lead_check_decay<<<nE, 256, 0, s>>>(l->arena, L.P.arena, w, L.off[par ? LB_ALPHA1 : LB_ALPHA0],
                                            L.off[par ? LB_BETA1 : LB_BETA0], L.off[LB_ES], L.off[LB_FIN], l->tol,
                                            sweep, l->d_conv, l->d_counters, l->d_counters + 1, e_base);
      ++l->launches;
    }
    int cnt[2];
    DevStatus h;
    ck(cudaMemcpyAsync(cnt, l->d_counters, sizeof cnt, cudaMemcpyDeviceToHost, s), "counter read");
    ck(cudaMemcpyAsync(&h, l->d_status, sizeof h, cudaMemcpyDeviceToHost, s), "status read");
    ck(cudaStreamSynchronize(s), "lead sweep");
    pending = cnt[0];
    lowest_open = cnt[1];
    if (h.singular_key != ~0ull) {
      const int e = static_cast<int>(h.singular_key >> 40);
      int c = -1;
      ck(cudaMemcpy(&c, l->d_conv + (e - e_base), sizeof c, cudaMemcpyDeviceToHost), "conv read");
      const int tag = static_cast<int>((h.singular_key >> 20) & 0xFFFFF);
      if ((c >= 0 && c < sweep) || (fixed_point && c == sweep && tag == 1)) {
        // the reference returned at sweep c before this inverse (frozen
        // energy, or m = (z - e)^-1 of the converging sweep): not an error
      } else if (fail_e < 0 || e < fail_e) {
        fail_e = e;
        fail_tag = tag;
        fail_pivot = static_cast<int>(h.singular_key & 0xFFFFF);
        fail_sweep = sweep;
      }
      ck(cudaMemcpyAsync(l->d_status, &clean, sizeof clean, cudaMemcpyHostToDevice, s), "status reset");
    }
    if (pending == 0) break;
    if (fail_e >= 0 && lowest_open >= fail_e) break;  // no lower energy can still fail
    if (fixed_point) {
      replay(l, b, L.gemm_c[par]);
      par ^= 1;
    }
  }
  std::vector<int> conv(static_cast<size_t>(nE));
  ck(cudaMemcpy(conv.data(), l->d_conv, sizeof(int) * nE, cudaMemcpyDeviceToHost), "conv read");
  l->sweeps.insert(l->sweeps.end(), conv.begin(), conv.end());
  if (fail_e >= 0 && (pending == 0 || lowest_open >= fail_e)) {
    static const char* what[4] = {"z - es", "z - e", "fixed-point rhs", "z - es (final)"};
    return set_status(st, NEGF_SINGULAR_BLOCK,
                      "energy point " + std::to_string(fail_e) + ": surface_self_energy: singular pivot " +
                          std::to_string(fail_pivot) + " in the " + std::to_string(w) + "x" + std::to_string(w) +
                          " " + what[std::min(fail_tag, 3)] + " block (sweep " + std::to_string(fail_sweep) + ")",
                      fail_e, -1, fail_pivot);
  }
  if (pending > 0)
    return set_status(st, NEGF_CONVERGENCE_ERROR,
                      "energy point " + std::to_string(lowest_open) +
                          (fixed_point ? ": surface self-energy decimation did not reach a 1e-10 fixed-point "
                                         "residual within 200 sweeps"
                                       : ": Sancho-Rubio decimation did not converge within 200 sweeps"),
                      lowest_open);
  if (!fixed_point) {
    k_lead_zfin<<<eg, 256, 0, s>>>(l->arena, L.P.arena, w, L.off[LB_FIN], d_E, l->eta);
    ++l->launches;
    replay(l, b, L.inv_fin);
    DevStatus h;
    ck(cudaMemcpyAsync(&h, l->d_status, sizeof h, cudaMemcpyDeviceToHost, s), "status read");
    ck(cudaStreamSynchronize(s), "lead final inverse");
    if (h.singular_key != ~0ull) {
      const int e = static_cast<int>(h.singular_key >> 40);
      const int pv = static_cast<int>(h.singular_key & 0xFFFFF);
      return set_status(st, NEGF_SINGULAR_BLOCK,
                        "energy point " + std::to_string(e) + ": Sancho-Rubio: singular pivot " + std::to_string(pv) +
                            " in the final surface block",
                        e, -1, pv);
    }
  }
  replay(l, b, L.fin1);
  replay(l, b, L.fin2);
  const dim3 sg(std::max(1, std::min(64, (w2 + 255) / 256)), nE);
  k_lead_sym<<<sg, 256, 0, s>>>(l->arena, L.P.arena, w, L.off[LB_SIG], d_out, ld);
  ++l->launches;
  ck(cudaGetLastError(), "lead launch");
  ck(cudaStreamSynchronize(s), "lead finish");
  return ok(st);
}

}  // namespace

extern "C" {

int negf_lead_create(int device, int w, const double* h00, const double* h01, double eta_ev, int criterion,
                     double tol, int max_energy_batch, negf_lead** out, negf_status* st) {
  if (!out || !h00 || !h01) return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  *out = nullptr;
  if (!(eta_ev > 0.0)) return set_status(st, NEGF_CONFIG_ERROR, "contact broadening eta must be positive");
  if (criterion != 0 && criterion != 1) return set_status(st, NEGF_CONTRACT_VIOLATION, "unknown lead criterion");
  if (criterion == 1 && !(tol > 0.0)) return set_status(st, NEGF_CONFIG_ERROR, "decimation tolerance must be positive");
  if (w <= 0)
    return set_status(st, NEGF_CONTRACT_VIOLATION,
                      "surface_self_energy: lead block size " + std::to_string(w) + " out of range");
  auto l = std::make_unique<negf_lead>();
  try {
    l->L = build_lead_plan(w);
    l->device = device;
    l->eta = eta_ev;
    l->criterion = criterion;
    l->tol = tol;
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&l->stream, cudaStreamNonBlocking), "stream");
    const Plan& P = l->L.P;
    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "meminfo");
    const int64_t per = P.arena * int64_t(sizeof(double2));
    int cap = max_energy_batch > 0 ? std::min(max_energy_batch, kMaxGridYZ) : 512;
    cap = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(cap, int64_t(0.4 * free_b) / per)));
    l->capacity = cap;
    l->arena = dev_alloc<double2>(static_cast<size_t>(P.arena) * cap, l->owned);
    std::vector<double2> a(static_cast<size_t>(w) * w), b(a.size());
    for (size_t k = 0; k < a.size(); ++k) {
      a[k] = make_double2(h00[2 * k], h00[2 * k + 1]);
      b[k] = make_double2(h01[2 * k], h01[2 * k + 1]);
    }
    l->d_h00 = dev_upload(a, l->owned);
    l->d_h01 = dev_upload(b, l->owned);
    l->d_tasks = dev_upload(P.gemm_tasks, l->owned);
    l->d_terms = dev_upload(P.gemm_terms, l->owned);
    l->d_tiles = dev_upload(P.gemm_tiles, l->owned);
    l->d_inv = dev_upload(P.inv_tasks, l->owned);
    l->d_big = dev_upload(P.big_tasks, l->owned);
    l->d_conv = dev_alloc<int>(static_cast<size_t>(cap), l->owned);
    l->d_counters = dev_alloc<int>(2, l->owned);
    l->d_status = dev_alloc<DevStatus>(1, l->owned);
    l->d_gemm_ctr = dev_alloc<unsigned long long>(2, l->owned);
    ck(cudaMemset(l->d_gemm_ctr, 0, 2 * sizeof(unsigned long long)), "memset");
    l->d_energies = dev_alloc<double>(static_cast<size_t>(cap), l->owned);
    l->d_out = dev_alloc<double2>(static_cast<size_t>(cap) * w * w, l->owned);
  } catch (const CudaFail& f) {
    for (void* p : l->owned) cudaFree(p);
    if (l->stream) cudaStreamDestroy(l->stream);
    return set_status(st, f.code, f.msg);
  } catch (const Failure& f) {
    return set_status(st, f.code == kContractViolation ? NEGF_CONTRACT_VIOLATION : NEGF_INTERNAL, f.what());
  }
  *out = l.release();
  return ok(st);
}

int negf_lead_sigma_device(negf_lead* l, int n_energies, const double* d_energies, int first_energy_index,
                           double* d_sigma_out, int64_t ld_out, negf_status* st) {
  if (!l || (n_energies > 0 && (!d_energies || !d_sigma_out)))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  const int w = l->L.w;
  if (ld_out < int64_t(w) * w) return set_status(st, NEGF_CONTRACT_VIOLATION, "ld_out < w*w");
  try {
    ck(cudaSetDevice(l->device), "cudaSetDevice");
    l->launches = 0;
    l->sweeps.clear();
    for (int e0 = 0; e0 < n_energies; e0 += l->capacity) {
      const int m = std::min(l->capacity, n_energies - e0);
      const int rc = lead_batch(l, m, first_energy_index + e0, d_energies + e0,
                                reinterpret_cast<double2*>(d_sigma_out) + int64_t(e0) * ld_out, ld_out, st);
      if (rc != NEGF_OK) return rc;
    }
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  } catch (const Failure& f) {
    return set_status(st, NEGF_INTERNAL, f.what());
  }
  return ok(st);
}

int negf_lead_sigma(negf_lead* l, int n_energies, const double* energies, int first_energy_index, double* sigma_out,
                    negf_status* st) {
  if (!l || (n_energies > 0 && (!energies || !sigma_out)))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  const int w = l->L.w;
  const int64_t w2 = int64_t(w) * w;
  try {
    ck(cudaSetDevice(l->device), "cudaSetDevice");
    l->launches = 0;
    l->sweeps.clear();
    int64_t total = 0;
    for (int e0 = 0; e0 < n_energies; e0 += l->capacity) {
      const int m = std::min(l->capacity, n_energies - e0);
      ck(cudaMemcpyAsync(l->d_energies, energies + e0, sizeof(double) * m, cudaMemcpyHostToDevice, l->stream),
         "energies upload");
      const int64_t before = l->launches;
      const int rc = lead_batch(l, m, first_energy_index + e0, l->d_energies, l->d_out, w2, st);
      total += l->launches - before;
      if (rc != NEGF_OK) return rc;
      ck(cudaMemcpyAsync(sigma_out + 2 * int64_t(e0) * w2, l->d_out, sizeof(double2) * m * w2,
                         cudaMemcpyDeviceToHost, l->stream),
         "sigma download");
      ck(cudaStreamSynchronize(l->stream), "sigma download");
    }
    l->launches = total;
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  } catch (const Failure& f) {
    return set_status(st, NEGF_INTERNAL, f.what());
  }
  return ok(st);
}

int negf_lead_last_sweeps(const negf_lead* l, int32_t* sweeps_out) {
  if (!l || !sweeps_out) return NEGF_CONTRACT_VIOLATION;
  for (size_t k = 0; k < l->sweeps.size(); ++k) sweeps_out[k] = l->sweeps[k];
  return NEGF_OK;
}

int64_t negf_lead_last_launches(const negf_lead* l) { return l ? l->launches : 0; }

void* negf_lead_stream(negf_lead* l) { return l ? static_cast<void*>(l->stream) : nullptr; }

void negf_lead_destroy(negf_lead* l) {
  if (!l) return;
  cudaSetDevice(l->device);
  if (l->stream) cudaStreamSynchronize(l->stream);
  for (void* p : l->owned) cudaFree(p);
  if (l->stream) cudaStreamDestroy(l->stream);
  delete l;
}

int negf_lead_modes_sigma_device(int w, double t_ev, double eta_ev, int n_energies, const double* d_energies,
                                 double* d_sigma_out, int64_t ld_out, void* stream, negf_status* st) {
  if (w <= 0 || (n_energies > 0 && (!d_energies || !d_sigma_out)))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "bad argument");
  if (!(eta_ev > 0.0)) return set_status(st, NEGF_CONFIG_ERROR, "contact broadening eta must be positive");
  if (ld_out < int64_t(w) * w) return set_status(st, NEGF_CONTRACT_VIOLATION, "ld_out < w*w");
  if (n_energies == 0) return ok(st);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  try {
    // Grow-only scratch (mode functions per width, lambda_m per energy): no
    // per-call allocation, so the call stays asynchronous on `stream`.
    struct Scratch {
      int device = -1, w = 0;
      double* phi = nullptr;
      double2* sig = nullptr;
      size_t sig_cap = 0;
    };
    static thread_local Scratch sc;
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    if (sc.device != dev) sc = Scratch{dev};
    if (sc.w != w) {
      if (sc.phi) ck(cudaFree(sc.phi), "cudaFree");
      sc.phi = nullptr;
      ck(cudaMalloc(&sc.phi, sizeof(double) * w * w), "phi");
      sc.w = w;
      k_modes_phi<<<(w * w + 255) / 256, 256, 0, s>>>(w, sc.phi);
      ck(cudaStreamSynchronize(s), "phi");  // later calls may use other streams
    }
    const size_t need = size_t(w) * n_energies;
    if (sc.sig_cap < need) {
      if (sc.sig) ck(cudaFree(sc.sig), "cudaFree");
      sc.sig = nullptr;
      ck(cudaMalloc(&sc.sig, sizeof(double2) * need), "sigma_m");
      sc.sig_cap = need;
    }
    // the energy index lives in gridDim.y / gridDim.z (<= 65535): chunk
    const int nb = (w + 31) / 32;
    for (int e0 = 0; e0 < n_energies; e0 += kMaxGridYZ) {
      const int m = std::min(kMaxGridYZ, n_energies - e0);
      k_modes_lambda<<<dim3((w + 127) / 128, m), 128, 0, s>>>(w, t_ev, eta_ev, d_energies + e0,
                                                             sc.sig + size_t(w) * e0);
      k_modes_sigma<<<dim3(nb, nb, m), dim3(32, 32), 0, s>>>(
          w, sc.phi, sc.sig + size_t(w) * e0, reinterpret_cast<double2*>(d_sigma_out) + size_t(ld_out) * e0, ld_out);
    }
    ck(cudaGetLastError(), "modes launch");
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  }
  return ok(st);
}

int negf_contacts_fill_device(int n_energies, const double* d_energies, double kT_ev, int n_contacts,
                              const negf_contact_desc* contacts, int n_phonon, const double* d_phonon_gamma,
                              int64_t ph_sr_off, int64_t ph_sl_off, double mu_phonon_ev, double* d_sigma_r,
                              int64_t sr_stride, double* d_sigma_lesser, int64_t sl_stride, void* stream,
                              negf_status* st) {
  if (n_energies <= 0) return ok(st);
  if (!d_energies || (n_contacts > 0 && !contacts))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  if (!(kT_ev > 0.0)) return set_status(st, NEGF_CONFIG_ERROR, "temperature must be positive");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  try {
    for (int c = 0; c < n_contacts; ++c) {
      const negf_contact_desc& cd = contacts[c];
      if (cd.w <= 0 || !cd.d_sigma || cd.ld < int64_t(cd.w) * cd.w)
        return set_status(st, NEGF_CONTRACT_VIOLATION, "contact block shape does not match its dof set");
      if ((cd.sr_off >= 0 && !d_sigma_r) || (cd.sl_off >= 0 && !d_sigma_lesser))
        return set_status(st, NEGF_CONTRACT_VIOLATION, "null pattern array");
      const int w2 = cd.w * cd.w;
      for (int e0 = 0; e0 < n_energies; e0 += kMaxGridYZ) {  // energies in gridDim.y: chunk
        const int m = std::min(kMaxGridYZ, n_energies - e0);
        k_fill_contact<<<dim3(std::max(1, std::min(64, (w2 + 255) / 256)), m), 256, 0, s>>>(
            cd.w, reinterpret_cast<const double2*>(cd.d_sigma) + size_t(cd.ld) * e0, cd.ld, cd.sr_off, cd.sl_off,
            cd.mu_ev, kT_ev, d_energies + e0,
            d_sigma_r ? reinterpret_cast<double2*>(d_sigma_r) + size_t(sr_stride) * e0 : nullptr, sr_stride,
            d_sigma_lesser ? reinterpret_cast<double2*>(d_sigma_lesser) + size_t(sl_stride) * e0 : nullptr,
            sl_stride);
      }
    }
    if (n_phonon > 0) {
      if (!d_phonon_gamma) return set_status(st, NEGF_CONTRACT_VIOLATION, "null phonon array");
      for (int e0 = 0; e0 < n_energies; e0 += kMaxGridYZ) {
        const int m = std::min(kMaxGridYZ, n_energies - e0);
        k_fill_phonon<<<dim3(std::max(1, std::min(256, (n_phonon + 255) / 256)), m), 256, 0, s>>>(
            n_phonon, d_phonon_gamma, ph_sr_off, ph_sl_off, mu_phonon_ev, kT_ev, d_energies + e0,
            d_sigma_r ? reinterpret_cast<double2*>(d_sigma_r) + size_t(sr_stride) * e0 : nullptr, sr_stride,
            d_sigma_lesser ? reinterpret_cast<double2*>(d_sigma_lesser) + size_t(sl_stride) * e0 : nullptr,
            sl_stride);
      }
    }
    ck(cudaGetLastError(), "fill launch");
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  }
  return ok(st);
}

}  // extern "C"
