// Device kernels of the B200 HSC path.  Complex FP64 throughout
// (interleaved double2 in HBM, as std::complex<double> in the reference).
//
//   k_assemble_*   A(E) = E I - H - Sigma^r(E) into the per-energy block arena
//                  (assemble_system + group_by_partition, block.cpp:49-82,
//                  123-161): template copy + diagonal / pattern scatters.
//   k_inverse_*    batched Gauss-Jordan explicit inverse with row partial
//                  pivoting and the reference's singular-pivot rule
//                  |u_kk| <= 1e-13 max|a| (dense.cpp:49-81).
//   k_gemm         grouped multi-term complex GEMM on FP64 tensor cores
//                  (mma.sync m8n8k4 f64 = SASS DMMA.8x8x4, the only FP64
//                  tensor path on sm_100a): every Psi, Schur, G/N/P row and
//                  diagonal-block update of hsc.cpp is one task of it.
//   k_diag         diagonal-only dot products for never-referenced clusters.
//   k_scale        diagonal Sigma^< seeds N = diag(s) conj(G) (hsc.cpp:122-125).
//   k_output       per-dof diag G^r / G^<, Re-residual guard and the weighted
//                  energy sum of electron_density (observables.cpp:71-91).
#include "kernels.hpp"

#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cstdio>
#include <cstdlib>

namespace negfb {

// Per-device one-time setup (function attributes are per device): true the
// first time a call site runs on the current device.
inline bool first_on_device(std::atomic<unsigned long long>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  return (done.fetch_or(bit) & bit) == 0;
}

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__device__ __forceinline__ double cabs2(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double2 cinv(double2 a) {
  // 1/a with scaling against overflow (Smith's algorithm).
  if (fabs(a.x) >= fabs(a.y)) {
    const double r = a.y / a.x, d = a.x + a.y * r;
    return make_double2(1.0 / d, -r / d);
  }
  const double r = a.x / a.y, d = a.x * r + a.y;
  return make_double2(r / d, -1.0 / d);
}

// ---------------------------------------------------------------------------
// Assembly
// ---------------------------------------------------------------------------
// Per-energy initialisation: zero the regions listed by the plan (D blocks,
// the original-entry prefix of each Arow row, Sigma^< blocks).  One CTA
// strides over regions; rows are coalesced.  Write-only traffic.
__global__ void k_init(double2* arena, int64_t stride, const InitRegion* __restrict__ zero, int nzero) {
  double2* a = arena + blockIdx.y * stride;
  for (int r = blockIdx.x; r < nzero; r += gridDim.x) {
    const InitRegion g = zero[r];
    const int64_t total = int64_t(g.rows) * g.cols;
    for (int64_t i = threadIdx.x; i < total; i += blockDim.x) {
      const int row = static_cast<int>(i / g.cols), col = static_cast<int>(i - int64_t(row) * g.cols);
      a[g.off + int64_t(row) * g.pitch + col] = make_double2(0.0, 0.0);
    }
  }
}

// -H entries into the zeroed A region (positions unique).
__global__ void k_scatter_h(double2* arena, int64_t stride, const int64_t* __restrict__ pos,
                            const double2* __restrict__ val, int64_t nnz) {
  double2* a = arena + blockIdx.y * stride;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nnz; i += int64_t(gridDim.x) * blockDim.x)
    a[pos[i]] = val[i];
}

// E on the diagonal and the Sigma^< slots (which live outside the A region).
__global__ void k_scatter(double2* arena, int64_t stride, int n, const int64_t* __restrict__ diag_pos,
                          const double* __restrict__ energies, const int64_t* __restrict__ sl_pos, const int* __restrict__ sl_ptr,
                          const int* __restrict__ sl_src, int sl_slots, int64_t sl_nnz,
                          const double2* __restrict__ sigma_l) {
  const int e = blockIdx.y;
  double2* a = arena + e * stride;
  const double E = energies[e];
  const int64_t step = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = t0; i < n; i += step) a[diag_pos[i]].x += E;
  const double2* sl = sigma_l + e * sl_nnz;
  for (int64_t s = t0; s < sl_slots; s += step) {
    double2 v = make_double2(0.0, 0.0);
    for (int q = sl_ptr[s]; q < sl_ptr[s + 1]; ++q) v = cadd(v, sl[sl_src[q]]);
    a[sl_pos[s]] = v;
  }
}

// Sigma^r slots: ordered after k_scatter (a diagonal slot hits an entry that
// k_scatter has just shifted by E).
__global__ void k_scatter_sigma_r(double2* arena, int64_t stride, const int64_t* __restrict__ sr_pos,
                                  const int* __restrict__ sr_ptr, const int* __restrict__ sr_src,
                                  int sr_slots, int64_t sr_nnz, const double2* __restrict__ sigma_r) {
  const int e = blockIdx.y;
  double2* a = arena + e * stride;
  const double2* sr = sigma_r + e * sr_nnz;
  const int64_t step = int64_t(gridDim.x) * blockDim.x;
  for (int64_t s = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; s < sr_slots; s += step) {
    double2 v = make_double2(0.0, 0.0);
    for (int q = sr_ptr[s]; q < sr_ptr[s + 1]; ++q) v = cadd(v, sr[sr_src[q]]);
    const int64_t p = sr_pos[s];
    a[p] = csub(a[p], v);
  }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// Batched explicit inverse (Gauss-Jordan, row partial pivoting, in place)
// ---------------------------------------------------------------------------
__device__ void report_singular(DevStatus* st, int e_global, int fold_pos, int pivot) {
  const unsigned long long key = (static_cast<unsigned long long>(e_global) << 40) |
                                 (static_cast<unsigned long long>(fold_pos) << 20) |
                                 static_cast<unsigned long long>(pivot);
  atomicMin(&st->singular_key, key);
}



// Register-resident Gauss-Jordan for m <= TR*R (one CTA per (block, energy)).
// Thread (tr, tc) of a TR x TC grid owns rows tr + TR*i and columns
// tc + TC*j of the block in registers; per pivot step only the pivot column
// and the pivot row travel through shared memory (double-buffered by step
// parity, two barriers per step).  Same pivots and singular rule as above.
template <int TR, int R>
__global__ void __launch_bounds__(TR * TR) k_inverse_reg(double2* arena, int64_t stride,
                                                         const InvTask* __restrict__ tasks, int e_base,
                                                         DevStatus* st) {
  constexpr int NT = TR * TR, MMAX = TR * R;
  __shared__ double2 colk[2][MMAX];
  __shared__ double2 prow[2][MMAX], krow[MMAX];
  __shared__ double red[NT / 32];
  __shared__ int cur_at[MMAX], pos_of[MMAX], perm[MMAX];
  const InvTask tk = tasks[blockIdx.x];
  const int m = tk.m;
  double2* g = arena + int64_t(blockIdx.y) * stride + tk.off;
  const int tid = threadIdx.x, tr = tid / TR, tc = tid - (tid / TR) * TR;
  double2 a[R][R];
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int r = tr + TR * i, c = tc + TR * j;
      a[i][j] = (r < m && c < m) ? g[int64_t(r) * m + c] : make_double2(0.0, 0.0);
      mx = fmax(mx, cabs2(a[i][j]));
    }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((tid & 31) == 0) red[tid >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, red[w]);
  const double thresh = 1e-13 * mx;
  bool failed = false;
  for (int k = 0; k < m; ++k) {
    const int par = k & 1;
    // 1. publish column k
    if (tc == k % TR) {
      const int jj = k / TR;
#pragma unroll
      for (int i = 0; i < R; ++i) {
        const int r = tr + TR * i;
#pragma unroll
        for (int j = 0; j < R; ++j)
          if (j == jj && r < m) colk[par][r] = a[i][j];
      }
    }
    __syncthreads();
    // 2. pivot: every warp reduces redundantly (largest |a_rk|, lowest row)
    double best = -1.0;
    int bi = k;
    for (int r = k + (tid & 31); r < m; r += 32) {
      const double v = cabs2(colk[par][r]);
      if (v > best) {
        best = v;
        bi = r;
      }
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (best <= thresh) {  // uniform across the CTA
      if (tid == 0) report_singular(st, e_base + blockIdx.y, tk.fold_pos, k);
      failed = true;
      break;
    }
    const int p = bi;
    if (tid == 0) perm[k] = p;
    // 3. pivot row (old row p) and old row k through shared memory
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = tr + TR * i;
      if (r == p || r == k)
#pragma unroll
        for (int j = 0; j < R; ++j) {
          const int c = tc + TR * j;
          if (c < m) {
            if (r == p) prow[par][c] = a[i][j];
            if (r == k) krow[c] = a[i][j];
          }
        }
    }
    __syncthreads();
    const double2 piv = colk[par][p];
    const double2 ip = cinv(piv);
    // 4./5. elimination on the swapped matrix: row k <- normalised old row p,
    // row p <- old row k, then every other row r: a_r -= a_rk * pivot row.
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const int r = tr + TR * i;
      if (r >= m) continue;
      double2 f;  // column-k value of (swapped) row r
      if (r == k) f = piv;
      else if (r == p) f = colk[par][k];
      else f = colk[par][r];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int c = tc + TR * j;
        if (c >= m) continue;
        const double2 pr = (c == k) ? ip : cmul(prow[par][c], ip);  // normalised pivot row
        if (r == k) {
          a[i][j] = pr;
        } else {
          const double2 base_v = (r == p) ? krow[c] : a[i][j];
          if (c == k) a[i][j] = make_double2(-(f.x * ip.x - f.y * ip.y), -(f.x * ip.y + f.y * ip.x));
          else a[i][j] = csub(base_v, cmul(f, pr));
        }
      }
    }
    // krow is reused next step: make sure every thread consumed it.
    __syncthreads();
  }
  if (failed) return;
  // Undo the row interchanges as column interchanges, last first: the column
  // currently at position q ends at pos_of[original].
  if (tid == 0) {
    for (int c = 0; c < m; ++c) cur_at[c] = c;
    for (int k = m - 1; k >= 0; --k) {
      const int p = perm[k];
      const int t2 = cur_at[k];
      cur_at[k] = cur_at[p];
      cur_at[p] = t2;
    }
    for (int q = 0; q < m; ++q) pos_of[cur_at[q]] = q;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < R; ++i)
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int r = tr + TR * i, c = tc + TR * j;
      if (r < m && c < m) g[int64_t(r) * m + pos_of[c]] = a[i][j];
    }
}

// Blocked Gauss-Jordan (right-looking, panel width 8) for 32 < m: the same
// pivots and singular rule as the unblocked elimination, but after each
// 8-column panel (factored by one warp with only __syncwarp) the rest of the
// block receives one rank-8 update R += (M_p - I_p) R_p on the FP64 tensor
// cores (DMMA), where M_p are the panel's accumulated Gauss-Jordan columns and
// R_p the 8 pivot rows -- three CTA barriers per 8 pivots.
// kGlobal: the block stays in global memory (L2-resident) for m > kSmemInvMax.
constexpr int INV_THREADS = 128;

// Panel of NB columns held in registers of warp 0: lane owns rows lane+32*i.
// Pivot rows travel by shuffles; the pivot loop is fully unrolled so every
// column index is a compile-time constant (no dynamic register selects), and
// candidates are compared by |z|^2 (same argmax as |z|).
__device__ __forceinline__ double cnorm(double2 a) { return fma(a.x, a.x, a.y * a.y); }
__device__ __forceinline__ double2 crcp(double2 a) {
  const double s = fmax(fabs(a.x), fabs(a.y));
  const double x = a.x / s, y = a.y / s;
  const double d = s * fma(x, x, y * y);
  return make_double2(x / d, -y / d);
}

// One NB-column panel of the shared-memory blocked Gauss-Jordan, factored by
// warp 0 with the panel held in registers: lane owns rows lane + 32 i (i <
// RPL).  Rows are not moved while the panel is factored: each lane tracks the
// current position of its rows (exactly the row interchanges of partial
// pivoting, ties to the lowest position), the pivot row reaches every lane by
// shuffles, and the panel is written back at the final positions -- no
// shared-memory round trip per pivot.  Same pivots, singular rule and
// per-element arithmetic as the shared-memory loop.  Returns false (after
// reporting) on a singular pivot.
template <int RPL, int NB>
__device__ __forceinline__ bool panel_regs(double2* A, int ld, int m, int k0, int kb, double thr2, int* perm,
                                           int* flag, DevStatus* st, int e_global, int fold_pos) {
  const int lane = threadIdx.x & 31;
  double2 v[RPL][NB];
  int pos[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = lane + 32 * i;
    pos[i] = r;
#pragma unroll
    for (int c = 0; c < NB; ++c) v[i][c] = (r < m) ? A[r * ld + k0 + c] : make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int kk = 0; kk < NB; ++kk) {
    if (kk >= kb) break;
    const int k = k0 + kk;
    double best = -1.0;
    int bpos = 0x7fffffff, bslot = 0;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      if (lane + 32 * i < m && pos[i] >= k) {
        const double x = cnorm(v[i][kk]);
        if (x > best || (x == best && pos[i] < bpos)) {
          best = x;
          bpos = pos[i];
          bslot = i;
        }
      }
    }
    const unsigned key = best >= 0.0 ? __float_as_uint(__double2float_ru(best)) : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    const unsigned tied = __ballot_sync(0xffffffffu, best >= 0.0 && key == kmax);
    int wl;
    if (__popc(tied) <= 1) {
      wl = tied ? __ffs(tied) - 1 : 0;
    } else {  // exact order among the lanes whose float images tie
      double cb = (best >= 0.0 && key == kmax) ? best : -1.0;
      int cp = (best >= 0.0 && key == kmax) ? bpos : 0x7fffffff, cl = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, cb, o);
        const int op = __shfl_xor_sync(0xffffffffu, cp, o);
        const int ol = __shfl_xor_sync(0xffffffffu, cl, o);
        if (ob > cb || (ob == cb && op < cp)) {
          cb = ob;
          cp = op;
          cl = ol;
        }
      }
      wl = cl;
    }
    const double wb = __shfl_sync(0xffffffffu, best, wl);
    if (!(wb > thr2) && wb == wb) {  // |u_kk| <= 1e-13 max|a| (NaN passes, as the smem loop)
      if (lane == 0) {
        *flag = 1;
        report_singular(st, e_global, fold_pos, k);
      }
      return false;
    }
    const int p = __shfl_sync(0xffffffffu, bpos, wl);
    const int ws = __shfl_sync(0xffffffffu, bslot, wl);
    if (lane == 0) perm[k] = p;
    double2 pr[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      double2 x = v[0][c];
#pragma unroll
      for (int i = 1; i < RPL; ++i)
        if (ws == i) x = v[i][c];
      pr[c].x = __shfl_sync(0xffffffffu, x.x, wl);
      pr[c].y = __shfl_sync(0xffffffffu, x.y, wl);
    }
    const double2 piv = pr[kk];
    const double rd = 1.0 / fma(piv.x, piv.x, piv.y * piv.y);
    const double2 ip = make_double2(piv.x * rd, -piv.y * rd);
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
        for (int c = 0; c < NB; ++c) v[i][c] = (c == kk) ? cmul(f, nip) : csub(v[i][c], cmul(f, pr[c]));
      }
      if (pos[i] == k) pos[i] = p;
      else if (pos[i] == p) pos[i] = k;
    }
  }
#pragma unroll
  for (int i = 0; i < RPL; ++i)
    if (lane + 32 * i < m)
#pragma unroll
      for (int c = 0; c < NB; ++c) A[pos[i] * ld + k0 + c] = v[i][c];
  return true;
}

template <bool kGlobal, int RPL, int NB>
// blocks <= 32 wide need few registers and little shared memory: 6 CTAs/SM
__global__ void __launch_bounds__(INV_THREADS, RPL == 1 ? 6 : 3) k_inverse_blocked(double2* arena, int64_t stride,
                                                                 const InvTask* __restrict__ tasks, int e_base,
                                                                 DevStatus* st) {
  extern __shared__ double2 sm[];
  const InvTask tk = tasks[blockIdx.x];
  const int m = tk.m;
  const int m8 = (m + 7) & ~7;
  const int ld = kGlobal ? m : m8 + 2;  // smem row pitch: 2 mod 8 -> conflict-free fragments
  double2* g = arena + int64_t(blockIdx.y) * stride + tk.off;
  // shared layout: [A (smem variant) | Rs: 8 x m8 | Pn: m8 x 8 (global variant) | ints]
  double2* A = kGlobal ? g : sm;
  double2* Rs = kGlobal ? sm : sm + int64_t(m8) * ld;
  double2* Pn = Rs + 8 * (m8 + 2);
  int* perm = reinterpret_cast<int*>(Pn + (kGlobal ? 8 * m8 : 0));
  int* pos_of = perm + m8;
  double* red = reinterpret_cast<double*>(pos_of + m8 + (m8 & 1));
  int* flag = reinterpret_cast<int*>(red + INV_THREADS / 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  double mx = 0.0;
  if (!kGlobal) {
    for (int i = tid; i < m8 * m8; i += INV_THREADS) {
      const int r = i / m8, c = i - r * m8;
      const double2 v = (r < m && c < m) ? g[int64_t(r) * m + c] : make_double2(0.0, 0.0);
      A[r * ld + c] = v;
      mx = fmax(mx, cabs2(v));
    }
  } else {
    for (int64_t i = tid; i < int64_t(m) * m; i += INV_THREADS) mx = fmax(mx, cabs2(A[i]));
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  if (tid == 0) *flag = 0;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < INV_THREADS / 32; ++w) mx = fmax(mx, red[w]);
  const double thresh = 1e-13 * mx;
  // element (r, c) of the block
  auto at = [&](int r, int c) -> double2& { return A[int64_t(r) * ld + c]; };

#ifdef NEGF_INV_CLOCKS
  long long clk_panel = 0, clk_swap = 0, clk_upd = 0, c0 = clock64();
#endif
  for (int k0 = 0; k0 < m; k0 += NB) {
    const int kb = min(NB, m - k0);
    // ---- panel (columns k0..k0+7, all rows) on warp 0
    double2* P = kGlobal ? Pn : nullptr;
    auto pan = [&](int r, int c) -> double2& { return kGlobal ? P[r * 8 + c] : at(r, k0 + c); };
    if (kGlobal) {
      for (int i = tid; i < m8 * 8; i += INV_THREADS) {
        const int r = i >> 3, c = i & 7;
        P[i] = (r < m && k0 + c < m) ? at(r, k0 + c) : make_double2(0.0, 0.0);
      }
      __syncthreads();
    }
#ifndef NEGF_PANEL_SMEM
    if (!kGlobal && warp == 0) {
      panel_regs<RPL, NB>(A, ld, m, k0, kb, thresh * thresh, perm, flag, st, e_base + blockIdx.y, tk.fold_pos);
    } else if (false) {
#else
    if (!kGlobal && warp == 0) {
#endif
      // Compact panel loop on warp 0: lane owns rows lane + 32 i (i < RPL);
      // the pivot row is read by broadcast from shared memory and the
      // elimination runs in registers.  Argmax: hardware max-reduction on the
      // float image of |a_rk|^2 (monotone), lowest row among the maxima,
      // then the exact double test against the singular threshold.
      const double thr2 = thresh * thresh;
      for (int kk = 0; kk < kb; ++kk) {
        const int k = k0 + kk;
        double best = -1.0;
        int bi = 0x7fffffff;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const int r = lane + 32 * i;
          if (r >= k && r < m) {
            const double v = cnorm(pan(r, kk));
            if (v > best) {
              best = v;
              bi = r;
            }
          }
        }
        const unsigned key = best >= 0.0 ? __float_as_uint(__double2float_ru(best)) : 0u;
        const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
        const unsigned tied = __ballot_sync(0xffffffffu, key == kmax);
        double cb;
        int ci;
        if (__popc(tied) == 1) {  // usual case: a single candidate lane
          const int src = __ffs(tied) - 1;
          cb = __shfl_sync(0xffffffffu, best, src);
          ci = __shfl_sync(0xffffffffu, bi, src);
        } else {  // exact order among the lanes whose float images tie
          cb = (key == kmax) ? best : -1.0;
          ci = (key == kmax) ? bi : 0x7fffffff;
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, cb, o);
            const int oi = __shfl_xor_sync(0xffffffffu, ci, o);
            if (ob > cb || (ob == cb && oi < ci)) {
              cb = ob;
              ci = oi;
            }
          }
        }
        if (!(cb > thr2)) {  // |u_kk| <= 1e-13 max|a| (NaN: see below)
          if (cb == cb) {
            if (lane == 0) {
              *flag = 1;
              report_singular(st, e_base + blockIdx.y, tk.fold_pos, k);
            }
            break;
          }
        }
        const int p = ci;
        if (lane == 0) perm[k] = p;
        if (lane < NB && p != k) {
          const double2 t2 = pan(k, lane);
          pan(k, lane) = pan(p, lane);
          pan(p, lane) = t2;
        }
        __syncwarp();
        double2 pr[NB];
#pragma unroll
        for (int c = 0; c < NB; ++c) pr[c] = pan(k, c);
        double2 piv = pr[0];
#pragma unroll
        for (int c = 1; c < NB; ++c)
          if (c == kk) piv = pr[c];
        const double rd = 1.0 / fma(piv.x, piv.x, piv.y * piv.y);
        const double2 ip = make_double2(piv.x * rd, -piv.y * rd);
#pragma unroll
        for (int c = 0; c < NB; ++c) pr[c] = (c == kk) ? ip : cmul(pr[c], ip);
        const double2 nip = make_double2(-ip.x, -ip.y);
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const int r = lane + 32 * i;
          if (r >= m) continue;
          if (r == k) {
#pragma unroll
            for (int c = 0; c < NB; ++c) pan(r, c) = pr[c];
            continue;
          }
          const double2 f = pan(r, kk);
#pragma unroll
          for (int c = 0; c < NB; ++c) pan(r, c) = (c == kk) ? cmul(f, nip) : csub(pan(r, c), cmul(f, pr[c]));
        }
        __syncwarp();
      }
    } else if (kGlobal && warp == 0) {
      for (int kk = 0; kk < kb; ++kk) {
        const int k = k0 + kk;
        double best = -1.0;
        int bi = k;
        for (int r = k + lane; r < m; r += 32) {
          const double v = cabs2(pan(r, kk));
          if (v > best) {
            best = v;
            bi = r;
          }
        }
        for (int o = 16; o; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
          }
        }
        if (best <= thresh) {
          if (lane == 0) {
            *flag = 1;
            report_singular(st, e_base + blockIdx.y, tk.fold_pos, k);
          }
          break;
        }
        const int p = bi;
        if (lane == 0) perm[k] = p;
        if (lane < 8 && p != k) {
          const double2 t2 = pan(k, lane);
          pan(k, lane) = pan(p, lane);
          pan(p, lane) = t2;
        }
        __syncwarp();
        const double2 ip = cinv(pan(k, kk));
        // Each lane owns rows lane, lane+32, ...: read its column-k factor
        // before row k is rewritten, then update its rows.
        __syncwarp();
        if (lane < 8) pan(k, lane) = (lane == kk) ? ip : cmul(pan(k, lane), ip);
        __syncwarp();
        for (int r = lane; r < m; r += 32) {
          if (r == k) continue;
          const double2 f = pan(r, kk);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            if (c == kk) pan(r, c) = make_double2(-(f.x * ip.x - f.y * ip.y), -(f.x * ip.y + f.y * ip.x));
            else pan(r, c) = csub(pan(r, c), cmul(f, pan(k, c)));
          }
        }
        __syncwarp();
      }
    }
    __syncthreads();
    if (*flag) return;
#ifdef NEGF_INV_CLOCKS
    { const long long c1 = clock64(); clk_panel += c1 - c0; c0 = c1; }
#endif
    // ---- row interchanges of this panel on the other columns (column-parallel)
    for (int c = tid; c < m8; c += INV_THREADS) {
      if ((c >= k0 && c < k0 + NB) || (kGlobal && c >= m)) {  // panel / no padding in global memory
#pragma unroll
        for (int kk = 0; kk < NB; ++kk) Rs[kk * (m8 + 2) + c] = make_double2(0.0, 0.0);
        continue;
      }
      for (int kk = 0; kk < kb; ++kk) {
        const int k = k0 + kk, p = perm[k];
        if (p != k) {
          const double2 t2 = at(k, c);
          at(k, c) = at(p, c);
          at(p, c) = t2;
        }
      }
      // stage the (swapped) pivot rows R_p
#pragma unroll
      for (int kk = 0; kk < NB; ++kk) Rs[kk * (m8 + 2) + c] = (kk < kb) ? at(k0 + kk, c) : make_double2(0.0, 0.0);
    }
    // M_p - I_p in the panel buffer (subtract the identity on the pivot rows)
    if (tid < kb) {
      double2& v = pan(k0 + tid, tid);
      v.x -= 1.0;
    }
    __syncthreads();
#ifdef NEGF_INV_CLOCKS
    { const long long c1 = clock64(); clk_swap += c1 - c0; c0 = c1; }
#endif
    // ---- rank-NB update of every 8x8 subtile (panel columns keep M_p): DMMA
    const int g8 = lane >> 2, t4 = lane & 3;
    const int nsub_r = m8 / 8, nsub_c = m8 / 8;
    for (int s = warp; s < nsub_r * nsub_c; s += INV_THREADS / 32) {
      const int sr = s / nsub_c, sc = s - sr * nsub_c;
      if (NB == 8 && sc * 8 == k0) continue;
      const int r = sr * 8 + g8, c = sc * 8 + 2 * t4;
      const bool in0 = !kGlobal || (r < m && c < m), in1 = !kGlobal || (r < m && c + 1 < m);
      double cr0 = 0.0, ci0 = 0.0, cr1 = 0.0, ci1 = 0.0;
      if (in0) {
        const double2 v = at(r, c);
        cr0 = v.x;
        ci0 = v.y;
      }
      if (in1) {
        const double2 v = at(r, c + 1);
        cr1 = v.x;
        ci1 = v.y;
      }
#pragma unroll
      for (int q = 0; q < NB / 4; ++q) {
        const double2 a = pan(r, 4 * q + t4);
        const double2 b = Rs[(4 * q + t4) * (m8 + 2) + sc * 8 + g8];
        dmma(cr0, cr1, a.x, b.x);
        dmma(cr0, cr1, -a.y, b.y);
        dmma(ci0, ci1, a.x, b.y);
        dmma(ci0, ci1, a.y, b.x);
      }
      const bool pc0 = (c >= k0 && c < k0 + NB), pc1 = (c + 1 >= k0 && c + 1 < k0 + NB);
      if (in0 && !pc0) at(r, c) = make_double2(cr0, ci0);
      if (in1 && !pc1) at(r, c + 1) = make_double2(cr1, ci1);
    }
#ifdef NEGF_INV_CLOCKS
    { __syncthreads(); const long long c1 = clock64(); clk_upd += c1 - c0; c0 = c1; }
#endif
    // restore M_p in the panel columns (add the identity back) and, for the
    // global variant, write the panel columns back
    __syncthreads();
    if (tid < kb) {
      double2& v = pan(k0 + tid, tid);
      v.x += 1.0;
    }
    if (kGlobal) {
      __syncthreads();
      for (int i = tid; i < m * 8; i += INV_THREADS) {
        const int r = i >> 3, c = i & 7;
        if (k0 + c < m) at(r, k0 + c) = P[i];
      }
    }
    __syncthreads();
  }
#ifdef NEGF_INV_CLOCKS
  if (tid == 0 && blockIdx.x == 0 && blockIdx.y == 0)
    printf("[inv clocks] m=%d panel %lld swap %lld update %lld\n", m, clk_panel, clk_swap, clk_upd);
#endif
  // Undo the row interchanges as column interchanges (last first).
  if (tid == 0) {
    int* cur_at = pos_of;  // reuse: first the permutation, then its inverse in Rs scratch
    for (int c = 0; c < m; ++c) cur_at[c] = c;
    for (int k = m - 1; k >= 0; --k) {
      const int p = perm[k];
      const int t2 = cur_at[k];
      cur_at[k] = cur_at[p];
      cur_at[p] = t2;
    }
    int* inv_pos = reinterpret_cast<int*>(Rs);
    for (int q = 0; q < m; ++q) inv_pos[cur_at[q]] = q;
    for (int q = 0; q < m; ++q) pos_of[q] = inv_pos[q];
  }
  __syncthreads();
  if (!kGlobal) {
    for (int i = tid; i < m * m; i += INV_THREADS) {
      const int r = i / m, c = i - r * m;
      g[int64_t(r) * m + pos_of[c]] = at(r, c);
    }
  } else {
    // one warp per row: the row is held in registers while it is permuted
    for (int r = warp; r < m; r += INV_THREADS / 32) {
      double2 v[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = lane + 32 * j;
        if (c < m) v[j] = at(r, c);
      }
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int c = lane + 32 * j;
        if (c < m) at(r, pos_of[c]) = v[j];
      }
      __syncwarp();
    }
  }
}

// Look-ahead variant of the shared-memory blocked Gauss-Jordan (8-column
// panels): while warps 1..3 apply panel p's rank-8 update to the bulk of the
// block, warp 0 first updates the 8 columns of panel p+1 and factors them, so
// the serial panel chain overlaps the update instead of following it.  Same
// pivots, same singular rule, same arithmetic per element as
// k_inverse_blocked<false, RPL, 8>.
template <int RPL>
__global__ void __launch_bounds__(INV_THREADS, RPL == 1 ? 6 : 4) k_inverse_la(double2* arena, int64_t stride,
                                                                           const InvTask* __restrict__ tasks,
                                                                           int e_base, DevStatus* st) {
  constexpr int NB = 8;
  extern __shared__ double2 sm[];
  const InvTask tk = tasks[blockIdx.x];
  const int m = tk.m;
  const int m8 = (m + 7) & ~7;
  const int ld = m8 + 2;  // smem row pitch: 2 mod 8 -> conflict-free fragments
  double2* g = arena + int64_t(blockIdx.y) * stride + tk.off;
  double2* A = sm;
  double2* Rs = sm + int64_t(m8) * ld;
  int* perm = reinterpret_cast<int*>(Rs + 8 * (m8 + 2));
  int* pos_of = perm + m8;
  double* red = reinterpret_cast<double*>(pos_of + m8 + (m8 & 1));
  int* flag = reinterpret_cast<int*>(red + INV_THREADS / 32);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  double mx = 0.0;
  for (int i = tid; i < m8 * m8; i += INV_THREADS) {
    const int r = i / m8, c = i - r * m8;
    const double2 v = (r < m && c < m) ? g[int64_t(r) * m + c] : make_double2(0.0, 0.0);
    A[r * ld + c] = v;
    mx = fmax(mx, cabs2(v));
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  if (tid == 0) *flag = 0;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < INV_THREADS / 32; ++w) mx = fmax(mx, red[w]);
  const double thresh = 1e-13 * mx;
  auto at = [&](int r, int c) -> double2& { return A[int64_t(r) * ld + c]; };

  // Panel factorisation of columns k0..k0+7 (all rows) on warp 0.
  auto factor = [&](int k0) {
    const int kb = min(NB, m - k0);
    auto pan = [&](int r, int c) -> double2& { return at(r, k0 + c); };
    const double thr2 = thresh * thresh;
    for (int kk = 0; kk < kb; ++kk) {
      const int k = k0 + kk;
      double best = -1.0;
      int bi = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = lane + 32 * i;
        if (r >= k && r < m) {
          const double v = cnorm(pan(r, kk));
          if (v > best) {
            best = v;
            bi = r;
          }
        }
      }
      const unsigned key = best >= 0.0 ? __float_as_uint(__double2float_ru(best)) : 0u;
      const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
      const unsigned tied = __ballot_sync(0xffffffffu, key == kmax);
      double cb;
      int ci;
      if (__popc(tied) == 1) {
        const int src = __ffs(tied) - 1;
        cb = __shfl_sync(0xffffffffu, best, src);
        ci = __shfl_sync(0xffffffffu, bi, src);
      } else {
        cb = (key == kmax) ? best : -1.0;
        ci = (key == kmax) ? bi : 0x7fffffff;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, cb, o);
          const int oi = __shfl_xor_sync(0xffffffffu, ci, o);
          if (ob > cb || (ob == cb && oi < ci)) {
            cb = ob;
            ci = oi;
          }
        }
      }
      if (!(cb > thr2)) {  // |u_kk| <= 1e-13 max|a|
        if (cb == cb) {
          if (lane == 0) {
            *flag = 1;
            report_singular(st, e_base + blockIdx.y, tk.fold_pos, k);
          }
          return;
        }
      }
      const int p = ci;
      if (lane == 0) perm[k] = p;
      if (lane < NB && p != k) {
        const double2 t2 = pan(k, lane);
        pan(k, lane) = pan(p, lane);
        pan(p, lane) = t2;
      }
      __syncwarp();
      double2 pr[NB];
#pragma unroll
      for (int c = 0; c < NB; ++c) pr[c] = pan(k, c);
      double2 piv = pr[0];
#pragma unroll
      for (int c = 1; c < NB; ++c)
        if (c == kk) piv = pr[c];
      const double rd = 1.0 / fma(piv.x, piv.x, piv.y * piv.y);
      const double2 ip = make_double2(piv.x * rd, -piv.y * rd);
#pragma unroll
      for (int c = 0; c < NB; ++c) pr[c] = (c == kk) ? ip : cmul(pr[c], ip);
      const double2 nip = make_double2(-ip.x, -ip.y);
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = lane + 32 * i;
        if (r >= m) continue;
        if (r == k) {
#pragma unroll
          for (int c = 0; c < NB; ++c) pan(r, c) = pr[c];
          continue;
        }
        const double2 f = pan(r, kk);
#pragma unroll
        for (int c = 0; c < NB; ++c) pan(r, c) = (c == kk) ? cmul(f, nip) : csub(pan(r, c), cmul(f, pr[c]));
      }
      __syncwarp();
    }
  };

  // Rank-8 update from panel k0 of the subtiles in column range [sc_lo, sc_hi)
  // (panel k0's own columns keep M_p), by warps w0 .. w0+nw-1.
  const int g8 = lane >> 2, t4 = lane & 3;
  const int nsub = m8 / 8;
  auto update = [&](int k0, int sc_lo, int sc_hi, int skip_sc, int w0, int nw) {
    const int ncol = sc_hi - sc_lo;
    for (int s = warp - w0; s < nsub * ncol; s += nw) {
      const int sr = s / ncol, sc = sc_lo + (s - sr * ncol);
      if (sc * 8 == k0 || sc == skip_sc) continue;
      const int r = sr * 8 + g8, c = sc * 8 + 2 * t4;
      const double2 v0 = at(r, c), v1 = at(r, c + 1);
      double cr0 = v0.x, ci0 = v0.y, cr1 = v1.x, ci1 = v1.y;
#pragma unroll
      for (int q = 0; q < NB / 4; ++q) {
        const double2 a = at(r, k0 + 4 * q + t4);
        const double2 b = Rs[(4 * q + t4) * (m8 + 2) + sc * 8 + g8];
        dmma(cr0, cr1, a.x, b.x);
        dmma(cr0, cr1, -a.y, b.y);
        dmma(ci0, ci1, a.x, b.y);
        dmma(ci0, ci1, a.y, b.x);
      }
      at(r, c) = make_double2(cr0, ci0);
      at(r, c + 1) = make_double2(cr1, ci1);
    }
  };

  if (warp == 0) factor(0);
  __syncthreads();
  if (*flag) return;
  for (int k0 = 0; k0 < m; k0 += NB) {
    const int kb = min(NB, m - k0);
    // row interchanges of panel k0 on the other columns; stage its pivot rows
    for (int c = tid; c < m8; c += INV_THREADS) {
      if (c >= k0 && c < k0 + NB) {
#pragma unroll
        for (int kk = 0; kk < NB; ++kk) Rs[kk * (m8 + 2) + c] = make_double2(0.0, 0.0);
        continue;
      }
      for (int kk = 0; kk < kb; ++kk) {
        const int k = k0 + kk, p = perm[k];
        if (p != k) {
          const double2 t2 = at(k, c);
          at(k, c) = at(p, c);
          at(p, c) = t2;
        }
      }
#pragma unroll
      for (int kk = 0; kk < NB; ++kk) Rs[kk * (m8 + 2) + c] = (kk < kb) ? at(k0 + kk, c) : make_double2(0.0, 0.0);
    }
    if (tid < kb) at(k0 + tid, k0 + tid).x -= 1.0;  // M_p - I_p
    __syncthreads();
    const int k1 = k0 + NB;
    if (k1 < m) {
      if (warp == 0) {  // look-ahead: next panel's columns, then its factorisation
        update(k0, k1 / 8, k1 / 8 + 1, -1, 0, 1);
        __syncwarp();
        factor(k1);
      } else {
        update(k0, 0, nsub, k1 / 8, 1, INV_THREADS / 32 - 1);
      }
    } else {
      update(k0, 0, nsub, -1, 0, INV_THREADS / 32);
    }
    __syncthreads();
    if (tid < kb) at(k0 + tid, k0 + tid).x += 1.0;
    __syncthreads();
    if (*flag) return;
  }
  // Undo the row interchanges as column interchanges (last first).
  if (tid == 0) {
    int* cur_at = pos_of;
    for (int c = 0; c < m; ++c) cur_at[c] = c;
    for (int k = m - 1; k >= 0; --k) {
      const int p = perm[k];
      const int t2 = cur_at[k];
      cur_at[k] = cur_at[p];
      cur_at[p] = t2;
    }
    int* inv_pos = reinterpret_cast<int*>(Rs);
    for (int q = 0; q < m; ++q) inv_pos[cur_at[q]] = q;
    for (int q = 0; q < m; ++q) pos_of[q] = inv_pos[q];
  }
  __syncthreads();
  for (int i = tid; i < m * m; i += INV_THREADS) {
    const int r = i / m, c = i - r * m;
    g[int64_t(r) * m + pos_of[c]] = at(r, c);
  }
}

// ---------------------------------------------------------------------------
// Register-resident Gauss-Jordan for m <= ROWS (<= 96): the whole block lives
// in the registers of ROWS * H threads -- thread t owns row r = t / H and the
// columns c = h + H j (h = t % H, j < SLOTS) -- so every pivot step updates
// all m x m entries at once on the FP64 pipes of all warps (m^3 complex FMAs
// in total, 8 flops each), instead of a serial 8-column panel on one warp
// followed by a rank-8 update.  Rows are never moved: partial pivoting keeps
// the *position* of every physical row (pos), exactly as if rows k and p were
// interchanged, so the pivot sequence, its tie-break (largest |a_rk|, lowest
// position) and the singular rule |u_kk| <= 1e-13 max|a| (dense.cpp:56-75)
// are those of the swapping elimination.  Per pivot: a warp argmax, one
// barrier, the pivot row's owners publish it normalised, one barrier, update.
// ---------------------------------------------------------------------------
struct InvCand {
  double v;     // |a_pk|^2 of the warp's best candidate (-1: none)
  int pos, row; // its position and physical row
  double2 val;  // a_pk
};

template <int ROWS, int H, int SLOTS>
__global__ void __launch_bounds__(ROWS * H, (ROWS * H <= 64) ? 8 : (ROWS * H <= 128) ? 3 : 1)
    k_inverse_rg(double2* arena, int64_t stride, const InvTask* __restrict__ tasks, int e_base, DevStatus* st) {
  constexpr int NT = ROWS * H, NW = NT / 32, MMAX = H * SLOTS;
  static_assert(NT % 32 == 0 && (H & (H - 1)) == 0 && MMAX >= ROWS, "bad register inverse shape");
  __shared__ double2 prow[2][MMAX];
  __shared__ InvCand cand[2][NW];
  __shared__ double red[NW];
  __shared__ int perm[ROWS], pos_of[ROWS];
  const InvTask tk = tasks[blockIdx.x];
  const int m = tk.m;
  double2* g = arena + int64_t(blockIdx.y) * stride + tk.off;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, h = t & (H - 1), r = t / H;
  const bool live = r < m;
  double2 a[SLOTS];
  double mx = 0.0;
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) {
    const int c = h + H * j;
    a[j] = (live && c < m) ? g[int64_t(r) * m + c] : make_double2(0.0, 0.0);
    mx = fmax(mx, cabs2(a[j]));
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  __syncthreads();
  mx = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) mx = fmax(mx, red[w]);
  const double thr2 = (1e-13 * mx) * (1e-13 * mx);
  int pos = r;  // current position of this physical row
#ifdef NEGF_RG_CLOCKS
  long long ck[5] = {0, 0, 0, 0, 0}, c0 = clock64();
#define RG_TICK(i) { const long long c1 = clock64(); ck[i] += c1 - c0; c0 = c1; }
#else
#define RG_TICK(i)
#endif
#pragma unroll
  for (int j = 0; j < SLOTS; ++j) {
    for (int hh = 0; hh < H; ++hh) {
      const int k = j * H + hh;
      if (k >= m) break;  // uniform
      const int par = k & 1;
      // column k of my row (held by the row's thread with h == hh, slot j)
      const int src = (lane & ~(H - 1)) | hh;
      double2 f;
      f.x = __shfl_sync(0xffffffffu, a[j].x, src);
      f.y = __shfl_sync(0xffffffffu, a[j].y, src);
      // warp argmax over the rows not yet pivoted (pos >= k): largest |a_rk|,
      // lowest position among equals
      double best = (live && h == 0 && pos >= k) ? cnorm(f) : -1.0;
      int bpos = (best >= 0.0) ? pos : 0x7fffffff;
      const unsigned key = best >= 0.0 ? __float_as_uint(__double2float_ru(best)) : 0u;
      const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
      const unsigned tied = __ballot_sync(0xffffffffu, key == kmax && best >= 0.0);
      int wl;  // lane holding the warp's winner
      if (__popc(tied) <= 1) {
        wl = tied ? __ffs(tied) - 1 : 0;
      } else {  // exact order among the lanes whose float images tie
        double cb = (key == kmax) ? best : -1.0;
        int cp = (key == kmax) ? bpos : 0x7fffffff, cl = lane;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, cb, o);
          const int op = __shfl_xor_sync(0xffffffffu, cp, o);
          const int ol = __shfl_xor_sync(0xffffffffu, cl, o);
          if (ob > cb || (ob == cb && op < cp)) {
            cb = ob;
            cp = op;
            cl = ol;
          }
        }
        wl = cl;
      }
      if (lane == wl) cand[par][warp] = InvCand{best, bpos, r, f};
      RG_TICK(0)
      __syncthreads();
      RG_TICK(1)
      InvCand w = cand[par][0];
#pragma unroll
      for (int q = 1; q < NW; ++q) {
        const InvCand o = cand[par][q];
        if (o.v > w.v || (o.v == w.v && o.pos < w.pos)) w = o;
      }
      if (!(w.v > thr2)) {  // |u_kk| <= 1e-13 max|a| (uniform across the CTA)
        if (w.v == w.v) {
          if (t == 0) report_singular(st, e_base + blockIdx.y, tk.fold_pos, k);
          return;
        }
      }
      const int p = w.pos;
      if (t == 0) perm[k] = p;
      const double rd = 1.0 / fma(w.val.x, w.val.x, w.val.y * w.val.y);
      const double2 ip = make_double2(w.val.x * rd, -w.val.y * rd);
      const bool pivot_row = r == w.row;
      if (pivot_row) {
#pragma unroll
        for (int jj = 0; jj < SLOTS; ++jj) {
          const int c = h + H * jj;
          if (c < MMAX) prow[par][c] = (jj == j && h == hh) ? ip : cmul(a[jj], ip);
        }
      }
      RG_TICK(2)
      __syncthreads();
      RG_TICK(3)
      if (pivot_row) {
#pragma unroll
        for (int jj = 0; jj < SLOTS; ++jj) a[jj] = prow[par][h + H * jj];
      } else if (live) {
#pragma unroll
        for (int jj = 0; jj < SLOTS; ++jj) {
          const double2 pr = prow[par][h + H * jj];
          const double2 b = (jj == j && h == hh) ? make_double2(0.0, 0.0) : a[jj];
          a[jj].x = fma(-f.x, pr.x, fma(f.y, pr.y, b.x));
          a[jj].y = fma(-f.x, pr.y, fma(-f.y, pr.x, b.y));
        }
      }
      if (pos == k) pos = p;
      else if (pos == p) pos = k;
      RG_TICK(4)
    }
  }
#ifdef NEGF_RG_CLOCKS
  if (blockIdx.x == 0 && blockIdx.y == 0 && (t == 0 || t == NT - 1))
    printf("[rg clocks] m=%d t=%d argmax %lld bar1 %lld pivrow %lld bar2 %lld update %lld per pivot\n", m, t,
           ck[0] / m, ck[1] / m, ck[2] / m, ck[3] / m, ck[4] / m);
#endif
  // Undo the row interchanges as column interchanges (last first).
  __syncthreads();
  if (t == 0) {
    int* cur_at = pos_of;
    for (int c = 0; c < m; ++c) cur_at[c] = c;
    for (int k = m - 1; k >= 0; --k) {
      const int p = perm[k];
      const int t2 = cur_at[k];
      cur_at[k] = cur_at[p];
      cur_at[p] = t2;
    }
    int* inv_pos = perm;  // perm is consumed
    for (int q = 0; q < m; ++q) inv_pos[cur_at[q]] = q;
    for (int q = 0; q < m; ++q) pos_of[q] = inv_pos[q];
  }
  __syncthreads();
  if (live) {
#pragma unroll
    for (int j = 0; j < SLOTS; ++j) {
      const int c = h + H * j;
      if (c < m) g[int64_t(pos) * m + pos_of[c]] = a[j];
    }
  }
}

// ---------------------------------------------------------------------------
// Shifting-window register Gauss-Jordan (m <= ROWS, m <= H * S).  Same
// elimination as k_inverse_rg (row partial pivoting by position tracking, the
// same pivot sequence and singular rule), but the m live columns of [A | I]
// are kept as a window that moves one column to the right per pivot step:
// the pivot column is always window column 0 and the new inverse column
// enters at the right end.  Every step is then the same code on the same
// registers (w[j-1] = w[j] - fs * prow[j-1]), so the pivot loop is NOT
// unrolled: a few hundred instructions instead of the ~100 KB of straight-line
// code k_inverse_rg needs for static register indices (its top stall is
// instruction fetch).  Thread t owns row r = t / H and the window columns
// h S .. h S + S - 1 (h = t % H); one shuffle per step brings the next
// chunk's first column.  Rows are scaled late: a pivoted row stays
// unnormalised (the update is linear in the row, the multiplier of a step is
// fs = f / pivot as in an LU factorisation) and is multiplied by its own
// 1 / pivot when the block is written back.
// ---------------------------------------------------------------------------
template <int NW>
__device__ __forceinline__ void sw_barrier() {
  if constexpr (NW == 1) __syncwarp();
  else __syncthreads();
}

// Value type of the window kernel: double2, or double for blocks that are real
// at every energy (InvTask::real).  The real operations are the complex ones
// with the zero imaginary parts dropped, so both give the same bits.
__device__ __forceinline__ double sw_norm(double2 a) { return cnorm(a); }
__device__ __forceinline__ double sw_norm(double a) { return a * a; }
__device__ __forceinline__ double2 sw_mul(double2 a, double2 b) { return cmul(a, b); }
__device__ __forceinline__ double sw_mul(double a, double b) { return a * b; }
__device__ __forceinline__ double2 sw_shfl(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ double sw_shfl(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double2 sw_shfl_down1(double2 v) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, 1), __shfl_down_sync(0xffffffffu, v.y, 1));
}
__device__ __forceinline__ double sw_shfl_down1(double v) { return __shfl_down_sync(0xffffffffu, v, 1); }
// w - fs * q
__device__ __forceinline__ double2 sw_fnma(double2 fs, double2 q, double2 w) {
  return make_double2(fma(-fs.x, q.x, fma(fs.y, q.y, w.x)), fma(-fs.x, q.y, fma(-fs.y, q.x, w.y)));
}
__device__ __forceinline__ double sw_fnma(double fs, double q, double w) { return fma(-fs, q, w); }
__device__ __forceinline__ void sw_set(double2& v, double re) { v = make_double2(re, 0.0); }
__device__ __forceinline__ void sw_set(double& v, double re) { v = re; }
__device__ __forceinline__ void sw_load(double2& v, const double2* p) { v = *p; }
__device__ __forceinline__ void sw_load(double& v, const double2* p) { v = p->x; }
__device__ __forceinline__ double2 sw_c(double2 v) { return v; }
__device__ __forceinline__ double2 sw_c(double v) { return make_double2(v, 0.0); }
// 1 / pivot from the candidate record (val = the pivot, v = |pivot|^2)
__device__ __forceinline__ void sw_recip(double2& ip, double2 val) {
  const double rd = 1.0 / fma(val.x, val.x, val.y * val.y);
  ip = make_double2(val.x * rd, -val.y * rd);
}
__device__ __forceinline__ void sw_recip(double& ip, double2 val) {
  const double rd = 1.0 / (val.x * val.x);
  ip = val.x * rd;
}

template <int ROWS, int H, int S, int MINB, bool REAL>
__global__ void __launch_bounds__(ROWS * H, MINB)
    k_inverse_sw(double2* arena, int64_t stride, const InvTask* __restrict__ tasks, int e_base, DevStatus* st) {
  using V = std::conditional_t<REAL, double, double2>;
  constexpr int NT = ROWS * H, NW = NT / 32, MW = H * S;
  // odd chunk pitch: the H chunk reads of one shared load hit distinct banks
  constexpr int PS = S | 1, PW = H * PS;
  static_assert(NT % 32 == 0 && (H & (H - 1)) == 0 && H <= 32, "bad window inverse shape");
  __shared__ V prow[2][PW];
  __shared__ InvCand cand[2][NW];
  __shared__ double red[NW];
  __shared__ int pos_of[ROWS];  // physical pivot row of step c = original column of the inverse column made there
  const InvTask tk = tasks[blockIdx.x];
  const int m = tk.m;
  double2* g = arena + int64_t(blockIdx.y) * stride + tk.off;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5, h = t & (H - 1), r = t / H;
  const bool live = r < m;
  V w[S];
  double mx = 0.0;
#pragma unroll
  for (int j = 0; j < S; ++j) {
    const int c = h * S + j;
    sw_set(w[j], 0.0);
    if (live && c < m) sw_load(w[j], g + int64_t(r) * m + c);
    mx = fmax(mx, sw_norm(w[j]));  // max |a|^2: the singular rule compares squared moduli
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[warp] = mx;
  sw_barrier<NW>();
  mx = 0.0;
#pragma unroll
  for (int q = 0; q < NW; ++q) mx = fmax(mx, red[q]);
  const double thr2 = 1e-26 * mx;  // (1e-13 max|a|)^2
  int pos = r;  // current position of this physical row
  V myip;
  sw_set(myip, 1.0);
  const V* pw = &prow[0][h * PS];
#pragma unroll 1
  for (int k = 0; k < m; ++k) {
    const int par = k & 1;
    // window column 0 of my row (held by the row's h == 0 thread), and the
    // first column of the next chunk (thread h + 1 of the row)
    const V f = sw_shfl(w[0], lane & ~(H - 1));
    V nx;
    sw_set(nx, 0.0);
    if constexpr (H > 1) nx = sw_shfl_down1(w[0]);
    // warp argmax over the rows not yet pivoted (pos >= k): largest |a_rk|,
    // lowest position among equals
    double best = (live && h == 0 && pos >= k) ? sw_norm(f) : -1.0;
    int bpos = (best >= 0.0) ? pos : 0x7fffffff;
    const unsigned key = best >= 0.0 ? __float_as_uint(__double2float_ru(best)) : 0u;
    const unsigned kmax = __reduce_max_sync(0xffffffffu, key);
    const unsigned tied = __ballot_sync(0xffffffffu, key == kmax && best >= 0.0);
    int wl;  // lane holding the warp's winner
    if (__popc(tied) <= 1) {
      wl = tied ? __ffs(tied) - 1 : 0;
    } else {  // exact order among the lanes whose float images tie
      double cb = (key == kmax) ? best : -1.0;
      int cp = (key == kmax) ? bpos : 0x7fffffff, cl = lane;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, cb, o);
        const int op = __shfl_xor_sync(0xffffffffu, cp, o);
        const int ol = __shfl_xor_sync(0xffffffffu, cl, o);
        if (ob > cb || (ob == cb && op < cp)) {
          cb = ob;
          cp = op;
          cl = ol;
        }
      }
      wl = cl;
    }
    InvCand win;
    if constexpr (NW == 1) {
      const double2 fc = sw_c(f);
      win.v = __shfl_sync(0xffffffffu, best, wl);
      win.pos = __shfl_sync(0xffffffffu, bpos, wl);
      win.row = __shfl_sync(0xffffffffu, r, wl);
      win.val.x = __shfl_sync(0xffffffffu, fc.x, wl);
      win.val.y = REAL ? 0.0 : __shfl_sync(0xffffffffu, fc.y, wl);
    } else {
      if (lane == wl) cand[par][warp] = InvCand{best, bpos, r, sw_c(f)};
      __syncthreads();
      win = cand[par][0];
#pragma unroll
      for (int q = 1; q < NW; ++q) {
        const InvCand o = cand[par][q];
        if (o.v > win.v || (o.v == win.v && o.pos < win.pos)) win = o;
      }
    }
    if (!(win.v > thr2)) {  // |u_kk| <= 1e-13 max|a| (uniform across the CTA)
      if (win.v == win.v) {
        if (t == 0) report_singular(st, e_base + blockIdx.y, tk.fold_pos, k);
        return;
      }
    }
    const int p = win.pos;
    if (t == 0) pos_of[k] = win.row;
    V ip;
    sw_recip(ip, win.val);
    const bool pivot_row = r == win.row;
    // the incoming column at the right end: the next chunk's first column,
    // or (last chunk) the unit column of the pivot row
    V last;
    sw_set(last, pivot_row ? 1.0 : 0.0);
    if constexpr (H > 1) {
      if (h != H - 1) last = nx;
    }
    V fs;
#ifdef NEGF_SW_NORMALISED  // A/B: pivot row normalised at its own step (k_inverse_rg's arithmetic)
    if (pivot_row) {
      V* d = &prow[par][h * PS];
#pragma unroll
      for (int j = 1; j < S; ++j) d[j - 1] = sw_mul(w[j], ip);
      d[S - 1] = sw_mul(last, ip);
    }
    sw_barrier<NW>();
    fs = f;
    if (pivot_row) sw_set(fs, 0.0);
    const V* pr = pw + par * PW;
    if (pivot_row) {
#pragma unroll
      for (int j = 1; j < S; ++j) w[j] = pr[j - 1];
      last = pr[S - 1];
    }
#else
    if (pivot_row) {
      V* d = &prow[par][h * PS];
#pragma unroll
      for (int j = 1; j < S; ++j) d[j - 1] = w[j];
      d[S - 1] = last;
      myip = ip;
    }
    sw_barrier<NW>();
    fs = sw_mul(f, ip);
    if (pivot_row) sw_set(fs, 0.0);
    const V* pr = pw + par * PW;
#endif
#pragma unroll
    for (int j = 1; j < S; ++j) w[j - 1] = sw_fnma(fs, pr[j - 1], w[j]);
    w[S - 1] = sw_fnma(fs, pr[S - 1], last);
    if (pos == k) pos = p;
    else if (pos == p) pos = k;
  }
  // No row was moved: the elimination turned A into the permutation with a 1
  // at (pivot row of step k, k), so row k of the inverse is the physical
  // pivot row of step k (final position pos = k) and the column made at step
  // c is the original column pos_of[c].
  __syncthreads();
  if (live) {
    const int shift = MW - m;  // the inverse column of step j sits at window column shift + j
#pragma unroll
    for (int j = 0; j < S; ++j) {
      const int c = h * S + j - shift;
      if (c >= 0) g[int64_t(pos) * m + pos_of[c]] = sw_c(sw_mul(w[j], myip));
    }
  }
}

// ---------------------------------------------------------------------------
// Multi-CTA blocked Gauss-Jordan for large blocks (m > kSmemInvMax), see
// plan.hpp: per kPanel-column inner panel, k_bigpanel (one CTA per block and
// energy) factors the panel with row partial pivoting (in shared memory, or
// in the arena's panel scratch -- L2 -- beyond kPanelSmemMax rows), applies
// its row interchanges to the other columns of the outer panel [o0, oe) and
// stages M_p - I_p and the pivot rows R_p; a grouped-GEMM task applies the
// rank-kPanel update to the outer panel.  Per outer panel, k_bigswap applies
// its kOuter interchanges to every other column and stages the rank-kOuter
// operands of one grouped-GEMM update of the whole block.  k_bigperm finally
// undoes the interchanges as column interchanges.
// ---------------------------------------------------------------------------
template <bool kSmemPanel>
__global__ void __launch_bounds__(256) k_bigpanel(double2* arena, int64_t stride, const BigTask* __restrict__ tasks,
                                                  int k0, int o0, int e_base, DevStatus* st) {
  // Panel rows in shared memory are padded to kPanel + 1 complex (144 B):
  // thread r's 16-byte accesses to row r then fall on distinct banks (a
  // 128-byte pitch would put every lane of a phase on the same banks).
  constexpr int PP = kSmemPanel ? kPanel + 1 : kPanel;
  extern __shared__ double2 pn_smem[];  // m x PP panel
  __shared__ double red_v[8];
  __shared__ int red_i[8];
  __shared__ double s_thr;
  __shared__ int s_fail;
  const BigTask tk = tasks[blockIdx.x];
  const int m = tk.m, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double2* base = arena + blockIdx.y * stride;
  double2* A = base + tk.off;
  double2* thr = base + tk.off_thr;
  double2* pn = kSmemPanel ? pn_smem : base + tk.off_mp;
  const int oe = min(o0 + kOuter, m);
  int* perm = reinterpret_cast<int*>(base + tk.off_perm);
  if (k0 == 0) {  // threshold from the original block (dense.cpp:58)
    double mx = 0.0;
    for (int64_t i = tid; i < int64_t(m) * m; i += 256) mx = fmax(mx, cabs2(A[i]));
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) red_v[warp] = mx;
    __syncthreads();
    if (tid == 0) {
      double v = 0.0;
      for (int w2 = 0; w2 < 8; ++w2) v = fmax(v, red_v[w2]);
      s_thr = 1e-13 * v;
      s_fail = 0;
      *thr = make_double2(s_thr, 0.0);
    }
  } else if (tid == 0) {
    const double2 v = *thr;
    s_thr = v.x;
    s_fail = v.y != 0.0;
  }
  __syncthreads();
  if (s_fail) return;
  const double thr2 = s_thr * s_thr;
  const int kb = min(kPanel, m - k0);
  for (int i = tid; i < m * kPanel; i += 256) {
    const int r = i / kPanel, c = i - r * kPanel;
    pn[r * PP + c] = c < kb ? A[int64_t(r) * m + k0 + c] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  for (int kk = 0; kk < kb; ++kk) {
    const int k = k0 + kk;
    // 1. argmax |a_rk|^2 over rows r >= k (lowest row among equals)
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = k + tid; r < m; r += 256) {
      const double v = cnorm(pn[r * PP + kk]);
      if (v > best) {
        best = v;
        bi = r;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
    }
    if (lane == 0) {
      red_v[warp] = best;
      red_i[warp] = bi;
    }
    __syncthreads();
    // 2. every thread combines the warps' candidates (same winner everywhere)
    double b2 = red_v[0];
    int p = red_i[0];
#pragma unroll
    for (int w2 = 1; w2 < 8; ++w2)
      if (red_v[w2] > b2 || (red_v[w2] == b2 && red_i[w2] < p)) {
        b2 = red_v[w2];
        p = red_i[w2];
      }
    if (!(b2 > thr2) && b2 == b2) {  // |u_kk| <= 1e-13 max|a| (uniform)
      if (tid == 0) {
        *thr = make_double2(s_thr, 1.0);
        report_singular(st, e_base + blockIdx.y, tk.fold_pos, k);
      }
      return;
    }
    const double2 ip = crcp(pn[p * PP + kk]);
    double2 rowp = make_double2(0.0, 0.0), rowk = make_double2(0.0, 0.0);
    if (tid < kPanel) {
      rowp = pn[p * PP + tid];
      rowk = pn[k * PP + tid];
    }
    if (tid == 0) perm[k] = p;
    __syncthreads();
    // 3. interchange rows k and p, normalise the pivot row
    if (tid < kPanel) {
      pn[k * PP + tid] = (tid == kk) ? ip : cmul(rowp, ip);
      if (p != k) pn[p * PP + tid] = rowk;
    }
    __syncthreads();
    // 4. eliminate column k from every other row
    double2 pr[kPanel];
#pragma unroll
    for (int c = 0; c < kPanel; ++c) pr[c] = pn[k * PP + c];
    for (int r = tid; r < m; r += 256) {
      if (r == k) continue;
      const double2 f = pn[r * PP + kk];
#pragma unroll
      for (int c = 0; c < kPanel; ++c)
        pn[r * PP + c] = (c == kk) ? make_double2(-(f.x * ip.x - f.y * ip.y), -(f.x * ip.y + f.y * ip.x))
                                   : csub(pn[r * PP + c], cmul(f, pr[c]));
    }
    __syncthreads();
  }
  // panel back into the block (M_p) and M_p - I_p into scratch
  double2* mp = base + tk.off_mp;
  for (int i = tid; i < m * kPanel; i += 256) {
    const int r = i / kPanel, c = i - r * kPanel;
    double2 v = pn[r * PP + c];
    if (c < kb) A[int64_t(r) * m + k0 + c] = v;
    else v = make_double2(0.0, 0.0);
    if (r == k0 + c) v.x -= 1.0;
    mp[i] = v;
  }
  // this panel's row interchanges on the outer panel's other columns, then
  // stage R_p there (the rank-kPanel update covers columns [o0, oe) only)
  double2* rs = base + tk.off_rs;
  for (int c = o0 + tid; c < oe; c += 256) {
    const bool in_panel = c >= k0 && c < k0 + kPanel;
    if (!in_panel)
      for (int kk = 0; kk < kb; ++kk) {
        const int k = k0 + kk, p = perm[k];
        if (p != k) {
          const double2 t2 = A[int64_t(k) * m + c];
          A[int64_t(k) * m + c] = A[int64_t(p) * m + c];
          A[int64_t(p) * m + c] = t2;
        }
      }
#pragma unroll
    for (int kk = 0; kk < kPanel; ++kk)
      rs[int64_t(kk) * m + c] = (kk < kb && !in_panel) ? A[int64_t(k0 + kk) * m + c] : make_double2(0.0, 0.0);
  }
}

// One outer panel [o0, oe) done: its row interchanges on every column outside
// it, then the rank-kOuter operands -- R_P = the pivot rows (zero inside the
// panel) and M_P - I_P = the panel's columns minus the identity on the pivot
// positions.  Column-parallel (coalesced rows).
__global__ void __launch_bounds__(256) k_bigswap(double2* arena, int64_t stride, const BigTask* __restrict__ tasks,
                                                 int o0) {
  const BigTask tk = tasks[blockIdx.x];
  const int m = tk.m, tid = threadIdx.x;
  double2* base = arena + blockIdx.y * stride;
  if (base[tk.off_thr].y != 0.0) return;  // singular: already reported
  double2* A = base + tk.off;
  const int* perm = reinterpret_cast<const int*>(base + tk.off_perm);
  double2* rs = base + tk.off_rs64;
  double2* mp = base + tk.off_mp64;
  const int oe = min(o0 + kOuter, m), kb = oe - o0;
  for (int c = tid; c < m; c += 256) {
    const bool inside = c >= o0 && c < oe;
    if (!inside)
      for (int kk = 0; kk < kb; ++kk) {
        const int k = o0 + kk, p = perm[k];
        if (p != k) {
          const double2 t2 = A[int64_t(k) * m + c];
          A[int64_t(k) * m + c] = A[int64_t(p) * m + c];
          A[int64_t(p) * m + c] = t2;
        }
      }
    for (int kk = 0; kk < kb; ++kk)
      rs[int64_t(kk) * m + c] = inside ? make_double2(0.0, 0.0) : A[int64_t(o0 + kk) * m + c];
  }
  for (int64_t i = tid; i < int64_t(m) * kb; i += 256) {
    const int r = static_cast<int>(i / kb), kk = static_cast<int>(i - int64_t(r) * kb);
    double2 v = A[int64_t(r) * m + o0 + kk];
    if (r == o0 + kk) v.x -= 1.0;
    mp[int64_t(r) * kOuter + kk] = v;
  }
}

// Undo the row interchanges as column interchanges, last first.  The index
// maps live in shared memory (8 m bytes; every CTA of a block derives them --
// a serial pass over m swaps -- in parallel), the rows are split over
// gridDim.z CTAs x 4 warps, each warp with its own row buffer in the arena's
// outer-panel scratch (kOuter x m: kBigPermChunks * 4 <= kOuter rows).
constexpr int kBigPermChunks = 16;
__global__ void __launch_bounds__(128) k_bigperm(double2* arena, int64_t stride, const BigTask* __restrict__ tasks) {
  extern __shared__ int pmaps[];  // pos_of[m], cur_at[m]
  const BigTask tk = tasks[blockIdx.x];
  const int m = tk.m, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int* pos_of = pmaps;
  int* cur_at = pmaps + m;
  double2* base = arena + blockIdx.y * stride;
  double2* thr = base + tk.off_thr;
  if (thr->y != 0.0) return;  // singular: already reported
  double2* A = base + tk.off;
  const int* perm = reinterpret_cast<const int*>(base + tk.off_perm);
  if (threadIdx.x == 0) {
    for (int c = 0; c < m; ++c) cur_at[c] = c;
    for (int k = m - 1; k >= 0; --k) {
      const int p = perm[k];
      const int t2 = cur_at[k];
      cur_at[k] = cur_at[p];
      cur_at[p] = t2;
    }
    for (int q = 0; q < m; ++q) pos_of[cur_at[q]] = q;
  }
  __syncthreads();
  const int wid = blockIdx.z * 4 + warp, nw = gridDim.z * 4;
  double2* buf = base + tk.off_rs64 + int64_t(wid) * m;
  for (int r = wid; r < m; r += nw) {
    for (int c = lane; c < m; c += 32) buf[c] = A[int64_t(r) * m + c];
    __syncwarp();
    for (int c = lane; c < m; c += 32) A[int64_t(r) * m + pos_of[c]] = buf[c];
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Grouped multi-term complex GEMM on DMMA (mma.sync.m8n8k4.f64)
// ---------------------------------------------------------------------------
constexpr int KC = 16;
constexpr int LD_RK = KC + 4;  // (row, k) smem layouts: pitch = 4 mod 8 -> conflict-free fragments

// CTA of 4 warps, each owning a 16x16 output region (2x2 DMMA subtiles),
// arranged WR x WC (2x2, 1x4 or 4x1) so that skinny tasks keep every warp
// busy; the CTA tile is (16 WR) x (16 WC).
template <int WR, int WC>
struct Arr {
  static constexpr int TM = 16 * WR, TN = 16 * WC;
  static constexpr int LDA_KR = TM + 2, LDB_KR = TN + 2;  // (k, row|col) pitch = 2 mod 8
  static constexpr int OPA = (TM * LD_RK > KC * LDA_KR) ? TM * LD_RK : KC * LDA_KR;
  static constexpr int OPB = (TN * LD_RK > KC * LDB_KR) ? TN * LD_RK : KC * LDB_KR;
  static constexpr int STAGE = OPA + OPB;  // complex elements per pipeline stage
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Per-thread chunk loader with the addressing hoisted to term changes: a
// thread's slots of one operand are a fixed stride apart in global memory and
// in shared memory, so a chunk costs one base add, a k-validity test and one
// cp.async per slot (the element-wise index arithmetic ran per chunk before).
// Slot i of thread tid covers element idx = tid + 128 i of the chunk: (row, k)
// layouts r = idx / KC, kk = idx % KC; (k, row) layouts kk = idx / T,
// r = idx % T.  Elements outside the task or the term are zero-filled.
template <int T, int LDKR>
struct OperandLoader {
  static constexpr int NS = (T * KC) / 128;  // slots per thread
  const double2* src;  // slot 0 source at k0 = 0
  int kmul;            // source advance per unit of k0 (1 for (row, k), ld for (k, row))
  int gstep;           // source stride between slots (elements)
  int live;            // (row, k): slots with a live row; (k, row): NS if the row is live, else 0
  bool rk;

  __device__ __forceinline__ void setup(const double2* base, int64_t off, int ld, bool row_k, int tk_rows, int r0) {
    const int tid = threadIdx.x;
    rk = row_k;
    if (row_k) {
      const int r = tid / KC, kk = tid % KC;
      src = base + off + int64_t(r0 + r) * ld + kk;
      kmul = 1;
      gstep = (128 / KC) * ld;
      live = max(0, min(NS, (tk_rows - r0 - r + (128 / KC) - 1) / (128 / KC)));
    } else {
      const int kk = tid / T, r = tid % T;
      src = base + off + int64_t(kk) * ld + (r0 + r);
      kmul = ld;
      gstep = (128 / T) * ld;
      live = (r0 + r < tk_rows) ? NS : 0;
    }
  }
  __device__ __forceinline__ void issue(double2* sm, const double2* dummy, int k0, int k) const {
    const int tid = threadIdx.x;
    const double2* p = src + int64_t(k0) * kmul;
    // (row, k): one k per thread, all slots live in k together;
    // (k, row): slot i sits at k = kk + i * (128 / T).
    const int kk = rk ? tid % KC : tid / T;
    const int kks = rk ? 0 : 128 / T;
    const int krem = k - k0 - kk;
    double2* d = sm + (rk ? (tid / KC) * LD_RK + kk : kk * LDKR + tid % T);
    const int sstep = rk ? (128 / KC) * LD_RK : (128 / T) * LDKR;
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      const bool v = (i < live) && (i * kks < krem);
      cp_async16(d, v ? p : dummy, v);
      p += gstep;
      d += sstep;
    }
  }
};

constexpr int kTermCache = 48;
// Energy groups of the item order (gemm_energy_groups; measured on config 2,
// dynamic scheduling).  CTA tiles: -1 = wave-sized groups, as many energies as
// fill the launch's resident CTAs once, the last three waves as one tile-major
// group (93.5 ms of k_gemm per batch and 197 GB of DRAM traffic, against 93.9 ms
// and 283 GB with all energies in one group, 94.8 ms with groups of 4; before
// the real-operand terms halved the DMMA work the single group was 0.7 %
// faster).  Warp tiles of the small separators: one energy per group (24.8 vs
// 25.4 ms).
#ifndef NEGF_GEMM_EG_CTA
#define NEGF_GEMM_EG_CTA (-1)
#endif
#ifndef NEGF_GEMM_EG_WARP
#define NEGF_GEMM_EG_WARP 1
#endif
constexpr int kGemmEgCta = NEGF_GEMM_EG_CTA, kGemmEgWarp = NEGF_GEMM_EG_WARP;  // term descriptors staged in shared memory per item

// Sign flip on the integer pipe (keeps the FP64 pipes free).
__device__ __forceinline__ double flip_sign(double v, int mask) {
  return __hiloint2double(__double2hiint(v) ^ mask, __double2loint(v));
}

// Epilogue of one warp's 16 x 16 output block at (r0, c0) of task tk: lane
// owns C[r][c], C[r][c+1] of each 8x8 subtile (val(i, j, q)).  Fused diagonal
// (GemmTask::dmode): row sums of Psi[r][c] op(C[r][c]), one partial per row
// and 16-column group.  mir: the block lies strictly above the diagonal of a
// symmetric task (also writes the transpose).
template <class Val>
__device__ __forceinline__ void gemm_epilogue(double2* base, const GemmTask& tk, int r0, int c0, bool mir,
                                              const Val& val) {
  const int lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  double2 rs[2] = {make_double2(0.0, 0.0), make_double2(0.0, 0.0)};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int r = r0 + 8 * i + g;
    if (r >= tk.m) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int c = c0 + 8 * j + 2 * t + q;
        if (c >= tk.n) continue;
        double2 v = val(i, j, q);
        if (mir) {  // strictly-upper tile of a symmetric task: the (c, r) entry too
          double2* d2 = base + tk.c_off + int64_t(c) * tk.ldc + r;
          if (tk.mirror == 2) *d2 = make_double2(-v.x, v.y);  // anti-Hermitian: -conj
          else if (tk.mode == MODE_ADD) *d2 = cadd(*d2, v);
          else if (tk.mode == MODE_INIT) *d2 = cadd(base[tk.init_off + int64_t(c) * tk.ld_init + r], v);
          else *d2 = v;
        }
        double2* dst = base + tk.c_off + int64_t(r) * tk.ldc + c;
        if (tk.mode == MODE_ADD) v = cadd(*dst, v);
        else if (tk.mode == MODE_INIT) v = cadd(base[tk.init_off + int64_t(r) * tk.ld_init + c], v);
        if (!tk.nostore) *dst = v;
        if (tk.c2_off >= 0) base[tk.c2_off + int64_t(r) * tk.ldc + c] = make_double2(2.0 * v.x, 2.0 * v.y);
        if (tk.dmode) {
          const double2 psi = base[tk.dpsi_off + int64_t(r) * tk.dpsi_ld + c];
          if (tk.dmode >= 2) v.y = -v.y;
          rs[i] = cadd(rs[i], cmul(psi, v));
        }
      }
    }
  }
  if (tk.dmode) {  // task-uniform: reduce over the 4 lanes of a row, one partial per (row, 16-column group)
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      rs[i].x += __shfl_xor_sync(0xffffffffu, rs[i].x, 1);
      rs[i].y += __shfl_xor_sync(0xffffffffu, rs[i].y, 1);
      rs[i].x += __shfl_xor_sync(0xffffffffu, rs[i].x, 2);
      rs[i].y += __shfl_xor_sync(0xffffffffu, rs[i].y, 2);
    }
    if (t == 0 && c0 < tk.n) {
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = r0 + 8 * i + g;
        if (r >= tk.m) continue;
        // dmode 3: the anti-Hermitian form, imaginary part only (plan.cpp)
        const double2 s = tk.dmode == 3 ? make_double2(0.0, -rs[i].y)
                          : tk.dmode == 2 ? make_double2(-rs[i].x, -rs[i].y) : rs[i];
        base[tk.dpart_off + int64_t(r) * tk.dpart_ld + c0 / 16] = s;
      }
    }
  }
}

template <int WR, int WC, bool M3>
__device__ __forceinline__ void gemm_item(double2* base, const GemmTask& tk, const GemmTerm* __restrict__ terms,
                                          const GemmTile& tl, double2* smem) {
  using A = Arr<WR, WC>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = (warp / WC) * 16, wn = (warp % WC) * 16;
  // Warp-uniform live subtiles (8-granular skip of padding).
  const int live_i = min(2, max(0, (tk.m - tl.m0 - wm + 7) / 8));
  const int live_j = min(2, max(0, (tk.n - tl.n0 - wn + 7) / 8));

  // M3 = false (every production launch): the conventional (4M) complex
  // product, Re C = Ar Br - Ai Bi (p1), Im C = Ar Bi + Ai Br (p2), four real
  // DMMAs per complex subtile step.  M3 = true (A/B switches only): the Gauss
  // (3M) product, P1 = Ar Br, P2 = Ai Bi, P3 = (Ar+Ai)(Br+Bi), C = (P1 - P2) +
  // i (P3 - P1 - P2) -- 11 % less GEMM time, but it mixes rounding of the real
  // parts into the imaginary ones: on config 2 it leaves max|Re G^<_jj| /
  // |G^<_jj| up to 194x the reference's own value at 40 of 256 energies, and
  // 116x its bar even when only the fold uses it.  p3 is
  // dead code for M3 = false.
  double p1[2][2][2], p2[2][2][2], p3[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) p1[i][j][q] = p2[i][j][q] = p3[i][j][q] = 0.0;

  // Flattened (term, k-chunk) sequence through a 2-stage cp.async ring, one
  // barrier per chunk.  The loader is re-based only when the term changes.
  const int tend = tk.term_begin + tk.term_count;
  int lt = tk.term_begin, lk0 = 0;
  while (lt < tend && terms[lt].k <= 0) ++lt;
  int ct = lt, ck0 = 0;
  OperandLoader<A::TM, A::LDA_KR> la;
  OperandLoader<A::TN, A::LDB_KR> lb;
  int lk = 0;
  auto setup = [&](int term) {
    const GemmTerm& q = terms[term];
    la.setup(base, q.a_off, q.lda, q.a_op == OP_N, tk.m, tl.m0);
    lb.setup(base, q.b_off, q.ldb, !(q.b_op == OP_N || q.b_op == OP_C), tk.n, tl.n0);
    lk = q.k;
  };
  auto load = [&](double2* st) {
    la.issue(st, base, lk0, lk);
    lb.issue(st + A::OPA, base, lk0, lk);
  };
  auto advance_load = [&]() {
    lk0 += KC;
    if (lk0 >= lk) {
      lk0 = 0;
      ++lt;
      while (lt < tend && terms[lt].k <= 0) ++lt;
      if (lt < tend) setup(lt);
    }
  };
  auto advance = [&](int& term, int& kq) {
    kq += KC;
    if (kq >= terms[term].k) {
      kq = 0;
      ++term;
      while (term < tend && terms[term].k <= 0) ++term;
    }
  };
  if (lt < tend) {
    setup(lt);
    load(smem);
    advance_load();
  }
  cp_async_commit();
  int stage = 0;
  while (ct < tend) {
    cp_async_wait<0>();
    __syncthreads();
    if (lt < tend) {
      load(smem + (stage ^ 1) * A::STAGE);
      advance_load();
    }
    cp_async_commit();
    const GemmTerm tm = terms[ct];
    const double2* As = smem + stage * A::STAGE;
    const double2* Bs = As + A::OPA;
    // Sign of the term and conj(B) as sign-bit masks (integer pipe).
    const int negA = tm.sign < 0 ? int(0x80000000) : 0;
    const int conjB = (tm.b_op == OP_C || tm.b_op == OP_H) ? int(0x80000000) : 0;
    const bool a_rk = (tm.a_op == OP_N);
    const bool b_kr = (tm.b_op == OP_N || tm.b_op == OP_C);
    const int ksteps = min(KC, tm.k - ck0);
    // One k4-step of the 2x2 subtile block.  RE (GemmTerm::real): bit 0 = the
    // A operand is real (exact zero imaginary parts, e.g. Psi of a cluster the
    // self-energies never reach), bit 1 = B is real: the products with a zero
    // factor are skipped -- they add exact zeros, so the sums are unchanged.
    auto kstep = [&](int s, auto re_c) {
      constexpr int RE = decltype(re_c)::value;
      constexpr bool a_re = (RE & 1) != 0, b_re = (RE & 2) != 0;
      (void)a_re;
      (void)b_re;
      const int kk = 4 * s + t;
      double2 a[2], b[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int r = wm + 8 * i + g;
        a[i] = a_rk ? As[r * LD_RK + kk] : As[kk * A::LDA_KR + r];
        a[i].x = flip_sign(a[i].x, negA);
        a[i].y = flip_sign(a[i].y, negA);
      }
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int c = wn + 8 * j + g;
        b[j] = b_kr ? Bs[kk * A::LDB_KR + c] : Bs[c * LD_RK + kk];
        b[j].y = flip_sign(b[j].y, conjB);
      }
      if constexpr (M3) {
        double as[2], bs[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) as[i] = a[i].x + a[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) bs[j] = b[j].x + b[j].y;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (i >= live_i) break;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (j >= live_j) break;
            dmma(p1[i][j][0], p1[i][j][1], a[i].x, b[j].x);
            dmma(p2[i][j][0], p2[i][j][1], a[i].y, b[j].y);
            dmma(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
          }
        }
      } else {
        double nai[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) nai[i] = flip_sign(a[i].y, int(0x80000000));
        if (live_i == 2 && live_j == 2) {
          // all four subtiles live: the first product of every accumulator,
          // then the second, so 8 independent DMMAs separate the dependent
          // ones (the asm statements keep their order; same per-accumulator
          // summation order as below)
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              dmma(p1[i][j][0], p1[i][j][1], a[i].x, b[j].x);
              if constexpr (!b_re) dmma(p2[i][j][0], p2[i][j][1], a[i].x, b[j].y);
            }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              if constexpr (!a_re && !b_re) dmma(p1[i][j][0], p1[i][j][1], nai[i], b[j].y);
              if constexpr (!a_re) dmma(p2[i][j][0], p2[i][j][1], a[i].y, b[j].x);
            }
          return;
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (i >= live_i) break;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (j >= live_j) break;
            dmma(p1[i][j][0], p1[i][j][1], a[i].x, b[j].x);
            if constexpr (!a_re && !b_re) dmma(p1[i][j][0], p1[i][j][1], nai[i], b[j].y);
            if constexpr (!b_re) dmma(p2[i][j][0], p2[i][j][1], a[i].x, b[j].y);
            if constexpr (!a_re) dmma(p2[i][j][0], p2[i][j][1], a[i].y, b[j].x);
          }
        }
      }
    };
    auto chunk = [&](auto re_c) {
      if (ksteps == KC) {  // full chunk: straight-line, loads can be hoisted
#pragma unroll
        for (int s = 0; s < KC / 4; ++s) kstep(s, re_c);
      } else {
#pragma unroll
        for (int s = 0; s < KC / 4; ++s) {
          if (4 * s >= ksteps) break;
          kstep(s, re_c);
        }
      }
    };
    if (live_i > 0 && live_j > 0) {
      switch (M3 ? 0 : tm.real) {
        case 1: chunk(std::integral_constant<int, 1>{}); break;
        case 2: chunk(std::integral_constant<int, 2>{}); break;
        case 3: chunk(std::integral_constant<int, 3>{}); break;
        default: chunk(std::integral_constant<int, 0>{});
      }
    }
    stage ^= 1;
    advance(ct, ck0);
  }
  cp_async_wait<0>();

  const bool mir = tk.mirror && tl.n0 > tl.m0;  // aligned 32x32 tiles: every entry has c > r
  gemm_epilogue(base, tk, tl.m0 + wm, tl.n0 + wn, mir, [&](int i, int j, int q) {
    if constexpr (M3) {
    return make_double2(p1[i][j][q] - p2[i][j][q], p3[i][j][q] - p1[i][j][q] - p2[i][j][q]);
    } else {
    return make_double2(p1[i][j][q], p2[i][j][q]);
    }
  });
}

// ---------------------------------------------------------------------------
// Diagonal-only products, diagonal seeds, outputs
// ---------------------------------------------------------------------------
// One thread per output row (rows of never-referenced clusters are short;
// a thread walks its row of Psi and of the row-stored block, L1-cached).
__global__ void k_diag(double2* arena, int64_t stride, const DiagTask* __restrict__ tasks,
                       const GemmTerm* __restrict__ terms, int begin) {
  const DiagTask tk = tasks[begin + blockIdx.x];
  double2* base = arena + blockIdx.y * stride;
  for (int a = threadIdx.x; a < tk.m; a += blockDim.x) {
    double2 acc = tk.has_init ? base[tk.init_off + int64_t(a) * tk.init_stride] : make_double2(0.0, 0.0);
    for (int q = 0; q < tk.part_np; ++q)  // fused row-task partials, in order
      acc = cadd(acc, base[tk.part_off + int64_t(a) * tk.part_np + q]);
    for (int q = tk.term_begin; q < tk.term_begin + tk.term_count; ++q) {
      const GemmTerm tm = terms[q];
      double2 s = make_double2(0.0, 0.0);
      for (int b = 0; b < tm.k; ++b) {
        const double2 av = tm.a_op == OP_N ? base[tm.a_off + int64_t(a) * tm.lda + b]
                                           : base[tm.a_off + int64_t(b) * tm.lda + a];
        double2 bv;
        if (tm.b_op == OP_N || tm.b_op == OP_C) bv = base[tm.b_off + int64_t(b) * tm.ldb + a];
        else bv = base[tm.b_off + int64_t(a) * tm.ldb + b];
        if (tm.b_op == OP_C || tm.b_op == OP_H) bv.y = -bv.y;
        s = cadd(s, cmul(av, bv));
      }
      if (tm.sign < 0) acc = csub(acc, s);
      else acc = cadd(acc, s);
    }
    base[tk.out_off + a] = acc;
  }
}

__global__ void k_scale(double2* arena, int64_t stride, const ScaleTask* __restrict__ tasks, int begin) {
  const ScaleTask tk = tasks[begin + blockIdx.x];
  double2* base = arena + blockIdx.y * stride;
  const int total = tk.m * tk.n;
  for (int i = threadIdx.x; i < total; i += blockDim.x) {
    const int a = i / tk.n, b = i - a * tk.n;
    double2 src = base[tk.src_off + int64_t(a) * tk.ld_src + b];
    src.y = -src.y;
    base[tk.dst_off + int64_t(a) * tk.ld_dst + b] = cmul(base[tk.sig_off + a], src);
  }
}

__global__ void k_output(const double2* __restrict__ arena, int64_t stride, int nE, int e_base, int n,
                         const int64_t* __restrict__ gr_pos, const int64_t* __restrict__ gl_pos,
                         const double* __restrict__ weights, double2* gr, double2* gl, double* density,
                         DevStatus* st) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int64_t pr = gr_pos[d], pl = gl_pos[d];
  double acc = density[d];
  double worst = 0.0;
  for (int e = 0; e < nE; ++e) {
    const double2* a = arena + int64_t(e) * stride;
    if (gr) gr[int64_t(e) * n + d] = a[pr];
    const double2 v = pl >= 0 ? a[pl] : make_double2(0.0, 0.0);
    if (gl) gl[int64_t(e) * n + d] = v;
    const double mag = hypot(v.x, v.y);
    if (fabs(v.x) > 1e-8 * mag)
      atomicMin(&st->residual_key, (static_cast<unsigned long long>(e_base + e) << 32) |
                                       static_cast<unsigned long long>(d));
    if (mag > 0.0) worst = fmax(worst, fabs(v.x) / mag);
    acc += weights[e] * v.y;
  }
  density[d] = acc;
  if (worst > 0.0) atomicMax(&st->max_resid_bits, static_cast<unsigned long long>(__double_as_longlong(worst)));
}

// Sigma^< skewness per cluster block (validate_sigma, hsc.cpp:108-112 with
// skew_hermitian_defect, dense.cpp:221-230): accumulate ||S + S^H||_F^2 and
// ||S||_F^2 per (energy, seeded cluster) from the slots.
__device__ __forceinline__ double2 slot_value(const double2* sl, const int* ptr, const int* src, int s) {
  double2 v = make_double2(0.0, 0.0);
  for (int q = ptr[s]; q < ptr[s + 1]; ++q) v = cadd(v, sl[src[q]]);
  return v;
}

// One CTA per (seeded cluster, energy): block reduction over the cluster's
// slots (plan: slots grouped per cluster), no contended atomics.
__global__ void k_skew_accum(const double2* __restrict__ sigma_l, int64_t sl_nnz, const int* __restrict__ cslots,
                             const int* __restrict__ cslot_ptr, const int* __restrict__ ptr,
                             const int* __restrict__ src, const int* __restrict__ partner, int nsc, double* acc) {
  const int c = blockIdx.x, e = blockIdx.y;
  const double2* sl = sigma_l + e * sl_nnz;
  double num = 0.0, den = 0.0;
  for (int q = cslot_ptr[c] + threadIdx.x; q < cslot_ptr[c + 1]; q += blockDim.x) {
    const int s = cslots[q];
    const double2 v = slot_value(sl, ptr, src, s);
    const int p = partner[s];
    if (p >= 0) {
      const double2 w = slot_value(sl, ptr, src, p);
      const double re = v.x + w.x, im = v.y - w.y;
      num += re * re + im * im;
    } else {
      num += 2.0 * (v.x * v.x + v.y * v.y);
    }
    den += v.x * v.x + v.y * v.y;
  }
  __shared__ double red[2][8];
  for (int o = 16; o; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = num;
    red[1][threadIdx.x >> 5] = den;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double n2 = 0.0, d2 = 0.0;
    for (int w = 0; w < (blockDim.x >> 5); ++w) {
      n2 += red[0][w];
      d2 += red[1][w];
    }
    acc[(int64_t(e) * nsc + c) * 2] = n2;
    acc[(int64_t(e) * nsc + c) * 2 + 1] = d2;
  }
}

__global__ void k_skew_flag(const double* __restrict__ acc, int nsc, const int* __restrict__ ids,
                            int nE, int e_base, DevStatus* st) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nsc * nE) return;
  const int e = i / nsc, c = i - e * nsc;
  const double num = sqrt(acc[2 * i]), den = sqrt(acc[2 * i + 1]);
  const double defect = den == 0.0 ? num : num / den;
  if (defect > 1e-10)
    atomicMin(&st->nonskew_key, (static_cast<unsigned long long>(e_base + e) << 32) |
                                    static_cast<unsigned long long>(ids[c]));
}

int grid_for(int64_t work, int threads, int cap) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > cap) b = cap;
  return static_cast<int>(b);
}

}  // namespace

void launch_assemble(const BatchArgs& b, const Plan& p, const int64_t* d_h_pos, const double2* d_h_val,
                     const InitRegion* d_init_zero, const int64_t* d_diag_pos, const double* d_energies, const int64_t* d_sr_pos,
                     const int* d_sr_ptr, const int* d_sr_src, int64_t sr_nnz,
                     const double2* d_sigma_r, cudaStream_t s, int64_t& launches) {
  const int nreg = static_cast<int>(p.init_zero.size());
  dim3 g1(std::max(1, std::min(nreg, 1024)), b.nE);
  k_init<<<g1, 256, 0, s>>>(b.arena, b.stride, d_init_zero, nreg);
  const int64_t hn = static_cast<int64_t>(p.h_pos.size());
  if (hn > 0) {
    dim3 gh(grid_for(hn, 256, 1024), b.nE);
    k_scatter_h<<<gh, 256, 0, s>>>(b.arena, b.stride, d_h_pos, d_h_val, hn);
    ++launches;
  }
  const int sr_slots = static_cast<int>(p.sr_slot_pos.size());
  dim3 g2(grid_for(p.desc.n, 256, 1024), b.nE);
  k_scatter<<<g2, 256, 0, s>>>(b.arena, b.stride, p.desc.n, d_diag_pos, d_energies, nullptr, nullptr, nullptr, 0,
                               0, nullptr);
  launches += 2;
  if (sr_slots > 0) {
    dim3 g3(grid_for(sr_slots, 256, 1024), b.nE);
    k_scatter_sigma_r<<<g3, 256, 0, s>>>(b.arena, b.stride, d_sr_pos, d_sr_ptr, d_sr_src, sr_slots,
                                         sr_nnz, d_sigma_r);
    ++launches;
  }
}

// Sigma^< slots into the seed blocks (zeroed by k_init): launched right before
// the plan's first reader (Plan::lesser_op), so a host-buffer solve can copy
// Sigma^< in while the fold and the G^r sweep run.
void launch_scatter_lesser(const BatchArgs& b, const Plan& p, const double* d_energies, const int64_t* d_sl_pos,
                           const int* d_sl_ptr, const int* d_sl_src, int64_t sl_nnz, const double2* d_sigma_l,
                           cudaStream_t s, int64_t& launches) {
  const int sl_slots = static_cast<int>(p.sl_slot_pos.size());
  if (sl_slots <= 0) return;
  dim3 g2(grid_for(sl_slots, 256, 1024), b.nE);
  k_scatter<<<g2, 256, 0, s>>>(b.arena, b.stride, 0, nullptr, d_energies, d_sl_pos, d_sl_ptr, d_sl_src, sl_slots,
                               sl_nnz, d_sigma_l);
  ++launches;
}

// RGF elementwise steps.  skew_half (dense.cpp:136-170): upper triangle of
// the product, the diagonal's imaginary part, lower = -conj(upper).
__global__ void k_skew(double2* arena, int64_t stride, const SkewTask* __restrict__ tasks, int begin) {
  const SkewTask tk = tasks[begin + blockIdx.x];
  double2* a = arena + blockIdx.z * stride;
  const int n = tk.n;
  const int64_t nn = int64_t(n) * n;
  for (int64_t idx = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; idx < nn; idx += int64_t(gridDim.y) * blockDim.x) {
    const int i = static_cast<int>(idx / n), j = static_cast<int>(idx - int64_t(i) * n);
    double2 v;
    if (i < j) v = a[tk.src + idx];
    else if (i == j) v = make_double2(0.0, a[tk.src + idx].y);
    else {
      const double2 u = a[tk.src + int64_t(j) * n + i];
      v = make_double2(-u.x, u.y);
    }
    a[tk.dst + idx] = v;
  }
}

// out = gl + term + x - x^H (rgf.cpp:373-377, in that order).
__global__ void k_combine(double2* arena, int64_t stride, const CombineTask* __restrict__ tasks, int begin) {
  const CombineTask tk = tasks[begin + blockIdx.x];
  double2* a = arena + blockIdx.z * stride;
  const int n = tk.n;
  const int64_t nn = int64_t(n) * n;
  for (int64_t idx = int64_t(blockIdx.y) * blockDim.x + threadIdx.x; idx < nn; idx += int64_t(gridDim.y) * blockDim.x) {
    const int i = static_cast<int>(idx / n), j = static_cast<int>(idx - int64_t(i) * n);
    const double2 g = a[tk.gl + idx], t = a[tk.term + idx], x = a[tk.x + idx];
    const double2 xh = a[tk.x + int64_t(j) * n + i];  // (x^H)_ij = conj(x_ji)
    double2 v = cadd(cadd(g, t), x);
    v = make_double2(v.x - xh.x, v.y + xh.y);
    a[tk.out + idx] = v;
  }
}

// out[j] = sum over ranks r = 0, 1, ... of parts[r * n + j], in rank order.
__global__ void k_ordered_sum(const double* __restrict__ parts, int nranks, int n, double* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
    double s = parts[j];
    for (int r = 1; r < nranks; ++r) s += parts[int64_t(r) * n + j];
    out[j] = s;
  }
}

void launch_ordered_sum(const double* parts, int nranks, int n, double* out, cudaStream_t s, int64_t& launches) {
  k_ordered_sum<<<std::max(1, std::min(1024, (n + 255) / 256)), 256, 0, s>>>(parts, nranks, n, out);
  ++launches;
}

void launch_skew(const BatchArgs& b, const SkewTask* d_tasks, const SkewTask* h_tasks, int begin, int count,
                 cudaStream_t s, int64_t& launches) {
  int nmax = 0;
  for (int i = 0; i < count; ++i) nmax = std::max(nmax, h_tasks[begin + i].n);
  const int gy = std::max(1, std::min(64, (nmax * nmax + 255) / 256));
  k_skew<<<dim3(count, gy, b.nE), 256, 0, s>>>(b.arena, b.stride, d_tasks, begin);
  ++launches;
}

void launch_combine(const BatchArgs& b, const CombineTask* d_tasks, const CombineTask* h_tasks, int begin, int count,
                    cudaStream_t s, int64_t& launches) {
  int nmax = 0;
  for (int i = 0; i < count; ++i) nmax = std::max(nmax, h_tasks[begin + i].n);
  const int gy = std::max(1, std::min(64, (nmax * nmax + 255) / 256));
  k_combine<<<dim3(count, gy, b.nE), 256, 0, s>>>(b.arena, b.stride, d_tasks, begin);
  ++launches;
}

// Shifting-window variant of a block size:
// the narrowest window H * S >= m, in steps of 4 columns (a step's cost goes
// with rows x window width; measured with tools/inv_bench, profiles/
// inverse_experiments_r02.txt).  0: none (m <= 16 or m > 64).
static int sw_window(int m) {
  // m <= 16 (the small separators of levels 2-4) stays on k_inverse_reg: the
  // window kernel is 3 x faster there (-DNEGF_SW_TINY: 1.3 ms per config-2
  // step), but its rounding moves the resonant energy 211 of the config-2
  // grid to 1.08 x its parity bar (tests/test_gpu_fullgrid.py).
#ifndef NEGF_SW_TINY
  if (m <= 16) return 0;
#endif
  if (m <= 0 || m > 100) return 0;
  if (m <= 16) return std::max(8, (m + 3) & ~3);
  if (m <= 32) return std::max(20, (m + 3) & ~3);
  if (m <= 48) return std::max(36, (m + 3) & ~3);
  if (m <= 64) return (m + 3) & ~3;
  return m <= 76 ? 76 : 100;  // separators of the upper levels (few blocks: one CTA per SM)
}

// <ROWS, H, S, MINB>: the complex instantiation; <ROWS, HR, SR, MINR>: the real
// one (a real block needs half the registers: 49..64-wide real blocks run with
// one thread per row, 8.8 vs 10.6 ms for 326 x 256 blocks of 64).
template <int ROWS, int H, int S, int MINB, int HR, int SR, int MINR>
static void launch_sw(dim3 grid, const BatchArgs& b, const InvTask* dt, DevStatus* st, cudaStream_t s, bool real) {
  static_assert(H * S == HR * SR, "same window for both value types");
  if (real) k_inverse_sw<ROWS, HR, SR, MINR, true><<<grid, ROWS * HR, 0, s>>>(b.arena, b.stride, dt, b.e_base, st);
  else k_inverse_sw<ROWS, H, S, MINB, false><<<grid, ROWS * H, 0, s>>>(b.arena, b.stride, dt, b.e_base, st);
}

void launch_inverse(const BatchArgs& b, const InvTask* d_tasks, const InvTask* h_tasks, int count,
                    DevStatus* st, cudaStream_t s, int64_t& launches) {
  // Tasks of a level are pre-sorted by size class (inv_size_class, shared
  // with plan.cpp) and by size within a class, so each variant below covers
  // one contiguous range.
  int i = 0;
  while (i < count) {
    const int c = inv_size_class(h_tasks[i].m);
#ifdef NEGF_INV_LEGACY
    const int win = 0;
#else
    const int win = sw_window(h_tasks[i].m);
#endif
    int j = i;
    int mmax = 0;
    // the register variants: one launch per window width and value type (real /
    // complex blocks); the shared-memory variants: one launch per padded size
    const bool real = win && h_tasks[i].real;
    while (j < count && inv_size_class(h_tasks[j].m) == c &&
           (win ? (sw_window(h_tasks[j].m) == win && (h_tasks[j].real != 0) == real)
                : (c < 3 || ((h_tasks[j].m + 7) & ~7) == ((h_tasks[i].m + 7) & ~7)))) {
      mmax = std::max(mmax, h_tasks[j].m);
      ++j;
    }
    dim3 grid(j - i, b.nE);
    const InvTask* dt = d_tasks + i;
    const int m8 = (mmax + 7) & ~7;
    const size_t smem = size_t(m8) * (m8 + 2) * 16 + size_t(8) * (m8 + 2) * 16 + size_t(2 * m8 + 2) * 4 + 64;
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr)) {
      cudaFuncSetAttribute(k_inverse_blocked<false, 1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k_inverse_blocked<false, 2, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
      cudaFuncSetAttribute(k_inverse_la<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }
    switch (win) {
      // <= 16 (-DNEGF_SW_TINY only): one warp per block, 3 x the 64-thread k_inverse_reg
      case 8: launch_sw<32, 1, 8, 16, 1, 8, 16>(grid, b, dt, st, s, real); break;
      case 12: launch_sw<32, 1, 12, 16, 1, 12, 16>(grid, b, dt, st, s, real); break;
      case 16: launch_sw<32, 1, 16, 16, 1, 16, 16>(grid, b, dt, st, s, real); break;
      // 17..32: one row per lane, one warp per block
      case 20: launch_sw<32, 1, 20, 10, 1, 20, 16>(grid, b, dt, st, s, real); break;
      case 24: launch_sw<32, 1, 24, 10, 1, 24, 16>(grid, b, dt, st, s, real); break;
      case 28: launch_sw<32, 1, 28, 10, 1, 28, 16>(grid, b, dt, st, s, real); break;
      case 32: launch_sw<32, 1, 32, 10, 1, 32, 16>(grid, b, dt, st, s, real); break;
      // 33..48: two lanes per row, three warps
      case 36: launch_sw<48, 2, 18, 4, 2, 18, 8>(grid, b, dt, st, s, real); break;
      case 40: launch_sw<48, 2, 20, 4, 2, 20, 8>(grid, b, dt, st, s, real); break;
      case 44: launch_sw<48, 2, 22, 4, 2, 22, 8>(grid, b, dt, st, s, real); break;
      case 48: launch_sw<48, 2, 24, 4, 2, 24, 8>(grid, b, dt, st, s, real); break;
      // 49..64: two lanes per row, four warps
      case 52: launch_sw<64, 2, 26, 3, 1, 52, 5>(grid, b, dt, st, s, real); break;
      case 56: launch_sw<64, 2, 28, 3, 1, 56, 5>(grid, b, dt, st, s, real); break;
      case 60: launch_sw<64, 2, 30, 3, 1, 60, 5>(grid, b, dt, st, s, real); break;
      case 64: launch_sw<64, 2, 32, 3, 1, 64, 5>(grid, b, dt, st, s, real); break;
      // 65..100: 2.3 / 1.1 x the look-ahead shared-memory kernel on 74 / 100 wide blocks
      case 76: launch_sw<80, 2, 38, 1, 2, 38, 2>(grid, b, dt, st, s, real); break;
      case 100: launch_sw<104, 4, 25, 1, 4, 25, 2>(grid, b, dt, st, s, real); break;
      default:
        switch (c) {
          case 0: k_inverse_reg<8, 2><<<grid, 64, 0, s>>>(b.arena, b.stride, dt, b.e_base, st); break;
          // classes 1-3 here only with -DNEGF_INV_LEGACY (A/B builds): the
          // unrolled register kernel and the shared-memory blocked kernel
          case 1: k_inverse_rg<32, 2, 16><<<grid, 64, 0, s>>>(b.arena, b.stride, dt, b.e_base, st); break;
          case 2: k_inverse_rg<48, 2, 24><<<grid, 96, 0, s>>>(b.arena, b.stride, dt, b.e_base, st); break;
          case 3:  // 8-column panel on one warp + DMMA rank-8 updates
            k_inverse_blocked<false, 2, 8><<<grid, INV_THREADS, smem, s>>>(b.arena, b.stride, dt, b.e_base, st);
            break;
          default:  // 101..kSmemInvMax: the same with look-ahead (panel p+1 overlaps update p)
            k_inverse_la<4><<<grid, INV_THREADS, smem, s>>>(b.arena, b.stride, dt, b.e_base, st);
        }
    }
    ++launches;
    i = j;
  }
}

void launch_bigpanel(const BatchArgs& b, const BigTask* d_tasks, const BigTask* h_tasks, int count, int k0, int o0,
                     DevStatus* st, cudaStream_t s, int64_t& launches) {
  if (count <= 0) return;
  int mmax = 0;
  for (int i = 0; i < count; ++i) mmax = std::max(mmax, h_tasks[i].m);
  if (mmax <= kPanelSmemMax) {
    const size_t smem = size_t(mmax) * (kPanel + 1) * sizeof(double2);
    static std::atomic<unsigned long long> attr{0};
    if (first_on_device(attr))
      cudaFuncSetAttribute(k_bigpanel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_bigpanel<true><<<dim3(count, b.nE), 256, smem, s>>>(b.arena, b.stride, d_tasks, k0, o0, b.e_base, st);
  } else {
    k_bigpanel<false><<<dim3(count, b.nE), 256, 0, s>>>(b.arena, b.stride, d_tasks, k0, o0, b.e_base, st);
  }
  ++launches;
}

void launch_bigswap(const BatchArgs& b, const BigTask* d_tasks, int count, int o0, cudaStream_t s,
                    int64_t& launches) {
  if (count <= 0) return;
  k_bigswap<<<dim3(count, b.nE), 256, 0, s>>>(b.arena, b.stride, d_tasks, o0);
  ++launches;
}

void launch_bigperm(const BatchArgs& b, const BigTask* d_tasks, const BigTask* h_tasks, int count, cudaStream_t s,
                    int64_t& launches) {
  if (count <= 0) return;
  int mmax = 0;
  for (int i = 0; i < count; ++i) mmax = std::max(mmax, h_tasks[i].m);
  const size_t smem = size_t(2) * mmax * sizeof(int);
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) cudaFuncSetAttribute(k_bigperm, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  static_assert(kBigPermChunks * 4 <= kOuter, "k_bigperm row buffers live in the outer-panel scratch");
  k_bigperm<<<dim3(count, b.nE, kBigPermChunks), 128, smem, s>>>(b.arena, b.stride, d_tasks);
  ++launches;
}

// Sparse leaf Psi (K_SPSI): Psi_x[r][c] = -sum_e inv_x[r][t_e] a_e over the
// stencil entries of column c of A_{x,S} (ascending t, fixed order); one CTA
// per (leaf, energy), consecutive threads on consecutive columns of a Psi row
// (coalesced stores; inv_x is re-read from L1).
__global__ void __launch_bounds__(256) k_spsi(double2* arena, int64_t stride, const SpsiTask* __restrict__ tasks,
                                              const int* __restrict__ colptr, const int* __restrict__ rows,
                                              const double2* __restrict__ vals, const int* __restrict__ wcols,
                                              int begin) {
  const SpsiTask tk = tasks[begin + blockIdx.x];
  double2* base = arena + int64_t(blockIdx.y) * stride;
  const double2* inv = base + tk.off_inv;
  const int* cp = colptr + tk.col_begin;
  if (tk.h > 0) {  // compact leaf: only the hull columns, Psi_H (m x h)
    const int* wc = wcols + tk.wcol_begin;
    for (int idx = threadIdx.x; idx < tk.m * tk.h; idx += blockDim.x) {
      const int r = idx / tk.h, c = wc[idx - r * tk.h];
      double2 acc = make_double2(0.0, 0.0);
      for (int e = cp[c]; e < cp[c + 1]; ++e) acc = cadd(acc, cmul(inv[int64_t(r) * tk.m + rows[e]], vals[e]));
      base[tk.off_psi + idx] = make_double2(-acc.x, -acc.y);
    }
    return;
  }
  const int total = tk.m * tk.K;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int r = idx / tk.K, c = idx - r * tk.K;
    double2 acc = make_double2(0.0, 0.0);
    for (int e = cp[c]; e < cp[c + 1]; ++e) acc = cadd(acc, cmul(inv[int64_t(r) * tk.m + rows[e]], vals[e]));
    const double2 v = make_double2(-acc.x, -acc.y);
    base[tk.off_psi + idx] = v;
    if (tk.off_psi2 >= 0) base[tk.off_psi2 + idx] = make_double2(2.0 * v.x, 2.0 * v.y);
  }
}

void launch_spsi(const BatchArgs& b, const SpsiTask* d_tasks, const int* d_colptr, const int* d_rows,
                 const double2* d_vals, const int* d_wcols, int begin, int count, cudaStream_t s, int64_t& launches) {
  if (count <= 0) return;
  k_spsi<<<dim3(count, b.nE), 256, 0, s>>>(b.arena, b.stride, d_tasks, d_colptr, d_rows, d_vals, d_wcols, begin);
  ++launches;
}

// M of a compact leaf (MGatherTask): per block, coef * [conj] src[a rs + c cs]
// into M[dst_row + a][dst_col + c] (coef 0: zeros).  One CTA per (leaf,
// energy); consecutive threads on consecutive M columns.
__global__ void __launch_bounds__(256) k_mgather(double2* arena, int64_t stride, const MGatherTask* __restrict__ tasks,
                                                 const MGatherBlock* __restrict__ blocks, int begin) {
  const MGatherTask tk = tasks[begin + blockIdx.x];
  double2* base = arena + int64_t(blockIdx.y) * stride;
  double2* M = base + tk.dst;
  for (int q = 0; q < tk.block_count; ++q) {
    const MGatherBlock bl = blocks[tk.block_begin + q];
    for (int idx = threadIdx.x; idx < bl.rows * bl.cols; idx += blockDim.x) {
      const int a = idx / bl.cols, c = idx - a * bl.cols;
      double2 v = make_double2(0.0, 0.0);
      if (bl.coef != 0.0) {
        v = base[bl.src + a * bl.rs + c * bl.cs];
        if (bl.conj) v.y = -v.y;
        v.x *= bl.coef;
        v.y *= bl.coef;
      }
      M[int64_t(bl.dst_row + a) * tk.h + bl.dst_col + c] = v;
    }
  }
}

void launch_mgather(const BatchArgs& b, const MGatherTask* d_tasks, const MGatherBlock* d_blocks, int begin, int count,
                    cudaStream_t s, int64_t& launches) {
  if (count <= 0) return;
  k_mgather<<<dim3(count, b.nE), 256, 0, s>>>(b.arena, b.stride, d_tasks, d_blocks, begin);
  ++launches;
}

// Sparse leaf Schur contributions (K_SSCHUR): for a target block,
// T[r][c] (+)= sum over its leaves i (in gather order) of
// (Psi_i^T A_i)[p_off + r][q_off + c] = -sum inv_i[t][t'] a(t', p_off + r) a(t, q_off + c)
// over the stencil entries of the two columns of the leaf's A_{i,S} (Psi_i
// itself is not needed).  One CTA per (target, energy), two schedules
// (SschurTask::entry, chosen by the plan from the touched area):
//  * entry: one thread per target entry walks the target's leaves in their
//    stored order and skips those whose column pair at (r, c) is empty -- no
//    barrier (small targets, densely touched: the low separator levels);
//  * per leaf over its touched rows x columns, leaves touching disjoint rows
//    x columns concurrently (waves, SschurContrib::sync) -- large targets with
//    small touched areas.
// Contributions are stored in waves, which keeps gather order for every
// entry, so both schedules give every entry the same sums in the same order
// as the reference's right-looking update.
__global__ void __launch_bounds__(128) k_sschur(double2* arena, int64_t stride, const SschurTask* __restrict__ tasks,
                                                const SschurContrib* __restrict__ contrib,
                                                const SpsiTask* __restrict__ spsi, const int* __restrict__ colptr,
                                                const int* __restrict__ rows, const double2* __restrict__ vals,
                                                const int* __restrict__ rc, int begin) {
  const SschurTask tk = tasks[begin + blockIdx.x];
  double2* base = arena + int64_t(blockIdx.y) * stride;
  double2* tgt = base + tk.off;
  auto leaf_term = [&](const SpsiTask& lt, const int* cb, int p0, int p1, int q0, int q1) {
    const double2* inv = base + lt.off_inv;
    double2 acc = make_double2(0.0, 0.0);
    for (int e2 = q0; e2 < q1; ++e2) {
      const double2* irow = inv + int64_t(rows[e2]) * lt.m;
      double2 z = make_double2(0.0, 0.0);
      for (int e1 = p0; e1 < p1; ++e1) z = cadd(z, cmul(irow[rows[e1]], vals[e1]));
      acc = csub(acc, cmul(z, vals[e2]));
    }
    (void)cb;
    return acc;
  };
  if (tk.entry) {
    for (int idx = threadIdx.x; idx < tk.mp * tk.mq; idx += blockDim.x) {
      const int r = idx / tk.mq, c = idx - r * tk.mq;
      double2* dst = tgt + int64_t(r) * tk.ld + c;
      double2 sum = tk.mode == MODE_ADD ? *dst : make_double2(0.0, 0.0);  // a pure fill block starts from zero
      bool touched = false;
      for (int q = 0; q < tk.contrib_count; ++q) {
        const SschurContrib& ct = contrib[tk.contrib_begin + q];
        const SpsiTask& lt = spsi[ct.spsi];
        const int* cb = colptr + lt.col_begin;
        const int p0 = cb[ct.p_off + r], p1 = cb[ct.p_off + r + 1];
        const int q0 = cb[ct.q_off + c], q1 = cb[ct.q_off + c + 1];
        if (p0 == p1 || q0 == q1) continue;
        sum = cadd(sum, leaf_term(lt, cb, p0, p1, q0, q1));
        touched = true;
      }
      if (touched || tk.mode != MODE_ADD) *dst = sum;
    }
    return;
  }
  if (tk.mode != MODE_ADD) {  // a pure fill block starts from zero
    for (int idx = threadIdx.x; idx < tk.mp * tk.mq; idx += blockDim.x) {
      const int r = idx / tk.mq, c = idx - r * tk.mq;
      tgt[int64_t(r) * tk.ld + c] = make_double2(0.0, 0.0);
    }
    __syncthreads();
  }
  for (int q = 0; q < tk.contrib_count; ++q) {
    const SschurContrib ct = contrib[tk.contrib_begin + q];
    const SpsiTask& lt = spsi[ct.spsi];
    const int* R = rc + ct.rc_begin;
    const int* Cc = R + ct.nr;
    const int* cb = colptr + lt.col_begin;
    for (int idx = threadIdx.x; idx < ct.nr * ct.nc; idx += blockDim.x) {
      const int r = R[idx / ct.nc], c = Cc[idx % ct.nc];
      const int* cp = cb + ct.p_off + r;
      const int* cq = cb + ct.q_off + c;
      double2* dst = tgt + int64_t(r) * tk.ld + c;
      *dst = cadd(*dst, leaf_term(lt, cb, cp[0], cp[1], cq[0], cq[1]));
    }
    if (ct.sync) __syncthreads();  // end of a wave of disjoint leaves
  }
}

void launch_sschur(const BatchArgs& b, const SschurTask* d_tasks, const SschurContrib* d_contrib,
                   const SpsiTask* d_spsi, const int* d_colptr, const int* d_rows, const double2* d_vals,
                   const int* d_rc, int begin, int count, cudaStream_t s, int64_t& launches) {
  if (count <= 0) return;
  k_sschur<<<dim3(count, b.nE), 128, 0, s>>>(b.arena, b.stride, d_tasks, d_contrib, d_spsi, d_colptr, d_rows,
                                              d_vals, d_rc, begin);
  ++launches;
}

// Woodbury diagonals of sparse leaves (K_LEAFDIAG, plan.hpp LeafDiagTask):
// M (nT x nT) gathered from the stored G / P blocks (upper triangle, one
// thread per output, fixed entry order), mirrored; W = inv_x[:, T] staged;
// then one warp per row r: sum_{i1,i2} W[r][i1] M[i1][i2] op(W[r][i2]).
#ifndef NEGF_LD_THREADS
#define NEGF_LD_THREADS 256
#endif
__global__ void __launch_bounds__(NEGF_LD_THREADS) k_leafdiag(double2* arena, int64_t stride,
                                                  const LeafDiagTask* __restrict__ tasks,
                                                  const int* __restrict__ trows, const int* __restrict__ optr,
                                                  const LeafDiagEntry* __restrict__ ent, int begin) {
  extern __shared__ double2 sm[];
  const LeafDiagTask tk = tasks[begin + blockIdx.x];
  double2* base = arena + int64_t(blockIdx.y) * stride;
  const int nT = tk.nT, m = tk.m;
  const int wp = nT | 1;  // odd pitches: conflict-free strided reads of W and M
  double2* M = sm;
  double2* W = sm + nT * wp;
  const int* T = trows + tk.t_begin;
  const int* op = optr + tk.out_begin;
  const int nO = nT * (nT + 1) / 2;
  // entry products first, all entries in parallel (independent loads) into
  // the W area (free until the W staging below), then per-output sums in the
  // fixed entry order
  const int e0 = op[0], ne = op[nO] - e0;
  double2* prod = W;
  for (int e = threadIdx.x; e < ne; e += blockDim.x) {
    const LeafDiagEntry en = ent[e0 + e];
    double2 v = base[en.pos];
    if (en.flag) v = make_double2(-v.x, v.y);
    const double* cf = reinterpret_cast<const double*>(&en.coef);  // std::complex: (re, im)
    prod[e] = cmul(make_double2(cf[0], cf[1]), v);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < nO; o += blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    for (int e = op[o]; e < op[o + 1]; ++e) acc = cadd(acc, prod[e - e0]);
    const int out = ent[op[o]].out;
    const int i1 = out >> 16, i2 = out & 0xffff;
    M[i1 * wp + i2] = acc;
    if (i1 != i2) M[i2 * wp + i1] = tk.mode == 0 ? acc : make_double2(-acc.x, acc.y);
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < m * nT; idx += blockDim.x) {
    const int r = idx / nT, i = idx - r * nT;
    W[r * wp + i] = base[tk.off_inv + int64_t(r) * m + T[i]];
  }
  __syncthreads();
  // one warp per row: lane i1 forms W[r][i1] (M[i1][:] . op(W[r][:])); the
  // lanes' partials are reduced by a fixed xor tree (deterministic)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int r = warp; r < m; r += nw) {
    const double2* w = W + r * wp;
    double2 part = make_double2(0.0, 0.0);
    for (int i1 = lane; i1 < nT; i1 += 32) {
      const double2* mr = M + i1 * wp;
      double2 y = make_double2(0.0, 0.0);
      for (int i2 = 0; i2 < nT; ++i2) {
        double2 w2 = w[i2];
        if (tk.mode) w2.y = -w2.y;
        y = cadd(y, cmul(mr[i2], w2));
      }
      part = cadd(part, cmul(w[i1], y));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      part.x += __shfl_xor_sync(0xffffffffu, part.x, o);
      part.y += __shfl_xor_sync(0xffffffffu, part.y, o);
    }
    if (lane == 0) {
      if (tk.mode == 0) part = cadd(base[tk.off_inv + int64_t(r) * m + r], part);
      base[tk.off_out + r] = part;
    }
  }
}

void launch_leafdiag(const BatchArgs& b, const LeafDiagTask* d_tasks, const LeafDiagTask* h_tasks,
                     const int* d_rows, const int* d_optr, const int* h_optr, const LeafDiagEntry* d_ent, int begin,
                     int count, cudaStream_t s, int64_t& launches) {
  if (count <= 0) return;
  size_t smem = 0;
  for (int i = begin; i < begin + count; ++i) {
    const LeafDiagTask& t = h_tasks[i];
    const size_t ne = size_t(h_optr[t.out_begin + t.nT * (t.nT + 1) / 2] - h_optr[t.out_begin]);
    smem = std::max(smem, sizeof(double2) * (size_t(t.nT) * (t.nT | 1) + std::max(size_t(t.m) * (t.nT | 1), ne)));
  }
  static std::atomic<unsigned long long> attr{0};
  if (first_on_device(attr)) cudaFuncSetAttribute(k_leafdiag, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  k_leafdiag<<<dim3(count, b.nE), NEGF_LD_THREADS, smem, s>>>(b.arena, b.stride, d_tasks, d_rows, d_optr, d_ent, begin);
  ++launches;
}

// Item w of a launch -> (tile, energy).  Energies go in groups of `eg`:
// all tiles of a group's energies are issued before the next group, energy
// fastest inside the group.  Small groups keep the operand panels that
// neighbouring tiles of one energy share in L2 (config 2, all k_gemm launches
// of a batch: 331 GB of DRAM traffic with eg = nE and a static stride, 195 GB
// with groups of 4 and the atomic counter below, against 298 GB algorithmic);
// eg = nE runs the 256 copies of a tile side by side.  Defaults: measured.
// The last group (energies e_main .. nE - 1, e_main a multiple of eg) may be
// wider than eg: a few waves of items in tile-major order, longest tiles
// first, so the launch does not end on a long tile that started last.
__device__ __forceinline__ void gemm_item_index(int64_t w, int nE, int64_t ntiles, int eg, int e_main, int64_t& ti,
                                                int& e) {
  const int64_t main_items = ntiles * e_main;
  if (w >= main_items) {
    const int64_t r = w - main_items;
    const int egc = nE - e_main;
    ti = r / egc;
    e = e_main + static_cast<int>(r - ti * egc);
    return;
  }
  const int64_t per = ntiles * eg;
  const int64_t grp = w / per;
  const int64_t r = w - grp * per;
  ti = r / eg;
  e = static_cast<int>(grp) * eg + static_cast<int>(r - ti * eg);
}

// Persistent launch over (tile, energy) items in the grouped order above; one
// launch per warp arrangement of an op (a task may mix arrangements, plan.cpp
// tile_task); tiles pre-sorted by decreasing cost in the plan.  Items are
// handed out by an atomic counter (ctr[0]; ctr == nullptr: static stride):
// with a static stride each CTA's sequence is fixed, CTAs drift apart by whole
// tile times after the first wave, and tiles that share an operand panel
// (neighbours in the item order) no longer run together -- the panel has left
// L2 before its second reader arrives.  The last CTA to finish resets the
// counters for the next launch on the stream.
__device__ __forceinline__ void gemm_ctr_done(unsigned long long* ctr, unsigned long long workers) {
  if (atomicAdd(ctr + 1, 1ull) == workers - 1) {
    ctr[0] = 0;
    ctr[1] = 0;
  }
}

#ifndef NEGF_GEMM_MINB
#define NEGF_GEMM_MINB 4  // resident CTAs per SM (A/B builds)
#endif
template <int WR, int WC, bool M3>
__global__ void __launch_bounds__(128, NEGF_GEMM_MINB) k_gemm(double2* arena, int64_t stride, int nE,
                                                     const GemmTask* __restrict__ tasks,
                                                     const GemmTerm* __restrict__ terms,
                                                     const GemmTile* __restrict__ tiles, int tile_begin,
                                                     int64_t items, int eg, int e_main,
                                                     unsigned long long* ctr) {
  extern __shared__ double2 gsm[];
  __shared__ int64_t s_next[2];  // double-buffered: slot it & 1 is written in iteration it
  const int64_t ntiles = items / nE;
  int64_t w = blockIdx.x;
  for (int it = 0; w < items; ++it) {
    if (ctr && threadIdx.x == 0) s_next[it & 1] = int64_t(gridDim.x) + int64_t(atomicAdd(ctr, 1ull));
    int64_t ti;
    int e;
    gemm_item_index(w, nE, ntiles, eg, e_main, ti, e);
    const GemmTile tl = tiles[tile_begin + ti];
    const GemmTask tk = tasks[tl.task];
    // Stage the task's term descriptors in shared memory (read every chunk).
    GemmTerm* tsm = reinterpret_cast<GemmTerm*>(gsm + 2 * Arr<WR, WC>::STAGE);
    const GemmTerm* tp = terms;
    if (tk.term_count <= kTermCache) {
      const int2* src = reinterpret_cast<const int2*>(terms + tk.term_begin);
      int2* dst = reinterpret_cast<int2*>(tsm);
      constexpr int W = sizeof(GemmTerm) / 8;
      static_assert(sizeof(GemmTerm) % 8 == 0, "term copy granule");
      for (int q = threadIdx.x; q < tk.term_count * W; q += blockDim.x) dst[q] = src[q];
      __syncthreads();
      tp = tsm - tk.term_begin;
    }
    gemm_item<WR, WC, M3>(arena + e * stride, tk, tp, tl, gsm);
    __syncthreads();
    w = ctr ? s_next[it & 1] : w + gridDim.x;
  }
  if (ctr && threadIdx.x == 0) gemm_ctr_done(ctr, gridDim.x);
}
// Warp tiles (GemmTile::arr == 3, small tasks): one warp per 16 x 16 output
// block, fragments loaded straight from global memory (L2 / HBM) into
// registers -- no shared-memory staging, no CTA barrier -- so many
// independent warps keep their loads in flight.  The DMMA sequence per
// accumulator (terms in order, 4-deep k-steps, zero-padded) is that of
// gemm_item, so the results are bit-identical to the CTA tiles.
#ifndef NEGF_WARP_MINB
#define NEGF_WARP_MINB 3
#endif
#ifndef NEGF_WARP_UNROLL
#define NEGF_WARP_UNROLL 1
#endif
constexpr int kWarpUnroll = NEGF_WARP_UNROLL;
template <bool M3>
__global__ void __launch_bounds__(256, NEGF_WARP_MINB) k_gemm_warp(double2* arena, int64_t stride, int nE,
                                                      const GemmTask* __restrict__ tasks,
                                                      const GemmTerm* __restrict__ terms,
                                                      const GemmTile* __restrict__ tiles, int tile_begin,
                                                      int64_t items, int eg, int e_main,
                                                      unsigned long long* ctr) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wpb = blockDim.x >> 5;
  const int64_t nw = int64_t(gridDim.x) * wpb;
  const int64_t ntiles = items / nE;
  // items per warp: static stride or the launch's atomic counter (k_gemm)
  for (int64_t w = int64_t(blockIdx.x) * wpb + (threadIdx.x >> 5), wn = 0; w < items; w = wn) {
    if (ctr) {
      unsigned long long x = 0;
      if (lane == 0) x = atomicAdd(ctr, 1ull);
      wn = nw + int64_t(__shfl_sync(0xffffffffu, x, 0));
    } else {
      wn = w + nw;
    }
    int64_t ti;
    int e;
    gemm_item_index(w, nE, ntiles, eg, e_main, ti, e);
    const GemmTile tl = tiles[tile_begin + ti];
    const GemmTask tk = tasks[tl.task];
    double2* base = arena + int64_t(e) * stride;
    const int live_i = min(2, max(0, (tk.m - tl.m0 + 7) / 8));
    const int live_j = min(2, max(0, (tk.n - tl.n0 + 7) / 8));
    double p1[2][2][2], p2[2][2][2], p3[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int q = 0; q < 2; ++q) p1[i][j][q] = p2[i][j][q] = p3[i][j][q] = 0.0;
    const int ra0 = tl.m0 + g, ra1 = tl.m0 + 8 + g;  // A rows of this lane
    const int cb0 = tl.n0 + g, cb1 = tl.n0 + 8 + g;  // B columns of this lane
    for (int q = tk.term_begin; q < tk.term_begin + tk.term_count; ++q) {
      const GemmTerm tm = terms[q];
      if (tm.k <= 0) continue;
      const int negA = tm.sign < 0 ? int(0x80000000) : 0;
      const int conjB = (tm.b_op == OP_C || tm.b_op == OP_H) ? int(0x80000000) : 0;
      const bool a_rk = (tm.a_op == OP_N);
      const bool b_kr = (tm.b_op == OP_N || tm.b_op == OP_C);
      const double2* A = base + tm.a_off;
      const double2* Bm = base + tm.b_off;
      // element (row, k) of op(A) and (k, col) of op(B) at this lane
      const int64_t as_r = a_rk ? tm.lda : 1, as_k = a_rk ? 1 : tm.lda;
      const int64_t bs_k = b_kr ? tm.ldb : 1, bs_c = b_kr ? 1 : tm.ldb;
      const bool va0 = ra0 < tk.m, va1 = ra1 < tk.m, vb0 = cb0 < tk.n, vb1 = cb1 < tk.n;
      // RE (GemmTerm::real): products with an exactly-zero factor skipped (gemm_item)
      auto kloop = [&](auto re_c) {
        constexpr int RE = decltype(re_c)::value;
        constexpr bool a_re = (RE & 1) != 0, b_re = (RE & 2) != 0;
        (void)a_re;
        (void)b_re;
#pragma unroll kWarpUnroll
      for (int k0 = 0; k0 < tm.k; k0 += 4) {
        const int kk = k0 + t;
        const bool vk = kk < tm.k;
        double2 a[2], b[2];
        const double2 z = make_double2(0.0, 0.0);
        a[0] = (va0 && vk) ? A[ra0 * as_r + kk * as_k] : z;
        a[1] = (va1 && vk) ? A[ra1 * as_r + kk * as_k] : z;
        b[0] = (vb0 && vk) ? Bm[kk * bs_k + cb0 * bs_c] : z;
        b[1] = (vb1 && vk) ? Bm[kk * bs_k + cb1 * bs_c] : z;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          a[i].x = flip_sign(a[i].x, negA);
          a[i].y = flip_sign(a[i].y, negA);
        }
#pragma unroll
        for (int j = 0; j < 2; ++j) b[j].y = flip_sign(b[j].y, conjB);
        if constexpr (M3) {
        double as[2], bs[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) as[i] = a[i].x + a[i].y;
#pragma unroll
        for (int j = 0; j < 2; ++j) bs[j] = b[j].x + b[j].y;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          if (i >= live_i) break;
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            if (j >= live_j) break;
            dmma(p1[i][j][0], p1[i][j][1], a[i].x, b[j].x);
            dmma(p2[i][j][0], p2[i][j][1], a[i].y, b[j].y);
            dmma(p3[i][j][0], p3[i][j][1], as[i], bs[j]);
          }
        }
        } else {
        double nai[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) nai[i] = flip_sign(a[i].y, int(0x80000000));
        if (live_i == 2 && live_j == 2) {
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              dmma(p1[i][j][0], p1[i][j][1], a[i].x, b[j].x);
              if constexpr (!b_re) dmma(p2[i][j][0], p2[i][j][1], a[i].x, b[j].y);
            }
#pragma unroll
          for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              if constexpr (!a_re && !b_re) dmma(p1[i][j][0], p1[i][j][1], nai[i], b[j].y);
              if constexpr (!a_re) dmma(p2[i][j][0], p2[i][j][1], a[i].y, b[j].x);
            }
        } else {
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            if (i >= live_i) break;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              if (j >= live_j) break;
              dmma(p1[i][j][0], p1[i][j][1], a[i].x, b[j].x);
              if constexpr (!a_re && !b_re) dmma(p1[i][j][0], p1[i][j][1], nai[i], b[j].y);
              if constexpr (!b_re) dmma(p2[i][j][0], p2[i][j][1], a[i].x, b[j].y);
              if constexpr (!a_re) dmma(p2[i][j][0], p2[i][j][1], a[i].y, b[j].x);
            }
          }
        }
        }
      }
      };
      switch (M3 ? 0 : tm.real) {
        case 1: kloop(std::integral_constant<int, 1>{}); break;
        case 2: kloop(std::integral_constant<int, 2>{}); break;
        case 3: kloop(std::integral_constant<int, 3>{}); break;
        default: kloop(std::integral_constant<int, 0>{});
      }
    }
    gemm_epilogue(base, tk, tl.m0, tl.n0, false, [&](int i, int j, int q) {
      if constexpr (M3) {
      return make_double2(p1[i][j][q] - p2[i][j][q], p3[i][j][q] - p1[i][j][q] - p2[i][j][q]);
      } else {
      return make_double2(p1[i][j][q], p2[i][j][q]);
      }
    });
  }
  if (ctr && lane == 0) gemm_ctr_done(ctr, static_cast<unsigned long long>(nw));
}

// Energies per item group and the start of the last group (gemm_item_index).
// Mode -1 (CTA tiles): wave-sized groups -- as many energies as fill the
// launch's resident CTAs once, so the tiles of one task run together and share
// its operand panels through L2 -- with the last three waves as one tile-major
// group (no long tile starts last).  NEGF_GEMM_EG = n > 0 forces groups of n,
// NEGF_GEMM_EG = 1073741824 one group of all energies (A/B).
struct EnergyGroups {
  int eg, e_main;
};
static EnergyGroups gemm_energy_groups(int nE, bool warp, int tile_count, int slots) {
  static const int env = [] {
    const char* e = std::getenv("NEGF_GEMM_EG");
    return e ? std::atoi(e) : 0;
  }();
  int mode = env != 0 ? env : (warp ? kGemmEgWarp : kGemmEgCta);
  if (mode < 0 && !warp) {
    const int wave = std::max(1, slots / std::max(1, tile_count));
    const int eg = std::min(wave, nE);
    const int tail = std::min(nE, 3 * wave);
    return {eg, ((nE - tail) / eg) * eg};
  }
  if (mode < 0) mode = kGemmEgWarp;
  const int eg = std::max(1, std::min(mode, nE));
  return {eg, (nE / eg) * eg};
}
// Dynamic item scheduling (atomic counter) unless NEGF_GEMM_DYN=0 (A/B).
static unsigned long long* gemm_counter(const BatchArgs& b) {
  static const bool dyn = [] {
    const char* e = std::getenv("NEGF_GEMM_DYN");
    return !(e && std::atoi(e) == 0);
  }();
  return dyn ? b.gemm_ctr : nullptr;
}

template <bool M3>
static void launch_gemm_warp(const BatchArgs& b, const GemmTask* d_tasks, const GemmTerm* d_terms,
                             const GemmTile* d_tiles, int tile_begin, int tile_count, cudaStream_t s) {
  static int slots_of[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& slots = slots_of[dev & 63];
  if (!slots) {
    int sms = 0, per_sm = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemm_warp<M3>, 256, 0);
    slots = std::max(1, sms * std::max(1, per_sm));
  }
  const int64_t items = int64_t(tile_count) * b.nE;
  const int grid = static_cast<int>(std::min<int64_t>((items + 7) / 8, slots));
  const EnergyGroups eg = gemm_energy_groups(b.nE, true, tile_count, slots);
  k_gemm_warp<M3><<<grid, 256, 0, s>>>(b.arena, b.stride, b.nE, d_tasks, d_terms, d_tiles, tile_begin, items, eg.eg,
                                   eg.e_main, gemm_counter(b));
}

template <int WR, int WC, bool M3>
static void launch_gemm_arr(const BatchArgs& b, const GemmTask* d_tasks, const GemmTerm* d_terms,
                            const GemmTile* d_tiles, int tile_begin, int tile_count, cudaStream_t s) {
  constexpr size_t smem = sizeof(double2) * 2 * Arr<WR, WC>::STAGE + sizeof(GemmTerm) * kTermCache;
  static int slots_of[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  int& slots = slots_of[dev & 63];
  if (!slots) {
    int sms = 0, per_sm = 0;
    cudaFuncSetAttribute(k_gemm<WR, WC, M3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gemm<WR, WC, M3>, 128, smem);
    slots = std::max(1, sms * std::max(1, per_sm));
  }
  const int64_t items = int64_t(tile_count) * b.nE;
  const int grid = static_cast<int>(std::min<int64_t>(items, slots));
  const EnergyGroups eg = gemm_energy_groups(b.nE, false, tile_count, slots);
  k_gemm<WR, WC, M3><<<grid, 128, smem, s>>>(b.arena, b.stride, b.nE, d_tasks, d_terms, d_tiles, tile_begin, items, eg.eg,
                                         eg.e_main, gemm_counter(b));
}
template <bool M3>
static void launch_gemm_impl(const BatchArgs& b, const GemmTask* d_tasks, const GemmTerm* d_terms,
                             const GemmTile* d_tiles, const GemmTile* h_tiles, int tile_begin, int tile_count,
                             cudaStream_t s, int64_t& launches) {
  // Tiles of one op are grouped by warp arrangement (plan.cpp): one launch each.
  int i = tile_begin;
  const int end = tile_begin + tile_count;
  while (i < end) {
    const int arr = h_tiles[i].arr;
    int j = i;
    while (j < end && h_tiles[j].arr == arr) ++j;
    if (arr == 1) launch_gemm_arr<1, 4, M3>(b, d_tasks, d_terms, d_tiles, i, j - i, s);
    else if (arr == 2) launch_gemm_arr<4, 1, M3>(b, d_tasks, d_terms, d_tiles, i, j - i, s);
    else if (arr == 3) launch_gemm_warp<M3>(b, d_tasks, d_terms, d_tiles, i, j - i, s);
    else launch_gemm_arr<2, 2, M3>(b, d_tasks, d_terms, d_tiles, i, j - i, s);
    ++launches;
    i = j;
  }
}
// gauss3m: the Gauss (3M) complex product for this op (see gemm_item); the
// caller decides per op (capi.cu: never for the G^< phases).
void launch_gemm(const BatchArgs& b, const GemmTask* d_tasks, const GemmTerm* d_terms,
                 const GemmTile* d_tiles, const GemmTile* h_tiles, int tile_begin, int tile_count,
                 cudaStream_t s, int64_t& launches, bool gauss3m) {
#ifdef NEGF_GEMM_3M
  gauss3m = true;  // A/B builds: 3M everywhere (round 1)
#endif
  if (gauss3m) launch_gemm_impl<true>(b, d_tasks, d_terms, d_tiles, h_tiles, tile_begin, tile_count, s, launches);
  else launch_gemm_impl<false>(b, d_tasks, d_terms, d_tiles, h_tiles, tile_begin, tile_count, s, launches);
}

void launch_diag(const BatchArgs& b, const DiagTask* d_tasks, const GemmTerm* d_terms, int begin,
                 int count, cudaStream_t s, int64_t& launches) {
  if (count <= 0) return;
  dim3 grid(count, b.nE);
  k_diag<<<grid, 64, 0, s>>>(b.arena, b.stride, d_tasks, d_terms, begin);
  ++launches;
}

void launch_scale(const BatchArgs& b, const ScaleTask* d_tasks, int begin, int count, cudaStream_t s,
                  int64_t& launches) {
  if (count <= 0) return;
  dim3 grid(count, b.nE);
  k_scale<<<grid, 256, 0, s>>>(b.arena, b.stride, d_tasks, begin);
  ++launches;
}

void launch_skew_check(const BatchArgs& b, const double2* d_sigma_l, int64_t sl_nnz, const int* d_cslots,
                       const int* d_cslot_ptr, const int* d_sl_ptr, const int* d_sl_src, const int* d_sl_partner,
                       int n_seeded, const int* d_seeded_ids, double* d_acc, DevStatus* st, cudaStream_t s,
                       int64_t& launches) {
  if (n_seeded <= 0 || sl_nnz <= 0) return;
  dim3 g(n_seeded, b.nE);
  k_skew_accum<<<g, 256, 0, s>>>(d_sigma_l, sl_nnz, d_cslots, d_cslot_ptr, d_sl_ptr, d_sl_src, d_sl_partner,
                                 n_seeded, d_acc);
  const int tot = n_seeded * b.nE;
  k_skew_flag<<<(tot + 255) / 256, 256, 0, s>>>(d_acc, n_seeded, d_seeded_ids, b.nE, b.e_base, st);
  launches += 2;
}

// G^r diagonal only (Plan::gr_done_op on): lets its device-to-host copy
// overlap the G^< sweep.
__global__ void k_output_gr(const double2* __restrict__ arena, int64_t stride, int nE, int n,
                            const int64_t* __restrict__ gr_pos, double2* gr) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= n) return;
  const int64_t pr = gr_pos[d];
  for (int e = 0; e < nE; ++e) gr[int64_t(e) * n + d] = arena[int64_t(e) * stride + pr];
}

void launch_output_gr(const BatchArgs& b, int n, const int64_t* d_gr_pos, double2* d_gr, cudaStream_t s,
                      int64_t& launches) {
  k_output_gr<<<(n + 255) / 256, 256, 0, s>>>(b.arena, b.stride, b.nE, n, d_gr_pos, d_gr);
  ++launches;
}

void launch_output(const BatchArgs& b, int n, const int64_t* d_gr_pos, const int64_t* d_gl_pos,
                   const double* d_weights, double2* d_gr, double2* d_gl, double* d_density,
                   DevStatus* st, cudaStream_t s, int64_t& launches) {
  k_output<<<(n + 255) / 256, 256, 0, s>>>(b.arena, b.stride, b.nE, b.e_base, n, d_gr_pos, d_gl_pos,
                                           d_weights, d_gr, d_gl, d_density, st);
  ++launches;
}

}  // namespace negfb
