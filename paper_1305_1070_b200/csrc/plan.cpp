// Host plan construction (see plan.hpp).  Reference anchors per step are
// given inline; all of this runs once per device, never per energy.
#include "plan.hpp"

#include <limits>

#include <cstdlib>

#include <algorithm>
#include <map>
#include <numeric>
#include <set>
#include <unordered_map>

namespace negfb {

namespace {

int64_t align8(int64_t x) { return (x + 7) & ~int64_t(7); }

int find_pos(const std::vector<int>& v, int x) {
  for (std::size_t i = 0; i < v.size(); ++i)
    if (v[i] == x) return static_cast<int>(i);
  return -1;
}

// Keeps `list` in ancestor order (nearest first) while inserting j.
void insert_anc_order(std::vector<int>& list, const Tree& t, int j) {
  if (find_pos(list, j) >= 0) return;
  const int lj = t.cluster(j).level;
  auto it = list.begin();
  while (it != list.end() && t.cluster(*it).level < lj) ++it;
  list.insert(it, j);
}

struct InvItem {
  int m, cluster, fold_pos;
  int64_t off;
};

struct Builder {
  Plan& P;
  const Tree& t;
  explicit Builder(Plan& p) : P(p), t(p.tree) {}

  int msz(int c) const { return t.cluster(c).size(); }
  int lev(int c) const { return t.cluster(c).level; }
  ClusterInfo& I(int c) { return P.ci[static_cast<std::size_t>(c)]; }

  int64_t col_of(const std::vector<int>& cols, const std::vector<int64_t>& offs, int j) const {
    const int p = find_pos(cols, j);
    if (p < 0) fail(kInternal, "plan: missing column block");
    return offs[static_cast<std::size_t>(p)];
  }

  int add_term(std::vector<GemmTerm>& terms, int k, int a_op, int64_t a_off, int lda, int b_op,
               int64_t b_off, int ldb, int sign) {
    GemmTerm g;
    g.k = k;
    g.a_op = a_op;
    g.b_op = b_op;
    g.sign = sign;
    g.lda = lda;
    g.ldb = ldb;
    g.a_off = a_off;
    g.b_off = b_off;
    g.real = 0;
    g.pad = 0;
    terms.push_back(g);
    return static_cast<int>(terms.size()) - 1;
  }

  // Open/close helpers for ops.
  Op cur{};
  void open(int kind, int phase, int level) {
    cur = Op{};
    cur.kind = kind;
    cur.phase = phase;
    cur.level = level;
    switch (kind) {
      case K_INVERSE: cur.begin = static_cast<int>(P.inv_tasks.size()); break;
      case K_GEMM:
        cur.begin = static_cast<int>(P.gemm_tiles.size());
        cur.task_begin = static_cast<int>(P.gemm_tasks.size());
        break;
      case K_DIAG: cur.begin = static_cast<int>(P.diag_tasks.size()); break;
      case K_PANEL:
      case K_BIGSWAP:
      case K_PERM: cur.begin = static_cast<int>(P.big_tasks.size()); break;
      case K_SPSI: cur.begin = static_cast<int>(P.spsi_tasks.size()); break;
      case K_SSCHUR: cur.begin = static_cast<int>(P.sschur_tasks.size()); break;
      case K_LEAFDIAG: cur.begin = static_cast<int>(P.ld_tasks.size()); break;
      case K_MGATHER: cur.begin = static_cast<int>(P.mg_tasks.size()); break;
      default: cur.begin = static_cast<int>(P.scale_tasks.size()); break;
    }
  }
  void close() {
    switch (cur.kind) {
      case K_INVERSE: cur.count = static_cast<int>(P.inv_tasks.size()) - cur.begin; break;
      case K_GEMM:
        cur.count = static_cast<int>(P.gemm_tiles.size()) - cur.begin;
        cur.task_count = static_cast<int>(P.gemm_tasks.size()) - cur.task_begin;
        break;
      case K_DIAG: cur.count = static_cast<int>(P.diag_tasks.size()) - cur.begin; break;
      case K_PANEL:
      case K_BIGSWAP:
      case K_PERM: cur.count = static_cast<int>(P.big_tasks.size()) - cur.begin; break;
      case K_SPSI: cur.count = static_cast<int>(P.spsi_tasks.size()) - cur.begin; break;
      case K_SSCHUR: cur.count = static_cast<int>(P.sschur_tasks.size()) - cur.begin; break;
      case K_LEAFDIAG: cur.count = static_cast<int>(P.ld_tasks.size()) - cur.begin; break;
      case K_MGATHER: cur.count = static_cast<int>(P.mg_tasks.size()) - cur.begin; break;
      default: cur.count = static_cast<int>(P.scale_tasks.size()) - cur.begin; break;
    }
    if (cur.kind == K_GEMM && cur.count > 1) {
      // Longest-processing-time first: the persistent kernel strides over
      // tiles in this order (8-granular live area x summed k).
      auto cost = [&](const GemmTile& tl) {
        const GemmTask& tk = P.gemm_tasks[tl.task];
        int64_t ks = 0;
        for (int q = tk.term_begin; q < tk.term_begin + tk.term_count; ++q) ks += P.gemm_terms[q].k;
        const int64_t lm = std::min(kArrTM[tl.arr], tk.m - tl.m0), ln = std::min(kArrTN[tl.arr], tk.n - tl.n0);
        return ((lm + 7) / 8) * ((ln + 7) / 8) * (ks + 16);
      };
      // one launch per op (tiles carry their arrangement), longest first
      // grouped by arrangement (one launch each), longest first within one
      std::stable_sort(P.gemm_tiles.begin() + cur.begin, P.gemm_tiles.end(),
                       [&](const GemmTile& a, const GemmTile& b) {
                         if (a.arr != b.arr) return a.arr < b.arr;
                         return cost(a) > cost(b);
                       });
    }
    if (cur.count > 0) {
      P.ops.push_back(cur);
      P.exec_cmul += cur.cmul;
    }
  }

  // Fused-diagonal / second-output settings for the next gemm_task.
  static GemmTask no_extra() {
    GemmTask t{};
    t.c2_off = -1;
    return t;
  }
  GemmTask pend_diag = no_extra();

  void gemm_task(int m, int n, int64_t c_off, int ldc, int mode, int64_t init_off, int ld_init,
                 int term_begin) {
    const GemmTask pd = pend_diag;
    pend_diag = no_extra();
    if (m <= 0 || n <= 0) {
      P.gemm_terms.resize(static_cast<std::size_t>(term_begin));
      return;
    }
    GemmTask tk = pd;
    tk.m = m;
    tk.n = n;
    tk.ldc = ldc;
    tk.mode = mode;
    tk.c_off = c_off;
    tk.init_off = init_off;
    tk.ld_init = ld_init;
    tk.term_begin = term_begin;
    tk.term_count = static_cast<int>(P.gemm_terms.size()) - term_begin;
    const int id = static_cast<int>(P.gemm_tasks.size());
    auto ksum_of = [&](const GemmTask& t2) {
      int ks = 0;
      for (int q = t2.term_begin; q < t2.term_begin + t2.term_count; ++q) ks += P.gemm_terms[q].k;
      return ks;
    };
    if (tk.mirror && (m != n || tk.nostore || tk.dmode || tk.c2_off >= 0 || (tk.mirror == 2 && mode != MODE_SET)))
      fail(kInternal, "plan: bad mirror task");
    P.gemm_tasks.push_back(tk);
    // executed work: the entries the tiles compute (a mirrored task computes
    // its upper triangle of 32x32 tiles)
    const double area = tk.mirror ? static_cast<double>(tile_task_sym(id, m, P.gemm_tiles))
                                  : (tile_task(id, m, n, ksum_of(tk), P.gemm_tiles), static_cast<double>(m) * n);
    for (int t2 = tk.term_begin; t2 < tk.term_begin + tk.term_count; ++t2)
      cur.cmul += area * P.gemm_terms[t2].k;
  }

  // Inverses of one group: shared-memory kernels by size class, then the
  // multi-CTA blocked Gauss-Jordan for the large blocks (kPanel-wide panels)
  // with its scratch from `scratch_off` on.
  void emit_inverses(int l, int phase, const std::vector<InvItem>& items, int64_t scratch_off) {
    auto& T = P.gemm_terms;
    open(K_INVERSE, phase, l);
    // Grouped by kernel variant (one launch each), largest blocks first
    // within a variant so the longest CTAs start first.
    std::vector<InvItem> order(items.begin(), items.end());
    std::stable_sort(order.begin(), order.end(), [&](const InvItem& a, const InvItem& b) {
      const int ca = inv_size_class(a.m), cb = inv_size_class(b.m);
      if (ca != cb) return ca < cb;
      return a.m > b.m;
    });
    for (const InvItem& it : order)
      if (it.m > 0 && it.m <= kSmemInvMax) {
        P.inv_tasks.push_back(InvTask{it.m, it.cluster, it.fold_pos, 0, it.off});
        cur.cmul += double(it.m) * it.m * it.m;
      }
    close();
    std::vector<BigTask> big;
    int64_t so = scratch_off;
    int mmax = 0;
    for (const InvItem& it : items) {
      const int m = it.m;
      if (m <= kSmemInvMax) continue;
      BigTask bt{};
      bt.m = m;
      bt.fold_pos = it.fold_pos;
      bt.cluster = it.cluster;
      bt.off = it.off;
      bt.off_mp = so;
      so += align8(int64_t(m) * kPanel);
      bt.off_rs = so;
      so += align8(int64_t(m) * kPanel);
      bt.off_mp64 = so;
      so += align8(int64_t(m) * kOuter);
      bt.off_rs64 = so;
      so += align8(int64_t(m) * kOuter);
      bt.off_perm = so;
      so += align8((3 * int64_t(m) + 3) / 4);
      bt.off_thr = so;
      so += 8;
      big.push_back(bt);
      mmax = std::max(mmax, m);
    }
    if (big.empty()) return;
    for (int o0 = 0; o0 < mmax; o0 += kOuter) {
      for (int k0 = o0; k0 < o0 + kOuter && k0 < mmax; k0 += kPanel) {
        open(K_PANEL, phase, l);
        cur.k0 = k0;
        cur.k1 = o0;
        for (const BigTask& bt : big)
          if (bt.m > k0) {
            P.big_tasks.push_back(bt);
            cur.cmul += double(bt.m) * kPanel * kPanel;
          }
        close();
        // rank-kPanel update of the outer panel's other columns:
        // A[:, o0:oe] += (M_p - I_p) R_p (R_p is zero on the inner panel)
        open(K_GEMM, phase, l);
        cur.inv_update = 1;
        for (const BigTask& bt : big) {
          const int oe = std::min(o0 + kOuter, bt.m);
          if (bt.m <= k0 || oe - o0 <= kPanel) continue;
          const int tb = static_cast<int>(T.size());
          add_term(T, kPanel, OP_N, bt.off_mp, kPanel, OP_N, bt.off_rs + o0, bt.m, +1);
          gemm_task(bt.m, oe - o0, bt.off + o0, bt.m, MODE_ADD, 0, 0, tb);
        }
        close();
      }
      open(K_BIGSWAP, phase, l);
      cur.k1 = o0;
      for (const BigTask& bt : big)
        if (bt.m > o0 && bt.m > kOuter) P.big_tasks.push_back(bt);
      close();
      // rank-kOuter update of every other column: A += (M_P - I_P) R_P
      open(K_GEMM, phase, l);
      cur.inv_update = 1;
      for (const BigTask& bt : big) {
        if (bt.m <= o0 || bt.m <= kOuter) continue;
        const int kb = std::min(kOuter, bt.m - o0);
        const int tb = static_cast<int>(T.size());
        add_term(T, kb, OP_N, bt.off_mp64, kOuter, OP_N, bt.off_rs64, bt.m, +1);
        gemm_task(bt.m, bt.m, bt.off, bt.m, MODE_ADD, 0, 0, tb);
      }
      close();
    }
    open(K_PERM, phase, l);
    for (const BigTask& bt : big) P.big_tasks.push_back(bt);
    close();
  }
};

}  // namespace

namespace {
// Tile cost in units of one full 32x32 tile-chunk: kTileFixed for issuing
// and synchronising the chunk regardless of content, the rest per live 8x8
// subtile (16 per tile).  Measured with tools/gemm_bench: an 8x8 live tile
// costs 0.40 of a full one.
double tile_fixed() {  // NEGF_TILE_FIXED overrides (A/B)
  static const double v = [] {
    const char* e = std::getenv("NEGF_TILE_FIXED");
    return e ? std::atof(e) : 0.36;
  }();
  return v;
}
double tile_cost(int arr, int m, int n, int m0, int n0) {
  const double kTileFixed = tile_fixed();
  const int wr = arr == 1 ? 1 : arr == 2 ? 4 : 2, wc = 4 / wr;
  int live = 0;
  for (int a = 0; a < wr; ++a)
    for (int b = 0; b < wc; ++b) {
      const int li = std::min(2, std::max(0, (m - m0 - 16 * a + 7) / 8));
      const int lj = std::min(2, std::max(0, (n - n0 - 16 * b + 7) / 8));
      live += li * lj;
    }
  return kTileFixed + (1.0 - kTileFixed) * live / 16.0;
}
// Tiles of arrangement `arr` over rows [r0, r1) x cols [c0, c1) of an m x n task.
double grid_tiles(int arr, int m, int n, int r0, int r1, int c0, int c1, int task, std::vector<GemmTile>* out) {
  double cost = 0.0;
  for (int y = r0; y < r1; y += kArrTM[arr])
    for (int x = c0; x < c1; x += kArrTN[arr]) {
      cost += tile_cost(arr, std::min(m, r1), std::min(n, c1), y, x);
      if (out) out->push_back(GemmTile{task, y, x, arr});
    }
  return cost;
}
}  // namespace

void tile_task(int task, int m, int n, int ksum, std::vector<GemmTile>& out) {
  // Small tasks (at most 16 rows, summed depth at most 256: the 6-13-dof
  // separators of levels 2-4 on config 2): warp tiles (arr 3), one warp per
  // 16 x 16 block with register fragments straight from L2 / HBM -- measured
  // 6.3 ms less per config-2 batch than the CTA tiles; the depth bound was 64
  // before the real-operand terms halved the DMMA work (256: another 0.9 ms;
  // 32- or 48-row tasks on warp tiles: 2 ms more).  Taller tasks keep the
  // staged CTA tiles.
  // NEGF_WARP_TILE_M / _K override the bounds (A/B experiments; M = 0 disables).
  static const int warp_m = [] {
    const char* e = std::getenv("NEGF_WARP_TILE_M");
    return e ? std::atoi(e) : 16;
  }();
  static const int warp_k = [] {
    const char* e = std::getenv("NEGF_WARP_TILE_K");
    return e ? std::atoi(e) : 256;
  }();
  if (m <= warp_m && ksum <= warp_k) {
    for (int y = 0; y < m; y += 16)
      for (int x = 0; x < n; x += 16) out.push_back(GemmTile{task, y, x, 3});
    return;
  }
  // Uniform grids.
  int best_arr = 0;
  double best = -1.0;
  for (int a : {0, 1, 2}) {
    const double c = grid_tiles(a, m, n, 0, m, 0, n, task, nullptr);
    if (best < 0 || c < best - 1e-9) {
      best = c;
      best_arr = a;
    }
  }
  // 32x32 core + remainder strips.
  const int M32 = (m / 32) * 32, N32 = (n / 32) * 32;
  int bot_arr = -1, rgt_arr = -1;
  double mixed = -1.0;
  if ((M32 > 0 || N32 > 0) && (M32 < m || N32 < n)) {
    mixed = grid_tiles(0, m, n, 0, M32, 0, N32, task, nullptr);
    if (M32 < m) {  // bottom strip, full width
      double bc = -1.0;
      for (int a : {0, 1}) {
        const double c = grid_tiles(a, m, n, M32, m, 0, n, task, nullptr);
        if (bc < 0 || c < bc - 1e-9) { bc = c; bot_arr = a; }
      }
      mixed += bc;
    }
    if (N32 < n && M32 > 0) {  // right strip above the bottom strip
      // 64x16 tiles must not reach into the bottom strip (MODE_ADD tasks
      // may not compute an entry twice): a 32-row remainder takes 32x32.
      const int M64 = (M32 / 64) * 64;
      const double c0 = grid_tiles(0, M32, n, 0, M32, N32, n, task, nullptr);
      const double c2 = grid_tiles(2, M32, n, 0, M64, N32, n, task, nullptr) +
                        grid_tiles(0, M32, n, M64, M32, N32, n, task, nullptr);
      rgt_arr = c2 < c0 - 1e-9 ? 2 : 0;
      mixed += std::min(c0, c2);
    }
  }
  if (mixed >= 0 && mixed < best - 1e-9) {
    grid_tiles(0, m, n, 0, M32, 0, N32, task, &out);
    if (M32 < m) grid_tiles(bot_arr, m, n, M32, m, 0, n, task, &out);
    if (N32 < n && M32 > 0) {
      if (rgt_arr == 2) {
        const int M64 = (M32 / 64) * 64;
        grid_tiles(2, M32, n, 0, M64, N32, n, task, &out);
        grid_tiles(0, M32, n, M64, M32, N32, n, task, &out);
      } else {
        grid_tiles(0, M32, n, 0, M32, N32, n, task, &out);
      }
    }
  } else {
    grid_tiles(best_arr, m, n, 0, m, 0, n, task, &out);
  }
}

int64_t tile_task_sym(int task, int m, std::vector<GemmTile>& out) {
  int64_t area = 0;
  for (int y = 0; y < m; y += 32)
    for (int x = y; x < m; x += 32) {
      out.push_back(GemmTile{task, y, x, 0});
      area += int64_t(std::min(32, m - y)) * std::min(32, m - x);
    }
  return area;
}

namespace {
// Exact-arithmetic rewrite forms of the plan.  On by default:
// symdiag_g / symdiag_p (each off-diagonal block pair of a diagonal-only
// quadratic form once, from 2 Psi), sparse (stencil-entry leaf Psi / Schur
// contributions), hull (structural zero columns skipped), compact (the
// diagonal-only rows of sparse leaves as one gathered Psi_H M Psi_H^T form per
// leaf, MGatherTask; hull only, so exact zeros are all it skips), real (blocks
// that are real for every energy -- mark_real_operands -- skip the products
// with their zero imaginary parts: bit-identical results).  Off by default,
// because they measurably lose accuracy against the dense truth at
// ill-conditioned energies (profiles/parity_forms_r02.txt):
// mirror_schur / mirror_g / mirror_p (upper triangle of a symmetric /
// anti-Hermitian block computed, the lower one copied) and woodbury (leaf
// diagonals from diag(inv) + diag(W M W^T)).  NEGF_PLAN_FORMS (a comma list)
// replaces the set for A/B experiments.
bool form_on(const char* name) {
  const char* e = std::getenv("NEGF_PLAN_FORMS");
  const std::string s = std::string(",") + (e ? e : "symdiag_g,symdiag_p,sparse,hull,compact,real") + ",";
  return s.find(std::string(",") + name + ",") != std::string::npos;
}
}  // namespace

// Real blocks.  With a real Hamiltonian, A(E) = E - H - Sigma^r(E) is complex
// only through Sigma^r, which touches the contact (and phonon) dofs.  A
// cluster none of whose dofs, and none of whose descendants' dofs, carries a
// Sigma^r entry is eliminated in real arithmetic: A_xx, A_{x,S}, their Schur
// fill (all from such descendants), A_xx^-1 and Psi_x have exactly zero
// imaginary parts at every energy, whatever values the caller passes.  GEMM
// terms reading those regions are flagged (GemmTerm::real) and skip the DMMAs
// whose factor is that zero; flagged inverses run the real kernel.  Skipped
// products are exact zeros, so every result is bit-identical to the complex
// evaluation.  The executed-work ledger counts a real x complex term at half
// and a real x real term or a real inverse at a quarter of the complex cost.
static void mark_real_operands(Plan& P) {
  const ProblemDesc& d = P.desc;
  for (const cplx& v : d.h_vals)
    if (v.imag() != 0.0) return;
  const Tree& t = P.tree;
  const int nc = t.num_clusters();
  std::vector<int> cl_of(static_cast<std::size_t>(d.n), -1);
  for (int c = 0; c < nc; ++c)
    for (int v : t.cluster(c).dofs) cl_of[static_cast<std::size_t>(v)] = c;
  std::vector<char> real(static_cast<std::size_t>(nc), 1);
  for (std::size_t k = 0; k < d.sr_rows.size(); ++k) {
    real[static_cast<std::size_t>(cl_of[static_cast<std::size_t>(d.sr_rows[k])])] = 0;
    real[static_cast<std::size_t>(cl_of[static_cast<std::size_t>(d.sr_cols[k])])] = 0;
  }
  // a complex cluster makes every ancestor complex (its Schur fill lands there)
  for (int c = 0; c < nc; ++c)
    if (!real[static_cast<std::size_t>(c)])
      for (int a : t.cluster(c).anc) real[static_cast<std::size_t>(a)] = 0;
  // arena regions that hold real data for the whole solve
  std::vector<std::pair<int64_t, int64_t>> iv;
  for (int c = 0; c < nc; ++c) {
    if (!real[static_cast<std::size_t>(c)]) continue;
    const ClusterInfo& X = P.ci[static_cast<std::size_t>(c)];
    const int64_t m = X.m;
    if (X.off_d >= 0) iv.push_back({X.off_d, X.off_d + m * m});
    if (X.off_arow >= 0 && X.K > 0) iv.push_back({X.off_arow, X.off_arow + m * X.K});
    if (X.off_psi >= 0 && X.K > 0) iv.push_back({X.off_psi, X.off_psi + m * X.K});
    if (X.off_psi2 >= 0 && X.K > 0) iv.push_back({X.off_psi2, X.off_psi2 + m * X.K});
    if (X.off_psic >= 0 && X.hc > 0) iv.push_back({X.off_psic, X.off_psic + m * X.hc});
  }
  if (iv.empty()) return;
  std::sort(iv.begin(), iv.end());
  auto is_real = [&](int64_t off) {
    auto it = std::upper_bound(iv.begin(), iv.end(), std::make_pair(off, std::numeric_limits<int64_t>::max()));
    if (it == iv.begin()) return false;
    --it;
    return off >= it->first && off < it->second;
  };
  for (GemmTerm& g : P.gemm_terms) g.real = (is_real(g.a_off) ? 1 : 0) | (is_real(g.b_off) ? 2 : 0);
  for (InvTask& it : P.inv_tasks) it.real = real[static_cast<std::size_t>(it.cluster)] ? 1 : 0;
  // executed work
  P.needed_cmul = P.exec_cmul;
  for (int c = 0; c < nc; ++c) P.n_real_clusters += real[static_cast<std::size_t>(c)] ? 1 : 0;
  P.exec_cmul = 0.0;
  for (Op& op : P.ops) {
    if (op.kind == K_GEMM && !op.inv_update) {
      std::vector<double> area(static_cast<std::size_t>(op.task_count), 0.0);
      for (int q = op.begin; q < op.begin + op.count; ++q) {
        const GemmTile& tl = P.gemm_tiles[static_cast<std::size_t>(q)];
        const GemmTask& tk = P.gemm_tasks[static_cast<std::size_t>(tl.task)];
        const int lm = std::min(kArrTM[tl.arr], tk.m - tl.m0), ln = std::min(kArrTN[tl.arr], tk.n - tl.n0);
        area[static_cast<std::size_t>(tl.task - op.task_begin)] += double(lm) * ln;
      }
      double cm = 0.0;
      for (int a = 0; a < op.task_count; ++a) {
        const GemmTask& tk = P.gemm_tasks[static_cast<std::size_t>(op.task_begin + a)];
        for (int q = tk.term_begin; q < tk.term_begin + tk.term_count; ++q) {
          const GemmTerm& g = P.gemm_terms[static_cast<std::size_t>(q)];
          const double wgt = g.real == 3 ? 0.25 : g.real ? 0.5 : 1.0;
          cm += area[static_cast<std::size_t>(a)] * g.k * wgt;
        }
      }
      op.cmul = cm;
    } else if (op.kind == K_INVERSE) {
      double cm = 0.0;
      for (int q = op.begin; q < op.begin + op.count; ++q) {
        const InvTask& it = P.inv_tasks[static_cast<std::size_t>(q)];
        cm += double(it.m) * it.m * it.m * (it.real ? 0.25 : 1.0);
      }
      op.cmul = cm;
    }
    P.exec_cmul += op.cmul;
  }
  P.exec_inv_cmul = 0.0;
  for (int c = 0; c < nc; ++c) {
    const double m = t.cluster(c).size();
    P.exec_inv_cmul += m * m * m * ((real[static_cast<std::size_t>(c)] && m <= kSmemInvMax) ? 0.25 : 1.0);
  }
}

Plan build_plan(ProblemDesc desc) {
  Plan P;
  P.desc = std::move(desc);
  // The symmetric forms need A(E) complex symmetric, as the reference's lean
  // fold already assumes (it reads only the (descendant, ancestor)
  // orientation, hsc.cpp:483-490): H symmetric in values, Sigma^r in pattern
  // (its values are the caller's, per energy).  Otherwise they stay off.
  bool a_symmetric = true;
  {
    std::map<std::pair<int, int>, cplx> hm;
    for (std::size_t k = 0; k < P.desc.h_rows.size(); ++k) hm[{P.desc.h_rows[k], P.desc.h_cols[k]}] += P.desc.h_vals[k];
    for (const auto& kv : hm) {
      auto it = hm.find({kv.first.second, kv.first.first});
      if (it == hm.end() || it->second != kv.second) {
        a_symmetric = false;
        break;
      }
    }
    std::set<std::pair<int, int>> sp;
    for (std::size_t k = 0; k < P.desc.sr_rows.size(); ++k) sp.insert({P.desc.sr_rows[k], P.desc.sr_cols[k]});
    for (const auto& e : sp)
      if (!sp.count({e.second, e.first})) a_symmetric = false;
  }
  const bool f_mirror_schur = a_symmetric && form_on("mirror_schur"), f_mirror_g = a_symmetric && form_on("mirror_g"),
             f_mirror_p = a_symmetric && form_on("mirror_p"), f_symdiag_g = a_symmetric && form_on("symdiag_g"),
             f_symdiag_p = a_symmetric && form_on("symdiag_p"), f_woodbury = form_on("woodbury"),
             f_sparse = form_on("sparse"), f_hull = form_on("hull"), f_compact = form_on("compact");
  const ProblemDesc& d = P.desc;
  const int n = d.n;
  if (n <= 0) fail(kContractViolation, "problem: no dofs");
  if (d.h_rows.size() != d.h_cols.size() || d.h_rows.size() != d.h_vals.size())
    fail(kContractViolation, "problem: H arrays disagree in length");
  if (d.sr_rows.size() != d.sr_cols.size() || d.sl_rows.size() != d.sl_cols.size())
    fail(kContractViolation, "problem: self-energy pattern arrays disagree in length");
  auto check_idx = [&](const std::vector<int>& v, const char* what) {
    for (int x : v)
      if (x < 0 || x >= n) fail(kContractViolation, std::string("problem: ") + what + " index out of range");
  };
  check_idx(d.h_rows, "H");
  check_idx(d.h_cols, "H");
  check_idx(d.sr_rows, "sigma_r");
  check_idx(d.sr_cols, "sigma_r");
  check_idx(d.sl_rows, "sigma_lesser");
  check_idx(d.sl_cols, "sigma_lesser");

  // ---- tree (run.cpp:123-133: graph of A's pattern, atomic contact groups)
  std::vector<std::pair<int, int>> pat;
  pat.reserve(d.h_rows.size() + d.sr_rows.size());
  for (std::size_t k = 0; k < d.h_rows.size(); ++k) pat.push_back({d.h_rows[k], d.h_cols[k]});
  for (std::size_t k = 0; k < d.sr_rows.size(); ++k) pat.push_back({d.sr_rows[k], d.sr_cols[k]});
  P.graph = graph_of_pattern(n, pat);
  if (d.explicit_tree) {
    if (d.tree_parent.size() != d.tree_dofs.size())
      fail(kContractViolation, "problem: explicit tree arrays disagree");
    std::vector<Cluster> cs(d.tree_parent.size());
    for (std::size_t i = 0; i < cs.size(); ++i) {
      cs[i].parent = d.tree_parent[i];
      cs[i].dofs = d.tree_dofs[i];
    }
    P.tree = Tree::build(std::move(cs), n);
  } else {
    P.tree = nested_dissection(P.graph, d.atomic_groups, d.max_leaf, d.coords);
  }
  const Tree& t = P.tree;
  const int nc = t.num_clusters();
  P.ci.assign(static_cast<std::size_t>(nc), ClusterInfo{});
  Builder B(P);
  for (int c = 0; c < nc; ++c) {
    B.I(c).m = t.cluster(c).size();
    P.max_block = std::max(P.max_block, B.I(c).m);
  }

  // ---- partition rule (block.cpp:55-72): every A entry joins related clusters
  {
    int bad = 0;
    for (const auto& e : pat) {
      const int ci = t.dof_cluster(e.first), cj = t.dof_cluster(e.second);
      if (ci == cj || t.is_ancestor(cj, ci) || t.is_ancestor(ci, cj)) continue;
      if (e.first < e.second) ++bad;
    }
    if (bad) fail(kPartitionViolation, std::to_string(bad) +
                                           " matrix entr(ies) join clusters that are not ancestor-related");
  }
  // Sigma^< must be cluster-block-diagonal (hsc.cpp:104-107).
  for (std::size_t k = 0; k < d.sl_rows.size(); ++k)
    if (t.dof_cluster(d.sl_rows[k]) != t.dof_cluster(d.sl_cols[k]))
      fail(kContractViolation, "sigma_lesser must be block diagonal on the cluster partition");

  // ---- symbolic fold (hsc.cpp:482-511): S0 from the (descendant, ancestor)
  // orientation of A's pattern, then fill of every ancestor pair.
  std::vector<std::set<int>> S0(static_cast<std::size_t>(nc));
  for (const auto& e : pat) {
    const int ci = t.dof_cluster(e.first), cj = t.dof_cluster(e.second);
    if (ci != cj && t.is_ancestor(cj, ci)) S0[ci].insert(cj);
  }
  for (int c = 0; c < nc; ++c)
    for (int j : t.cluster(c).anc)
      if (S0[c].count(j)) B.I(c).S.push_back(j);
  for (int i : t.fold_order()) {
    const std::vector<int> js = B.I(i).S;  // complete: all descendants folded
    for (std::size_t p = 0; p < js.size(); ++p)
      for (std::size_t q = p + 1; q < js.size(); ++q) insert_anc_order(B.I(js[p]).S, t, js[q]);
  }
  // Column layout of Arow_x / Psi_x: blocks holding original entries of A
  // first (initialised per energy), pure fill blocks after them (written by
  // their gather task, never initialised).  S itself stays in ancestor order.
  for (int c = 0; c < nc; ++c) {
    ClusterInfo& ci = B.I(c);
    ci.s_col.assign(ci.S.size(), 0);
    ci.s_orig.assign(ci.S.size(), 0);
    int64_t off = 0;
    for (int pass = 0; pass < 2; ++pass)
      for (std::size_t q = 0; q < ci.S.size(); ++q) {
        const bool orig = S0[c].count(ci.S[q]) != 0;
        if (orig != (pass == 0)) continue;
        ci.s_col[q] = off;
        ci.s_orig[q] = orig ? 1 : 0;
        off += B.msz(ci.S[q]);
        if (orig) ci.K0 = static_cast<int>(off);
      }
    for (int j : ci.S) B.I(j).referenced = true;
    ci.K = static_cast<int>(off);
  }

  // ---- Sigma^< structure (hsc.cpp:89-125): seeded clusters, dense or diagonal
  for (std::size_t k = 0; k < d.sl_rows.size(); ++k) {
    const int c = t.dof_cluster(d.sl_rows[k]);
    B.I(c).seeded = true;
    if (d.sl_rows[k] != d.sl_cols[k]) B.I(c).seed_dense = true;
    P.any_seed = true;
  }

  // ---- needed-block closure for the top-down sweeps
  const int root = t.root();
  {
    std::vector<std::set<int>> needG(static_cast<std::size_t>(nc)), needP(static_cast<std::size_t>(nc));
    for (int c = 0; c < nc; ++c) {
      if (c == root) continue;
      for (int j : B.I(c).S) {
        needG[c].insert(j);
        needP[c].insert(j);
      }
      if (B.I(c).seeded)
        for (int j : t.cluster(c).anc) needG[c].insert(j);
    }
    auto propagate = [&](std::vector<std::set<int>>& need, int y) {
      for (int j : need[y])
        for (int k : B.I(y).S) {
          if (k == j) continue;
          if (B.lev(k) < B.lev(j)) need[k].insert(j);
          else need[j].insert(k);
        }
    };
    for (int y : t.fold_order()) {
      propagate(needG, y);
      propagate(needP, y);
    }
    for (int c = 0; c < nc; ++c) {
      ClusterInfo& ci = B.I(c);
      for (int j : t.cluster(c).anc) {
        if (needG[c].count(j)) ci.gcols.push_back(j);
        if (needP[c].count(j)) ci.pcols.push_back(j);
      }
      ci.full_g = ci.referenced || ci.seeded || c == root;
      ci.full_p = ci.referenced || c == root;
    }
  }
  // ---- N structure (hsc.cpp:229-266)
  {
    std::vector<std::vector<int>> ncols(static_cast<std::size_t>(nc));
    for (int c = 0; c < nc; ++c)
      if (B.I(c).seeded) {
        ncols[c] = t.cluster(c).anc;
        B.I(c).has_nd = true;
      }
    for (int i : t.fold_order()) {
      if (ncols[i].empty()) continue;
      for (int j : B.I(i).S)
        for (int k : ncols[i]) {
          if (B.lev(k) < B.lev(j)) continue;
          if (k == j) B.I(j).has_nd = true;
          else insert_anc_order(ncols[j], t, k);
        }
    }
    for (int c = 0; c < nc; ++c) B.I(c).ncols = ncols[c];
  }
  for (int c = 0; c < nc; ++c) {
    ClusterInfo& ci = B.I(c);
    auto offs = [&](const std::vector<int>& cols, std::vector<int64_t>& o, int& w) {
      int64_t acc = 0;
      for (int j : cols) {
        o.push_back(acc);
        acc += B.msz(j);
      }
      w = static_cast<int>(acc);
    };
    offs(ci.gcols, ci.gcol_off, ci.WG);
    offs(ci.ncols, ci.ncol_off, ci.WN);
    offs(ci.pcols, ci.pcol_off, ci.WP);
  }

  // ---- arena layout (complex elements per energy)
  int64_t cur = 0;
  auto take = [&](int64_t cnt) {
    const int64_t o = cur;
    cur = align8(cur + cnt);
    return o;
  };
  for (int c = 0; c < nc; ++c) B.I(c).off_d = take(int64_t(B.msz(c)) * B.msz(c));
  for (int c = 0; c < nc; ++c)
    if (B.I(c).K) B.I(c).off_arow = take(int64_t(B.msz(c)) * B.I(c).K);
  P.a_region = cur;
  P.z_begin = cur;
  for (int c = 0; c < nc; ++c) {
    ClusterInfo& ci = B.I(c);
    if (!ci.seeded) continue;
    ci.off_sig = take(ci.seed_dense ? int64_t(ci.m) * ci.m : int64_t(ci.m));
  }
  for (int c = 0; c < nc; ++c) {
    ClusterInfo& ci = B.I(c);
    if (ci.has_nd) ci.off_nd = take(int64_t(ci.m) * ci.m);
    if (ci.WN) ci.off_nrow = take(int64_t(ci.m) * ci.WN);
  }
  if (P.any_seed) B.I(root).off_pd = take(int64_t(B.msz(root)) * B.msz(root));
  P.z_end = cur;
  for (int c = 0; c < nc; ++c) {
    ClusterInfo& ci = B.I(c);
    if (ci.K) ci.off_psi = take(int64_t(ci.m) * ci.K);
    // 2 Psi for never-referenced, unseeded clusters: diag(G_xx) = diag(inv) +
    // diag(Psi G_SS Psi^T) with G_SS complex symmetric, so each off-diagonal
    // block pair enters once, doubled (see the G-row loop)
    if (ci.K && !ci.full_g && c != root) ci.off_psi2 = take(int64_t(ci.m) * ci.K);
    if (c == root) ci.off_gd = ci.off_d;  // G_rr = (A_rr folded)^-1 (hsc.cpp:148-150)
    else ci.off_gd = take(ci.full_g ? int64_t(ci.m) * ci.m : int64_t(ci.m));
    if (P.any_seed && c != root) ci.off_pd = take(ci.full_p ? int64_t(ci.m) * ci.m : int64_t(ci.m));
  }
  // Row storage, by liveness.  The multi-CTA inverse scratch lives only in
  // the fold, G rows from the G^r sweep to the seeds (hsc.cpp:229-237), P rows
  // from the P sweep on -- so all three share one region.  Rows of
  // never-referenced clusters feed only their diagonal (fused into the row
  // tasks' epilogue, GemmTask::dmode): never stored, no storage.
  const int64_t rows_begin = cur;
  for (int c = 0; c < nc; ++c) {
    ClusterInfo& ci = B.I(c);
    const bool g_fused = !ci.full_g && c != root;
    if (ci.WG) ci.off_grow = g_fused ? 0 : take(int64_t(ci.m) * ci.WG);
  }
  {
    int64_t pc = rows_begin;
    for (int c = 0; c < nc; ++c) {
      ClusterInfo& ci = B.I(c);
      const bool p_fused = !ci.full_p && c != root;
      if (P.any_seed && ci.WP && !p_fused) {
        ci.off_prow = pc;
        pc = align8(pc + int64_t(ci.m) * ci.WP);
      } else if (P.any_seed && ci.WP) {
        ci.off_prow = 0;
      }
    }
    cur = std::max(cur, pc);
  }
  // Scratch of the multi-CTA inverse (fold only), reused level after level.
  {
    std::vector<int64_t> need(static_cast<std::size_t>(t.levels()) + 1, 0);
    for (int c = 0; c < nc; ++c) {
      const int64_t m = B.msz(c);
      if (m <= kSmemInvMax) continue;
      need[B.lev(c)] += big_scratch_elems(m);
    }
    P.big_scratch = rows_begin;
    cur = std::max(cur, align8(rows_begin + *std::max_element(need.begin(), need.end())));
  }
  P.arena = std::max<int64_t>(cur, 8);
  // Per-energy initialisation: D blocks and the original-entry prefix of each
  // Arow row come from the template; Sigma^< blocks and (without N_rr) the
  // root's P block are zeroed.  Everything else is written before it is read.
  for (int c = 0; c < nc; ++c) {
    const ClusterInfo& I = B.I(c);
    if (I.m == 0) continue;
    P.init_zero.push_back(InitRegion{I.off_d, 1, I.m * I.m, I.m * I.m});
    if (I.K0 > 0) P.init_zero.push_back(InitRegion{I.off_arow, I.m, I.K0, I.K});
    if (I.seeded) P.init_zero.push_back(InitRegion{I.off_sig, 1, I.seed_dense ? I.m * I.m : I.m, 0});
  }
  if (P.any_seed && !B.I(root).has_nd && B.msz(root) > 0)
    P.init_zero.push_back(InitRegion{B.I(root).off_pd, 1, B.msz(root) * B.msz(root), 0});

  // ---- -H as (position, value) pairs in the descendant-row orientation (the
  // only one the lean fold reads, hsc.cpp:483-490); duplicates summed.
  auto a_pos = [&](int r, int c) -> int64_t {
    const int ci = t.dof_cluster(r), cj = t.dof_cluster(c);
    const int lr = t.local_index(r), lc = t.local_index(c);
    const ClusterInfo& I = P.ci[ci];
    if (ci == cj) return I.off_d + int64_t(lr) * I.m + lc;
    const int p = find_pos(I.S, cj);
    if (p < 0) return -1;  // ancestor-row orientation: never read
    return I.off_arow + int64_t(lr) * I.K + I.s_col[p] + lc;
  };
  {
    std::vector<std::pair<int64_t, cplx>> hv;
    hv.reserve(d.h_rows.size());
    for (std::size_t k = 0; k < d.h_rows.size(); ++k) {
      const int64_t pos = a_pos(d.h_rows[k], d.h_cols[k]);
      if (pos >= 0) hv.push_back({pos, -d.h_vals[k]});
    }
    std::stable_sort(hv.begin(), hv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& e : hv) {
      if (!P.h_pos.empty() && P.h_pos.back() == e.first) P.h_val.back() += e.second;
      else {
        P.h_pos.push_back(e.first);
        P.h_val.push_back(e.second);
      }
    }
  }
  P.diag_pos.resize(static_cast<std::size_t>(n));
  for (int dof = 0; dof < n; ++dof) {
    const ClusterInfo& I = P.ci[t.dof_cluster(dof)];
    P.diag_pos[dof] = I.off_d + int64_t(t.local_index(dof)) * (I.m + 1);
  }
  // Sigma^r slots (duplicates summed, coo_normalize semantics).
  {
    std::map<int64_t, std::vector<int>> by_pos;
    for (std::size_t k = 0; k < d.sr_rows.size(); ++k) {
      const int64_t pos = a_pos(d.sr_rows[k], d.sr_cols[k]);
      if (pos >= 0) by_pos[pos].push_back(static_cast<int>(k));
    }
    P.sr_slot_ptr.push_back(0);
    for (const auto& kv : by_pos) {
      P.sr_slot_pos.push_back(kv.first);
      for (int s : kv.second) P.sr_slot_src.push_back(s);
      P.sr_slot_ptr.push_back(static_cast<int>(P.sr_slot_src.size()));
    }
  }
  // Sigma^< slots: one per distinct (r, c); partner = slot of (c, r).
  {
    std::map<std::pair<int, int>, std::vector<int>> by_rc;
    for (std::size_t k = 0; k < d.sl_rows.size(); ++k)
      by_rc[{d.sl_rows[k], d.sl_cols[k]}].push_back(static_cast<int>(k));
    std::map<std::pair<int, int>, int> slot_of;
    P.sl_slot_ptr.push_back(0);
    for (const auto& kv : by_rc) {
      const int r = kv.first.first, c = kv.first.second;
      const ClusterInfo& I = P.ci[t.dof_cluster(r)];
      const int lr = t.local_index(r), lc = t.local_index(c);
      slot_of[kv.first] = static_cast<int>(P.sl_slot_pos.size());
      P.sl_slot_pos.push_back(I.seed_dense ? I.off_sig + int64_t(lr) * I.m + lc : I.off_sig + lr);
      P.sl_cluster.push_back(t.dof_cluster(r));
      for (int s : kv.second) P.sl_slot_src.push_back(s);
      P.sl_slot_ptr.push_back(static_cast<int>(P.sl_slot_src.size()));
    }
    for (const auto& kv : by_rc) {
      auto it = slot_of.find({kv.first.second, kv.first.first});
      P.sl_partner.push_back(it == slot_of.end() ? -1 : it->second);
    }
    std::vector<int> cidx(static_cast<std::size_t>(nc), -1);
    for (int c = 0; c < nc; ++c)
      if (B.I(c).seeded) {
        cidx[c] = static_cast<int>(P.seeded_ids.size());
        P.seeded_ids.push_back(c);
      }
    for (int c : P.sl_cluster) P.sl_cidx.push_back(cidx[c]);
    P.cslot_ptr.assign(P.seeded_ids.size() + 1, 0);
    for (int ci2 : P.sl_cidx) ++P.cslot_ptr[ci2 + 1];
    for (std::size_t q = 1; q < P.cslot_ptr.size(); ++q) P.cslot_ptr[q] += P.cslot_ptr[q - 1];
    P.cslots.assign(P.sl_cidx.size(), 0);
    std::vector<int> fillp(P.cslot_ptr.begin(), P.cslot_ptr.end() - 1);
    for (std::size_t s2 = 0; s2 < P.sl_cidx.size(); ++s2) P.cslots[fillp[P.sl_cidx[s2]]++] = static_cast<int>(s2);
  }
  P.out_gr_pos.resize(static_cast<std::size_t>(n));
  P.out_gl_pos.resize(static_cast<std::size_t>(n));
  for (int dof = 0; dof < n; ++dof) {
    const int c = t.dof_cluster(dof);
    const ClusterInfo& I = P.ci[c];
    const int l = t.local_index(dof);
    P.out_gr_pos[dof] = I.off_gd + (I.full_g ? int64_t(l) * (I.m + 1) : l);
    P.out_gl_pos[dof] = P.any_seed ? I.off_pd + (I.full_p ? int64_t(l) * (I.m + 1) : l) : -1;
  }

  // ---- schedule
  std::vector<std::vector<int>> by_level(static_cast<std::size_t>(t.levels()) + 1);
  for (int c : t.fold_order()) by_level[B.lev(c)].push_back(c);
  std::vector<int> fold_pos(static_cast<std::size_t>(nc), nc - 1);
  for (std::size_t k = 0; k < t.fold_order().size(); ++k) fold_pos[t.fold_order()[k]] = static_cast<int>(k);
  auto& T = P.gemm_terms;

  // Fold (hsc.cpp:473-526), level by level, in left-looking form: right
  // before the clusters of level l are inverted, every Schur contribution
  // they will ever receive is gathered in one task per target block,
  //   A_{x,q} += sum_{y : x,q in S(y)} Psi_{y,x}^T A_{y,q}     (q = x or q in S(x)),
  // with the contributors y (all below x, already folded, rows final) in
  // fold order.  The sum is the reference's right-looking update
  // (hsc.cpp:501-511) reassociated: the same terms, each target written once.
  std::vector<std::map<std::pair<int, int>, std::vector<std::array<int, 3>>>> schur(
      static_cast<std::size_t>(t.levels()) + 1);
  for (int y : t.fold_order()) {
    const auto& js = B.I(y).S;
    for (std::size_t p = 0; p < js.size(); ++p)
      for (std::size_t q = p; q < js.size(); ++q)
        schur[B.lev(js[p])][{js[p], js[q]}].push_back({y, static_cast<int>(p), static_cast<int>(q)});
  }
  // Inverses of one level: shared-memory kernels by size class, then the
  // multi-CTA blocked Gauss-Jordan for the large blocks (kPanel-wide panels).
  auto emit_inverses = [&](int l, const std::vector<int>& xs) {
    std::vector<InvItem> items;
    for (int x : xs) items.push_back(InvItem{B.msz(x), x, fold_pos[x], B.I(x).off_d});
    B.emit_inverses(l, 0, items, P.big_scratch);
  };
  // Leaves whose coupling block A_{x,S(x)} is the -H template alone: no Schur
  // fill (no descendants), every S entry original, no Sigma^r slot inside it.
  // Their Psi is formed from the stencil entries (K_SPSI).
  std::vector<char> leaf_sparse(static_cast<std::size_t>(nc), 0);
  std::vector<std::vector<std::vector<std::pair<int, cplx>>>> leaf_cols(static_cast<std::size_t>(nc));
  {
    std::vector<std::pair<int64_t, int>> arows;  // (off_arow, cluster) of candidate leaves
    for (int c = 0; c < nc; ++c) {
      const ClusterInfo& I = B.I(c);
      if (!t.cluster(c).children.empty() || c == root || I.K == 0 || I.K0 != I.K) continue;
      bool orig = true;
      for (char o : I.s_orig) orig = orig && o;
      if (!orig) continue;
      if (!f_sparse) continue;
      leaf_sparse[static_cast<std::size_t>(c)] = 1;
      leaf_cols[static_cast<std::size_t>(c)].resize(static_cast<std::size_t>(I.K));
      arows.push_back({I.off_arow, c});
    }
    std::sort(arows.begin(), arows.end());
    auto owner = [&](int64_t pos) -> int {  // candidate leaf whose Arow holds pos, or -1
      auto it = std::upper_bound(arows.begin(), arows.end(), std::make_pair(pos, std::numeric_limits<int>::max()));
      if (it == arows.begin()) return -1;
      --it;
      const ClusterInfo& I = B.I(it->second);
      return pos < I.off_arow + int64_t(I.m) * I.K ? it->second : -1;
    };
    for (int64_t pos : P.sr_slot_pos) {
      const int c = owner(pos);
      if (c >= 0) leaf_sparse[static_cast<std::size_t>(c)] = 0;
    }
    for (std::size_t q = 0; q < P.h_pos.size(); ++q) {
      const int c = owner(P.h_pos[q]);
      if (c < 0 || !leaf_sparse[static_cast<std::size_t>(c)]) continue;
      const ClusterInfo& I = B.I(c);
      const int64_t rel = P.h_pos[q] - I.off_arow;
      leaf_cols[static_cast<std::size_t>(c)][static_cast<std::size_t>(rel % I.K)].push_back(
          {static_cast<int>(rel / I.K), P.h_val[q]});
    }
  }
  // Structural nonzero column hull [lo, hi) of every coupling block A_{x,S[q]}
  // (and so of Psi_{x,S[q]} = -inv_x A_{x,S[q]}): the original -H / Sigma^r
  // entries, then, in fold order, the Schur fill A_{jp,jq} += Psi_{x,jp}^T
  // A_{x,jq} whose columns are those of A_{x,jq}.  Columns outside it are
  // exact zeros, so the row products' inner sums skip them.
  std::vector<std::vector<std::array<int, 2>>> nzr(static_cast<std::size_t>(nc));
  {
    std::vector<std::pair<int64_t, int>> ar;
    for (int c = 0; c < nc; ++c) {
      const ClusterInfo& I = B.I(c);
      nzr[static_cast<std::size_t>(c)].resize(I.S.size());
      for (std::size_t q = 0; q < I.S.size(); ++q) nzr[static_cast<std::size_t>(c)][q] = {B.msz(I.S[q]), 0};
      if (I.K > 0 && I.m > 0) ar.push_back({I.off_arow, c});
    }
    std::sort(ar.begin(), ar.end());
    auto mark = [&](int64_t pos) {
      auto it = std::upper_bound(ar.begin(), ar.end(), std::make_pair(pos, std::numeric_limits<int>::max()));
      if (it == ar.begin()) return;
      --it;
      const ClusterInfo& I = B.I(it->second);
      if (pos >= I.off_arow + int64_t(I.m) * I.K) return;
      const int col = static_cast<int>((pos - I.off_arow) % I.K);
      for (std::size_t q = 0; q < I.S.size(); ++q)
        if (col >= I.s_col[q] && col < I.s_col[q] + B.msz(I.S[q])) {
          auto& r = nzr[static_cast<std::size_t>(it->second)][q];
          const int l = static_cast<int>(col - I.s_col[q]);
          r[0] = std::min(r[0], l);
          r[1] = std::max(r[1], l + 1);
          return;
        }
    };
    for (int64_t pos : P.h_pos) mark(pos);
    for (int64_t pos : P.sr_slot_pos) mark(pos);
    for (int x : t.fold_order()) {
      const ClusterInfo& X = B.I(x);
      for (std::size_t p = 0; p < X.S.size(); ++p)
        for (std::size_t q = p + 1; q < X.S.size(); ++q) {
          const auto& src = nzr[static_cast<std::size_t>(x)][q];
          if (src[0] >= src[1]) continue;
          const int jp = X.S[p];
          const int qq = find_pos(B.I(jp).S, X.S[q]);
          if (qq < 0) fail(kInternal, "plan: fill block missing from S");
          auto& r = nzr[static_cast<std::size_t>(jp)][static_cast<std::size_t>(qq)];
          r[0] = std::min(r[0], src[0]);
          r[1] = std::max(r[1], src[1]);
        }
    }
  }
  if (!f_hull)
    for (int c = 0; c < nc; ++c)
      for (std::size_t q = 0; q < B.I(c).S.size(); ++q) nzr[static_cast<std::size_t>(c)][q] = {0, B.msz(B.I(c).S[q])};
  // Fused-diagonal row tasks (rows of never-referenced clusters feed only
  // diag(G_xx) / diag(P_xx) = sum_c Psi[r][c] op(C[r][c])) need only the
  // output columns where Psi_{x,j} can be nonzero: the hull of its coupling
  // block.  The other columns are multiplied by exact zeros, so the task is
  // restricted to the hull (empty hull: no task).  Partials: one per row and
  // 16-column group of each restricted task.
  auto out_hull = [&](int x, int j) -> std::array<int, 2> {
    const int p = find_pos(B.I(x).S, j);
    return p < 0 ? std::array<int, 2>{0, 0} : nzr[static_cast<std::size_t>(x)][static_cast<std::size_t>(p)];
  };
  auto same_set = [](std::vector<int> x, std::vector<int> y) {
    std::sort(x.begin(), x.end());
    std::sort(y.begin(), y.end());
    return x == y;
  };
  for (int c = 0; c < nc; ++c) {
    ClusterInfo& ci = B.I(c);
    const bool wood = f_woodbury && leaf_sparse[static_cast<std::size_t>(c)] && !ci.full_g && !ci.full_p &&
                      !ci.seeded && !ci.has_nd && ci.ncols.empty() && ci.m > 0;
    if (f_compact && f_hull && leaf_sparse[static_cast<std::size_t>(c)] && !wood && c != root && ci.m > 0 && ci.K > 0 &&
        !ci.full_g && !ci.seeded && !ci.has_nd && ci.ncols.empty() && same_set(ci.gcols, ci.S) &&
        (!P.any_seed || (!ci.full_p && same_set(ci.pcols, ci.S)))) {
      int h = 0;
      ci.hoff.assign(ci.S.size(), 0);
      for (std::size_t q = 0; q < ci.S.size(); ++q) {
        ci.hoff[q] = h;
        const auto& r = nzr[static_cast<std::size_t>(c)][q];
        if (r[1] > r[0]) h += r[1] - r[0];
      }
      if (h > 0) {
        ci.compact = true;
        ci.hc = h;
        ci.gpart_np = (h + 15) / 16;
        ci.off_gpart = take(int64_t(ci.m) * ci.gpart_np);
        if (P.any_seed) {
          ci.ppart_np = ci.gpart_np;
          ci.off_ppart = take(int64_t(ci.m) * ci.ppart_np);
        }
        ci.off_psic = take(int64_t(ci.m) * h);
        ci.off_mg = take(int64_t(h) * h);
        continue;
      }
    }
    if (!ci.full_g && c != root && ci.m > 0) {
      for (int j : ci.gcols) {
        const auto h = out_hull(c, j);
        if (h[1] > h[0]) ci.gpart_np += (h[1] - h[0] + 15) / 16;
      }
      if (ci.gpart_np) ci.off_gpart = take(int64_t(ci.m) * ci.gpart_np);
    }
    if (P.any_seed && !ci.full_p && c != root && ci.m > 0) {
      for (int j : ci.pcols) {
        const auto h = out_hull(c, j);
        if (h[1] > h[0]) ci.ppart_np += (h[1] - h[0] + 15) / 16;
      }
      if (ci.ppart_np) ci.off_ppart = take(int64_t(ci.m) * ci.ppart_np);
    }
  }
  P.arena = std::max(P.arena, cur);
  // Woodbury diagonals of the sparse, never-referenced, unseeded leaves
  // (LeafDiagTask): per leaf its boundary rows T and, per mode, the gathered
  // upper triangle of M.
  std::vector<char> leaf_wood(static_cast<std::size_t>(nc), 0);
  auto emit_leafdiag = [&](int x, int mode) {
    const ClusterInfo& X = B.I(x);
    // rows of A_{x,S}: (column in S space, value), from the column lists
    std::vector<std::vector<std::pair<int, cplx>>> rows(static_cast<std::size_t>(X.m));
    const auto& cols = leaf_cols[static_cast<std::size_t>(x)];
    for (int c = 0; c < X.K; ++c)
      for (const auto& e : cols[static_cast<std::size_t>(c)]) rows[static_cast<std::size_t>(e.first)].push_back({c, e.second});
    std::vector<int> T;
    for (int r = 0; r < X.m; ++r)
      if (!rows[static_cast<std::size_t>(r)].empty()) T.push_back(r);
    auto where = [&](int cc, int& k, int& l) {  // S-space column -> (cluster, local index)
      for (std::size_t q = 0; q < X.S.size(); ++q)
        if (cc >= X.s_col[q] && cc < X.s_col[q] + B.msz(X.S[q])) {
          k = X.S[q];
          l = static_cast<int>(cc - X.s_col[q]);
          return;
        }
      fail(kInternal, "plan: leaf coupling column outside S");
    };
    // arena position of G_SS / P_SS (k1, l1; k2, l2); flag: -conj of that entry
    auto at = [&](int k1, int l1, int k2, int l2, int& flag) -> int64_t {
      flag = 0;
      const ClusterInfo& K1 = B.I(k1);
      const ClusterInfo& K2 = B.I(k2);
      if (mode == 0) {
        if (k1 == k2) return K1.off_gd + int64_t(l1) * K1.m + l2;
        if (B.lev(k1) < B.lev(k2)) return K1.off_grow + int64_t(l1) * K1.WG + B.col_of(K1.gcols, K1.gcol_off, k2) + l2;
        return K2.off_grow + int64_t(l2) * K2.WG + B.col_of(K2.gcols, K2.gcol_off, k1) + l1;  // G symmetric
      }
      if (k1 == k2) return K1.off_pd + int64_t(l1) * K1.m + l2;
      if (B.lev(k1) < B.lev(k2)) return K1.off_prow + int64_t(l1) * K1.WP + B.col_of(K1.pcols, K1.pcol_off, k2) + l2;
      flag = 1;  // P_{k1,k2} = -P_{k2,k1}^H (hsc.cpp:204-206)
      return K2.off_prow + int64_t(l2) * K2.WP + B.col_of(K2.pcols, K2.pcol_off, k1) + l1;
    };
    LeafDiagTask lt{};
    lt.m = X.m;
    lt.nT = static_cast<int>(T.size());
    lt.t_begin = static_cast<int>(P.ld_rows.size());
    lt.out_begin = static_cast<int>(P.ld_optr.size());
    lt.mode = mode;
    lt.off_inv = X.off_d;
    lt.off_out = mode == 0 ? X.off_gd : X.off_pd;
    for (int r : T) P.ld_rows.push_back(r);
    double cm = 0.0;
    for (int i1 = 0; i1 < lt.nT; ++i1)
      for (int i2 = i1; i2 < lt.nT; ++i2) {
        P.ld_optr.push_back(static_cast<int>(P.ld_entries.size()));
        for (const auto& e1 : rows[static_cast<std::size_t>(T[static_cast<std::size_t>(i1)])])
          for (const auto& e2 : rows[static_cast<std::size_t>(T[static_cast<std::size_t>(i2)])]) {
            int k1, l1, k2, l2, flag;
            where(e1.first, k1, l1);
            where(e2.first, k2, l2);
            LeafDiagEntry en{};
            en.pos = at(k1, l1, k2, l2, flag);
            en.flag = flag;
            en.out = (i1 << 16) | i2;
            en.coef = mode == 0 ? e1.second * e2.second : e1.second * std::conj(e2.second);
            P.ld_entries.push_back(en);
            cm += 1.0;
          }
      }
    P.ld_optr.push_back(static_cast<int>(P.ld_entries.size()));
    B.cur.cmul += cm + double(X.m) * lt.nT * (lt.nT + 1);  // gather + W M W^T per row
    P.ld_tasks.push_back(lt);
  };
  for (int c = 0; c < nc; ++c) {
    const ClusterInfo& I = B.I(c);
    leaf_wood[static_cast<std::size_t>(c)] = f_woodbury && leaf_sparse[static_cast<std::size_t>(c)] && !I.full_g && !I.full_p &&
                                             !I.seeded && !I.has_nd && I.ncols.empty() && I.m > 0 && I.m < 65536;
  }
  // A sparse leaf's coupling block A_{x,S} is read only through its stencil
  // entries (the plan's CSC: K_SPSI, K_SSCHUR, K_LEAFDIAG, the hulls above),
  // never from the arena: its Arow region is neither zeroed nor scattered
  // per energy.
  {
    std::vector<std::pair<int64_t, int64_t>> skip;  // [begin, end) arena ranges
    for (int c = 0; c < nc; ++c) {
      const ClusterInfo& I = B.I(c);
      if (leaf_sparse[static_cast<std::size_t>(c)] && I.K > 0 && I.m > 0)
        skip.push_back({I.off_arow, I.off_arow + int64_t(I.m) * I.K});
    }
    std::sort(skip.begin(), skip.end());
    auto skipped = [&](int64_t pos) {
      auto it = std::upper_bound(skip.begin(), skip.end(), std::make_pair(pos, std::numeric_limits<int64_t>::max()));
      return it != skip.begin() && pos < std::prev(it)->second;
    };
    std::vector<InitRegion> iz;
    for (const InitRegion& r : P.init_zero)
      if (!skipped(r.off)) iz.push_back(r);
    P.init_zero.swap(iz);
    std::vector<int64_t> hp;
    std::vector<cplx> hv;
    for (std::size_t q = 0; q < P.h_pos.size(); ++q)
      if (!skipped(P.h_pos[q])) {
        hp.push_back(P.h_pos[q]);
        hv.push_back(P.h_val[q]);
      }
    P.h_pos.swap(hp);
    P.h_val.swap(hv);
  }
  // Leaf -> SpsiTask index (leaves' Psi tasks are emitted at level 1, before
  // any gather that reads them).
  std::vector<int> spsi_of(static_cast<std::size_t>(nc), -1);
  auto gather_schur = [&](int l) {
    // sparse leaf contributions first (their own op), then the dense gather
    std::vector<char> had_sparse;
    B.open(K_SSCHUR, 0, l);
    for (const auto& kv : schur[l]) {
      const int jp = kv.first.first, jq = kv.first.second;
      const ClusterInfo& J = B.I(jp);
      SschurTask st{};
      st.contrib_begin = static_cast<int>(P.sschur_contrib.size());
      double cm = 0.0;
      for (const auto& c3 : kv.second) {
        const int i = c3[0];
        const int sp = spsi_of[static_cast<std::size_t>(i)];
        if (sp < 0) continue;
        const ClusterInfo& X = B.I(i);
        SschurContrib ct{};
        ct.spsi = sp;
        ct.p_off = static_cast<int>(X.s_col[c3[1]]);
        ct.q_off = static_cast<int>(X.s_col[c3[2]]);
        ct.rc_begin = static_cast<int>(P.sschur_rc.size());
        const int* cb = P.spsi_colptr.data() + P.spsi_tasks[static_cast<std::size_t>(sp)].col_begin;
        for (int r = 0; r < B.msz(jp); ++r)
          if (cb[ct.p_off + r + 1] > cb[ct.p_off + r]) P.sschur_rc.push_back(r);
        ct.nr = static_cast<int>(P.sschur_rc.size()) - ct.rc_begin;
        for (int c = 0; c < B.msz(jq); ++c)
          if (cb[ct.q_off + c + 1] > cb[ct.q_off + c]) P.sschur_rc.push_back(c);
        ct.nc = static_cast<int>(P.sschur_rc.size()) - ct.rc_begin - ct.nr;
        P.sschur_contrib.push_back(ct);
        const int* cpp = cb + ct.p_off;
        const int* cpq = cb + ct.q_off;
        cm += double(cpp[B.msz(jp)] - cpp[0]) * (cpq[B.msz(jq)] - cpq[0]);  // entry pairs
      }
      st.contrib_count = static_cast<int>(P.sschur_contrib.size()) - st.contrib_begin;
      if (st.contrib_count > 0) {  // waves of row x column-disjoint contributions
        auto* cb0 = P.sschur_contrib.data() + st.contrib_begin;
        const int nq = st.contrib_count;
        std::vector<int> wave(static_cast<std::size_t>(nq), 0);
        auto overlap = [&](int a, int b, int off_a, int off_b, int na, int nb) {
          const int* x = P.sschur_rc.data() + cb0[a].rc_begin + off_a;
          const int* y = P.sschur_rc.data() + cb0[b].rc_begin + off_b;
          for (int i = 0; i < na; ++i)
            for (int j = 0; j < nb; ++j)
              if (x[i] == y[j]) return true;
          return false;
        };
        for (int q2 = 0; q2 < nq; ++q2)
          for (int q1 = 0; q1 < q2; ++q1)
            if (overlap(q1, q2, 0, 0, cb0[q1].nr, cb0[q2].nr) &&
                overlap(q1, q2, cb0[q1].nr, cb0[q2].nr, cb0[q1].nc, cb0[q2].nc))
              wave[q2] = std::max(wave[q2], wave[q1] + 1);
        std::vector<int> ord(static_cast<std::size_t>(nq));
        std::iota(ord.begin(), ord.end(), 0);
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return wave[a] < wave[b]; });
        std::vector<SschurContrib> sorted;
        for (int q2 : ord) sorted.push_back(cb0[q2]);
        for (int q2 = 0; q2 < nq; ++q2)
          sorted[q2].sync = (q2 + 1 == nq || wave[ord[q2 + 1]] != wave[ord[q2]]) ? 1 : 0;
        std::copy(sorted.begin(), sorted.end(), cb0);
      }
      had_sparse.push_back(st.contrib_count > 0);
      if (!st.contrib_count) continue;
      st.mp = J.m;
      st.mq = B.msz(jq);
      {
        int64_t touched = 0;
        for (int q2 = 0; q2 < st.contrib_count; ++q2) {
          const SschurContrib& c2 = P.sschur_contrib[static_cast<std::size_t>(st.contrib_begin + q2)];
          touched += int64_t(c2.nr) * c2.nc;
        }
        st.entry = int64_t(st.mp) * st.mq <= 2 * touched ? 1 : 0;
      }
      if (jp == jq) {
        st.ld = J.m;
        st.mode = MODE_ADD;
        st.off = J.off_d;
      } else {
        const int p = find_pos(J.S, jq);
        if (p < 0) fail(kInternal, "plan: fill block missing from S");
        st.ld = J.K;
        st.mode = J.s_orig[p] ? MODE_ADD : MODE_SET;
        st.off = J.off_arow + J.s_col[p];
      }
      P.sschur_tasks.push_back(st);
      B.cur.cmul += cm;
    }
    B.close();
    B.open(K_GEMM, 0, l);
    std::size_t q = 0;
    for (const auto& kv : schur[l]) {
      const int jp = kv.first.first, jq = kv.first.second;
      const bool sparse_done = had_sparse[q++];
      const ClusterInfo& J = B.I(jp);
      const int tb = static_cast<int>(T.size());
      const int pq = jp == jq ? -1 : find_pos(J.S, jq);
      if (jp != jq && pq < 0) fail(kInternal, "plan: fill block missing from S");
      const bool add = jp == jq || J.s_orig[static_cast<std::size_t>(pq)] || sparse_done;
      // An accumulating target is updated only on the hull of its terms'
      // nonzero rows (columns of Psi_{i,jp}) x columns (of A_{i,jq}); a pure
      // fill block written by this task alone keeps its full extent (zeros).
      int rlo = B.msz(jp), rhi = 0, clo = B.msz(jq), chi = 0;
      for (const auto& c3 : kv.second) {
        if (spsi_of[static_cast<std::size_t>(c3[0])] >= 0) continue;
        const auto& nr = nzr[static_cast<std::size_t>(c3[0])][static_cast<std::size_t>(c3[1])];
        const auto& nq = nzr[static_cast<std::size_t>(c3[0])][static_cast<std::size_t>(c3[2])];
        rlo = std::min(rlo, nr[0]); rhi = std::max(rhi, nr[1]);
        clo = std::min(clo, nq[0]); chi = std::max(chi, nq[1]);
      }
      if (jp == jq) {  // square diagonal sub-block (mirror)
        rlo = clo = std::min(rlo, clo);
        rhi = chi = std::max(rhi, chi);
      }
      if (!add || rlo >= rhi || clo >= chi) {
        rlo = 0; rhi = B.msz(jp); clo = 0; chi = B.msz(jq);
      }
      for (const auto& c3 : kv.second) {
        if (spsi_of[static_cast<std::size_t>(c3[0])] >= 0) continue;
        const ClusterInfo& X = B.I(c3[0]);
        B.add_term(T, X.m, OP_T, X.off_psi + X.s_col[c3[1]] + rlo, X.K, OP_N, X.off_arow + X.s_col[c3[2]] + clo, X.K,
                   +1);
      }
      if (static_cast<int>(T.size()) == tb) continue;  // leaves only: done by the sparse op
      if (jp == jq) {  // A_jj += sum Psi^T A_{i,j}: complex symmetric
        B.pend_diag.mirror = f_mirror_schur ? 1 : 0;
        B.gemm_task(rhi - rlo, rhi - rlo, J.off_d + int64_t(rlo) * J.m + rlo, J.m, MODE_ADD, 0, 0, tb);
      } else {
        // a pure fill block is produced by this single gather task (or
        // started by the sparse op, then accumulated)
        B.gemm_task(rhi - rlo, chi - clo, J.off_arow + int64_t(rlo) * J.K + J.s_col[static_cast<std::size_t>(pq)] + clo,
                    J.K, add ? MODE_ADD : MODE_SET, 0, 0, tb);
      }
    }
    B.close();
  };
  for (int l = 1; l <= t.levels() - 1; ++l) {
    const auto& xs = by_level[l];
    gather_schur(l);
    emit_inverses(l, xs);
    std::vector<int> sparse;  // leaves whose coupling block is the -H template alone
    B.open(K_GEMM, 0, l);  // Psi_x = -inv_x A_{x,S(x)}
    for (int x : xs) {
      const ClusterInfo& I = B.I(x);
      if (!I.K) continue;
      if (leaf_sparse[static_cast<std::size_t>(x)]) {
        sparse.push_back(x);
        continue;
      }
      const int tb = static_cast<int>(T.size());
      B.add_term(T, I.m, OP_N, I.off_d, I.m, OP_N, I.off_arow, I.K, -1);
      if (I.off_psi2 >= 0) B.pend_diag.c2_off = I.off_psi2;
      B.gemm_task(I.m, I.K, I.off_psi, I.K, MODE_SET, 0, 0, tb);
    }
    B.close();
    if (!sparse.empty()) {
      // leaves whose Psi is read (G / P rows) first: the op launches them;
      // the Woodbury leaves only keep their CSC record (K_SSCHUR reads
      // A_{x,S} and inv_x directly)
      std::stable_partition(sparse.begin(), sparse.end(),
                            [&](int x) { return !leaf_wood[static_cast<std::size_t>(x)]; });
      bool closed = false;
      B.open(K_SPSI, 0, l);
      for (int x : sparse) {
        if (!closed && leaf_wood[static_cast<std::size_t>(x)]) {
          B.close();
          closed = true;
        }
        const ClusterInfo& I = B.I(x);
        const auto& cols = leaf_cols[static_cast<std::size_t>(x)];
        SpsiTask st{};
        st.m = I.m;
        st.K = I.K;
        st.col_begin = static_cast<int>(P.spsi_colptr.size());
        st.off_inv = I.off_d;
        st.off_psi = I.off_psi;
        st.off_psi2 = leaf_wood[static_cast<std::size_t>(x)] ? -1 : I.off_psi2;  // 2 Psi: the row forms only
        if (I.compact) {  // only the hull columns, compacted (Psi_H); no 2 Psi
          st.h = I.hc;
          st.wcol_begin = static_cast<int>(P.spsi_wcols.size());
          st.off_psi = I.off_psic;
          st.off_psi2 = -1;
          for (std::size_t q = 0; q < I.S.size(); ++q) {
            const auto& r = nzr[static_cast<std::size_t>(x)][q];
            for (int a = r[0]; a < r[1]; ++a) P.spsi_wcols.push_back(static_cast<int>(I.s_col[q]) + a);
          }
        }
        for (int c = 0; c < I.K; ++c) {
          P.spsi_colptr.push_back(static_cast<int>(P.spsi_row.size()));
          for (const auto& e : cols[static_cast<std::size_t>(c)]) {
            P.spsi_row.push_back(e.first);
            P.spsi_val.push_back(e.second);
          }
        }
        P.spsi_colptr.push_back(static_cast<int>(P.spsi_row.size()));
        if (!closed && I.compact) {
          for (int q = 0; q < I.hc; ++q) {
            const int c = P.spsi_wcols[static_cast<std::size_t>(st.wcol_begin + q)];
            B.cur.cmul += double(I.m) * (P.spsi_colptr[static_cast<std::size_t>(st.col_begin + c + 1)] -
                                         P.spsi_colptr[static_cast<std::size_t>(st.col_begin + c)]);
          }
        } else if (!closed) {
          B.cur.cmul += double(I.m) * (P.spsi_colptr.back() - P.spsi_colptr[static_cast<std::size_t>(st.col_begin)]);
        }
        spsi_of[static_cast<std::size_t>(x)] = static_cast<int>(P.spsi_tasks.size());
        P.spsi_tasks.push_back(st);
      }
      if (!closed) B.close();
    }
  }
  gather_schur(t.levels());
  emit_inverses(t.levels(), std::vector<int>{root});

  P.exec_inv_cmul = 0;
  for (int c = 0; c < nc; ++c) P.exec_inv_cmul += double(B.msz(c)) * B.msz(c) * B.msz(c);

  // M of a compact leaf (MGatherTask): the G_SS (mode 0) / P_SS (mode 1)
  // blocks on the hull columns H, exactly the B operands of the row tasks it
  // replaces -- block pair (k, j) at (hoff[k], hoff[j]).  Every pair is
  // gathered (the reference's own sum, hsc.cpp:210-227 / 275-303): in this one
  // product the symmetric forms would only turn half of M into zeros.
  auto emit_mgather = [&](int x, int mode) {
    const ClusterInfo& X = B.I(x);
    const bool sym = false;
    MGatherTask mt{};
    mt.h = X.hc;
    mt.dst = X.off_mg;
    mt.block_begin = static_cast<int>(P.mg_blocks.size());
    for (std::size_t qa = 0; qa < X.S.size(); ++qa) {
      const auto ra = nzr[static_cast<std::size_t>(x)][qa];
      if (ra[0] >= ra[1]) continue;
      for (std::size_t qc = 0; qc < X.S.size(); ++qc) {
        const auto rc = nzr[static_cast<std::size_t>(x)][qc];
        if (rc[0] >= rc[1]) continue;
        MGatherBlock mb{};
        mb.dst_row = X.hoff[qa];
        mb.dst_col = X.hoff[qc];
        mb.rows = ra[1] - ra[0];
        mb.cols = rc[1] - rc[0];
        if (sym && qa > qc) {
          mb.coef = 0.0;
        } else {
          const int k = X.S[qa], j = X.S[qc];
          const double two = (sym && qa < qc) ? 2.0 : 1.0;
          const ClusterInfo& Kc = B.I(k);
          const ClusterInfo& Jc = B.I(j);
          if (k == j) {
            mb.src = (mode == 0 ? Jc.off_gd : Jc.off_pd) + int64_t(ra[0]) * B.msz(j) + rc[0];
            mb.rs = B.msz(j);
            mb.cs = 1;
            mb.coef = two;
          } else if (B.lev(k) < B.lev(j)) {
            if (mode == 0) {
              mb.src = Kc.off_grow + int64_t(ra[0]) * Kc.WG + B.col_of(Kc.gcols, Kc.gcol_off, j) + rc[0];
              mb.rs = Kc.WG;
            } else {
              mb.src = Kc.off_prow + int64_t(ra[0]) * Kc.WP + B.col_of(Kc.pcols, Kc.pcol_off, j) + rc[0];
              mb.rs = Kc.WP;
            }
            mb.cs = 1;
            mb.coef = two;
          } else {  // G_{k,j} = G_{j,k}^T;  P_{k,j} = -P_{j,k}^H
            if (mode == 0) {
              mb.src = Jc.off_grow + int64_t(rc[0]) * Jc.WG + B.col_of(Jc.gcols, Jc.gcol_off, k) + ra[0];
              mb.cs = Jc.WG;
              mb.coef = two;
            } else {
              mb.src = Jc.off_prow + int64_t(rc[0]) * Jc.WP + B.col_of(Jc.pcols, Jc.pcol_off, k) + ra[0];
              mb.cs = Jc.WP;
              mb.coef = -two;
              mb.conj = 1;
            }
            mb.rs = 1;
          }
        }
        P.mg_blocks.push_back(mb);  // a copy: no flops charged
      }
    }
    mt.block_count = static_cast<int>(P.mg_blocks.size()) - mt.block_begin;
    P.mg_tasks.push_back(mt);
  };
  // The single GEMM task of a compact leaf: Psi_H (m x h) M (h x h), only
  // the fused diagonal kept (dmode 1: G, 2 / 3: P).
  auto emit_compact_rows = [&](int x, int mode) {
    const ClusterInfo& X = B.I(x);
    const int tb = static_cast<int>(T.size());
    B.add_term(T, X.hc, OP_N, X.off_psic, X.hc, OP_N, X.off_mg, X.hc, +1);
    // P: diag(P_xx) of an anti-Hermitian P is imaginary; with the symdiag_p
    // form the sum keeps only its imaginary part (dmode 3), as the row tasks do
    B.pend_diag.dmode = mode == 0 ? 1 : (f_symdiag_p ? 3 : 2);
    B.pend_diag.nostore = 1;
    B.pend_diag.dpsi_off = X.off_psic;
    B.pend_diag.dpsi_ld = X.hc;
    B.pend_diag.dpart_off = mode == 0 ? X.off_gpart : X.off_ppart;
    B.pend_diag.dpart_ld = mode == 0 ? X.gpart_np : X.ppart_np;
    B.gemm_task(X.m, X.hc, X.off_mg, X.hc, MODE_SET, 0, 0, tb);
  };

  // G^r extraction top-down (hsc.cpp:171-227).
  for (int l = t.levels() - 1; l >= 1; --l) {
    const auto& xs = by_level[l];
    B.open(K_MGATHER, 1, l);
    for (int x : xs)
      if (B.I(x).compact) emit_mgather(x, 0);
    B.close();
    B.open(K_GEMM, 1, l);
    for (int x : xs) {
      const ClusterInfo& X = B.I(x);
      if (leaf_wood[static_cast<std::size_t>(x)]) continue;  // K_LEAFDIAG below
      if (X.compact) {
        emit_compact_rows(x, 0);
        continue;
      }
      const bool fused = !X.full_g && x != root;  // rows feed only diag(G_xx): not stored
      const bool sym = f_symdiag_g && fused && X.off_gpart >= 0 && X.off_psi2 >= 0;
      int gb = 0;  // partial group of this task
      for (std::size_t jj = 0; jj < X.gcols.size(); ++jj) {
        const int j = X.gcols[jj];
        const auto oh = fused ? out_hull(x, j) : std::array<int, 2>{0, B.msz(j)};
        if (oh[0] >= oh[1]) continue;  // Psi_{x,j} == 0: no diagonal contribution
        const int c0 = oh[0], nw = oh[1] - oh[0];
        const int tb = static_cast<int>(T.size());
        const int jpos = find_pos(X.S, j);
        for (std::size_t kk = 0; kk < X.S.size(); ++kk) {
          const int k = X.S[kk];
          // symmetric form: block pair (k, j) once, in the task of the later
          // one, from 2 Psi_k; the diagonal block from Psi_j
          if (sym && static_cast<int>(kk) > jpos) continue;
          const auto nz = nzr[static_cast<std::size_t>(x)][kk];
          if (nz[0] >= nz[1]) continue;  // Psi_{x,k} == 0
          const int lo = nz[0], kn = nz[1] - nz[0];
          const int64_t a = (sym && static_cast<int>(kk) < jpos ? X.off_psi2 : X.off_psi) + X.s_col[kk] + lo;
          if (k == j)
            B.add_term(T, kn, OP_N, a, X.K, OP_N, B.I(j).off_gd + int64_t(lo) * B.msz(j) + c0, B.msz(j), +1);
          else if (B.lev(k) < B.lev(j))
            B.add_term(T, kn, OP_N, a, X.K, OP_N,
                       B.I(k).off_grow + int64_t(lo) * B.I(k).WG + B.col_of(B.I(k).gcols, B.I(k).gcol_off, j) + c0,
                       B.I(k).WG, +1);
          else
            B.add_term(T, kn, OP_N, a, X.K, OP_T,
                       B.I(j).off_grow + int64_t(c0) * B.I(j).WG + B.col_of(B.I(j).gcols, B.I(j).gcol_off, k) + lo,
                       B.I(j).WG, +1);
        }
        if (fused) {
          if (X.off_gpart < 0 || jpos < 0) fail(kInternal, "plan: diagonal-only row outside the fill set");
          B.pend_diag.dmode = 1;
          B.pend_diag.nostore = 1;
          B.pend_diag.dpsi_off = X.off_psi + X.s_col[static_cast<std::size_t>(jpos)] + c0;
          B.pend_diag.dpsi_ld = X.K;
          B.pend_diag.dpart_off = X.off_gpart + gb;
          B.pend_diag.dpart_ld = X.gpart_np;
          gb += (nw + 15) / 16;
        }
        B.gemm_task(X.m, nw, X.off_grow + X.gcol_off[jj] + c0, X.WG, MODE_SET, 0, 0, tb);
      }
    }
    B.close();
    B.open(K_GEMM, 1, l);  // full diagonal blocks
    for (int x : xs) {
      const ClusterInfo& X = B.I(x);
      if (!X.full_g) continue;
      const int tb = static_cast<int>(T.size());
      for (std::size_t kk = 0; kk < X.S.size(); ++kk)
      {
        const auto nz = nzr[static_cast<std::size_t>(x)][kk];
        if (nz[0] >= nz[1]) continue;
        B.add_term(T, nz[1] - nz[0], OP_N, X.off_psi + X.s_col[kk] + nz[0], X.K, OP_T,
                   X.off_grow + B.col_of(X.gcols, X.gcol_off, X.S[kk]) + nz[0], X.WG, +1);
      }
      B.pend_diag.mirror = f_mirror_g ? 1 : 0;  // G_xx = inv_x + Psi G_{x,S}^T: complex symmetric
      B.gemm_task(X.m, X.m, X.off_gd, X.m, MODE_INIT, X.off_d, X.m, tb);
    }
    B.close();
    B.open(K_DIAG, 1, l);  // diagonal entries only (never-referenced, unseeded)
    for (int x : xs) {
      const ClusterInfo& X = B.I(x);
      if (X.full_g || X.m == 0 || leaf_wood[static_cast<std::size_t>(x)]) continue;
      DiagTask dt{};
      dt.m = X.m;
      dt.init_stride = X.m + 1;
      dt.has_init = 1;
      dt.out_off = X.off_gd;
      dt.init_off = X.off_d;
      dt.term_begin = static_cast<int>(P.diag_terms.size());
      if (X.off_gpart >= 0) {  // sum of the fused row-task partials
        dt.part_off = X.off_gpart;
        dt.part_np = X.gpart_np;
      }
      dt.term_count = static_cast<int>(P.diag_terms.size()) - dt.term_begin;
      P.diag_tasks.push_back(dt);
    }
    B.close();
    B.open(K_LEAFDIAG, 1, l);
    for (int x : xs)
      if (leaf_wood[static_cast<std::size_t>(x)]) emit_leafdiag(x, 0);
    B.close();
  }

  if (P.any_seed) {
    // Seeds N = Sigma^<_x conj(G_x.) (hsc.cpp:229-237), all clusters at once.
    B.open(K_GEMM, 2, 0);
    for (int x = 0; x < nc; ++x) {
      const ClusterInfo& X = B.I(x);
      if (!X.seeded || !X.seed_dense || X.m == 0) continue;
      int tb = static_cast<int>(T.size());
      B.add_term(T, X.m, OP_N, X.off_sig, X.m, OP_C, X.off_gd, X.m, +1);
      B.gemm_task(X.m, X.m, X.off_nd, X.m, MODE_SET, 0, 0, tb);
      if (X.WN) {
        tb = static_cast<int>(T.size());
        B.add_term(T, X.m, OP_N, X.off_sig, X.m, OP_C, X.off_grow, X.WG, +1);
        B.gemm_task(X.m, X.WN, X.off_nrow, X.WN, MODE_SET, 0, 0, tb);
      }
    }
    B.close();
    B.open(K_SCALE, 2, 0);
    for (int x = 0; x < nc; ++x) {
      const ClusterInfo& X = B.I(x);
      if (!X.seeded || X.seed_dense || X.m == 0) continue;
      P.scale_tasks.push_back(ScaleTask{X.m, X.m, X.m, X.m, X.off_gd, X.off_nd, X.off_sig});
      B.cur.cmul += double(X.m) * X.m;
      if (X.WN) {
        P.scale_tasks.push_back(ScaleTask{X.m, X.WN, X.WG, X.WN, X.off_grow, X.off_nrow, X.off_sig});
        B.cur.cmul += double(X.m) * X.WN;
      }
    }
    B.close();
    // N fold bottom-up (hsc.cpp:246-266), left-looking like the Schur fold:
    // N_{j,k} += sum_{y : j in S(y)} Psi_{y,j}^T N_{y,k}, level(k) >= level(j),
    // gathered per target right after the targets' own contributors are final.
    std::vector<std::map<std::pair<int, int>, std::vector<std::array<int, 3>>>> nf(
        static_cast<std::size_t>(t.levels()) + 1);
    for (int y : t.fold_order()) {
      const ClusterInfo& Y = B.I(y);
      if (Y.ncols.empty()) continue;
      for (std::size_t jj = 0; jj < Y.S.size(); ++jj)
        for (std::size_t kk = 0; kk < Y.ncols.size(); ++kk) {
          const int j = Y.S[jj], k = Y.ncols[kk];
          if (B.lev(k) < B.lev(j)) continue;
          nf[B.lev(j)][{j, k}].push_back({y, static_cast<int>(jj), static_cast<int>(kk)});
        }
    }
    for (int l = 2; l <= t.levels(); ++l) {
      B.open(K_GEMM, 3, l);
      for (const auto& kv : nf[l]) {
        const int j = kv.first.first, k = kv.first.second;
        const ClusterInfo& J = B.I(j);
        const int tb = static_cast<int>(T.size());
        for (const auto& c3 : kv.second) {
          const ClusterInfo& X = B.I(c3[0]);
          B.add_term(T, X.m, OP_T, X.off_psi + X.s_col[c3[1]], X.K, OP_N, X.off_nrow + X.ncol_off[c3[2]], X.WN,
                     +1);
        }
        // seeded targets already hold their seed; otherwise this task is the
        // block's only writer
        const int mode = J.seeded ? MODE_ADD : MODE_SET;
        if (k == j) B.gemm_task(J.m, J.m, J.off_nd, J.m, mode, 0, 0, tb);
        else B.gemm_task(J.m, B.msz(k), J.off_nrow + B.col_of(J.ncols, J.ncol_off, k), J.WN, mode, 0, 0, tb);
      }
      B.close();
    }
    // P = G^< extraction top-down (hsc.cpp:190-208, 275-319).
    B.open(K_GEMM, 4, t.levels());
    {
      const ClusterInfo& R = B.I(root);
      if (R.has_nd && R.m > 0) {
        const int tb = static_cast<int>(T.size());
        B.add_term(T, R.m, OP_N, R.off_d, R.m, OP_N, R.off_nd, R.m, +1);
        B.gemm_task(R.m, R.m, R.off_pd, R.m, MODE_SET, 0, 0, tb);
      }
    }
    B.close();
    for (int l = t.levels() - 1; l >= 1; --l) {
      const auto& xs = by_level[l];
      B.open(K_MGATHER, 4, l);
      for (int x : xs)
        if (B.I(x).compact) emit_mgather(x, 1);
      B.close();
      B.open(K_GEMM, 4, l);
      for (int x : xs) {
        const ClusterInfo& X = B.I(x);
        if (leaf_wood[static_cast<std::size_t>(x)]) continue;  // K_LEAFDIAG below
        if (X.compact) {
          emit_compact_rows(x, 1);
          continue;
        }
        // Symmetric form of a diagonal-only, unseeded P row set:
        // diag(P_xx) = diag(Psi P_SS Psi^H) with P_SS anti-Hermitian (P_{j,k} =
        // -P_{k,j}^H, hsc.cpp:204-206), so the (k, j) and (j, k) block pairs sum to
        // w - conj(w) = 2i Im(w): each pair once from 2 Psi, imaginary part kept
        // (dmode 3).  The diagonal blocks' own real parts are rounding noise
        // (G^< is anti-Hermitian), so the whole sum keeps only its imaginary part.
        const bool pfused = !X.full_p && x != root;  // rows feed only diag(P_xx): not stored
        const bool psym = f_symdiag_p && pfused && X.off_ppart >= 0 && X.off_psi2 >= 0 && X.ncols.empty() && !X.has_nd;
        int gb = 0;  // partial group of this task
        for (std::size_t jj = 0; jj < X.pcols.size(); ++jj) {
          const int j = X.pcols[jj];
          const auto oh = pfused ? out_hull(x, j) : std::array<int, 2>{0, B.msz(j)};
          if (oh[0] >= oh[1]) continue;  // Psi_{x,j} == 0: no diagonal contribution
          const int c0 = oh[0], nw = oh[1] - oh[0];
          const int tb = static_cast<int>(T.size());
          const int np = find_pos(X.ncols, j);
          const int jpos = find_pos(X.S, j);
          if (np >= 0) B.add_term(T, X.m, OP_N, X.off_d, X.m, OP_N, X.off_nrow + X.ncol_off[np] + c0, X.WN, +1);
          for (std::size_t kk = 0; kk < X.S.size(); ++kk) {
            const int k = X.S[kk];
            if (psym && static_cast<int>(kk) > jpos) continue;
            const auto nz = nzr[static_cast<std::size_t>(x)][kk];
            if (nz[0] >= nz[1]) continue;  // Psi_{x,k} == 0
            const int lo = nz[0], kn = nz[1] - nz[0];
            const int64_t a = (psym && static_cast<int>(kk) < jpos ? X.off_psi2 : X.off_psi) + X.s_col[kk] + lo;
            if (k == j)
              B.add_term(T, kn, OP_N, a, X.K, OP_N, B.I(j).off_pd + int64_t(lo) * B.msz(j) + c0, B.msz(j), +1);
            else if (B.lev(k) < B.lev(j))
              B.add_term(T, kn, OP_N, a, X.K, OP_N,
                         B.I(k).off_prow + int64_t(lo) * B.I(k).WP + B.col_of(B.I(k).pcols, B.I(k).pcol_off, j) + c0,
                         B.I(k).WP, +1);
            else
              B.add_term(T, kn, OP_N, a, X.K, OP_H,
                         B.I(j).off_prow + int64_t(c0) * B.I(j).WP + B.col_of(B.I(j).pcols, B.I(j).pcol_off, k) + lo,
                         B.I(j).WP, -1);
          }
          if (pfused) {
            if (X.off_ppart < 0 || jpos < 0) fail(kInternal, "plan: diagonal-only row outside the fill set");
            B.pend_diag.dmode = psym ? 3 : 2;
            B.pend_diag.nostore = 1;
            B.pend_diag.dpsi_off = X.off_psi + X.s_col[static_cast<std::size_t>(jpos)] + c0;
            B.pend_diag.dpsi_ld = X.K;
            B.pend_diag.dpart_off = X.off_ppart + gb;
            B.pend_diag.dpart_ld = X.ppart_np;
            gb += (nw + 15) / 16;
          }
          B.gemm_task(X.m, nw, X.off_prow + X.pcol_off[jj] + c0, X.WP, MODE_SET, 0, 0, tb);
        }
      }
      B.close();
      B.open(K_GEMM, 4, l);
      for (int x : xs) {
        const ClusterInfo& X = B.I(x);
        if (!X.full_p) continue;
        const int tb = static_cast<int>(T.size());
        if (X.has_nd) B.add_term(T, X.m, OP_N, X.off_d, X.m, OP_N, X.off_nd, X.m, +1);
        for (std::size_t kk = 0; kk < X.S.size(); ++kk)
        {
          const auto nz = nzr[static_cast<std::size_t>(x)][kk];
          if (nz[0] >= nz[1]) continue;
          B.add_term(T, nz[1] - nz[0], OP_N, X.off_psi + X.s_col[kk] + nz[0], X.K, OP_H,
                     X.off_prow + B.col_of(X.pcols, X.pcol_off, X.S[kk]) + nz[0], X.WP, -1);
        }
        B.pend_diag.mirror = f_mirror_p ? 2 : 0;  // P_xx = G^<_xx: anti-Hermitian
        B.gemm_task(X.m, X.m, X.off_pd, X.m, MODE_SET, 0, 0, tb);
      }
      B.close();
      B.open(K_DIAG, 4, l);
      for (int x : xs) {
        const ClusterInfo& X = B.I(x);
        if (X.full_p || X.m == 0 || leaf_wood[static_cast<std::size_t>(x)]) continue;
        DiagTask dt{};
        dt.m = X.m;
        dt.init_stride = 0;
        dt.has_init = 0;
        dt.out_off = X.off_pd;
        dt.term_begin = static_cast<int>(P.diag_terms.size());
        if (X.has_nd) {
          B.add_term(P.diag_terms, X.m, OP_N, X.off_d, X.m, OP_N, X.off_nd, X.m, +1);
          B.cur.cmul += double(X.m) * X.m;
        }
        if (X.off_ppart >= 0) {  // sum of the fused row-task partials
          dt.part_off = X.off_ppart;
          dt.part_np = X.ppart_np;
        }
        dt.term_count = static_cast<int>(P.diag_terms.size()) - dt.term_begin;
        P.diag_tasks.push_back(dt);
      }
      B.close();
      B.open(K_LEAFDIAG, 4, l);
      for (int x : xs)
        if (leaf_wood[static_cast<std::size_t>(x)]) emit_leafdiag(x, 1);
      B.close();
    }
  }

  // ---- reference ledger (lean mode, dense.hpp charges)
  {
    Ledger& f = P.ref_fold;
    for (int i : t.fold_order()) {
      const int64_t m = B.msz(i);
      f.inverse_ops += m * m * m;
      const auto& js = B.I(i).S;
      for (int j : js) f.multiply_ops += m * m * B.msz(j);
      for (std::size_t p = 0; p < js.size(); ++p)
        for (std::size_t q = p; q < js.size(); ++q) f.multiply_ops += int64_t(B.msz(js[p])) * m * B.msz(js[q]);
    }
    f.inverse_ops += int64_t(B.msz(root)) * B.msz(root) * B.msz(root);
    Ledger& g = P.ref_gless;
    int64_t sum_anc_cache = 0;
    (void)sum_anc_cache;
    for (int x = 0; x < nc; ++x) {
      const int64_t m = B.msz(x);
      int64_t wanc = 0;
      for (int j : t.cluster(x).anc) wanc += B.msz(j);
      if (x != root) {
        for (int k : B.I(x).S) {
          g.multiply_ops += m * B.msz(k) * wanc;  // rows
          g.multiply_ops += m * B.msz(k) * m;     // diagonal
        }
      }
      if (B.I(x).seeded) {
        if (B.I(x).seed_dense) g.multiply_ops += m * m * m + m * m * wanc;
        else g.multiply_ops += m * m + m * wanc;
      }
    }
    if (P.any_seed) {
      for (int i : t.fold_order()) {
        const auto& ncl = B.I(i).ncols;
        for (int j : B.I(i).S)
          for (int k : ncl)
            if (B.lev(k) >= B.lev(j)) g.multiply_ops += int64_t(B.msz(j)) * B.msz(i) * B.msz(k);
      }
      for (int x = 0; x < nc; ++x) {
        const int64_t m = B.msz(x);
        const ClusterInfo& X = B.I(x);
        if (x == root) {
          if (X.has_nd) g.multiply_ops += m * m * m;
          continue;
        }
        for (int j : t.cluster(x).anc) {
          if (find_pos(X.ncols, j) >= 0) g.multiply_ops += m * m * B.msz(j);
          for (int k : X.S) g.multiply_ops += m * B.msz(k) * B.msz(j);
        }
        if (X.has_nd) g.multiply_ops += m * m * m;
        for (int k : X.S) g.multiply_ops += m * B.msz(k) * m;
      }
    }
  }
  // seeds (phase 2) are the first readers of the Sigma^< slots; phases >= 2
  // never write G^r blocks
  P.lesser_op = static_cast<int>(P.ops.size());
  for (std::size_t i = 0; i < P.ops.size(); ++i)
    if (P.ops[i].phase >= 2) {
      P.lesser_op = static_cast<int>(i);
      break;
    }
  P.gr_done_op = P.lesser_op;
  if (form_on("real")) mark_real_operands(P);
  return P;
}

LeadPlan build_lead_plan(int w) {
  if (w <= 0) fail(kContractViolation, "lead: block size out of range");
  LeadPlan L;
  L.w = w;
  Plan& P = L.P;
  const int64_t w2 = align8(int64_t(w) * w);
  for (int b = 0; b < LB_COUNT; ++b) L.off[b] = b * w2;
  P.big_scratch = LB_COUNT * w2;
  // scratch for two simultaneous big inverses (g and m)
  const int64_t per = w > kSmemInvMax ? big_scratch_elems(w) : 0;
  P.arena = P.big_scratch + 2 * per;
  Builder B(P);
  auto& T = P.gemm_terms;
  auto mark = [&](int* r, auto&& body) {
    r[0] = static_cast<int>(P.ops.size());
    body();
    r[1] = static_cast<int>(P.ops.size());
  };
  auto prod = [&](int c, int a, int b2, int mode, int sign, int init = -1) {
    const int tb = static_cast<int>(T.size());
    B.add_term(T, w, OP_N, L.off[a], w, OP_N, L.off[b2], w, sign);
    B.gemm_task(w, w, L.off[c], w, mode, init >= 0 ? L.off[init] : 0, w, tb);
  };
  mark(L.inv_gm, [&] {
    B.emit_inverses(0, 10, {InvItem{w, 0, 0, L.off[LB_G]}, InvItem{w, 0, 1, L.off[LB_M]}}, P.big_scratch);
  });
  for (int par = 0; par < 2; ++par) {
    mark(L.gemm_a[par], [&] {
      B.open(K_GEMM, 10, 0);
      prod(LB_T1, LB_H01CT, LB_G, MODE_SET, +1);
      prod(LB_AM, par ? LB_ALPHA1 : LB_ALPHA0, LB_M, MODE_SET, +1);
      prod(LB_BM, par ? LB_BETA1 : LB_BETA0, LB_M, MODE_SET, +1);
      B.close();
    });
  }
  for (int par = 0; par < 2; ++par) {
    mark(L.gemm_a2[par], [&] {
      B.open(K_GEMM, 10, 0);
      prod(LB_AM, par ? LB_ALPHA1 : LB_ALPHA0, LB_M, MODE_SET, +1);
      prod(LB_BM, par ? LB_BETA1 : LB_BETA0, LB_M, MODE_SET, +1);
      B.close();
    });
  }
  mark(L.gemm_b, [&] {
    B.open(K_GEMM, 10, 0);
    prod(LB_RHS, LB_T1, LB_H01, MODE_INIT, -1, LB_ZH);
    B.close();
  });
  mark(L.inv_rhs, [&] { B.emit_inverses(0, 10, {InvItem{w, 0, 2, L.off[LB_RHS]}}, P.big_scratch); });
  mark(L.inv_m, [&] { B.emit_inverses(0, 10, {InvItem{w, 0, 1, L.off[LB_M]}}, P.big_scratch); });
  mark(L.inv_fin, [&] { B.emit_inverses(0, 10, {InvItem{w, 0, 3, L.off[LB_FIN]}}, P.big_scratch); });
  for (int par = 0; par < 2; ++par) {
    const int al = par ? LB_ALPHA1 : LB_ALPHA0, be = par ? LB_BETA1 : LB_BETA0;
    const int al2 = par ? LB_ALPHA0 : LB_ALPHA1, be2 = par ? LB_BETA0 : LB_BETA1;
    mark(L.gemm_c[par], [&] {
      B.open(K_GEMM, 10, 0);
      prod(LB_ES, LB_AM, be, MODE_ADD, +1);
      {
        const int tb = static_cast<int>(T.size());
        B.add_term(T, w, OP_N, L.off[LB_AM], w, OP_N, L.off[be], w, +1);
        B.add_term(T, w, OP_N, L.off[LB_BM], w, OP_N, L.off[al], w, +1);
        B.gemm_task(w, w, L.off[LB_E], w, MODE_ADD, 0, 0, tb);
      }
      prod(al2, LB_AM, al, MODE_SET, +1);
      prod(be2, LB_BM, be, MODE_SET, +1);
      B.close();
    });
  }
  mark(L.fin1, [&] {
    B.open(K_GEMM, 10, 0);
    prod(LB_T1, LB_H01CT, LB_FIN, MODE_SET, +1);
    B.close();
  });
  mark(L.fin2, [&] {
    B.open(K_GEMM, 10, 0);
    prod(LB_SIG, LB_T1, LB_H01, MODE_SET, +1);
    B.close();
  });
  return L;
}

Plan build_rgf_plan(ProblemDesc desc, std::vector<std::vector<int>> layers) {
  struct {
    int max_layer = 0;
  } R;
  Plan P;
  P.desc = std::move(desc);
  const ProblemDesc& d = P.desc;
  const int n = d.n;
  if (n <= 0) fail(kContractViolation, "problem: no dofs");
  if (layers.empty()) fail(kContractViolation, "layer map is empty");
  // layered_from_coo (rgf.cpp:69-150): sorted layers, disjoint cover.
  const int L = static_cast<int>(layers.size());
  std::vector<int> layer_of(static_cast<size_t>(n), -1), local_of(static_cast<size_t>(n), -1);
  for (int l = 0; l < L; ++l) {
    auto& dofs = layers[static_cast<size_t>(l)];
    std::sort(dofs.begin(), dofs.end());
    for (size_t k = 0; k < dofs.size(); ++k) {
      const int x = dofs[k];
      if (x < 0 || x >= n || layer_of[static_cast<size_t>(x)] != -1)
        fail(kContractViolation, "layer map is not a disjoint cover");
      layer_of[static_cast<size_t>(x)] = l;
      local_of[static_cast<size_t>(x)] = static_cast<int>(k);
    }
  }
  for (int x = 0; x < n; ++x)
    if (layer_of[static_cast<size_t>(x)] == -1) fail(kContractViolation, "layer map does not cover every dof");
  std::vector<int> nl(static_cast<size_t>(L));
  for (int l = 0; l < L; ++l) {
    nl[static_cast<size_t>(l)] = static_cast<int>(layers[static_cast<size_t>(l)].size());
    if (nl[static_cast<size_t>(l)] == 0) fail(kContractViolation, "layer map has an empty layer");
    R.max_layer = std::max(R.max_layer, nl[static_cast<size_t>(l)]);
  }
  // Entries coupling non-adjacent layers (H and Sigma^r are A's pattern).
  {
    std::vector<std::pair<int, int>> viol;
    auto scan = [&](const std::vector<int>& rows, const std::vector<int>& cols) {
      for (size_t k = 0; k < rows.size(); ++k) {
        const int lr = layer_of[static_cast<size_t>(rows[k])], lc = layer_of[static_cast<size_t>(cols[k])];
        if (std::abs(lr - lc) > 1) viol.push_back({std::min(rows[k], cols[k]), std::max(rows[k], cols[k])});
      }
    };
    scan(d.h_rows, d.h_cols);
    scan(d.sr_rows, d.sr_cols);
    if (!viol.empty()) {
      std::sort(viol.begin(), viol.end());
      viol.erase(std::unique(viol.begin(), viol.end()), viol.end());
      fail(kPartitionViolation, std::to_string(viol.size()) + " entr(ies) couple non-adjacent layers");
    }
    // lower coupling == transpose of the upper one (rgf.cpp:137-147), on H
    std::map<std::pair<int, int>, cplx> inter;
    for (size_t k = 0; k < d.h_rows.size(); ++k)
      if (layer_of[static_cast<size_t>(d.h_rows[k])] != layer_of[static_cast<size_t>(d.h_cols[k])])
        inter[{d.h_rows[k], d.h_cols[k]}] += d.h_vals[k];
    for (const auto& kv : inter) {
      auto it = inter.find({kv.first.second, kv.first.first});
      const cplx mirror = it == inter.end() ? cplx(0.0, 0.0) : it->second;
      if (mirror != kv.second) {
        const int l = std::min(layer_of[static_cast<size_t>(kv.first.first)], layer_of[static_cast<size_t>(kv.first.second)]);
        fail(kContractViolation, "lower coupling " + std::to_string(l) + " is not the transpose of the upper coupling");
      }
    }
    for (size_t k = 0; k < d.sl_rows.size(); ++k)
      if (layer_of[static_cast<size_t>(d.sl_rows[k])] != layer_of[static_cast<size_t>(d.sl_cols[k])])
        fail(kContractViolation, "sigma_lesser is not block diagonal on the layer map");
  }
  // ---- arena
  int64_t cur = 0;
  auto take = [&](int64_t count) {
    const int64_t o = cur;
    cur += align8(std::max<int64_t>(count, 1));
    return o;
  };
  std::vector<int64_t> og(L), osl(L), ogl(L), ob(L, -1), ogb(L, -1), oxc(L, -1), ogrd(L), oout(L);
  for (int l = 0; l < L; ++l) {
    const int64_t a = nl[l], b = l + 1 < L ? nl[l + 1] : 0;
    og[l] = take(a * a);
    osl[l] = take(a * a);
    ogl[l] = take(a * a);
    if (l + 1 < L) {
      ob[l] = take(a * b);
      ogb[l] = take(a * b);
      oxc[l] = take(a * a);
      ogrd[l] = take(a * a);
      oout[l] = take(a * a);
    }
  }
  ogrd[L - 1] = og[L - 1];
  oout[L - 1] = ogl[L - 1];
  const int64_t nm2 = int64_t(R.max_layer) * R.max_layer;
  const int64_t oT = take(nm2), oM = take(nm2), oPP = take(nm2), oTERM = take(nm2), oX = take(nm2);
  P.big_scratch = cur;
  if (R.max_layer > kSmemInvMax) take(big_scratch_elems(R.max_layer));
  P.arena = cur;
  P.a_region = 0;
  for (int l = 0; l < L; ++l) {
    P.init_zero.push_back(InitRegion{og[l], 1, nl[l] * nl[l], 0});
    P.init_zero.push_back(InitRegion{osl[l], 1, nl[l] * nl[l], 0});
    if (l + 1 < L) P.init_zero.push_back(InitRegion{ob[l], 1, nl[l] * nl[l + 1], 0});
  }
  // ---- assembly maps (same kernels as the HSC path)
  auto a_pos = [&](int r, int c) -> int64_t {
    const int lr = layer_of[static_cast<size_t>(r)], lc = layer_of[static_cast<size_t>(c)];
    const int ir = local_of[static_cast<size_t>(r)], ic = local_of[static_cast<size_t>(c)];
    if (lr == lc) return og[lr] + int64_t(ir) * nl[lr] + ic;
    if (lc == lr + 1) return ob[lr] + int64_t(ir) * nl[lc] + ic;
    return -1;  // lower coupling: the transpose of the upper one
  };
  {
    std::vector<std::pair<int64_t, cplx>> hv;
    for (size_t k = 0; k < d.h_rows.size(); ++k) {
      const int64_t pos = a_pos(d.h_rows[k], d.h_cols[k]);
      if (pos >= 0) hv.push_back({pos, -d.h_vals[k]});
    }
    std::stable_sort(hv.begin(), hv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& e : hv) {
      if (!P.h_pos.empty() && P.h_pos.back() == e.first) P.h_val.back() += e.second;
      else {
        P.h_pos.push_back(e.first);
        P.h_val.push_back(e.second);
      }
    }
  }
  P.diag_pos.resize(static_cast<size_t>(n));
  for (int x = 0; x < n; ++x) {
    const int l = layer_of[static_cast<size_t>(x)];
    P.diag_pos[static_cast<size_t>(x)] = og[l] + int64_t(local_of[static_cast<size_t>(x)]) * (nl[l] + 1);
  }
  {
    std::map<int64_t, std::vector<int>> by_pos;
    for (size_t k = 0; k < d.sr_rows.size(); ++k) {
      const int64_t pos = a_pos(d.sr_rows[k], d.sr_cols[k]);
      if (pos >= 0) by_pos[pos].push_back(static_cast<int>(k));
    }
    P.sr_slot_ptr.push_back(0);
    for (const auto& kv : by_pos) {
      P.sr_slot_pos.push_back(kv.first);
      for (int s : kv.second) P.sr_slot_src.push_back(s);
      P.sr_slot_ptr.push_back(static_cast<int>(P.sr_slot_src.size()));
    }
  }
  {
    std::map<std::pair<int, int>, std::vector<int>> by_rc;
    for (size_t k = 0; k < d.sl_rows.size(); ++k) by_rc[{d.sl_rows[k], d.sl_cols[k]}].push_back(static_cast<int>(k));
    std::map<std::pair<int, int>, int> slot_of;
    P.sl_slot_ptr.push_back(0);
    for (const auto& kv : by_rc) {
      const int r = kv.first.first, c = kv.first.second;
      const int l = layer_of[static_cast<size_t>(r)];
      slot_of[kv.first] = static_cast<int>(P.sl_slot_pos.size());
      P.sl_slot_pos.push_back(osl[l] + int64_t(local_of[static_cast<size_t>(r)]) * nl[l] + local_of[static_cast<size_t>(c)]);
      P.sl_cluster.push_back(l);
      for (int s : kv.second) P.sl_slot_src.push_back(s);
      P.sl_slot_ptr.push_back(static_cast<int>(P.sl_slot_src.size()));
    }
    for (const auto& kv : by_rc) {
      auto it = slot_of.find({kv.first.second, kv.first.first});
      P.sl_partner.push_back(it == slot_of.end() ? -1 : it->second);
    }
    std::vector<int> lidx(static_cast<size_t>(L), -1);
    for (int l : P.sl_cluster)
      if (lidx[l] < 0) lidx[l] = 0;
    for (int l = 0; l < L; ++l)
      if (lidx[l] == 0) {
        lidx[l] = static_cast<int>(P.seeded_ids.size());
        P.seeded_ids.push_back(l);
      }
    for (int l : P.sl_cluster) P.sl_cidx.push_back(lidx[l]);
    P.cslot_ptr.assign(P.seeded_ids.size() + 1, 0);
    for (int c : P.sl_cidx) ++P.cslot_ptr[c + 1];
    for (size_t q = 1; q < P.cslot_ptr.size(); ++q) P.cslot_ptr[q] += P.cslot_ptr[q - 1];
    P.cslots.assign(P.sl_cidx.size(), 0);
    std::vector<int> fillp(P.cslot_ptr.begin(), P.cslot_ptr.end() - 1);
    for (size_t s2 = 0; s2 < P.sl_cidx.size(); ++s2) P.cslots[fillp[P.sl_cidx[s2]]++] = static_cast<int>(s2);
  }
  P.out_gr_pos.resize(static_cast<size_t>(n));
  P.out_gl_pos.resize(static_cast<size_t>(n));
  for (int x = 0; x < n; ++x) {
    const int l = layer_of[static_cast<size_t>(x)];
    const int64_t dd = int64_t(local_of[static_cast<size_t>(x)]) * (nl[l] + 1);
    P.out_gr_pos[static_cast<size_t>(x)] = ogrd[l] + dd;
    P.out_gl_pos[static_cast<size_t>(x)] = oout[l] + dd;
  }
  // ---- schedule
  Builder B(P);
  auto& T = P.gemm_terms;
  auto term = [&](int k, int aop, int64_t a, int lda, int bop, int64_t b, int ldb, int sign) {
    B.add_term(T, k, aop, a, lda, bop, b, ldb, sign);
  };
  auto skew = [&](int sz, int64_t src, int64_t dst) {
    Op op{};
    op.kind = K_SKEW;
    op.phase = 11;
    op.begin = static_cast<int>(P.skew_tasks.size());
    op.count = 1;
    P.skew_tasks.push_back(SkewTask{sz, 0, src, dst});
    P.ops.push_back(op);
  };
  // rgf_gr forward sweep (rgf.cpp:198-225), dense couplings
  for (int l = 0; l < L; ++l) {
    if (l > 0) {
      const int a = nl[l - 1], b = nl[l];
      B.open(K_GEMM, 10, l);  // GB_{l-1} = g_{l-1} B_{l-1}
      int tb = static_cast<int>(T.size());
      term(a, OP_N, og[l - 1], a, OP_N, ob[l - 1], b, +1);
      B.gemm_task(a, b, ogb[l - 1], b, MODE_SET, 0, 0, tb);
      B.close();
      B.open(K_GEMM, 10, l);  // m = D_l - GB^T B
      tb = static_cast<int>(T.size());
      term(a, OP_T, ogb[l - 1], b, OP_N, ob[l - 1], b, -1);
      B.gemm_task(b, b, og[l], b, MODE_ADD, 0, 0, tb);
      B.close();
    }
    B.emit_inverses(l, 10, {InvItem{nl[l], l, l, og[l]}}, P.big_scratch);
  }
  // backward sweep (rgf.cpp:227-282)
  for (int l = L - 2; l >= 0; --l) {
    const int a = nl[l], b = nl[l + 1];
    B.open(K_GEMM, 10, l);  // goff = -G_{l+1,l+1} GB_l^T   (b x a)
    int tb = static_cast<int>(T.size());
    term(b, OP_N, ogrd[l + 1], b, OP_T, ogb[l], b, -1);
    B.gemm_task(b, a, oT, a, MODE_SET, 0, 0, tb);
    B.close();
    B.open(K_GEMM, 10, l);
    tb = static_cast<int>(T.size());  // G_ll = g_l - GB_l goff
    term(b, OP_N, ogb[l], b, OP_N, oT, a, -1);
    B.gemm_task(a, a, ogrd[l], a, MODE_INIT, og[l], a, tb);
    tb = static_cast<int>(T.size());  // xcoef_l = -goff^T B_l^T
    term(b, OP_T, oT, a, OP_T, ob[l], b, -1);
    B.gemm_task(a, a, oxc[l], a, MODE_SET, 0, 0, tb);
    B.close();
  }
  P.rgf_gr_ops = static_cast<int>(P.ops.size());
  // rgf_gless forward sweep (rgf.cpp:310-345)
  for (int l = 0; l < L; ++l) {
    const int b = nl[l];
    if (l > 0) {
      const int a = nl[l - 1];
      B.open(K_GEMM, 11, l);  // t = B^T g<_{l-1}   (b x a)
      int tb = static_cast<int>(T.size());
      term(a, OP_T, ob[l - 1], b, OP_N, ogl[l - 1], a, +1);
      B.gemm_task(b, a, oT, a, MODE_SET, 0, 0, tb);
      B.close();
      B.open(K_GEMM, 11, l);  // S_l += t conj(B)
      tb = static_cast<int>(T.size());
      term(a, OP_N, oT, a, OP_C, ob[l - 1], b, +1);
      B.gemm_task(b, b, osl[l], b, MODE_ADD, 0, 0, tb);
      B.close();
    }
    B.open(K_GEMM, 11, l);  // m = g_l S_l
    int tb = static_cast<int>(T.size());
    term(b, OP_N, og[l], b, OP_N, osl[l], b, +1);
    B.gemm_task(b, b, oM, b, MODE_SET, 0, 0, tb);
    B.close();
    B.open(K_GEMM, 11, l);  // m g_l^H
    tb = static_cast<int>(T.size());
    term(b, OP_N, oM, b, OP_H, og[l], b, +1);
    B.gemm_task(b, b, oPP, b, MODE_SET, 0, 0, tb);
    B.close();
    skew(b, oPP, ogl[l]);
  }
  // backward sweep (rgf.cpp:347-378)
  for (int l = L - 2; l >= 0; --l) {
    const int a = nl[l], b = nl[l + 1];
    B.open(K_GEMM, 11, l);
    int tb = static_cast<int>(T.size());  // m = W G<_{l+1}, W = GB_l
    term(b, OP_N, ogb[l], b, OP_N, oout[l + 1], b, +1);
    B.gemm_task(a, b, oM, b, MODE_SET, 0, 0, tb);
    tb = static_cast<int>(T.size());  // x = xcoef_l g<_l
    term(a, OP_N, oxc[l], a, OP_N, ogl[l], a, +1);
    B.gemm_task(a, a, oX, a, MODE_SET, 0, 0, tb);
    B.close();
    B.open(K_GEMM, 11, l);  // m W^H
    tb = static_cast<int>(T.size());
    term(b, OP_N, oM, b, OP_H, ogb[l], b, +1);
    B.gemm_task(a, a, oPP, a, MODE_SET, 0, 0, tb);
    B.close();
    skew(a, oPP, oTERM);
    Op op{};
    op.kind = K_COMBINE;
    op.phase = 11;
    op.begin = static_cast<int>(P.comb_tasks.size());
    op.count = 1;
    P.comb_tasks.push_back(CombineTask{a, 0, ogl[l], oTERM, oX, oout[l]});
    P.ops.push_back(op);
  }
  P.max_block = R.max_layer;
  for (int l = 0; l < L; ++l) P.exec_inv_cmul += double(nl[l]) * nl[l] * nl[l];
  P.rgf_layers = std::move(layers);
  P.lesser_op = P.rgf_gr_ops;
  P.gr_done_op = static_cast<int>(P.ops.size());
  return P;
}

}  // namespace negfb
