// C ABI of the B200 HSC path (include/negf_gpu.h): host plan handles, device
// handles, the per-batch schedule replay and the NCCL density exchange.
#include "negf_gpu.h"

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <memory>
#include <string>
#include <functional>
#include <vector>

#include "capi_util.hpp"
#include "kernels.hpp"
#include "plan.hpp"
#include "tree.hpp"

using namespace negfb;

struct negf_plan {
  Plan plan;
};

namespace {

// --- NCCL, resolved at run time so the process reuses whichever libnccl the
// framework (torch) already loaded.
typedef int (*nccl_get_id_t)(void*);
typedef int (*nccl_allreduce_t)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef int (*nccl_allgather_t)(const void*, void*, size_t, int, void*, cudaStream_t);
typedef int (*nccl_destroy_t)(void*);
typedef const char* (*nccl_err_t)(int);
struct NcclApi {
  bool ok = false;
  nccl_get_id_t get_id = nullptr;
  void* init = nullptr;
  nccl_allreduce_t allreduce = nullptr;
  nccl_allgather_t allgather = nullptr;
  nccl_destroy_t destroy = nullptr;
  nccl_err_t err = nullptr;
};
struct NcclId {
  char internal[128];
};
typedef int (*nccl_init_by_value_t)(void**, int, NcclId, int);

NcclApi load_nccl() {
  NcclApi api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.get_id = reinterpret_cast<nccl_get_id_t>(dlsym(h, "ncclGetUniqueId"));
  api.init = dlsym(h, "ncclCommInitRank");
  api.allreduce = reinterpret_cast<nccl_allreduce_t>(dlsym(h, "ncclAllReduce"));
  api.allgather = reinterpret_cast<nccl_allgather_t>(dlsym(h, "ncclAllGather"));
  api.destroy = reinterpret_cast<nccl_destroy_t>(dlsym(h, "ncclCommDestroy"));
  api.err = reinterpret_cast<nccl_err_t>(dlsym(h, "ncclGetErrorString"));
  api.ok = api.get_id && api.init && api.allreduce && api.destroy;
  return api;
}

NcclApi& nccl() {
  static NcclApi api = load_nccl();  // thread-safe one-time resolution
  return api;
}

constexpr double kTwoPi = 6.283185307179586476925286766559;

}  // namespace

struct negf_gpu {
  const Plan* plan = nullptr;
  int device = 0;
  cudaStream_t stream = nullptr;
  // host-buffer solves: Sigma^< in and G^r out on a copy stream, overlapping
  // the fold / the G^< sweep (created on first use)
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_sl = nullptr, ev_gr = nullptr;
  std::vector<void*> owned;
  int capacity = 1;
  double2* arena = nullptr;
  int64_t* d_h_pos = nullptr;
  double2* d_h_val = nullptr;
  InitRegion* d_init_zero = nullptr;
  int64_t* d_diag_pos = nullptr;
  int64_t *d_sr_pos = nullptr, *d_sl_pos = nullptr, *d_gr_pos = nullptr, *d_gl_pos = nullptr;
  int *d_sr_ptr = nullptr, *d_sr_src = nullptr, *d_sl_ptr = nullptr, *d_sl_src = nullptr;
  int *d_sl_partner = nullptr, *d_sl_cidx = nullptr, *d_seeded = nullptr;
  int *d_cslots = nullptr, *d_cslot_ptr = nullptr;
  GemmTask* d_tasks = nullptr;
  GemmTerm* d_terms = nullptr;
  GemmTile* d_tiles = nullptr;
  DiagTask* d_diag = nullptr;
  GemmTerm* d_diag_terms = nullptr;
  ScaleTask* d_scale = nullptr;
  InvTask* d_inv = nullptr;
  BigTask* d_big = nullptr;
  SkewTask* d_skew_tasks = nullptr;
  SpsiTask* d_spsi = nullptr;
  int* d_spsi_colptr = nullptr;
  int* d_spsi_wcols = nullptr;
  MGatherTask* d_mg = nullptr;
  MGatherBlock* d_mg_blocks = nullptr;
  int* d_spsi_row = nullptr;
  double2* d_spsi_val = nullptr;
  SschurTask* d_sschur = nullptr;
  SschurContrib* d_sschur_contrib = nullptr;
  int* d_sschur_rc = nullptr;
  LeafDiagTask* d_ld = nullptr;
  int* d_ld_rows = nullptr;
  int* d_ld_optr = nullptr;
  LeafDiagEntry* d_ld_entries = nullptr;
  CombineTask* d_comb_tasks = nullptr;
  // per-batch staging
  double *d_energies = nullptr, *d_weights = nullptr;
  double2 *d_sigma_r = nullptr, *d_sigma_l = nullptr, *d_gr = nullptr, *d_gl = nullptr;
  double* d_density = nullptr;
  double* d_skew = nullptr;
  DevStatus* d_status = nullptr;
  unsigned long long* d_gemm_ctr = nullptr;  // persistent-GEMM work counters (BatchArgs::gemm_ctr)
  void* comm = nullptr;
  int nranks = 1;
  double* d_gather = nullptr;  // nranks x n partial densities (ordered reduction)
  // Cross-rank sum of the partials (negf_gpu_allreduce_density); d_density
  // itself stays this rank's running partial, so later solves and reductions
  // never count an earlier contribution twice.
  double* d_reduced = nullptr;
  bool reduced_valid = false;       // d_reduced is newer than every solve
  unsigned long long resid_first = ~0ull;  // lowest (energy << 32 | dof) residual key seen
  int64_t launches = 0;
  int residual_mode = 1;
  int ordered_reduce = 1;
  double max_resid = 0.0;
  // profiling
  bool profiling = false;
  std::vector<cudaEvent_t> ev;
  struct Rec {
    int kind;
    double cmul;
    int64_t launches;
    int op;
  };
  std::vector<Rec> recs;
  negf_kernel_stat stats[NEGF_KSTAT_COUNT] = {};
  std::vector<double> op_ms;  // per plan op, summed over profiled solves
};

namespace {

// Event bracket around one launch group (profiling mode only).
struct Bracket {
  negf_gpu* g;
  int kind;
  double cmul;
  int64_t before;
  int op;
  Bracket(negf_gpu* gg, int k, double c, int o = -1) : g(gg), kind(k), cmul(c), before(gg->launches), op(o) {
    if (!g->profiling) return;
    const size_t i = 2 * g->recs.size();
    while (g->ev.size() < i + 2) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      g->ev.push_back(e);
    }
    cudaEventRecord(g->ev[i], g->stream);
  }
  ~Bracket() {
    if (!g->profiling) return;
    const size_t i = 2 * g->recs.size();
    cudaEventRecord(g->ev[i + 1], g->stream);
    g->recs.push_back({kind, cmul, g->launches - before, op});
  }
};

void flush_profile(negf_gpu* g) {
  if (!g->profiling || g->recs.empty()) return;
  cudaStreamSynchronize(g->stream);
  static const bool verbose = [] {
    const char* e = std::getenv("NEGF_PROFILE_VERBOSE");
    return e && e[0] == '1';
  }();
  for (size_t r = 0; r < g->recs.size(); ++r) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, g->ev[2 * r], g->ev[2 * r + 1]);
    if (verbose && g->recs[r].op >= 0) {
      const Op& op = g->plan->ops[g->recs[r].op];
      std::fprintf(stderr, "[negf-prof] op %3d kind %d phase %d level %2d count %6d ms %9.3f TF/s %7.2f\n",
                   g->recs[r].op, op.kind, op.phase, op.level, op.count, ms,
                   ms > 0 ? 8.0 * g->recs[r].cmul / (ms * 1e-3) / 1e12 : 0.0);
    }
    if (g->recs[r].op >= 0) {
      if (g->op_ms.size() < g->plan->ops.size()) g->op_ms.assign(g->plan->ops.size(), 0.0);
      g->op_ms[g->recs[r].op] += ms;
    }
    negf_kernel_stat& s = g->stats[g->recs[r].kind];
    s.ms += ms;
    s.cmul += g->recs[r].cmul;
    s.launches += g->recs[r].launches;
  }
  g->recs.clear();
}

}  // namespace

namespace {

void reset_status(negf_gpu* g) {
  DevStatus h{~0ull, ~0ull, ~0ull, 0ull};
  ck(cudaMemcpyAsync(g->d_status, &h, sizeof h, cudaMemcpyHostToDevice, g->stream), "status reset");
}

// Phases (Op::phase bit mask) whose GEMM ops use the Gauss (3M) complex
// product.  Default 0: the conventional product everywhere.  NEGF_GEMM_3M_PHASES
// (e.g. 3 = fold + G^r sweep) is an A/B switch: the G^< phases (seeds, N fold,
// P rows) must keep the conventional product, whose rounding keeps diag G^<
// imaginary to the reference's level.
unsigned gauss3m_phases() {
  static const unsigned m = [] {
    const char* e = std::getenv("NEGF_GEMM_3M_PHASES");
    return e ? static_cast<unsigned>(std::atoi(e)) : 0u;
  }();
  return m;
}

// Host-side hooks of a batch replay: `lesser_in` enqueues the Sigma^< upload
// (it runs right before the first Sigma^< reader is enqueued, so the fold is
// already queued while a pageable copy stages); with `gr_early`, the G^r
// diagonal is written as soon as it is final and `gr_ready` recorded after it.
struct BatchHooks {
  std::function<void()> lesser_in;
  bool gr_early = false;
  cudaEvent_t gr_ready = nullptr;
};

// Replays the plan's schedule for one batch (all inputs on device).
void run_batch(negf_gpu* g, int nE, int e_base, const double* d_E, const double* d_w,
               const double2* d_sr, const double2* d_sl, double2* d_gr, double2* d_gl,
               const BatchHooks* hk = nullptr) {
  const Plan& P = *g->plan;
  BatchArgs b{g->arena, P.arena, nE, e_base, g->d_gemm_ctr};
  cudaStream_t s = g->stream;
  int64_t& L = g->launches;
  {
    Bracket br(g, NEGF_KSTAT_ASSEMBLE, 0.0);
    launch_assemble(b, P, g->d_h_pos, g->d_h_val, g->d_init_zero, g->d_diag_pos, d_E, g->d_sr_pos, g->d_sr_ptr,
                    g->d_sr_src, static_cast<int64_t>(P.desc.sr_rows.size()), d_sr, s, L);
  }
  const auto lesser = [&] {
    if (hk && hk->lesser_in) hk->lesser_in();
    Bracket br(g, NEGF_KSTAT_ASSEMBLE, 0.0);
    const int64_t sl_nnz = static_cast<int64_t>(P.desc.sl_rows.size());
    launch_scatter_lesser(b, P, d_E, g->d_sl_pos, g->d_sl_ptr, g->d_sl_src, sl_nnz, d_sl, s, L);
    launch_skew_check(b, d_sl, sl_nnz, g->d_cslots, g->d_cslot_ptr, g->d_sl_ptr, g->d_sl_src, g->d_sl_partner,
                      static_cast<int>(P.seeded_ids.size()), g->d_seeded, g->d_skew, g->d_status, s, L);
  };
  const bool gr_early = hk && hk->gr_early && d_gr;
  const auto gr_out = [&] {
    if (!gr_early) return;
    Bracket br(g, NEGF_KSTAT_OUTPUT, 0.0);
    launch_output_gr(b, P.desc.n, g->d_gr_pos, d_gr, s, L);
    if (hk->gr_ready) ck(cudaEventRecord(hk->gr_ready, s), "event");
  };
  static const int kind_stat[13] = {NEGF_KSTAT_INVERSE, NEGF_KSTAT_GEMM,    NEGF_KSTAT_DIAG,
                                    NEGF_KSTAT_SCALE,   NEGF_KSTAT_INVERSE, NEGF_KSTAT_INVERSE,
                                    NEGF_KSTAT_SCALE,   NEGF_KSTAT_SCALE,   NEGF_KSTAT_SCALE,
                                    NEGF_KSTAT_SCALE,   NEGF_KSTAT_DIAG,    NEGF_KSTAT_INVERSE,
                                    NEGF_KSTAT_DIAG};
  // K_SPSI / K_SSCHUR: sparse, with the scalings; K_LEAFDIAG: diagonals;
  // K_BIGSWAP: part of the multi-CTA inverse
  for (size_t oi = 0; oi < P.ops.size(); ++oi) {
    if (static_cast<int>(oi) == P.gr_done_op) gr_out();
    if (static_cast<int>(oi) == P.lesser_op) lesser();
    const Op& op = P.ops[oi];
    Bracket br(g, kind_stat[op.kind], op.cmul * nE, static_cast<int>(oi));
    switch (op.kind) {
      case K_INVERSE:
        launch_inverse(b, g->d_inv + op.begin, P.inv_tasks.data() + op.begin, op.count, g->d_status, s, L);
        break;
      case K_GEMM:
        launch_gemm(b, g->d_tasks, g->d_terms, g->d_tiles, P.gemm_tiles.data(), op.begin, op.count, s, L,
                    gauss3m_phases() & (1u << op.phase));
        break;
      case K_DIAG:
        launch_diag(b, g->d_diag, g->d_diag_terms, op.begin, op.count, s, L);
        break;
      case K_PANEL:
        launch_bigpanel(b, g->d_big + op.begin, P.big_tasks.data() + op.begin, op.count, op.k0, op.k1, g->d_status, s, L);
        break;
      case K_PERM:
        launch_bigperm(b, g->d_big + op.begin, P.big_tasks.data() + op.begin, op.count, s, L);
        break;
      case K_BIGSWAP:
        launch_bigswap(b, g->d_big + op.begin, op.count, op.k1, s, L);
        break;
      case K_SKEW:
        launch_skew(b, g->d_skew_tasks, P.skew_tasks.data(), op.begin, op.count, s, L);
        break;
      case K_COMBINE:
        launch_combine(b, g->d_comb_tasks, P.comb_tasks.data(), op.begin, op.count, s, L);
        break;
      case K_SPSI:
        launch_spsi(b, g->d_spsi, g->d_spsi_colptr, g->d_spsi_row, g->d_spsi_val, g->d_spsi_wcols, op.begin, op.count,
                    s, L);
        break;
      case K_MGATHER:
        launch_mgather(b, g->d_mg, g->d_mg_blocks, op.begin, op.count, s, L);
        break;
      case K_LEAFDIAG:
        launch_leafdiag(b, g->d_ld, P.ld_tasks.data(), g->d_ld_rows, g->d_ld_optr, P.ld_optr.data(),
                        g->d_ld_entries, op.begin, op.count, s, L);
        break;
      case K_SSCHUR:
        launch_sschur(b, g->d_sschur, g->d_sschur_contrib, g->d_spsi, g->d_spsi_colptr, g->d_spsi_row,
                      g->d_spsi_val, g->d_sschur_rc, op.begin, op.count, s, L);
        break;
      default:
        launch_scale(b, g->d_scale, op.begin, op.count, s, L);
        break;
    }
  }
  if (P.gr_done_op >= static_cast<int>(P.ops.size())) gr_out();
  if (P.lesser_op >= static_cast<int>(P.ops.size())) lesser();
  {
    Bracket br(g, NEGF_KSTAT_OUTPUT, 0.0);
    launch_output(b, P.desc.n, g->d_gr_pos, g->d_gl_pos, d_w, gr_early ? nullptr : d_gr, d_gl, g->d_density,
                  g->d_status, s, L);
  }
  ck(cudaGetLastError(), "kernel launch");
}

// Reads the device status and maps it to the reference's precedence: the
// lowest energy index wins; within one energy the fold's SingularBlock comes
// before validate_sigma's NonSkewHermitianInput (hsc_fold runs first,
// run.cpp:164-169); ResidualTooLarge is raised only when every energy solved
// (electron_density runs after solve_all, run.cpp:285-291).
//
// The device status is sticky: every solve since the last collect() merges
// into it (atomicMin keys), so errors of asynchronous calls (sync = 0) are
// reported by the next negf_gpu_check / synchronous solve; it is cleared only
// here, once read.
int collect(negf_gpu* g, negf_status* st) {
  DevStatus h;
  ck(cudaMemcpyAsync(&h, g->d_status, sizeof h, cudaMemcpyDeviceToHost, g->stream), "status read");
  ck(cudaStreamSynchronize(g->stream), "stream sync");
  reset_status(g);
  const unsigned long long none = ~0ull;
  double worst;
  std::memcpy(&worst, &h.max_resid_bits, sizeof worst);
  g->max_resid = std::max(g->max_resid, worst);
  g->resid_first = std::min<unsigned long long>(g->resid_first, h.residual_key);
  const long long es = h.singular_key == none ? -1 : static_cast<long long>(h.singular_key >> 40);
  const long long en = h.nonskew_key == none ? -1 : static_cast<long long>(h.nonskew_key >> 32);
  if (es >= 0 && (en < 0 || es <= en)) {
    const int fold_pos = static_cast<int>((h.singular_key >> 20) & 0xFFFFF);
    const int pivot = static_cast<int>(h.singular_key & 0xFFFFF);
    if (!g->plan->rgf_layers.empty()) {  // RGF: fold_pos is the layer
      const int sz = static_cast<int>(g->plan->rgf_layers[static_cast<size_t>(fold_pos)].size());
      return set_status(st, NEGF_SINGULAR_BLOCK,
                        "energy point " + std::to_string(es) + ": inverse: singular pivot " + std::to_string(pivot) +
                            " in " + std::to_string(sz) + "x" + std::to_string(sz) + " block of layer " +
                            std::to_string(fold_pos),
                        static_cast<int>(es), fold_pos, pivot);
    }
    const Tree& t = g->plan->tree;
    const int cluster = fold_pos < static_cast<int>(t.fold_order().size()) ? t.fold_order()[fold_pos] : t.root();
    return set_status(st, NEGF_SINGULAR_BLOCK,
                      "energy point " + std::to_string(es) + ": inverse: singular pivot " +
                          std::to_string(pivot) + " in " + std::to_string(t.cluster(cluster).size()) + "x" +
                          std::to_string(t.cluster(cluster).size()) + " block of cluster " +
                          std::to_string(cluster),
                      static_cast<int>(es), cluster, pivot);
  }
  if (en >= 0) {
    const int cluster = static_cast<int>(h.nonskew_key & 0xFFFFFFFFull);
    return set_status(st, NEGF_NON_SKEW_HERMITIAN,
                      "energy point " + std::to_string(en) + ": sigma_lesser block of cluster " +
                          std::to_string(cluster) + " is not skew-Hermitian",
                      static_cast<int>(en), cluster);
  }
  if (h.residual_key != none && g->residual_mode != 0) {
    const int e = static_cast<int>(h.residual_key >> 32);
    const int d = static_cast<int>(h.residual_key & 0xFFFFFFFFull);
    return set_status(st, NEGF_RESIDUAL_TOO_LARGE,
                      "G^< diagonal entry has a real part beyond the skew-Hermitian tolerance at "
                      "energy index " + std::to_string(e) + ", dof " + std::to_string(d),
                      e, -1, -1, d);
  }
  return ok(st);
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

ProblemDesc desc_from_c(const negf_problem* p) {
  ProblemDesc d;
  d.n = p->n_dofs;
  d.h_rows.assign(p->h_rows, p->h_rows + p->h_nnz);
  d.h_cols.assign(p->h_cols, p->h_cols + p->h_nnz);
  d.h_vals.resize(static_cast<size_t>(p->h_nnz));
  for (int64_t k = 0; k < p->h_nnz; ++k) d.h_vals[k] = cplx(p->h_vals[2 * k], p->h_vals[2 * k + 1]);
  if (p->sr_nnz) {
    d.sr_rows.assign(p->sr_rows, p->sr_rows + p->sr_nnz);
    d.sr_cols.assign(p->sr_cols, p->sr_cols + p->sr_nnz);
  }
  if (p->sl_nnz) {
    d.sl_rows.assign(p->sl_rows, p->sl_rows + p->sl_nnz);
    d.sl_cols.assign(p->sl_cols, p->sl_cols + p->sl_nnz);
  }
  if (p->coords) {
    d.coords.resize(static_cast<size_t>(p->n_dofs));
    for (int i = 0; i < p->n_dofs; ++i) d.coords[i] = {p->coords[2 * i], p->coords[2 * i + 1]};
  }
  for (int gi = 0; gi < p->n_groups; ++gi)
    d.atomic_groups.emplace_back(p->group_dofs + p->group_ptr[gi], p->group_dofs + p->group_ptr[gi + 1]);
  d.max_leaf = p->max_leaf;
  if (p->n_tree_clusters > 0) {
    d.explicit_tree = true;
    d.tree_parent.assign(p->tree_parent, p->tree_parent + p->n_tree_clusters);
    for (int c = 0; c < p->n_tree_clusters; ++c)
      d.tree_dofs.emplace_back(p->tree_dofs + p->tree_ptr[c], p->tree_dofs + p->tree_ptr[c + 1]);
  }
  return d;
}

}  // namespace

extern "C" {

int negf_plan_create(const negf_problem* p, negf_plan** out, negf_status* st) {
  if (!p || !out) return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  try {
    *out = new negf_plan{build_plan(desc_from_c(p))};
    return ok(st);
  } catch (const Failure& f) {
    return set_status(st, f.code, f.what());
  } catch (const std::exception& e) {
    return set_status(st, NEGF_INTERNAL, e.what());
  }
}

int negf_rgf_plan_create(const negf_problem* p, int n_layers, const int32_t* layer_ptr, const int32_t* layer_dofs,
                         negf_plan** out, negf_status* st) {
  if (!p || !out || n_layers < 0 || (n_layers > 0 && (!layer_ptr || !layer_dofs)))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  try {
    std::vector<std::vector<int>> layers;
    for (int l = 0; l < n_layers; ++l) layers.emplace_back(layer_dofs + layer_ptr[l], layer_dofs + layer_ptr[l + 1]);
    *out = new negf_plan{build_rgf_plan(desc_from_c(p), std::move(layers))};
    return ok(st);
  } catch (const Failure& f) {
    return set_status(st, f.code, f.what());
  } catch (const std::exception& e) {
    return set_status(st, NEGF_INTERNAL, e.what());
  }
}

int negf_plan_info_get(const negf_plan* h, negf_plan_info* info) {
  if (!h || !info) return NEGF_CONTRACT_VIOLATION;
  const Plan& P = h->plan;
  info->n_dofs = P.desc.n;
  const bool rgf = !P.rgf_layers.empty();
  info->n_clusters = rgf ? static_cast<int>(P.rgf_layers.size()) : P.tree.num_clusters();
  info->levels = rgf ? 0 : P.tree.levels();
  info->root = rgf ? -1 : P.tree.root();
  info->max_block = P.max_block;
  info->arena_bytes_per_energy = P.arena * 16;
  info->ref_fold_mul = P.ref_fold.multiply_ops;
  info->ref_fold_inv = P.ref_fold.inverse_ops;
  info->ref_gless_mul = P.ref_gless.multiply_ops;
  info->ref_gless_inv = P.ref_gless.inverse_ops;
  info->exec_cmul = P.exec_cmul;
  info->exec_inv_cmul = P.exec_inv_cmul;
  info->needed_cmul = P.needed_cmul > 0.0 ? P.needed_cmul : P.exec_cmul;
  info->n_real_clusters = P.n_real_clusters;
  info->pad_ = 0;
  info->n_ops = static_cast<int>(P.ops.size());
  info->n_gemm_tasks = static_cast<int>(P.gemm_tasks.size());
  info->n_gemm_tiles = static_cast<int>(P.gemm_tiles.size());
  info->n_inv_tasks = static_cast<int>(P.inv_tasks.size());
  return NEGF_OK;
}

int negf_plan_tree(const negf_plan* h, int32_t* parent, int32_t* level, int32_t* dof_ptr, int32_t* dofs,
                   int32_t* fold_order) {
  if (h && !h->plan.rgf_layers.empty()) return NEGF_CONTRACT_VIOLATION;
  if (!h) return NEGF_CONTRACT_VIOLATION;
  const Tree& t = h->plan.tree;
  int32_t off = 0;
  for (int c = 0; c < t.num_clusters(); ++c) {
    const Cluster& cl = t.cluster(c);
    if (parent) parent[c] = cl.parent;
    if (level) level[c] = cl.level;
    if (dof_ptr) dof_ptr[c] = off;
    if (dofs) std::copy(cl.dofs.begin(), cl.dofs.end(), dofs + off);
    off += cl.size();
  }
  if (dof_ptr) dof_ptr[t.num_clusters()] = off;
  if (fold_order) std::copy(t.fold_order().begin(), t.fold_order().end(), fold_order);
  return NEGF_OK;
}

int negf_plan_fill(const negf_plan* h, int32_t* ptr, int32_t* ids) {
  if (h && !h->plan.rgf_layers.empty()) return NEGF_CONTRACT_VIOLATION;
  if (!h) return NEGF_CONTRACT_VIOLATION;
  int32_t off = 0;
  const auto& ci = h->plan.ci;
  for (size_t c = 0; c < ci.size(); ++c) {
    if (ptr) ptr[c] = off;
    if (ids) std::copy(ci[c].S.begin(), ci[c].S.end(), ids + off);
    off += static_cast<int32_t>(ci[c].S.size());
  }
  if (ptr) ptr[ci.size()] = off;
  return NEGF_OK;
}

int negf_plan_gemm_tasks(const negf_plan* h, int32_t* m, int32_t* n, int64_t* k_total, int32_t* phase,
                         int32_t* level) {
  if (!h) return NEGF_CONTRACT_VIOLATION;
  const Plan& P = h->plan;
  for (const Op& op : P.ops) {
    if (op.kind != K_GEMM) continue;
    for (int t = op.task_begin; t < op.task_begin + op.task_count; ++t) {
      const GemmTask& tk = P.gemm_tasks[t];
      int64_t ks = 0;
      for (int q = tk.term_begin; q < tk.term_begin + tk.term_count; ++q) ks += P.gemm_terms[q].k;
      if (m) m[t] = tk.m;
      if (n) n[t] = tk.n;
      if (k_total) k_total[t] = ks;
      if (phase) phase[t] = op.phase;
      if (level) level[t] = op.level;
    }
  }
  return NEGF_OK;
}

int negf_plan_gemm_tiles(const negf_plan* h, int32_t* task, int32_t* m0, int32_t* n0, int32_t* arr,
                         int32_t* mirrored) {
  if (!h) return NEGF_CONTRACT_VIOLATION;
  const Plan& P = h->plan;
  for (std::size_t i = 0; i < P.gemm_tiles.size(); ++i) {
    const GemmTile& t = P.gemm_tiles[i];
    if (task) task[i] = t.task;
    if (m0) m0[i] = t.m0;
    if (n0) n0[i] = t.n0;
    if (arr) arr[i] = t.arr;
    if (mirrored) mirrored[i] = (P.gemm_tasks[t.task].mirror && t.n0 > t.m0) ? 1 : 0;
  }
  return NEGF_OK;
}

int negf_plan_ops(const negf_plan* h, int32_t* kind, int32_t* phase, int32_t* level, int32_t* begin,
                  int32_t* count, double* cmul) {
  if (!h) return NEGF_CONTRACT_VIOLATION;
  const Plan& P = h->plan;
  for (std::size_t i = 0; i < P.ops.size(); ++i) {
    const Op& o = P.ops[i];
    if (kind) kind[i] = o.kind;
    if (phase) phase[i] = o.kind == K_GEMM && o.inv_update ? 6 : o.phase;
    if (level) level[i] = o.level;
    if (begin) begin[i] = o.begin;
    if (count) count[i] = o.count;
    if (cmul) cmul[i] = o.cmul;
  }
  return NEGF_OK;
}

void negf_plan_destroy(negf_plan* p) { delete p; }

int negf_gpu_create(const negf_plan* hp, int device, int max_energy_batch, negf_gpu** out,
                    negf_status* st) {
  if (!hp || !out) return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  auto g = std::make_unique<negf_gpu>();
  try {
    const Plan& P = hp->plan;
    g->plan = &P;
    g->device = device;
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking), "stream");
    auto& o = g->owned;
    g->d_h_pos = dev_upload(P.h_pos, o);
    g->d_h_val = reinterpret_cast<double2*>(dev_upload(P.h_val, o));
    g->d_diag_pos = dev_upload(P.diag_pos, o);
    g->d_init_zero = dev_upload(P.init_zero, o);
    g->d_sr_pos = dev_upload(P.sr_slot_pos, o);
    g->d_sr_ptr = dev_upload(P.sr_slot_ptr, o);
    g->d_sr_src = dev_upload(P.sr_slot_src, o);
    g->d_sl_pos = dev_upload(P.sl_slot_pos, o);
    g->d_sl_ptr = dev_upload(P.sl_slot_ptr, o);
    g->d_sl_src = dev_upload(P.sl_slot_src, o);
    g->d_sl_partner = dev_upload(P.sl_partner, o);
    g->d_sl_cidx = dev_upload(P.sl_cidx, o);
    g->d_seeded = dev_upload(P.seeded_ids, o);
    g->d_cslots = dev_upload(P.cslots, o);
    g->d_cslot_ptr = dev_upload(P.cslot_ptr, o);
    g->d_gr_pos = dev_upload(P.out_gr_pos, o);
    g->d_gl_pos = dev_upload(P.out_gl_pos, o);
    g->d_tasks = dev_upload(P.gemm_tasks, o);
    g->d_terms = dev_upload(P.gemm_terms, o);
    g->d_tiles = dev_upload(P.gemm_tiles, o);
    g->d_diag = dev_upload(P.diag_tasks, o);
    g->d_diag_terms = dev_upload(P.diag_terms, o);
    g->d_scale = dev_upload(P.scale_tasks, o);
    g->d_inv = dev_upload(P.inv_tasks, o);
    g->d_big = dev_upload(P.big_tasks, o);
    g->d_skew_tasks = dev_upload(P.skew_tasks, o);
    g->d_spsi = dev_upload(P.spsi_tasks, o);
    g->d_spsi_colptr = dev_upload(P.spsi_colptr, o);
    g->d_spsi_wcols = dev_upload(P.spsi_wcols, o);
    g->d_mg = dev_upload(P.mg_tasks, o);
    g->d_mg_blocks = dev_upload(P.mg_blocks, o);
    g->d_spsi_row = dev_upload(P.spsi_row, o);
    g->d_spsi_val = reinterpret_cast<double2*>(dev_upload(P.spsi_val, o));
    g->d_sschur = dev_upload(P.sschur_tasks, o);
    g->d_sschur_contrib = dev_upload(P.sschur_contrib, o);
    g->d_sschur_rc = dev_upload(P.sschur_rc, o);
    g->d_ld = dev_upload(P.ld_tasks, o);
    g->d_ld_rows = dev_upload(P.ld_rows, o);
    g->d_ld_optr = dev_upload(P.ld_optr, o);
    g->d_ld_entries = dev_upload(P.ld_entries, o);
    g->d_comb_tasks = dev_upload(P.comb_tasks, o);
    const int n = P.desc.n;
    const size_t sr = P.desc.sr_rows.size(), sl = P.desc.sl_rows.size();
    const size_t per_energy = size_t(P.arena) * 16 + (sr + sl) * 16 + size_t(n) * 32 + 16 +
                              P.seeded_ids.size() * 16;
    size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
    // energies of a batch go in gridDim.y / gridDim.z: at most kMaxGridYZ
    int cap = static_cast<int>(std::min<size_t>(size_t(0.85 * double(free_b)) / per_energy, kMaxGridYZ));
    if (max_energy_batch > 0) cap = std::min(cap, max_energy_batch);
    if (cap < 1)
      throw CudaFail{NEGF_OUT_OF_MEMORY, "one energy point needs " + std::to_string(per_energy) +
                                             " bytes of device memory; " + std::to_string(free_b) + " free"};
    g->capacity = cap;
    g->arena = dev_alloc<double2>(size_t(P.arena) * cap, o);
    g->d_energies = dev_alloc<double>(cap, o);
    g->d_weights = dev_alloc<double>(cap, o);
    g->d_sigma_r = dev_alloc<double2>(sr * cap, o);
    g->d_sigma_l = dev_alloc<double2>(sl * cap, o);
    g->d_gr = dev_alloc<double2>(size_t(n) * cap, o);
    g->d_gl = dev_alloc<double2>(size_t(n) * cap, o);
    g->d_density = dev_alloc<double>(n, o);
    g->d_skew = dev_alloc<double>(2 * std::max<size_t>(1, P.seeded_ids.size()) * cap, o);
    g->d_status = dev_alloc<DevStatus>(1, o);
    g->d_gemm_ctr = dev_alloc<unsigned long long>(2, o);
    ck(cudaMemsetAsync(g->d_gemm_ctr, 0, 2 * sizeof(unsigned long long), g->stream), "memset");
    ck(cudaMemsetAsync(g->d_density, 0, sizeof(double) * n, g->stream), "memset");
    reset_status(g.get());
    ck(cudaStreamSynchronize(g->stream), "sync");
    *out = g.release();
    return ok(st);
  } catch (const CudaFail& f) {
    for (void* p : g->owned) cudaFree(p);
    if (g->stream) cudaStreamDestroy(g->stream);
    return set_status(st, f.code, f.msg);
  }
}

int negf_gpu_batch_capacity(const negf_gpu* g) { return g ? g->capacity : 0; }

int negf_gpu_solve_batch(negf_gpu* g, int nE, const double* energies, const double* weights,
                         const double* sigma_r, const double* sigma_lesser, int first, double* gr,
                         double* gless, negf_status* st) {
  if (!g || nE < 0 || (nE > 0 && (!energies || !weights)))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  try {
    const Plan& P = *g->plan;
    const size_t sr = P.desc.sr_rows.size(), sl = P.desc.sl_rows.size();
    const int n = P.desc.n;
    if ((sr && !sigma_r) || (sl && !sigma_lesser))
      return set_status(st, NEGF_CONTRACT_VIOLATION, "self-energy values missing");
    g->launches = 0;
    g->reduced_valid = false;
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    if (!g->copy_stream) {
      ck(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking), "stream");
      ck(cudaEventCreateWithFlags(&g->ev_sl, cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&g->ev_gr, cudaEventDisableTiming), "event");
    }
    for (int e0 = 0; e0 < nE; e0 += g->capacity) {
      const int m = std::min(g->capacity, nE - e0);
      cudaStream_t s = g->stream, cs = g->copy_stream;
      ck(cudaMemcpyAsync(g->d_energies, energies + e0, sizeof(double) * m, cudaMemcpyHostToDevice, s), "h2d");
      ck(cudaMemcpyAsync(g->d_weights, weights + e0, sizeof(double) * m, cudaMemcpyHostToDevice, s), "h2d");
      if (sr)
        ck(cudaMemcpyAsync(g->d_sigma_r, sigma_r + 2 * sr * size_t(e0), 16 * sr * m, cudaMemcpyHostToDevice, s),
           "h2d");
      // Sigma^< goes in on the copy stream while the fold and the G^r sweep
      // run; G^r comes out on it while the G^< sweep runs.
      BatchHooks hk;
      hk.lesser_in = [&] {
        if (!sl) return;
        ck(cudaMemcpyAsync(g->d_sigma_l, sigma_lesser + 2 * sl * size_t(e0), 16 * sl * m, cudaMemcpyHostToDevice,
                           cs),
           "h2d");
        ck(cudaEventRecord(g->ev_sl, cs), "event");
        ck(cudaStreamWaitEvent(s, g->ev_sl, 0), "event wait");
      };
      hk.gr_early = gr != nullptr;
      hk.gr_ready = g->ev_gr;
      run_batch(g, m, first + e0, g->d_energies, g->d_weights, g->d_sigma_r, g->d_sigma_l,
                gr ? g->d_gr : nullptr, gless ? g->d_gl : nullptr, &hk);
      if (gr) {
        ck(cudaStreamWaitEvent(cs, g->ev_gr, 0), "event wait");
        ck(cudaMemcpyAsync(gr + 2 * size_t(n) * e0, g->d_gr, 16 * size_t(n) * m, cudaMemcpyDeviceToHost, cs),
           "d2h");
      }
      if (gless)
        ck(cudaMemcpyAsync(gless + 2 * size_t(n) * e0, g->d_gl, 16 * size_t(n) * m, cudaMemcpyDeviceToHost, s),
           "d2h");
      // Stop at the first batch holding a solver failure (its energies are the
      // lowest failing ones); residual checks are deferred to the end.
      DevStatus h;
      ck(cudaMemcpyAsync(&h, g->d_status, sizeof h, cudaMemcpyDeviceToHost, s), "status");
      ck(cudaStreamSynchronize(s), "sync");
      ck(cudaStreamSynchronize(cs), "sync");
      flush_profile(g);
      if (h.singular_key != ~0ull || h.nonskew_key != ~0ull) break;
    }
    return collect(g, st);
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  }
}

int negf_gpu_solve_batch_device(negf_gpu* g, int nE, const double* d_E, const double* d_w,
                                const double* d_sr, const double* d_sl, int first, double* d_gr,
                                double* d_gless, int sync, negf_status* st) {
  if (!g || nE < 0) return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  try {
    const Plan& P = *g->plan;
    const size_t sr = P.desc.sr_rows.size(), sl = P.desc.sl_rows.size();
    const int n = P.desc.n;
    g->launches = 0;
    g->reduced_valid = false;
    ck(cudaSetDevice(g->device), "cudaSetDevice");
    for (int e0 = 0; e0 < nE; e0 += g->capacity) {
      const int m = std::min(g->capacity, nE - e0);
      run_batch(g, m, first + e0, d_E + e0, d_w + e0,
                reinterpret_cast<const double2*>(d_sr) + sr * size_t(e0),
                reinterpret_cast<const double2*>(d_sl) + sl * size_t(e0),
                d_gr ? reinterpret_cast<double2*>(d_gr) + size_t(n) * e0 : nullptr,
                d_gless ? reinterpret_cast<double2*>(d_gless) + size_t(n) * e0 : nullptr);
    }
    if (!sync) return ok(st);  // profile events are read later (profile_read): no host sync here
    flush_profile(g);
    return collect(g, st);
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  }
}

int negf_gpu_check(negf_gpu* g, negf_status* st) {
  if (!g) return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  try {
    return collect(g, st);
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  }
}

int negf_gpu_density(negf_gpu* g, double* out, int reset, negf_status* st) {
  if (!g || !out) return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  try {
    const int n = g->plan->desc.n;
    const double* src = g->reduced_valid ? g->d_reduced : g->d_density;
    ck(cudaMemcpyAsync(out, src, sizeof(double) * n, cudaMemcpyDeviceToHost, g->stream), "d2h");
    if (reset) {
      ck(cudaMemsetAsync(g->d_density, 0, sizeof(double) * n, g->stream), "memset");
      g->reduced_valid = false;
    }
    ck(cudaStreamSynchronize(g->stream), "sync");
    for (int i = 0; i < n; ++i) out[i] /= kTwoPi;  // observables.cpp:91
    return ok(st);
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  }
}

int negf_gpu_set_residual_check(negf_gpu* g, int mode) {
  if (!g) return NEGF_CONTRACT_VIOLATION;
  g->residual_mode = mode;
  return NEGF_OK;
}

double negf_gpu_max_real_residual(negf_gpu* g) { return g ? g->max_resid : 0.0; }

int negf_gpu_residual_violation(negf_gpu* g, int32_t* energy_index, int32_t* dof, int reset) {
  if (!g) return 0;
  const unsigned long long k = g->resid_first;
  if (reset) g->resid_first = ~0ull;
  if (k == ~0ull) return 0;
  if (energy_index) *energy_index = static_cast<int32_t>(k >> 32);
  if (dof) *dof = static_cast<int32_t>(k & 0xFFFFFFFFull);
  return 1;
}

int negf_gpu_profile(negf_gpu* g, int enable) {
  if (!g) return NEGF_CONTRACT_VIOLATION;
  flush_profile(g);
  g->profiling = enable != 0;
  return NEGF_OK;
}

int negf_gpu_profile_read(negf_gpu* g, negf_kernel_stat* out, int reset) {
  if (!g || !out) return NEGF_CONTRACT_VIOLATION;
  flush_profile(g);
  for (int k = 0; k < NEGF_KSTAT_COUNT; ++k) out[k] = g->stats[k];
  if (reset)
    for (auto& s : g->stats) s = negf_kernel_stat{};
  return NEGF_OK;
}

int negf_gpu_profile_ops(negf_gpu* g, double* ms_out, int reset) {
  if (!g || !ms_out) return NEGF_CONTRACT_VIOLATION;
  flush_profile(g);
  const std::size_t n = g->plan->ops.size();
  for (std::size_t i = 0; i < n; ++i) ms_out[i] = i < g->op_ms.size() ? g->op_ms[i] : 0.0;
  if (reset) g->op_ms.assign(n, 0.0);
  return NEGF_OK;
}

void* negf_gpu_stream(negf_gpu* g) { return g ? g->stream : nullptr; }
void* negf_gpu_density_device(negf_gpu* g) { return g ? g->d_density : nullptr; }
int64_t negf_gpu_last_launches(const negf_gpu* g) { return g ? g->launches : 0; }

void negf_gpu_destroy(negf_gpu* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->comm && nccl().ok) nccl().destroy(g->comm);
  if (g->stream) cudaStreamSynchronize(g->stream);
  for (cudaEvent_t e : g->ev) cudaEventDestroy(e);
  for (void* p : g->owned) cudaFree(p);
  if (g->copy_stream) {
    cudaStreamSynchronize(g->copy_stream);
    cudaStreamDestroy(g->copy_stream);
    cudaEventDestroy(g->ev_sl);
    cudaEventDestroy(g->ev_gr);
  }
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

int negf_nccl_unique_id(char id_out[128], negf_status* st) {
  NcclApi& api = nccl();
  if (!api.ok) return set_status(st, NEGF_NCCL_ERROR, "libnccl.so.2 could not be loaded");
  NcclId id;
  const int r = api.get_id(&id);
  if (r != 0) return set_status(st, NEGF_NCCL_ERROR, api.err ? api.err(r) : "ncclGetUniqueId failed");
  std::memcpy(id_out, id.internal, 128);
  return ok(st);
}

int negf_gpu_nccl_init(negf_gpu* g, const char id[128], int nranks, int rank, negf_status* st) {
  NcclApi& api = nccl();
  if (!g) return set_status(st, NEGF_CONTRACT_VIOLATION, "null argument");
  if (!api.ok) return set_status(st, NEGF_NCCL_ERROR, "libnccl.so.2 could not be loaded");
  cudaSetDevice(g->device);
  NcclId nid;
  std::memcpy(nid.internal, id, 128);
  const int r = reinterpret_cast<nccl_init_by_value_t>(api.init)(&g->comm, nranks, nid, rank);
  if (r != 0) return set_status(st, NEGF_NCCL_ERROR, api.err ? api.err(r) : "ncclCommInitRank failed");
  g->nranks = nranks;
  try {
    g->d_gather = dev_alloc<double>(size_t(nranks) * g->plan->desc.n, g->owned);
    g->d_reduced = dev_alloc<double>(size_t(g->plan->desc.n), g->owned);
  } catch (const CudaFail& f) {
    return set_status(st, f.code, f.msg);
  }
  return ok(st);
}

int negf_gpu_set_ordered_reduce(negf_gpu* g, int ordered) {
  if (!g) return NEGF_CONTRACT_VIOLATION;
  g->ordered_reduce = ordered != 0;
  return NEGF_OK;
}

int negf_gpu_allreduce_density(negf_gpu* g, negf_status* st) {
  NcclApi& api = nccl();
  if (!g || !g->comm) return set_status(st, NEGF_CONTRACT_VIOLATION, "no NCCL communicator");
  cudaSetDevice(g->device);
  const int n = g->plan->desc.n;
  if (g->ordered_reduce && api.allgather) {
    // Deterministic for any rank count and NCCL algorithm: gather the
    // partials, then sum them in rank order on the device.
    const int r = api.allgather(g->d_density, g->d_gather, size_t(n), 8, g->comm, g->stream);
    if (r != 0) return set_status(st, NEGF_NCCL_ERROR, api.err ? api.err(r) : "ncclAllGather failed");
    int64_t L = 0;
    launch_ordered_sum(g->d_gather, g->nranks, n, g->d_reduced, g->stream, L);
    if (cudaStreamSynchronize(g->stream) != cudaSuccess)
      return set_status(st, NEGF_CUDA_ERROR, "sync after allgather failed");
    g->reduced_valid = true;
    return ok(st);
  }
  // ncclFloat64 = 8, ncclSum = 0 (nccl.h)
  const int r = api.allreduce(g->d_density, g->d_reduced, size_t(n), 8, 0, g->comm, g->stream);
  if (r != 0) return set_status(st, NEGF_NCCL_ERROR, api.err ? api.err(r) : "ncclAllReduce failed");
  if (cudaStreamSynchronize(g->stream) != cudaSuccess)
    return set_status(st, NEGF_CUDA_ERROR, "sync after allreduce failed");
  g->reduced_valid = true;
  return ok(st);
}

}  // extern "C"
