// TEST INFRASTRUCTURE ONLY (oracle/): drives the UNMODIFIED reference solver
// sources under /root/reference/proj/src (compiled by oracle/Makefile into
// oracle/_ref/) so that
//   * the committed golden vectors are the reference's own outputs, and
//   * bench.py --impl reference / cpu_baseline time the reference's own CPU
//     path on the same seeded inputs the GPU path consumes.
// Nothing in the product links this file.
//
// Modes
//   ref_driver cli solve|bench|partition <config.json>
//       the reference's own commands (run.cpp:283-447) -> golden CSVs
//   ref_driver solve <problem.bin> <out.bin> [--threads T] [--solver hsc|dense|rgf|tree]
//                    [--energies i,j,...]
//       per-energy pipeline of solve_energy (run.cpp:141-192) over a binary
//       problem (format in oracle/refio.py), energy pool as solve_all
//       (run.cpp:218-264): atomic work counter, lowest failing index wins.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "negf/block.hpp"
#include "negf/config.hpp"
#include "negf/dense.hpp"
#include "negf/errors.hpp"
#include "negf/hsc.hpp"
#include "negf/observables.hpp"
#include "negf/oracle.hpp"
#include "negf/partition.hpp"
#include "negf/rgf.hpp"
#include "negf/run.hpp"
#include "negf/sparse.hpp"
#include "negf/device.hpp"
#include "negf/synthetic.hpp"

extern "C" void scipy_openblas_set_num_threads64_(int);

using namespace negf;

namespace {

struct Reader {
  std::ifstream in;
  explicit Reader(const std::string& p) : in(p, std::ios::binary) {
    if (!in) throw std::runtime_error("cannot open " + p);
  }
  template <class T> T get() {
    T v;
    in.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!in) throw std::runtime_error("truncated problem file");
    return v;
  }
  template <class T> std::vector<T> vec(std::size_t n) {
    std::vector<T> v(n);
    if (n) in.read(reinterpret_cast<char*>(v.data()), sizeof(T) * n);
    if (!in) throw std::runtime_error("truncated problem file");
    return v;
  }
  std::vector<int> ivec() { return vec<int>(static_cast<std::size_t>(get<int32_t>())); }
};

struct Problem {
  int n = 0;
  SparseCoo h;
  std::vector<std::vector<int>> layers;
  std::vector<std::array<double, 2>> coords;
  std::vector<std::vector<int>> groups;
  int max_leaf = 64;
  std::vector<int> dofs_l, dofs_r;
  bool has_ph = false, has_ph_less = false;
  std::vector<double> energies, weights;
  // per energy
  std::vector<std::vector<cplx>> sig_l, sig_r, ph, less_l, less_r, ph_less;
};

Problem read_problem(const std::string& path) {
  Reader r(path);
  char magic[8];
  r.in.read(magic, 8);
  if (std::memcmp(magic, "NEGFPRB1", 8) != 0) throw std::runtime_error("bad magic");
  Problem p;
  p.n = r.get<int32_t>();
  p.h.n = p.n;
  const int64_t nnz = r.get<int64_t>();
  auto rows = r.vec<int32_t>(static_cast<std::size_t>(nnz));
  auto cols = r.vec<int32_t>(static_cast<std::size_t>(nnz));
  auto vals = r.vec<cplx>(static_cast<std::size_t>(nnz));
  for (int64_t k = 0; k < nnz; ++k) p.h.add(rows[k], cols[k], vals[k]);
  coo_normalize(p.h);
  const int nl = r.get<int32_t>();
  for (int l = 0; l < nl; ++l) p.layers.push_back(r.ivec());
  if (r.get<int32_t>()) {
    auto c = r.vec<double>(2 * static_cast<std::size_t>(p.n));
    p.coords.resize(static_cast<std::size_t>(p.n));
    for (int d = 0; d < p.n; ++d) p.coords[d] = {c[2 * d], c[2 * d + 1]};
  }
  const int ng = r.get<int32_t>();
  for (int g = 0; g < ng; ++g) p.groups.push_back(r.ivec());
  p.max_leaf = r.get<int32_t>();
  p.dofs_l = r.ivec();
  p.dofs_r = r.ivec();
  p.has_ph = r.get<int32_t>() != 0;
  p.has_ph_less = r.get<int32_t>() != 0;
  const int ne = r.get<int32_t>();
  p.energies = r.vec<double>(static_cast<std::size_t>(ne));
  p.weights = r.vec<double>(static_cast<std::size_t>(ne));
  const std::size_t wl2 = p.dofs_l.size() * p.dofs_l.size();
  const std::size_t wr2 = p.dofs_r.size() * p.dofs_r.size();
  for (int e = 0; e < ne; ++e) {
    p.sig_l.push_back(r.vec<cplx>(wl2));
    p.sig_r.push_back(r.vec<cplx>(wr2));
    p.ph.push_back(p.has_ph ? r.vec<cplx>(static_cast<std::size_t>(p.n))
                            : std::vector<cplx>(static_cast<std::size_t>(p.n)));
    p.less_l.push_back(r.vec<cplx>(wl2));
    p.less_r.push_back(r.vec<cplx>(wr2));
    p.ph_less.push_back(p.has_ph_less ? r.vec<cplx>(static_cast<std::size_t>(p.n))
                                      : std::vector<cplx>());
  }
  return p;
}

ContactBlock contact(const std::vector<int>& dofs, const std::vector<cplx>& v) {
  ContactBlock c;
  c.dofs = dofs;
  const int w = static_cast<int>(dofs.size());
  c.sigma = CMatrix(w, w);
  for (int i = 0; i < w; ++i)
    for (int j = 0; j < w; ++j) c.sigma(i, j) = v[static_cast<std::size_t>(i) * w + j];
  return c;
}

// Sigma^< as the reference's producers emit it (device.cpp:322-360,
// synthetic.cpp:124-144): nonzero entries only, canonical order.
SparseCoo lesser_coo(const Problem& p, int e) {
  SparseCoo s;
  s.n = p.n;
  auto add_block = [&](const std::vector<int>& dofs, const std::vector<cplx>& v) {
    const std::size_t w = dofs.size();
    for (std::size_t i = 0; i < w; ++i)
      for (std::size_t j = 0; j < w; ++j)
        if (v[i * w + j] != cplx(0.0, 0.0)) s.add(dofs[i], dofs[j], v[i * w + j]);
  };
  add_block(p.dofs_l, p.less_l[e]);
  add_block(p.dofs_r, p.less_r[e]);
  if (p.has_ph_less)
    for (int d = 0; d < p.n; ++d)
      if (p.ph_less[e][d] != cplx(0.0, 0.0)) s.add(d, d, p.ph_less[e][d]);
  coo_normalize(s);
  return s;
}

SparseCoo system_at(const Problem& p, int e) {
  const std::vector<cplx> none;
  return assemble_system(p.h, contact(p.dofs_l, p.sig_l[e]), contact(p.dofs_r, p.sig_r[e]),
                         p.has_ph ? p.ph[e] : none, p.energies[e], p.layers);
}

struct EnergyOut {
  std::vector<cplx> gr, gless;
  FlopLedger ledger;
};

EnergyOut solve_one(const Problem& p, const std::shared_ptr<const SeparatorTree>& tree,
                    const std::string& solver, int e) {
  const SparseCoo a = system_at(p, e);
  const SparseCoo sl = lesser_coo(p, e);
  EnergyOut out;
  GreensDiagonal d;
  d.n_dofs = p.n;
  if (solver == "hsc") {
    ClusterBlockMatrix am = group_by_partition(a, tree);
    HscFactorization fact = hsc_fold(std::move(am), out.ledger);
    ClusterBlockMatrix sig = group_by_partition(sl, tree, BlockSymmetry::SkewHermitian);
    HscGlessResult res = hsc_gless(fact, sig, out.ledger);
    for (int c = 0; c < tree->num_clusters(); ++c) d.dof_sets.push_back(tree->cluster(c).dofs);
    d.gr_diag = std::move(res.gr_diag);
    d.gless_diag = std::move(res.gless_diag);
  } else if (solver == "rgf") {
    LayeredSystem sys = layered_from_coo(a, p.layers);
    attach_sigma_lesser(sys, sl);
    RgfGrResult r = rgf_gr(sys, RgfGrOptions{}, out.ledger);
    std::vector<CMatrix> gl = rgf_gless(sys, r, out.ledger);
    d.dof_sets = p.layers;
    d.gr_diag = std::move(r.gr_diag);
    d.gless_diag = std::move(gl);
  } else {
    const CMatrix gr = dense_gr(a);
    const CMatrix gl = dense_gless(gr, dense_from_coo(sl));
    out.gr.resize(static_cast<std::size_t>(p.n));
    out.gless.resize(static_cast<std::size_t>(p.n));
    for (int j = 0; j < p.n; ++j) {
      out.gr[j] = gr(j, j);
      out.gless[j] = gl(j, j);
    }
    return out;
  }
  out.gr = d.gr_dof_diagonal();
  out.gless = d.gless_dof_diagonal();
  return out;
}

int error_code(std::exception_ptr ep, std::string& msg) {
  try {
    std::rethrow_exception(ep);
  } catch (const SingularBlock& e) {
    msg = e.what();
    return 1;
  } catch (const NonSkewHermitianInput& e) {
    msg = e.what();
    return 2;
  } catch (const ContractViolation& e) {
    msg = e.what();
    return 3;
  } catch (const ConfigError& e) {
    msg = e.what();
    return 7;
  } catch (const PartitionViolation& e) {
    msg = e.what();
    return 8;
  } catch (const ResidualTooLarge& e) {
    msg = e.what();
    return 9;
  } catch (const std::exception& e) {
    msg = e.what();
    return 10;
  }
}

template <class T> void put(std::ofstream& o, const T& v) {
  o.write(reinterpret_cast<const char*>(&v), sizeof(T));
}

int cmd_problem(int argc, char** argv) {
  const std::string in = argv[2], outp = argv[3];
  int threads = 1;
  std::string solver = "hsc";
  std::vector<int> subset;
  for (int i = 4; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    if (k == "--threads") threads = std::stoi(argv[i + 1]);
    else if (k == "--solver") solver = argv[i + 1];
    else if (k == "--energies") {
      std::stringstream ss(argv[i + 1]);
      std::string tok;
      while (std::getline(ss, tok, ',')) subset.push_back(std::stoi(tok));
    }
  }
  scipy_openblas_set_num_threads64_(1);
  const Problem p = read_problem(in);
  if (subset.empty())
    for (int e = 0; e < static_cast<int>(p.energies.size()); ++e) subset.push_back(e);
  // --solver tree: build_tree only (the separator tree of the HSC path, no
  // energy solved)
  const bool tree_only = solver == "tree";
  const int m = tree_only ? 0 : static_cast<int>(subset.size());

  int status = 0, err_energy = -1;
  std::string msg;
  std::shared_ptr<const SeparatorTree> tree;
  std::vector<EnergyOut> res(static_cast<std::size_t>(m));
  double wall = 0.0, tree_wall = 0.0;
  try {
    const auto t0 = std::chrono::steady_clock::now();
    if (solver == "hsc" || tree_only) {
      // build_tree (run.cpp:123-133): graph of A(E0), contact atomic groups.
      const Graph g = graph_of_pattern(system_at(p, subset.front()));
      tree = std::make_shared<SeparatorTree>(nested_dissection(g, p.groups, p.max_leaf, p.coords));
    }
    const auto t1 = std::chrono::steady_clock::now();
    tree_wall = std::chrono::duration<double>(t1 - t0).count();
    std::vector<std::exception_ptr> errs(static_cast<std::size_t>(m));
    std::atomic<int> next{0};
    auto work = [&] {
      for (;;) {
        const int k = next.fetch_add(1);
        if (k >= m) return;
        try {
          res[k] = solve_one(p, tree, solver, subset[k]);
        } catch (...) {
          errs[k] = std::current_exception();
        }
      }
    };
    std::vector<std::thread> pool;
    const int nt = m == 0 ? 0 : std::max(1, std::min(threads, m));
    for (int t = 0; t < nt; ++t) pool.emplace_back(work);
    for (auto& th : pool) th.join();
    wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    for (int k = 0; k < m; ++k)
      if (errs[k]) {
        status = error_code(errs[k], msg);
        err_energy = subset[k];
        break;
      }
  } catch (...) {
    status = error_code(std::current_exception(), msg);
  }

  std::ofstream o(outp, std::ios::binary);
  o.write("NEGFOUT1", 8);
  put<int32_t>(o, status);
  put<int32_t>(o, err_energy);
  char buf[512] = {0};
  std::strncpy(buf, msg.c_str(), sizeof buf - 1);
  o.write(buf, sizeof buf);
  put<int32_t>(o, tree ? tree->num_clusters() : 0);
  if (tree)
    for (int c = 0; c < tree->num_clusters(); ++c) {
      const auto& cl = tree->cluster(c);
      put<int32_t>(o, cl.parent);
      put<int32_t>(o, cl.level);
      put<int32_t>(o, static_cast<int32_t>(cl.dofs.size()));
      o.write(reinterpret_cast<const char*>(cl.dofs.data()), 4 * cl.dofs.size());
    }
  FlopLedger tot;
  for (const auto& r : res) tot.merge(r.ledger);
  put<int64_t>(o, tot.multiply_ops);
  put<int64_t>(o, tot.inverse_ops);
  put<double>(o, wall);
  put<double>(o, tree_wall);
  put<int32_t>(o, threads);
  put<int32_t>(o, status == 0 ? m : 0);
  if (status == 0) {
    for (int k = 0; k < m; ++k) put<int32_t>(o, subset[k]);
    for (int k = 0; k < m; ++k) o.write(reinterpret_cast<const char*>(res[k].gr.data()), 16 * p.n);
    for (int k = 0; k < m; ++k) o.write(reinterpret_cast<const char*>(res[k].gless.data()), 16 * p.n);
  }
  return 0;
}

// ---- problem dumps from the reference's own input builders ---------------

void put_ivec(std::ofstream& o, const std::vector<int>& v) {
  put<int32_t>(o, static_cast<int32_t>(v.size()));
  o.write(reinterpret_cast<const char*>(v.data()), 4 * v.size());
}

void put_cvec(std::ofstream& o, const std::vector<cplx>& v) {
  o.write(reinterpret_cast<const char*>(v.data()), 16 * v.size());
}

std::vector<cplx> flat(const CMatrix& m) {
  return std::vector<cplx>(m.data(), m.data() + static_cast<std::size_t>(m.rows()) * m.cols());
}

struct Dump {
  SparseCoo h;
  std::vector<std::vector<int>> layers;
  std::vector<std::array<double, 2>> coords;
  std::vector<std::vector<int>> groups;
  int max_leaf = 64;
  std::vector<int> dl, dr;
  bool has_ph = false, has_ph_less = false;
  std::vector<double> energies, weights;
  std::vector<std::vector<cplx>> sl, sr, ph, ll, lr, phl;
};

void write_dump(const Dump& d, const std::string& path) {
  std::ofstream o(path, std::ios::binary);
  o.write("NEGFPRB1", 8);
  put<int32_t>(o, d.h.n);
  put<int64_t>(o, static_cast<int64_t>(d.h.entries.size()));
  for (const auto& e : d.h.entries) put<int32_t>(o, e.row);
  for (const auto& e : d.h.entries) put<int32_t>(o, e.col);
  for (const auto& e : d.h.entries) put<cplx>(o, e.val);
  put<int32_t>(o, static_cast<int32_t>(d.layers.size()));
  for (const auto& l : d.layers) put_ivec(o, l);
  put<int32_t>(o, d.coords.empty() ? 0 : 1);
  for (const auto& c : d.coords) {
    put<double>(o, c[0]);
    put<double>(o, c[1]);
  }
  put<int32_t>(o, static_cast<int32_t>(d.groups.size()));
  for (const auto& g : d.groups) put_ivec(o, g);
  put<int32_t>(o, d.max_leaf);
  put_ivec(o, d.dl);
  put_ivec(o, d.dr);
  put<int32_t>(o, d.has_ph ? 1 : 0);
  put<int32_t>(o, d.has_ph_less ? 1 : 0);
  put<int32_t>(o, static_cast<int32_t>(d.energies.size()));
  for (double e : d.energies) put<double>(o, e);
  for (double w : d.weights) put<double>(o, w);
  for (std::size_t e = 0; e < d.energies.size(); ++e) {
    put_cvec(o, d.sl[e]);
    put_cvec(o, d.sr[e]);
    if (d.has_ph) put_cvec(o, d.ph[e]);
    put_cvec(o, d.ll[e]);
    put_cvec(o, d.lr[e]);
    if (d.has_ph_less) put_cvec(o, d.phl[e]);
  }
}

// Splits a block-diagonal COO lesser self-energy back into the two contact
// blocks and the diagonal remainder.
void split_lesser(const SparseCoo& s, const std::vector<int>& dl, const std::vector<int>& dr, int n,
                  std::vector<cplx>& ll, std::vector<cplx>& lr, std::vector<cplx>& diag) {
  std::vector<int> li(static_cast<std::size_t>(n), -1), ri(static_cast<std::size_t>(n), -1);
  for (std::size_t k = 0; k < dl.size(); ++k) li[dl[k]] = static_cast<int>(k);
  for (std::size_t k = 0; k < dr.size(); ++k) ri[dr[k]] = static_cast<int>(k);
  ll.assign(dl.size() * dl.size(), cplx(0.0, 0.0));
  lr.assign(dr.size() * dr.size(), cplx(0.0, 0.0));
  diag.assign(static_cast<std::size_t>(n), cplx(0.0, 0.0));
  for (const auto& e : s.entries) {
    if (li[e.row] >= 0 && li[e.col] >= 0) ll[li[e.row] * dl.size() + li[e.col]] += e.val;
    else if (ri[e.row] >= 0 && ri[e.col] >= 0) lr[ri[e.row] * dr.size() + ri[e.col]] += e.val;
    else if (e.row == e.col) diag[e.row] += e.val;
    else throw std::runtime_error("lesser entry outside the contact blocks and the diagonal");
  }
}

// ref_driver synthetic nx ny seed fuzz coupling max_leaf out.bin E...
int cmd_synthetic(int argc, char** argv) {
  SyntheticSpec spec;
  spec.nx = std::stoi(argv[2]);
  spec.ny = std::stoi(argv[3]);
  spec.seed = std::stoull(argv[4]);
  spec.fuzz = std::stoi(argv[5]) != 0;
  spec.coupling_t = std::stod(argv[6]);
  const SyntheticSystem sys = make_synthetic_system(spec);
  Dump d;
  d.h = sys.h;
  d.layers = sys.layers;
  d.coords = sys.coords;
  d.groups = {sys.layers.front()};
  if (sys.layers.size() > 1) d.groups.push_back(sys.layers.back());
  d.max_leaf = std::stoi(argv[7]);
  d.dl = sys.sigma_r_left.dofs;
  d.dr = sys.sigma_r_right.dofs;
  d.has_ph = false;
  d.has_ph_less = spec.fuzz;
  for (int i = 9; i < argc; ++i) d.energies.push_back(std::stod(argv[i]));
  d.weights = make_energy_grid(d.energies).weights;
  for (std::size_t e = 0; e < d.energies.size(); ++e) {
    d.sl.push_back(flat(sys.sigma_r_left.sigma));
    d.sr.push_back(sys.sigma_r_right.empty() ? std::vector<cplx>() : flat(sys.sigma_r_right.sigma));
    d.ph.push_back({});
    std::vector<cplx> ll, lr, dg;
    split_lesser(sys.sigma_lesser, d.dl, d.dr, sys.h.n, ll, lr, dg);
    d.ll.push_back(ll);
    d.lr.push_back(lr);
    d.phl.push_back(dg);
  }
  write_dump(d, argv[8]);
  return 0;
}

// ref_driver device config.json max_leaf_override out.bin : the physical
// devices of run.cpp build_problem / sigma_for_energy (run.cpp:45-109).
int cmd_device(int argc, char** argv) {
  (void)argc;
  const RunConfig cfg = load_run_config(argv[2]);
  DeviceSystem dev;
  double mu = 0.0, temp = 300.0;
  if (cfg.device_kind == DeviceKind::Superlattice) {
    dev = build_superlattice_hamiltonian(cfg.superlattice);
    mu = cfg.superlattice.fermi_energy_ev;
    temp = cfg.superlattice.temperature_k;
  } else if (cfg.device_kind == DeviceKind::Graphene) {
    dev = build_graphene_hamiltonian(cfg.graphene);
    mu = cfg.graphene.fermi_energy_ev;
  } else {
    throw std::runtime_error("device dump supports superlattice and graphene");
  }
  Dump d;
  d.h = dev.h;
  d.layers = dev.layers;
  d.coords = dev.coords;
  if (cfg.contact.model == ContactModel::DenseLead) {
    d.groups = {dev.layers.front()};
    if (dev.layers.size() > 1) d.groups.push_back(dev.layers.back());
  }
  d.max_leaf = cfg.max_leaf;
  d.dl = dev.layers.front();
  d.dr = dev.layers.back();
  d.has_ph = true;
  d.has_ph_less = true;
  d.energies = cfg.energy.energies_ev;
  d.weights = cfg.energy.weights;
  for (double E : d.energies) {
    SelfEnergySet s;
    attach_contacts(dev, cfg.contact.model, E, cfg.contact.eta_ev, s);
    s.sigma_r_phonon = phonon_self_energy(dev, cfg.contact.eta_phonon_ev);
    s.sigma_lesser = lesser_self_energy(s.sigma_r_left, s.sigma_r_right, s.sigma_r_phonon, dev.h.n, E, mu,
                                        mu, temp);
    d.sl.push_back(flat(s.sigma_r_left.sigma));
    d.sr.push_back(flat(s.sigma_r_right.sigma));
    d.ph.push_back(s.sigma_r_phonon);
    std::vector<cplx> ll, lr, dg;
    split_lesser(s.sigma_lesser, d.dl, d.dr, dev.h.n, ll, lr, dg);
    d.ll.push_back(ll);
    d.lr.push_back(lr);
    d.phl.push_back(dg);
  }
  write_dump(d, argv[3]);
  return 0;
}

// ref_driver lead in.bin out.bin : surface_self_energy (device.cpp:195-251)
// of one dense lead at nE energies.  in: "NEGFLED1", int32 w, int32 nE,
// f64 eta, h00[w*w], h01[w*w] (complex, row-major), f64 energies[nE].
// out: "NEGFLEO1", int32 nE, then per energy int32 code (0 ok, 1
// ConvergenceError, 2 SingularBlock, 3 other) and w*w complex (zeros on error).
int cmd_lead(char** argv) {
  std::ifstream in(argv[2], std::ios::binary);
  char magic[8];
  in.read(magic, 8);
  if (std::memcmp(magic, "NEGFLED1", 8) != 0) throw std::runtime_error("bad lead input");
  int32_t w = 0, ne = 0;
  double eta = 0.0;
  in.read(reinterpret_cast<char*>(&w), 4);
  in.read(reinterpret_cast<char*>(&ne), 4);
  in.read(reinterpret_cast<char*>(&eta), 8);
  CMatrix h00(w, w), h01(w, w);
  in.read(reinterpret_cast<char*>(h00.data()), sizeof(cplx) * w * w);
  in.read(reinterpret_cast<char*>(h01.data()), sizeof(cplx) * w * w);
  std::vector<double> es(static_cast<std::size_t>(ne));
  in.read(reinterpret_cast<char*>(es.data()), 8 * ne);
  if (!in) throw std::runtime_error("short lead input");
  std::ofstream out(argv[3], std::ios::binary);
  out.write("NEGFLEO1", 8);
  out.write(reinterpret_cast<const char*>(&ne), 4);
  for (double e : es) {
    int32_t code = 0;
    CMatrix s(w, w);
    try {
      s = surface_self_energy(h00, h01, e, eta);
    } catch (const ConvergenceError&) {
      code = 1;
    } catch (const SingularBlock&) {
      code = 2;
    } catch (const Error&) {
      code = 3;
    }
    out.write(reinterpret_cast<const char*>(&code), 4);
    out.write(reinterpret_cast<const char*>(s.data()), sizeof(cplx) * w * w);
  }
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc >= 10 && std::string(argv[1]) == "synthetic") return cmd_synthetic(argc, argv);
  if (argc >= 4 && std::string(argv[1]) == "device") return cmd_device(argc, argv);
  if (argc >= 4 && std::string(argv[1]) == "lead") return cmd_lead(argv);
  if (argc >= 4 && std::string(argv[1]) == "cli") {
    scipy_openblas_set_num_threads64_(1);
    try {
      const RunConfig cfg = load_run_config(argv[3]);
      const std::string c = argv[2];
      if (c == "solve") cmd_solve(cfg);
      else if (c == "bench") cmd_bench(cfg);
      else cmd_partition(cfg);
    } catch (const ConfigError& e) {
      std::fprintf(stderr, "config error: %s\n", e.what());
      return 2;
    } catch (const PartitionViolation& e) {
      std::fprintf(stderr, "partition error: %s\n", e.what());
      return 2;
    } catch (const Error& e) {
      std::fprintf(stderr, "error: %s\n", e.what());
      return 3;
    }
    return 0;
  }
  if (argc >= 4 && std::string(argv[1]) == "solve") return cmd_problem(argc, argv);
  std::fprintf(stderr, "usage: ref_driver cli solve|bench|partition cfg.json | solve in out [opts]\n");
  return 1;
}
