// negf_solve -- a C++ host program on the C ABI alone (include/negf_gpu.h):
// what the reference's solve_all / cmd_solve (proj/src/run.cpp:218-326)
// becomes when its HSC energy loop is routed to the B200 library.  No CUDA
// headers or torch types: plain pointers and sizes, as a maintainer would
// bind it from run.cpp.
//
//   negf_solve problem.bin out_dir [--nx NX --ny NY] [--device D] [--batch B]
//
// problem.bin is the reference's own problem dump (NEGFPRB1, written by
// oracle/ref_driver: H, layers, coords, atomic contact groups, per-energy
// contact Sigma^r / Sigma^< blocks and phonon diagonals).  Outputs:
// out_dir/diag.bin (per-energy diag G^r, diag G^<, negf_shard_writer format),
// out_dir/density.csv, ldos.csv, line_density.csv when --nx/--ny are given
// (cmd_solve's artefacts), else out_dir/density.bin.  Exit codes follow the
// reference CLI (negf_main.cpp:65-77): 2 for ConfigError/PartitionViolation,
// 3 for every other solver error.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "negf_gpu.h"

namespace {

struct Reader {
  std::vector<char> buf;
  size_t pos = 0;
  template <class T>
  T get() {
    T v;
    std::memcpy(&v, buf.data() + pos, sizeof(T));
    pos += sizeof(T);
    return v;
  }
  template <class T>
  std::vector<T> arr(size_t n) {
    std::vector<T> v(n);
    std::memcpy(v.data(), buf.data() + pos, sizeof(T) * n);
    pos += sizeof(T) * n;
    return v;
  }
};

struct Problem {
  int n = 0, max_leaf = 64, has_ph = 0, has_ph_less = 0;
  std::vector<int32_t> h_rows, h_cols;
  std::vector<double> h_vals;  // complex interleaved
  std::vector<std::vector<int32_t>> layers, groups;
  std::vector<double> coords;  // 2n or empty
  std::vector<int32_t> dl, dr;
  std::vector<double> energies, weights;
  // per energy, complex interleaved
  std::vector<std::vector<double>> sig_l, sig_r, ph, less_l, less_r, ph_less;
};

Problem read_problem(const char* path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error(std::string("cannot open ") + path);
  Reader r;
  r.buf.assign(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
  if (r.buf.size() < 8 || std::memcmp(r.buf.data(), "NEGFPRB1", 8) != 0)
    throw std::runtime_error("not a NEGFPRB1 problem file");
  r.pos = 8;
  Problem p;
  p.n = r.get<int32_t>();
  const int64_t nnz = r.get<int64_t>();
  p.h_rows = r.arr<int32_t>(nnz);
  p.h_cols = r.arr<int32_t>(nnz);
  p.h_vals = r.arr<double>(2 * nnz);
  const int nl = r.get<int32_t>();
  for (int l = 0; l < nl; ++l) p.layers.push_back(r.arr<int32_t>(r.get<int32_t>()));
  if (r.get<int32_t>()) p.coords = r.arr<double>(2 * size_t(p.n));
  const int ng = r.get<int32_t>();
  for (int g = 0; g < ng; ++g) p.groups.push_back(r.arr<int32_t>(r.get<int32_t>()));
  p.max_leaf = r.get<int32_t>();
  p.dl = r.arr<int32_t>(r.get<int32_t>());
  p.dr = r.arr<int32_t>(r.get<int32_t>());
  p.has_ph = r.get<int32_t>();
  p.has_ph_less = r.get<int32_t>();
  const int ne = r.get<int32_t>();
  p.energies = r.arr<double>(ne);
  p.weights = r.arr<double>(ne);
  const size_t wl = p.dl.size(), wr = p.dr.size();
  for (int e = 0; e < ne; ++e) {
    p.sig_l.push_back(r.arr<double>(2 * wl * wl));
    p.sig_r.push_back(r.arr<double>(2 * wr * wr));
    if (p.has_ph) p.ph.push_back(r.arr<double>(2 * size_t(p.n)));
    p.less_l.push_back(r.arr<double>(2 * wl * wl));
    p.less_r.push_back(r.arr<double>(2 * wr * wr));
    if (p.has_ph_less) p.ph_less.push_back(r.arr<double>(2 * size_t(p.n)));
  }
  return p;
}

// Sigma pattern: the entries of the two contact blocks and of the phonon
// diagonal that are nonzero at some energy (the reference's producers drop
// exact zeros, device.cpp:344-356), each with its source position.
struct Pattern {
  std::vector<int32_t> rows, cols;
  std::vector<std::pair<int, size_t>> src;  // (0 left | 1 right | 2 diag, element index)
};

Pattern pattern(const Problem& p, bool lesser) {
  Pattern pt;
  const auto& L = lesser ? p.less_l : p.sig_l;
  const auto& R = lesser ? p.less_r : p.sig_r;
  const auto& D = lesser ? p.ph_less : p.ph;
  auto nz = [](const std::vector<std::vector<double>>& blocks, size_t i) {
    for (const auto& b : blocks)
      if (b[2 * i] != 0.0 || b[2 * i + 1] != 0.0) return true;
    return false;
  };
  int tag = 0;
  for (const auto* dofs : {&p.dl, &p.dr}) {
    const auto& blocks = tag == 0 ? L : R;
    const size_t w = dofs->size();
    for (size_t a = 0; a < w; ++a)
      for (size_t b = 0; b < w; ++b)
        if (nz(blocks, a * w + b)) {
          pt.rows.push_back((*dofs)[a]);
          pt.cols.push_back((*dofs)[b]);
          pt.src.push_back({tag, a * w + b});
        }
    ++tag;
  }
  if (!D.empty())
    for (int x = 0; x < p.n; ++x)
      if (nz(D, size_t(x))) {
        pt.rows.push_back(x);
        pt.cols.push_back(x);
        pt.src.push_back({2, size_t(x)});
      }
  return pt;
}

void values(const Problem& p, const Pattern& pt, bool lesser, int e, double* out) {
  const auto& L = lesser ? p.less_l : p.sig_l;
  const auto& R = lesser ? p.less_r : p.sig_r;
  const auto& D = lesser ? p.ph_less : p.ph;
  for (size_t q = 0; q < pt.src.size(); ++q) {
    const auto& s = pt.src[q];
    const std::vector<double>& b = s.first == 0 ? L[e] : s.first == 1 ? R[e] : D[e];
    out[2 * q] = b[2 * s.second];
    out[2 * q + 1] = b[2 * s.second + 1];
  }
}

int exit_code(const negf_status& st) {
  std::fprintf(stderr, "error: %s\n", st.msg);
  return (st.code == NEGF_CONFIG_ERROR || st.code == NEGF_PARTITION_VIOLATION) ? 2 : 3;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: negf_solve problem.bin out_dir [--nx NX --ny NY] [--device D] [--batch B]\n");
    return 1;
  }
  int nx = 0, ny = 0, device = 0, batch = 0;
  for (int i = 3; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    if (k == "--nx") nx = std::atoi(argv[i + 1]);
    else if (k == "--ny") ny = std::atoi(argv[i + 1]);
    else if (k == "--device") device = std::atoi(argv[i + 1]);
    else if (k == "--batch") batch = std::atoi(argv[i + 1]);
  }
  Problem p;
  try {
    p = read_problem(argv[1]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  }
  const int n = p.n, ne = static_cast<int>(p.energies.size());

  const Pattern spr = pattern(p, false), spl = pattern(p, true);
  std::vector<int32_t> gptr{0}, gdofs;
  for (const auto& g : p.groups) {
    gdofs.insert(gdofs.end(), g.begin(), g.end());
    gptr.push_back(static_cast<int32_t>(gdofs.size()));
  }
  negf_problem d{};
  d.n_dofs = n;
  d.h_nnz = static_cast<int64_t>(p.h_rows.size());
  d.h_rows = p.h_rows.data();
  d.h_cols = p.h_cols.data();
  d.h_vals = p.h_vals.data();
  d.sr_nnz = static_cast<int64_t>(spr.rows.size());
  d.sr_rows = spr.rows.data();
  d.sr_cols = spr.cols.data();
  d.sl_nnz = static_cast<int64_t>(spl.rows.size());
  d.sl_rows = spl.rows.data();
  d.sl_cols = spl.cols.data();
  d.coords = p.coords.empty() ? nullptr : p.coords.data();
  d.n_groups = static_cast<int>(p.groups.size());
  d.group_ptr = gptr.data();
  d.group_dofs = gdofs.data();
  d.max_leaf = p.max_leaf;

  // Per-energy pattern values, in the order of the patterns above.
  const size_t srn = spr.rows.size(), sln = spl.rows.size();
  std::vector<double> sr(2 * srn * ne), sl(2 * sln * ne);
  for (int e = 0; e < ne; ++e) {
    values(p, spr, false, e, sr.data() + 2 * srn * e);
    values(p, spl, true, e, sl.data() + 2 * sln * e);
  }

  negf_status st{};
  negf_plan* plan = nullptr;
  if (negf_plan_create(&d, &plan, &st) != NEGF_OK) return exit_code(st);
  negf_gpu* g = nullptr;
  if (negf_gpu_create(plan, device, batch, &g, &st) != NEGF_OK) return exit_code(st);
  std::vector<double> gr(2 * size_t(n) * ne), gl(2 * size_t(n) * ne), dens(n);
  const int rc = negf_gpu_solve_batch(g, ne, p.energies.data(), p.weights.data(), sr.data(), sl.data(), 0,
                                      gr.data(), gl.data(), &st);
  if (rc != NEGF_OK) return exit_code(st);
  if (negf_gpu_density(g, dens.data(), 0, &st) != NEGF_OK) return exit_code(st);

  const std::string out = argv[2];
  std::string cmd = "mkdir -p '" + out + "'";
  if (std::system(cmd.c_str()) != 0) {
    std::fprintf(stderr, "config error: cannot create %s\n", out.c_str());
    return 2;
  }
  negf_shard_writer* w = nullptr;
  if (negf_shard_writer_open((out + "/diag.bin").c_str(), n, 0, 1, 3, &w, &st) != NEGF_OK) return exit_code(st);
  negf_shard_writer_append(w, ne, 0, p.energies.data(), gr.data(), gl.data(), &st);
  if (negf_shard_writer_close(w, &st) != NEGF_OK) return exit_code(st);
  if (nx > 0 && ny > 0 && nx * ny == n) {
    if (negf_write_solve_csv(out.c_str(), nx, ny, ne, p.energies.data(), dens.data(), gr.data(), &st) != NEGF_OK)
      return exit_code(st);
  } else {
    std::ofstream f(out + "/density.bin", std::ios::binary);
    f.write(reinterpret_cast<const char*>(dens.data()), sizeof(double) * n);
  }
  negf_plan_info info{};
  negf_plan_info_get(plan, &info);
  std::printf("solved %d energy points, %d dofs, %d clusters, %lld launches\n", ne, n, info.n_clusters,
              static_cast<long long>(negf_gpu_last_launches(g)));
  negf_gpu_destroy(g);
  negf_plan_destroy(plan);
  return 0;
}
