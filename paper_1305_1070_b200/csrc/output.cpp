// Output path, C ABI in include/negf_gpu.h:
//   * negf_format_double / negf_write_solve_csv: cmd_solve's CSV artefacts
//     (density.csv, ldos.csv, line_density.csv; proj/src/run.cpp:276-326)
//     with the reference's 17-significant-digit format_double;
//   * negf_shard_writer_*: a binary per-shard writer for the per-energy
//     diag G^r / G^< (the reference writes ldos.csv per energy x dof, 537 M
//     lines for config 5).  Records are written by a background thread;
//     device-resident diagonals are staged through pinned buffers with one
//     D2H copy + event per append, so file I/O overlaps the next batch.
#include <cuda_runtime.h>

#include <charconv>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <deque>
#include <filesystem>
#include <fstream>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_util.hpp"

using namespace negfb;

namespace {

constexpr double kPi = 3.14159265358979323846;

std::string fmt(double v) {
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::general, 17);
  return std::string(buf, res.ptr);
}

}  // namespace

struct negf_shard_writer {
  std::FILE* f = nullptr;
  int n = 0, what = 0;
  int64_t records = 0;
  int64_t record_bytes = 0;
  // background writer
  struct Job {
    std::vector<char> host;      // host-owned record bytes (host appends)
    char* pinned = nullptr;      // staged device copy (device appends)
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;
    int slot = -1;
  };
  std::mutex mu;
  std::condition_variable cv;
  std::deque<Job> q;
  bool stop = false;
  int error = 0;
  std::string error_msg;
  std::thread th;
  // pinned staging slots for device appends
  static constexpr int kSlots = 2;
  char* slot_buf[kSlots] = {nullptr, nullptr};
  size_t slot_cap[kSlots] = {0, 0};
  bool slot_busy[kSlots] = {false, false};
  cudaEvent_t slot_ev[kSlots] = {nullptr, nullptr};
  int next_slot = 0;

  void run() {
    for (;;) {
      Job j;
      {
        std::unique_lock<std::mutex> lk(mu);
        cv.wait(lk, [&] { return stop || !q.empty(); });
        if (q.empty()) return;
        j = std::move(q.front());
        q.pop_front();
      }
      const char* p = j.pinned ? j.pinned : j.host.data();
      if (j.ready) cudaEventSynchronize(j.ready);
      const size_t wrote = error ? 0 : std::fwrite(p, 1, j.bytes, f);
      std::lock_guard<std::mutex> lk(mu);
      if (!error && wrote != j.bytes) {
        error = NEGF_CONFIG_ERROR;
        error_msg = "shard writer: short write";
      }
      if (j.slot >= 0) slot_busy[j.slot] = false;
      cv.notify_all();
    }
  }
};

namespace {

void write_header(negf_shard_writer* w, int rank, int world) {
  char h[64] = {};
  std::memcpy(h, "NEGFSHD1", 8);
  const int32_t v[6] = {1, w->n, rank, world, w->what, 0};
  std::memcpy(h + 8, v, sizeof v);
  std::memcpy(h + 32, &w->records, 8);
  std::fwrite(h, 1, sizeof h, w->f);
}

// Record layout: int32 energy_index, int32 0, f64 energy, [n c128 gr], [n c128 gless].
void pack(char* dst, int energy_index, double energy) {
  const int32_t hdr[2] = {energy_index, 0};
  std::memcpy(dst, hdr, 8);
  std::memcpy(dst + 8, &energy, 8);
}

}  // namespace

extern "C" {

int negf_format_double(double v, char* buf, int len) {
  const std::string s = fmt(v);
  if (!buf || len <= static_cast<int>(s.size())) return -1;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return static_cast<int>(s.size());
}

int negf_write_solve_csv(const char* out_dir, int nx, int ny, int n_energies, const double* energies,
                         const double* density, const double* gr_diag, negf_status* st) {
  namespace fs = std::filesystem;
  if (!out_dir || nx < 1 || ny < 1 || (n_energies > 0 && !energies) || !density)
    return set_status(st, NEGF_CONTRACT_VIOLATION, "write_solve_csv: bad argument");
  try {
    fs::create_directories(out_dir);
  } catch (const std::exception& e) {
    return set_status(st, NEGF_CONFIG_ERROR, std::string("cannot create output directory: ") + e.what());
  }
  auto open = [&](const char* name, std::ofstream& out) {
    const fs::path path = fs::path(out_dir) / name;
    out.open(path, std::ios::binary);
    return static_cast<bool>(out);
  };
  const size_t n = static_cast<size_t>(nx) * ny;
  {
    std::ofstream out;
    if (!open("density.csv", out)) return set_status(st, NEGF_CONFIG_ERROR, "cannot open output file 'density.csv'");
    out << "x_index,y_index,density\n";
    for (int y = 0; y < ny; ++y)
      for (int x = 0; x < nx; ++x) out << x << ',' << y << ',' << fmt(density[static_cast<size_t>(y) * nx + x]) << '\n';
  }
  if (gr_diag) {
    std::ofstream out;
    if (!open("ldos.csv", out)) return set_status(st, NEGF_CONFIG_ERROR, "cannot open output file 'ldos.csv'");
    out << "x_index,y_index,energy_eV,ldos\n";
    for (int k = 0; k < n_energies; ++k) {
      const std::string e = fmt(energies[k]);
      const double* g = gr_diag + 2 * static_cast<size_t>(k) * n;
      for (int y = 0; y < ny; ++y)
        for (int x = 0; x < nx; ++x) {
          const size_t j = static_cast<size_t>(y) * nx + x;
          out << x << ',' << y << ',' << e << ',' << fmt(-g[2 * j + 1] / kPi) << '\n';  // ldos (observables.cpp:50-55)
        }
    }
  }
  {
    std::ofstream out;
    if (!open("line_density.csv", out))
      return set_status(st, NEGF_CONFIG_ERROR, "cannot open output file 'line_density.csv'");
    out << "y_index,density\n";
    for (int y = 0; y < ny; ++y) {
      double s = 0.0;  // line_density_y (observables.cpp:96-110)
      for (int x = 0; x < nx; ++x) s += density[static_cast<size_t>(y) * nx + x];
      out << y << ',' << fmt(s) << '\n';
    }
  }
  return ok(st);
}

int negf_shard_writer_open(const char* path, int n_dofs, int rank, int world, int what, negf_shard_writer** out,
                           negf_status* st) {
  if (!path || !out || n_dofs < 1 || what < 1 || what > 3)
    return set_status(st, NEGF_CONTRACT_VIOLATION, "shard writer: bad argument");
  *out = nullptr;
  auto* w = new negf_shard_writer;
  w->f = std::fopen(path, "wb");
  if (!w->f) {
    delete w;
    return set_status(st, NEGF_CONFIG_ERROR, std::string("cannot open output file '") + path + "'");
  }
  w->n = n_dofs;
  w->what = what;
  w->record_bytes = 16 + ((what & 1) ? 16 * int64_t(n_dofs) : 0) + ((what & 2) ? 16 * int64_t(n_dofs) : 0);
  write_header(w, rank, world);
  w->th = std::thread([w] { w->run(); });
  *out = w;
  return ok(st);
}

int negf_shard_writer_append(negf_shard_writer* w, int n_energies, int first_energy_index, const double* energies,
                             const double* gr, const double* gless, negf_status* st) {
  if (!w || (n_energies > 0 && !energies) || ((w->what & 1) && !gr) || ((w->what & 2) && !gless))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "shard writer: bad argument");
  negf_shard_writer::Job j;
  j.bytes = static_cast<size_t>(w->record_bytes) * n_energies;
  j.host.resize(j.bytes);
  const size_t nb = 16 * static_cast<size_t>(w->n);
  for (int k = 0; k < n_energies; ++k) {
    char* r = j.host.data() + static_cast<size_t>(k) * w->record_bytes;
    pack(r, first_energy_index + k, energies[k]);
    char* p = r + 16;
    if (w->what & 1) {
      std::memcpy(p, reinterpret_cast<const char*>(gr) + k * nb, nb);
      p += nb;
    }
    if (w->what & 2) std::memcpy(p, reinterpret_cast<const char*>(gless) + k * nb, nb);
  }
  {
    std::lock_guard<std::mutex> lk(w->mu);
    if (w->error) return set_status(st, w->error, w->error_msg);
    w->q.push_back(std::move(j));
    w->records += n_energies;
  }
  w->cv.notify_all();
  return ok(st);
}

int negf_shard_writer_append_device(negf_shard_writer* w, int n_energies, int first_energy_index,
                                    const double* energies, const double* d_gr, const double* d_gless, void* stream,
                                    negf_status* st) {
  if (!w || (n_energies > 0 && !energies) || ((w->what & 1) && !d_gr) || ((w->what & 2) && !d_gless))
    return set_status(st, NEGF_CONTRACT_VIOLATION, "shard writer: bad argument");
  if (n_energies == 0) return ok(st);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int slot = -1;
  try {
    const size_t bytes = static_cast<size_t>(w->record_bytes) * n_energies;
    {
      std::unique_lock<std::mutex> lk(w->mu);
      slot = w->next_slot;
      w->cv.wait(lk, [&] { return !w->slot_busy[slot] || w->error; });
      if (w->error) return set_status(st, w->error, w->error_msg);
      w->slot_busy[slot] = true;
      w->next_slot = (slot + 1) % negf_shard_writer::kSlots;
    }
    if (w->slot_cap[slot] < bytes) {
      if (w->slot_buf[slot]) ck(cudaFreeHost(w->slot_buf[slot]), "cudaFreeHost");
      w->slot_buf[slot] = nullptr;
      ck(cudaHostAlloc(reinterpret_cast<void**>(&w->slot_buf[slot]), bytes, cudaHostAllocDefault), "cudaHostAlloc");
      w->slot_cap[slot] = bytes;
    }
    if (!w->slot_ev[slot]) ck(cudaEventCreateWithFlags(&w->slot_ev[slot], cudaEventDisableTiming), "event");
    char* buf = w->slot_buf[slot];
    const size_t nb = 16 * static_cast<size_t>(w->n);
    for (int k = 0; k < n_energies; ++k) pack(buf + static_cast<size_t>(k) * w->record_bytes,
                                              first_energy_index + k, energies[k]);
    // Strided D2H: one 2-D copy per array straight into the record layout.
    const size_t pitch = static_cast<size_t>(w->record_bytes);
    size_t at = 16;
    if (w->what & 1) {
      ck(cudaMemcpy2DAsync(buf + at, pitch, d_gr, nb, nb, n_energies, cudaMemcpyDeviceToHost, s), "gr D2H");
      at += nb;
    }
    if (w->what & 2)
      ck(cudaMemcpy2DAsync(buf + at, pitch, d_gless, nb, nb, n_energies, cudaMemcpyDeviceToHost, s), "gless D2H");
    ck(cudaEventRecord(w->slot_ev[slot], s), "event record");
    negf_shard_writer::Job j;
    j.pinned = buf;
    j.bytes = bytes;
    j.ready = w->slot_ev[slot];
    j.slot = slot;
    {
      std::lock_guard<std::mutex> lk(w->mu);
      w->q.push_back(std::move(j));
      w->records += n_energies;
    }
    w->cv.notify_all();
  } catch (const CudaFail& f) {
    if (slot >= 0) {
      std::lock_guard<std::mutex> lk(w->mu);
      w->slot_busy[slot] = false;
    }
    return set_status(st, f.code, f.msg);
  }
  return ok(st);
}

int negf_shard_writer_close(negf_shard_writer* w, negf_status* st) {
  if (!w) return ok(st);
  {
    std::lock_guard<std::mutex> lk(w->mu);
    w->stop = true;
  }
  w->cv.notify_all();
  w->th.join();
  int rc = NEGF_OK;
  std::string msg;
  if (w->error) {
    rc = w->error;
    msg = w->error_msg;
  } else {
    std::fseek(w->f, 32, SEEK_SET);  // patch the record count
    std::fwrite(&w->records, 8, 1, w->f);
  }
  if (std::fclose(w->f) != 0 && rc == NEGF_OK) {
    rc = NEGF_CONFIG_ERROR;
    msg = "shard writer: close failed";
  }
  for (int k = 0; k < negf_shard_writer::kSlots; ++k) {
    if (w->slot_buf[k]) cudaFreeHost(w->slot_buf[k]);
    if (w->slot_ev[k]) cudaEventDestroy(w->slot_ev[k]);
  }
  delete w;
  return rc == NEGF_OK ? ok(st) : set_status(st, rc, msg);
}

}  // extern "C"
