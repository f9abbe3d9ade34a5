// Device kernels of the B200 HSC path (sm_100a, complex FP64).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "plan.hpp"

namespace negfb {

// Device-side error record (lowest key wins, like run.cpp:258-262).
struct DevStatus {
  unsigned long long singular_key;   // energy<<40 | fold_pos<<20 | pivot
  unsigned long long residual_key;   // energy<<32 | dof
  unsigned long long nonskew_key;    // energy<<32 | cluster
  unsigned long long max_resid_bits; // max |Re g<|/|g<| as non-negative double bits
};

struct BatchArgs {
  double2* arena;
  int64_t stride;     // complex elements per energy arena
  int nE;
  int e_base;         // global index of energy 0 of this batch
  // Work counters of the persistent GEMM launches: {next item, finished CTAs},
  // zero between launches (the last CTA of a launch resets them; launches on
  // the solver stream are ordered).
  unsigned long long* gemm_ctr;
};

void launch_assemble(const BatchArgs& b, const Plan& p, const int64_t* d_h_pos, const double2* d_h_val,
                     const InitRegion* d_init_zero, const int64_t* d_diag_pos, const double* d_energies,
                     const int64_t* d_sr_pos, const int* d_sr_ptr, const int* d_sr_src,
                     int64_t sr_nnz, const double2* d_sigma_r, cudaStream_t s, int64_t& launches);
void launch_scatter_lesser(const BatchArgs& b, const Plan& p, const double* d_energies, const int64_t* d_sl_pos,
                           const int* d_sl_ptr, const int* d_sl_src, int64_t sl_nnz, const double2* d_sigma_l,
                           cudaStream_t s, int64_t& launches);
void launch_inverse(const BatchArgs& b, const InvTask* d_tasks, const InvTask* h_tasks, int count,
                    DevStatus* st, cudaStream_t s, int64_t& launches);
void launch_bigpanel(const BatchArgs& b, const BigTask* d_tasks, const BigTask* h_tasks, int count, int k0, int o0,
                     DevStatus* st, cudaStream_t s, int64_t& launches);
void launch_bigswap(const BatchArgs& b, const BigTask* d_tasks, int count, int o0, cudaStream_t s,
                    int64_t& launches);
void launch_bigperm(const BatchArgs& b, const BigTask* d_tasks, const BigTask* h_tasks, int count, cudaStream_t s,
                    int64_t& launches);
void launch_gemm(const BatchArgs& b, const GemmTask* d_tasks, const GemmTerm* d_terms,
                 const GemmTile* d_tiles, const GemmTile* h_tiles, int tile_begin, int tile_count,
                 cudaStream_t s, int64_t& launches, bool gauss3m = false);
void launch_spsi(const BatchArgs& b, const SpsiTask* d_tasks, const int* d_colptr, const int* d_rows,
                 const double2* d_vals, const int* d_wcols, int begin, int count, cudaStream_t s, int64_t& launches);
void launch_mgather(const BatchArgs& b, const MGatherTask* d_tasks, const MGatherBlock* d_blocks, int begin, int count,
                    cudaStream_t s, int64_t& launches);
void launch_sschur(const BatchArgs& b, const SschurTask* d_tasks, const SschurContrib* d_contrib,
                   const SpsiTask* d_spsi, const int* d_colptr, const int* d_rows, const double2* d_vals,
                   const int* d_rc, int begin, int count, cudaStream_t s, int64_t& launches);
void launch_leafdiag(const BatchArgs& b, const LeafDiagTask* d_tasks, const LeafDiagTask* h_tasks,
                     const int* d_rows, const int* d_optr, const int* h_optr, const LeafDiagEntry* d_ent, int begin,
                     int count, cudaStream_t s, int64_t& launches);
void launch_diag(const BatchArgs& b, const DiagTask* d_tasks, const GemmTerm* d_terms, int begin,
                 int count, cudaStream_t s, int64_t& launches);
void launch_scale(const BatchArgs& b, const ScaleTask* d_tasks, int begin, int count,
                  cudaStream_t s, int64_t& launches);
void launch_skew_check(const BatchArgs& b, const double2* d_sigma_l, int64_t sl_nnz, const int* d_cslots,
                       const int* d_cslot_ptr, const int* d_sl_ptr, const int* d_sl_src, const int* d_sl_partner,
                       int n_seeded, const int* d_seeded_ids, double* d_acc, DevStatus* st, cudaStream_t s,
                       int64_t& launches);
void launch_skew(const BatchArgs& b, const SkewTask* d_tasks, const SkewTask* h_tasks, int begin, int count,
                 cudaStream_t s, int64_t& launches);
void launch_combine(const BatchArgs& b, const CombineTask* d_tasks, const CombineTask* h_tasks, int begin, int count,
                    cudaStream_t s, int64_t& launches);
void launch_ordered_sum(const double* parts, int nranks, int n, double* out, cudaStream_t s, int64_t& launches);
void launch_output_gr(const BatchArgs& b, int n, const int64_t* d_gr_pos, double2* d_gr, cudaStream_t s,
                      int64_t& launches);
void launch_output(const BatchArgs& b, int n, const int64_t* d_gr_pos, const int64_t* d_gl_pos,
                   const double* d_weights, double2* d_gr, double2* d_gl, double* d_density,
                   DevStatus* st, cudaStream_t s, int64_t& launches);

}  // namespace negfb
