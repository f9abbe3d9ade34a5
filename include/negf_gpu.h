/* negf_gpu.h -- C ABI of the B200 HSC selected-inversion path.
 *
 * Drop-in for the per-energy HSC solve of the reference C++ library
 * (/root/reference/proj).  The reference has no C ABI and no plugin
 * mechanism; each entry point below names the C++ interface it replaces:
 *
 *   negf_plan_create      build_tree            proj/src/run.cpp:123-133
 *                         nested_dissection     proj/include/negf/partition.hpp:84-87
 *                         (+ the structural half of group_by_partition
 *                          block.hpp:61-63 and hsc_fold hsc.hpp:65-66)
 *   negf_plan_tree        SeparatorTree accessors partition.hpp:19-68
 *   negf_plan_ledger      FlopLedger of hsc_fold + hsc_gless dense.hpp:69-82
 *   negf_gpu_create       (new) device arena + schedule upload, one per GPU
 *   negf_gpu_solve_batch  solve_energy's HSC branch, batched over energies
 *                         proj/src/run.cpp:141-192: assemble_system
 *                         block.cpp:123-161 -> hsc_fold hsc.cpp:447-534 ->
 *                         hsc_gless hsc.cpp:552-577 -> GreensDiagonal
 *                         flattening block.cpp:163-205 -> the energy sum of
 *                         electron_density observables.cpp:58-93
 *   negf_gpu_density      electron_density's result (before the caller's
 *                         geometric scaling, run.cpp:291-292)
 *   negf_gpu_nccl_*       (new) the one cross-GPU exchange: allreduce of the
 *                         energy-partial density over NCCL
 *
 * Conventions: complex values are interleaved (re, im) float64 -- the layout
 * of std::complex<double>; all pointers are caller-owned host memory unless
 * the name says _device; calls on one handle are not thread-safe (one host
 * thread or one process per GPU, like the reference's per-thread energy
 * solves).  Every call returns a NEGF_* status code and, when
 * `st` is non-null, fills it.  Codes mirror proj/include/negf/errors.hpp.
 */
#ifndef NEGF_GPU_H
#define NEGF_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  NEGF_OK = 0,
  NEGF_SINGULAR_BLOCK = 1,       /* SingularBlock (errors.hpp:36-42)        */
  NEGF_NON_SKEW_HERMITIAN = 2,   /* NonSkewHermitianInput (errors.hpp:61-65)*/
  NEGF_CONTRACT_VIOLATION = 3,   /* ContractViolation (errors.hpp:27-31)    */
  NEGF_CUDA_ERROR = 4,
  NEGF_NCCL_ERROR = 5,
  NEGF_OUT_OF_MEMORY = 6,
  NEGF_CONFIG_ERROR = 7,         /* ConfigError (errors.hpp:21-25)          */
  NEGF_PARTITION_VIOLATION = 8,  /* PartitionViolation (errors.hpp:44-53)   */
  NEGF_RESIDUAL_TOO_LARGE = 9,   /* ResidualTooLarge (errors.hpp:67-71)     */
  NEGF_INTERNAL = 10,
  NEGF_CONVERGENCE_ERROR = 11    /* ConvergenceError (errors.hpp:56-61)     */
};

typedef struct {
  int code;
  int energy_index; /* lowest failing energy index (run.cpp:258-262), or -1 */
  int cluster;      /* cluster being eliminated (SingularBlock), or -1      */
  int pivot;        /* pivot index within the block (SingularBlock), or -1  */
  int dof;          /* offending dof (ResidualTooLarge), or -1              */
  char msg[256];
} negf_status;

/* Problem description: the inputs of build_tree/solve_energy.
 * A(E) = E*I - H - Sigma^r(E)   (assemble_system, block.cpp:123-161)
 * Sigma^r(E) and Sigma^<(E) have fixed patterns; their values are supplied
 * per energy in pattern order.  Contacts are dense sub-blocks of these
 * patterns, the phonon self-energy their diagonal entries (device.cpp). */
typedef struct {
  int n_dofs;
  int64_t h_nnz;
  const int32_t* h_rows;
  const int32_t* h_cols;
  const double* h_vals;          /* complex, h_nnz                          */
  int64_t sr_nnz;                /* Sigma^r pattern                         */
  const int32_t* sr_rows;
  const int32_t* sr_cols;
  int64_t sl_nnz;                /* Sigma^< pattern (cluster-block-diagonal)*/
  const int32_t* sl_rows;
  const int32_t* sl_cols;
  const double* coords;          /* 2*n_dofs (x, y) or NULL: BFS surrogate  */
  int n_groups;                  /* atomic groups (dense contacts)          */
  const int32_t* group_ptr;      /* n_groups+1                              */
  const int32_t* group_dofs;
  int max_leaf;
  /* Optional explicit tree instead of nested dissection (fixture tests). */
  int n_tree_clusters;           /* 0 = use nested dissection               */
  const int32_t* tree_parent;    /* n_tree_clusters (-1 = root)             */
  const int32_t* tree_ptr;       /* n_tree_clusters+1                       */
  const int32_t* tree_dofs;
} negf_problem;

typedef struct negf_plan negf_plan;
typedef struct negf_gpu negf_gpu;

typedef struct {
  int n_dofs, n_clusters, levels, root, max_block;
  int64_t arena_bytes_per_energy;
  int64_t ref_fold_mul, ref_fold_inv;    /* reference ledger, per energy */
  int64_t ref_gless_mul, ref_gless_inv;
  double exec_cmul;                      /* executed work / energy in complex MACs (8 real flops):
                                            a product with a real operand counts 1/2, real x real
                                            and real inverses 1/4 (what the FP64 pipes execute) */
  double exec_inv_cmul;
  int n_ops, n_gemm_tasks, n_gemm_tiles, n_inv_tasks;
  double needed_cmul;                    /* the same needed-only work counted as complex throughout
                                            (8 m n k per product, 8 m^3 per inverse) */
  int n_real_clusters, pad_;             /* clusters eliminated in real arithmetic */
} negf_plan_info;

int negf_plan_create(const negf_problem* p, negf_plan** out, negf_status* st);
int negf_plan_info_get(const negf_plan* p, negf_plan_info* info);
/* Tree export: parent[nc], level[nc], dof_ptr[nc+1], dofs[n] (ascending per
 * cluster), fold_order[nc-1].  Any pointer may be NULL. */
int negf_plan_tree(const negf_plan* p, int32_t* parent, int32_t* level, int32_t* dof_ptr,
                   int32_t* dofs, int32_t* fold_order);
/* Fill sets S(i) (the Psi lists, nearest ancestor first): ptr[nc+1], ids. */
int negf_plan_fill(const negf_plan* p, int32_t* ptr, int32_t* ids);
/* Schedule introspection: per grouped-GEMM task its m, n, summed k, phase
 * (0 fold, 1 G^r, 2 seed, 3 N fold, 4 G^<) and level.  Arrays of
 * n_gemm_tasks entries (negf_plan_info); any pointer may be NULL. */
int negf_plan_gemm_tasks(const negf_plan* p, int32_t* m, int32_t* n, int64_t* k_total, int32_t* phase,
                         int32_t* level);
/* CTA tiles of the grouped-GEMM launches (introspection): task index, tile
 * origin, warp arrangement (0: 32x32, 1: 16x64, 2: 64x16) and whether the
 * tile also writes its transpose (symmetric tasks), n_gemm_tiles entries;
 * any pointer may be NULL. */
int negf_plan_gemm_tiles(const negf_plan* p, int32_t* task, int32_t* m0, int32_t* n0, int32_t* arr,
                         int32_t* mirrored);
/* The replayed op list (introspection, n_ops entries): kind (0 inverse,
 * 1 grouped GEMM, 2 diagonal, 3 seed scaling, 4 panel, 5 permutation, 6 skew,
 * 7 combine, 8 sparse leaf Psi, 9 sparse leaf Schur contributions, 10 leaf
 * Woodbury diagonals, 11 outer-panel interchanges of a multi-CTA inverse),
 * phase (0 fold, 1 G^r, 2 seed, 3 N fold, 4 G^<, 6 a GEMM update inside a
 * multi-CTA block inverse), tree level, range in the
 * kind's task (GEMM: tile) array, executed complex MACs per energy; any
 * pointer may be NULL. */
int negf_plan_ops(const negf_plan* p, int32_t* kind, int32_t* phase, int32_t* level, int32_t* begin,
                  int32_t* count, double* cmul);
void negf_plan_destroy(negf_plan* p);

/* Layered RGF plan: rgf_gr + rgf_gless
 * (proj/src/rgf.cpp:181-380) on layered_from_coo's layer map
 * (rgf.cpp:69-150; n_layers lists of dofs, layer_ptr[n_layers+1]) of the same
 * problem, as a plan the negf_gpu_* device calls solve exactly like an HSC
 * plan (diag G^r, diag G^<, density).  Every coupling is handled as a dense
 * block.  Errors: NEGF_CONTRACT_VIOLATION for a layer map that is not a
 * disjoint cover, a non-transposed lower coupling or a Sigma^< that is not
 * layer-block-diagonal; NEGF_PARTITION_VIOLATION for entries coupling
 * non-adjacent layers.  negf_plan_tree / negf_plan_fill do not apply. */
int negf_rgf_plan_create(const negf_problem* p, int n_layers, const int32_t* layer_ptr,
                         const int32_t* layer_dofs, negf_plan** out, negf_status* st);

/* Device side: allocates the per-energy arenas for up to max_energy_batch
 * energies (0 = as many as fit in 85% of free HBM) on `device`. */
int negf_gpu_create(const negf_plan* plan, int device, int max_energy_batch, negf_gpu** out,
                    negf_status* st);
int negf_gpu_batch_capacity(const negf_gpu* g);

/* Solves n_energies energy points (chunked internally by the batch
 * capacity).  Host inputs:
 *   energies[nE], weights[nE] (trapezoid weights, observables.cpp:14-32),
 *   sigma_r[nE][sr_nnz], sigma_lesser[nE][sl_nnz] (complex),
 *   first_energy_index: global index of energies[0] for error reports.
 * Host outputs (nullable): gr_diag[nE][n], gless_diag[nE][n] (complex, per
 * dof in global order).  The weighted Im G^< sum is accumulated on device
 * into the handle's density (negf_gpu_density). */
int negf_gpu_solve_batch(negf_gpu* g, int n_energies, const double* energies,
                         const double* weights, const double* sigma_r,
                         const double* sigma_lesser, int first_energy_index, double* gr_diag,
                         double* gless_diag, negf_status* st);
/* Same, with every input and output already resident in device memory
 * (d_gr/d_gless nullable).  Runs on the handle's stream; no host sync unless
 * `sync` is nonzero (errors are then reported by negf_gpu_check).  The device
 * status is sticky: every solve since the last negf_gpu_check / synchronous
 * solve merges into it (lowest energy index first), and only reading it
 * clears it. */
int negf_gpu_solve_batch_device(negf_gpu* g, int n_energies, const double* d_energies,
                                const double* d_weights, const double* d_sigma_r,
                                const double* d_sigma_lesser, int first_energy_index,
                                double* d_gr, double* d_gless, int sync, negf_status* st);
int negf_gpu_check(negf_gpu* g, negf_status* st);
/* density_out[n] = (1/2pi) sum_k w_k Im G^<_jj(E_k) over all solved energies
 * (observables.cpp:71-91): this rank's partial, or the cross-rank sum when
 * negf_gpu_allreduce_density ran after the last solve.  reset != 0 zeroes
 * the accumulator afterwards. */
int negf_gpu_density(negf_gpu* g, double* density_out, int reset, negf_status* st);
void* negf_gpu_stream(negf_gpu* g);       /* cudaStream_t of the handle */
void* negf_gpu_density_device(negf_gpu* g); /* double[n] this rank's partial (unscaled) */
/* electron_density's Re-residual guard (observables.cpp:79-84): mode 1
 * (default) raises NEGF_RESIDUAL_TOO_LARGE like the reference; mode 0 only
 * records the largest |Re G^<_jj| / |G^<_jj| (DensityMap::max_real_residual). */
int negf_gpu_set_residual_check(negf_gpu* g, int mode);
double negf_gpu_max_real_residual(negf_gpu* g);
/* Lowest (energy index, dof) whose |Re G^<_jj| > 1e-8 |G^<_jj| since the last
 * reset, whatever the mode (the quantity electron_density checks first,
 * observables.cpp:79-84): returns 1 and fills the (nullable) outputs, else 0.
 * Lets a multi-rank sweep raise ResidualTooLarge only after every rank's
 * solver errors are settled (run.cpp:258-291). */
int negf_gpu_residual_violation(negf_gpu* g, int32_t* energy_index, int32_t* dof, int reset);

/* Kernel launches issued by the last solve call (ours only). */
int64_t negf_gpu_last_launches(const negf_gpu* g);

/* Optional per-kernel timing: CUDA events recorded on the handle's stream
 * around every launch of subsequent solves (a host sync is added at the end
 * of each solve).  Totals accumulate until reset. */
typedef struct {
  double ms;            /* summed event time of the launches             */
  double cmul;          /* executed complex multiply-adds (8 flops each)  */
  int64_t launches;
} negf_kernel_stat;
enum { NEGF_KSTAT_GEMM = 0, NEGF_KSTAT_INVERSE = 1, NEGF_KSTAT_DIAG = 2, NEGF_KSTAT_SCALE = 3,
       NEGF_KSTAT_ASSEMBLE = 4, NEGF_KSTAT_OUTPUT = 5, NEGF_KSTAT_COUNT = 6 };
int negf_gpu_profile(negf_gpu* g, int enable);
int negf_gpu_profile_read(negf_gpu* g, negf_kernel_stat* out /* [NEGF_KSTAT_COUNT] */, int reset);
/* Per plan op (negf_plan_ops order): summed CUDA-event milliseconds of the
 * profiled solves (n_ops entries). */
int negf_gpu_profile_ops(negf_gpu* g, double* ms_out, int reset);
void negf_gpu_destroy(negf_gpu* g);

/* NCCL: one communicator per handle, bootstrapped by the caller (e.g. a
 * torch.distributed broadcast of the 128-byte id). */
int negf_nccl_unique_id(char id_out[128], negf_status* st);
int negf_gpu_nccl_init(negf_gpu* g, const char id[128], int nranks, int rank, negf_status* st);
/* Sum of the ranks' unscaled density partials into a separate buffer (the
 * partials keep accumulating; negf_gpu_density returns the sum until the
 * next solve).  Default
 * (ordered): ncclAllGather of the partials + a device sum in
 * rank order, bit-reproducible for any rank count and NCCL algorithm;
 * negf_gpu_set_ordered_reduce(g, 0) selects a plain ncclAllReduce. */
int negf_gpu_allreduce_density(negf_gpu* g, negf_status* st);
int negf_gpu_set_ordered_reduce(negf_gpu* g, int ordered);

/* ---- Contact self-energies on the GPU -------------
 *
 *   negf_lead_*                surface_self_energy  proj/src/device.cpp:195-251
 *                              (energy-doubling decimation, fixed-point test
 *                              ||refined - g||_F <= 1e-10, <= 200 sweeps), the
 *                              per-energy call of attach_contacts
 *                              device.cpp:262-304 / sigma_for_energy
 *                              run.cpp:90-109, batched over energies
 *   negf_lead_modes_sigma_device  analytic transverse-mode Sigma of a uniform
 *                              hard-wall 2-D effective-mass lead (the lead model
 *                              BASELINE.json names for configs 1/2/4/5)
 *   negf_contacts_fill_device  lesser_self_energy device.cpp:322-366 and the
 *                              placement of the contact / phonon
 *                              (phonon_self_energy device.cpp:306-320) values
 *                              into the Sigma^r / Sigma^< pattern arrays of
 *                              negf_gpu_solve_batch_device
 */
typedef struct negf_lead negf_lead;
/* One dense lead: onsite block h00 and coupling h01 (w x w complex,
 * row-major).  criterion 0 = the reference's surface_self_energy: h01 couples
 * a lead cell to the next one away from the device, the fixed-point test
 * ||refined - g||_F <= 1e-10 ends the sweeps and Sigma = h01^H g h01.
 * criterion 1 = decay test max|alpha|, max|beta| < tol (alpha_0 = h01,
 * beta_0 = h01^T) and Sigma = h01^T (z - es)^-1 h01 (the convention of
 * paper_1305_1070_b200/devices.py sancho_rubio, used for config 3).
 * Errors as the reference: eta <= 0 -> NEGF_CONFIG_ERROR; w out of range ->
 * NEGF_CONTRACT_VIOLATION. */
int negf_lead_create(int device, int w, const double* h00, const double* h01, double eta_ev, int criterion,
                     double tol, int max_energy_batch, negf_lead** out, negf_status* st);
/* Sigma^r(E_k) = h01^H g_s(E_k) h01 (made exactly complex symmetric), for
 * n_energies energies.  Host variant: energies[nE] -> sigma_out[nE][w][w].
 * Errors report the lowest failing energy (first_energy_index + k):
 * NEGF_SINGULAR_BLOCK from an inverse, NEGF_CONVERGENCE_ERROR after 200
 * sweeps. */
int negf_lead_sigma(negf_lead* l, int n_energies, const double* energies, int first_energy_index,
                    double* sigma_out, negf_status* st);
/* Device variant: d_energies[nE] -> d_sigma_out + k*ld_out (complex
 * elements, ld_out >= w*w).  Synchronous on the handle's stream. */
int negf_lead_sigma_device(negf_lead* l, int n_energies, const double* d_energies, int first_energy_index,
                           double* d_sigma_out, int64_t ld_out, negf_status* st);
/* Decimation sweeps each energy of the last call needed (index of the
 * converged sweep, as the reference's loop counter), sweeps_out[nE]. */
int negf_lead_last_sweeps(const negf_lead* l, int32_t* sweeps_out);
int64_t negf_lead_last_launches(const negf_lead* l);
void* negf_lead_stream(negf_lead* l);
void negf_lead_destroy(negf_lead* l);

/* Analytic lead: Sigma_ab(E) = sum_m phi_am (-t lambda_m) phi_bm with
 * phi_ym = sqrt(2/(w+1)) sin(y m pi/(w+1)), eps_m = 4t - 2t cos(m pi/(w+1)),
 * z = (eps_m - E - i eta)/(2t), lambda_m = z -+ sqrt(z^2 - 1) with
 * |lambda_m| <= 1; symmetrised like surface_self_energy.  Runs on `stream`
 * (a cudaStream_t, NULL = legacy default stream) without host sync; it uses
 * a per-thread scratch buffer, so calls from one host thread on different
 * streams must not overlap. */
int negf_lead_modes_sigma_device(int w, double t_ev, double eta_ev, int n_energies, const double* d_energies,
                                 double* d_sigma_out, int64_t ld_out, void* stream, negf_status* st);

/* One dense contact block in the pattern arrays: its w*w entries are
 * consecutive, row-major, starting at sr_off in Sigma^r and sl_off in
 * Sigma^< (-1 = absent). */
typedef struct {
  int w;
  const double* d_sigma;   /* device, complex, energy k at d_sigma + 2*k*ld */
  int64_t ld;              /* complex elements between energies           */
  int64_t sr_off, sl_off;
  double mu_ev;            /* contact chemical potential                  */
} negf_contact_desc;
/* Fills, per energy k, the contact blocks of Sigma^r (copy) and Sigma^<
 * (-f(E_k; mu) (S - S^H), device.cpp:335-342) and the phonon diagonal
 * (Sigma^r = -i gamma_d; Sigma^< = -f(E_k; mu_ph) (s - conj s),
 * device.cpp:356-362) with f the Fermi function of device.cpp:253-260 at
 * kT_ev (= kBoltzmannEvPerK * temperature_k).  Phonon entries are n_phonon
 * consecutive pattern entries from ph_sr_off / ph_sl_off (-1 = absent).
 * Pattern entries not named here are left untouched. */
int negf_contacts_fill_device(int n_energies, const double* d_energies, double kT_ev, int n_contacts,
                              const negf_contact_desc* contacts, int n_phonon, const double* d_phonon_gamma,
                              int64_t ph_sr_off, int64_t ph_sl_off, double mu_phonon_ev, double* d_sigma_r,
                              int64_t sr_stride, double* d_sigma_lesser, int64_t sl_stride, void* stream,
                              negf_status* st);

/* ---- Output path -----------------------------------
 *
 *   negf_format_double     format_double   proj/src/run.cpp:276-281
 *                          (std::to_chars, general, 17 significant digits)
 *   negf_write_solve_csv   cmd_solve's artefacts run.cpp:284-326:
 *                          density.csv, ldos.csv (ldos observables.cpp:50-55),
 *                          line_density.csv (line_density_y
 *                          observables.cpp:96-110); dof j = y*nx + x
 *   negf_shard_writer_*    (new) binary per-shard diag G^r / G^< writer,
 *                          replacing ldos.csv's per-energy x dof text for
 *                          large runs
 */
/* Writes v into buf (NUL-terminated); returns its length or -1. */
int negf_format_double(double v, char* buf, int len);
/* density[nx*ny] already scaled (density_scale, run.cpp:55-56); gr_diag
 * (nE x nx*ny complex) or NULL to skip ldos.csv.  Creates out_dir. */
int negf_write_solve_csv(const char* out_dir, int nx, int ny, int n_energies, const double* energies,
                         const double* density, const double* gr_diag, negf_status* st);

/* Shard file: 64-byte header "NEGFSHD1", int32 version, n_dofs, rank, world,
 * what (1 = G^r, 2 = G^<, 3 = both), int32 0, int64 record count; then one
 * record per energy: int32 energy_index, int32 0, f64 energy, [n c128 diag
 * G^r], [n c128 diag G^<].  Records are written by a background thread in
 * append order. */
typedef struct negf_shard_writer negf_shard_writer;
int negf_shard_writer_open(const char* path, int n_dofs, int rank, int world, int what,
                           negf_shard_writer** out, negf_status* st);
/* Host diagonals (nE x n complex each; the array `what` excludes may be NULL). */
int negf_shard_writer_append(negf_shard_writer* w, int n_energies, int first_energy_index,
                             const double* energies, const double* gr, const double* gless, negf_status* st);
/* Device diagonals: one strided D2H copy per array on `stream` into pinned
 * staging (two slots, reused when written), file write off the caller's
 * thread.  The device buffers may be reused once the stream passes. */
int negf_shard_writer_append_device(negf_shard_writer* w, int n_energies, int first_energy_index,
                                    const double* energies, const double* d_gr, const double* d_gless,
                                    void* stream, negf_status* st);
/* Drains the queue, patches the record count, closes the file. */
int negf_shard_writer_close(negf_shard_writer* w, negf_status* st);

#ifdef __cplusplus
}
#endif
#endif /* NEGF_GPU_H */
