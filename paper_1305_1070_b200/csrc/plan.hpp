// Host plan: everything about one device that does not depend on the energy.
//
// Built once (reference analogue: build_tree + the structural half of
// group_by_partition / hsc_fold / LeanSolver, proj/src/run.cpp:123-133,
// block.cpp:49-82, hsc.cpp:131-327,447-534) and replayed for every energy
// batch:
//   * the separator tree (tree.hpp, bit-exact with the reference),
//   * the symbolic fold: fill sets S(i) (hsc.cpp:482-511),
//   * the needed-block closure for the top-down sweeps (SURVEY App. A.4,
//     generalised to the exact transitive rule),
//   * the per-energy HBM arena layout of every block,
//   * the level-synchronous task lists (inverse / grouped GEMM / diagonal
//     dot / seed scaling) in a deterministic order,
//   * the reference's operation ledger (dense.hpp:69-82 rules) and the
//     executed (needed-only) ledger that is the roofline numerator.
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <vector>

#include "common.hpp"
#include "tree.hpp"

namespace negfb {

struct ProblemDesc {
  int n = 0;
  // Energy-independent Hamiltonian, COO (duplicates summed).
  std::vector<int> h_rows, h_cols;
  std::vector<cplx> h_vals;
  // Energy-dependent retarded self-energy pattern (values per energy):
  // A(E) = E I - H - Sigma^r(E)  (block.cpp:123-161).
  std::vector<int> sr_rows, sr_cols;
  // Lesser self-energy pattern; must be cluster-block-diagonal.
  std::vector<int> sl_rows, sl_cols;
  // Partition inputs (run.cpp:113-133) ...
  std::vector<std::array<double, 2>> coords;
  std::vector<std::vector<int>> atomic_groups;
  int max_leaf = 64;
  // ... or an explicit tree (parent per cluster + dof lists).
  bool explicit_tree = false;
  std::vector<int> tree_parent;
  std::vector<std::vector<int>> tree_dofs;
};

// Operand transforms.
enum : int { OP_N = 0, OP_T = 1, OP_C = 2, OP_H = 3 };
// Epilogue modes.
enum : int { MODE_SET = 0, MODE_ADD = 1, MODE_INIT = 2 };

// One output block C (m x n) = [Init +] sum_t sign_t op(A_t) op(B_t).
// Offsets are complex-element offsets inside one energy's arena.
struct GemmTask {
  int m, n;
  int ldc;
  int mode;
  int64_t c_off;
  int64_t init_off;
  int ld_init;
  int term_begin, term_count;
  // Fused diagonal (rows of never-referenced clusters, whose G / P rows feed
  // only diag(G_xx) / diag(P_xx)): the epilogue forms, per output row r and
  // 16-column warp group, sum_c Psi[r][c] * op(C[r][c]) (dmode 1: +C, 2:
  // -conj(C), 3: i Im(-conj(C)) -- the anti-Hermitian symmetric form) into
  // partials[dpart_off + r * dpart_ld + group]; nostore skips writing C itself.
  int dmode, nostore;
  int dpsi_ld, dpart_ld;
  // Symmetric output (m == n): only 32x32 tiles on or above the diagonal
  // run; a tile strictly above it also writes the lower triangle.  mirror 1:
  // C = C^T up to rounding (the Schur update of a diagonal block, a full
  // G_xx), written with the task's mode (ADD / INIT read their own (c, r)
  // entry); mirror 2: C = -C^H (a full P_xx = G^<_xx), MODE_SET only.
  int mirror;
  int64_t dpsi_off, dpart_off;
  // Second output 2*C at c2_off (same ldc) when >= 0: the doubled Psi of
  // clusters whose symmetric diagonal quadratic form uses each block pair once.
  int64_t c2_off;
};

struct GemmTerm {
  int k;
  int a_op;        // OP_N: A stored m x k; OP_T: stored k x m
  int b_op;        // OP_N/OP_C: stored k x n; OP_T/OP_H: stored n x k
  int sign;        // +1 / -1
  int lda, ldb;
  int64_t a_off, b_off;
  // bit 0: the A operand is real for every energy (zero imaginary parts,
  // exactly), bit 1: B is -- set by mark_real_operands (plan.cpp)
  int real;
  int pad;
};

// CTA tile of a grouped GEMM launch.
struct GemmTile {
  int task;
  int m0, n0;
  int arr;  // warp arrangement of the CTA: 0 = 2x2 (32x32), 1 = 1x4 (16x64), 2 = 4x1 (64x16), 3 = one warp (16x16)
};

// Diagonal-only output: out[a] = [init[a*init_stride]] + sum_t sign_t
// sum_b A_t[a][b] * opB_t[b][a]   (a < m).
struct DiagTask {
  int m;
  int init_stride;   // m+1 when init is a full m x m block, 1 for a vector
  int has_init;
  int term_begin, term_count;
  int part_np;       // fused-epilogue partials per row (0: none), summed in order
  int64_t out_off;   // vector of m
  int64_t init_off;
  int64_t part_off;
};

// dst[a][b] = sig[a] * conj(src[a][b]), a < m, b < n (diagonal Sigma^< seed).
struct ScaleTask {
  int m, n;
  int ld_src, ld_dst;
  int64_t src_off, dst_off, sig_off;
};

struct InvTask {
  int m;
  int cluster;
  int fold_pos;   // position in fold order (root = nc-1): error precedence
  int real;       // the block is real for every energy (mark_real_operands)
  int64_t off;
};

// Blocks above kSmemInvMax are inverted by the multi-CTA blocked
// Gauss-Jordan, in outer panels of kOuter columns, each factored as kPanel-
// wide inner panels: per inner panel one K_PANEL launch (factor it with row
// partial pivoting, apply its interchanges inside the outer panel, stage
// M_p - I_p and the pivot rows) and one grouped-GEMM rank-kPanel update of the
// outer panel's columns; per outer panel one K_BIGSWAP launch (its
// interchanges on every other column, staging of the rank-kOuter operands)
// and ONE grouped-GEMM rank-kOuter update of the whole block (K = 64: the
// bulk of the m^3 work runs as compute-bound GEMM); finally one K_PERM launch
// undoes the interchanges.  Any block size: the panel lives in shared memory
// up to kPanelSmemMax rows, in arena scratch (L2) beyond.  Scratch lives in
// the arena.
constexpr int kPanel = 8;
constexpr int kOuter = 64;
constexpr int kPanelSmemMax = 1400;  // m x (kPanel + 1) complex panel in shared memory (<= 197 KB)

struct BigTask {
  int m;
  int fold_pos;
  int cluster;
  int pad;
  int64_t off;       // the block (m x m)
  int64_t off_mp;    // inner panel M_p - I_p (m x kPanel); the working panel when m > kPanelSmemMax
  int64_t off_rs;    // inner staged pivot rows (kPanel x m)
  int64_t off_mp64;  // outer panel M_p - I_p (m x kOuter)
  int64_t off_rs64;  // outer staged pivot rows (kOuter x m); row buffers of K_PERM
  int64_t off_perm;  // 3 m ints: perm, and K_PERM's two index maps
  int64_t off_thr;   // (threshold, failed flag)
};
// Complex elements of arena scratch one BigTask of size m needs.
inline int64_t big_scratch_elems(int64_t m) {
  auto a8 = [](int64_t x) { return (x + 7) & ~int64_t(7); };
  return a8(m * kPanel) * 2 + a8(m * kOuter) * 2 + a8((3 * m + 3) / 4) + 8;
}

enum OpKind : int { K_INVERSE = 0, K_GEMM = 1, K_DIAG = 2, K_SCALE = 3, K_PANEL = 4, K_PERM = 5, K_SKEW = 6,
                    K_COMBINE = 7, K_SPSI = 8, K_SSCHUR = 9, K_LEAFDIAG = 10, K_BIGSWAP = 11, K_MGATHER = 12 };

// Compact leaves (sparse, never referenced, unseeded): their G / P rows feed
// only diag(G_xx) / diag(P_xx) = sum_{a,c} Psi[r][a] M[a][c] Psi[r][c] over the
// hull columns H of Psi_x (concatenated over S(x)), with M the G_SS / P_SS
// blocks restricted to H x H (block pairs of the symmetric forms doubled, the
// skipped ones zero).  K_MGATHER builds M per (leaf, energy); one grouped-GEMM
// task per leaf then forms Psi_H M with the fused-diagonal epilogue.
struct MGatherBlock {
  int dst_row, dst_col;   // block origin in M (h x h, row-major)
  int rows, cols;
  int conj;               // 1: conjugate the source
  int pad;
  double coef;            // 0: zero block (no source)
  int64_t src;            // source element (0, 0)
  int64_t rs, cs;         // source strides per M row / column
};
struct MGatherTask {
  int h;
  int block_begin, block_count;
  int pad;
  int64_t dst;            // M (h x h)
};

// Psi_x = -inv_x A_{x,S(x)} for a leaf whose coupling block holds only the
// energy-independent -H entries (no Schur fill below a leaf; contact and
// phonon self-energies never leave a cluster): A_{x,S} is a few stencil
// entries per column, so Psi is formed column by column from those entries
// (CSC in SpsiTask's ranges) instead of a dense m x m x K product.
struct SpsiTask {
  int m, K;
  int col_begin;      // K + 1 entries of Plan::spsi_colptr from here
  int h;              // > 0: compact Psi_H (m x h, the hull columns of Plan::spsi_wcols from
  int wcol_begin;     //      wcol_begin) is written instead of the full m x K Psi
  int pad;
  int64_t off_inv;    // inv_x (m x m, row-major; the D block after inversion)
  int64_t off_psi;    // Psi_x (m x K)
  int64_t off_psi2;   // 2 Psi_x, or -1
};

// The leaves' share of a gathered Schur update (hsc.cpp:501-511):
// A_{jp,jq} (+)= sum over leaves i of Psi_{i,jp}^T A_{i,jq}, with A_{i,jq} the
// leaf's stencil entries (SpsiTask CSC): m_p x m_q outputs, a few products
// each.  Runs before the block's dense gather GEMM (which then accumulates).
struct SschurTask {
  int mp, mq, ld, mode;         // mode: MODE_ADD or MODE_SET
  int contrib_begin, contrib_count;
  int entry;                    // 1: one thread per target entry over all leaves (small, densely
                                //    touched targets); 0: per leaf over its touched rows x columns,
                                //    waves of disjoint leaves between barriers (large targets)
  int pad;
  int64_t off;                  // target block
};
// diag(G_xx) / diag(P_xx) of a never-referenced, unseeded sparse leaf by the
// Woodbury form of hsc.cpp:220-226 / 289-300: with Psi = -inv_x A_{x,S} and
// A_{x,S} nonzero only on the rows T of boundary dofs,
//   diag(G_xx) = diag(inv_x) + diag(W M W^T),  M = A_{T,S} G_SS A_{T,S}^T,
//   diag(P_xx) =               diag(W M W^H),  M = A_{T,S} P_SS A_{T,S}^H,
// W = inv_x[:, T]: |T|^2 entries of M gathered from the stored G / P blocks
// instead of the m x K x K row products.  M is complex symmetric (G) /
// anti-Hermitian (P): its upper triangle is gathered (CSR over the
// |T|(|T|+1)/2 outputs of LeafDiagTask), the lower one mirrored.
struct LeafDiagTask {
  int m, nT;
  int t_begin;        // nT local rows in Plan::ld_rows
  int out_begin;      // nT(nT+1)/2 + 1 entries of Plan::ld_optr
  int mode;           // 0: G (symmetric, + diag inv), 1: P (anti-Hermitian)
  int pad;
  int64_t off_inv;    // inv_x (m x m)
  int64_t off_out;    // diag vector (m)
};
struct LeafDiagEntry {
  int64_t pos;        // arena position of the G / P entry
  int flag;           // 1: use -conj(value) (P block read in the other orientation)
  int out;            // packed (i1 << 16) | i2 of the output (redundant, for checks)
  cplx coef;          // a1 a2 (G) or a1 conj(a2) (P)
};

struct SschurContrib {
  int spsi;                     // the leaf's SpsiTask (inv_i, CSC of A_{i,S})
  int p_off, q_off;             // column offsets of jp and of jq in A_{i,S}
  int nr, nc;                   // target rows / columns the leaf touches (nonempty columns)
  int rc_begin;                 // nr row then nc column indices in Plan::sschur_rc
  int sync;                     // 1: last of its wave (a barrier follows).  Contributions are
                                // ordered by wave: a contribution is in the wave after the
                                // latest earlier one (gather order) whose rows x columns it
                                // overlaps, so every target entry still receives its leaves
                                // in gather order while disjoint leaves run concurrently
  int pad;
};

struct Op {
  int kind;
  int begin, count;  // range in the kind's array (tiles for K_GEMM)
  int task_begin, task_count;  // K_GEMM: task range (for accounting)
  int phase;         // 0 fold, 1 G, 2 seed, 3 N fold, 4 P
  int level;
  int k0;            // K_PANEL: first column of the panel
  int k1;            // K_PANEL / K_BIGSWAP: first column of the outer panel
  int inv_update;    // K_GEMM: 1 = a rank-kPanel / rank-kOuter update inside a multi-CTA block inverse
  double cmul;       // executed complex multiply-adds per energy
};

// Elementwise steps of the RGF path (K_SKEW / K_COMBINE ops).
struct SkewTask {      // dst = skew_half(src): upper triangle of src, Im of
  int n, pad;          // the diagonal, lower = -conj(upper) (dense.cpp:136-170)
  int64_t src, dst;
};
struct CombineTask {   // out = gl + term + x - x^H (rgf.cpp:373-377)
  int n, pad;
  int64_t gl, term, x, out;
};

struct Ledger {
  int64_t multiply_ops = 0;
  int64_t inverse_ops = 0;
};

struct ClusterInfo {
  int m = 0;
  std::vector<int> S;                 // fill set, nearest first (Psi list)
  std::vector<int64_t> s_col;         // column offset of each S entry in Arow/Psi
  std::vector<char> s_orig;           // S entry holds original entries of A (else pure fill)
  int K0 = 0;                         // width of the original-entry column prefix
  int K = 0;                          // sum of |S|
  bool referenced = false, seeded = false, seed_dense = false;
  bool full_g = false, full_p = false, has_nd = false;
  std::vector<int> gcols, ncols, pcols;          // anc order
  std::vector<int64_t> gcol_off, ncol_off, pcol_off;
  int WG = 0, WN = 0, WP = 0;
  int64_t off_d = -1, off_arow = -1, off_psi = -1, off_sig = -1;
  int64_t off_gd = -1, off_grow = -1, off_nd = -1, off_nrow = -1, off_pd = -1, off_prow = -1;
  int64_t off_gpart = -1, off_ppart = -1;  // fused-diagonal partials (m x NP)
  int64_t off_psi2 = -1;                   // 2 Psi (symmetric fused G diagonal)
  int gpart_np = 0, ppart_np = 0;
  // compact leaf (see MGatherTask): hull width h, offsets of S's hull blocks in H
  bool compact = false;
  int hc = 0;
  std::vector<int> hoff;
  int64_t off_psic = -1, off_mg = -1;  // Psi_H (m x h), M (h x h)
};

// Region [off, off + rows*pitch) with `cols` leading elements per row.
struct InitRegion {
  int64_t off;
  int rows, cols, pitch;
};

struct Plan {
  ProblemDesc desc;
  Tree tree;
  Graph graph;
  std::vector<ClusterInfo> ci;

  int64_t arena = 0;         // complex elements per energy
  int64_t a_region = 0;      // [0, a_region): D + Arow (template copied per energy)
  int64_t big_scratch = 0;   // arena offset of the multi-CTA inverse scratch
  int64_t z_begin = 0, z_end = 0;  // region zeroed per energy (Sigma^<, N, root P)
  std::vector<int64_t> h_pos;       // -H entries of the A region: positions ...
  std::vector<cplx> h_val;          // ... and values (duplicates summed)
  std::vector<InitRegion> init_zero;  // zeroed per energy (D, original Arow prefix, Sigma^<)

  // Per-energy scatter maps.
  std::vector<int64_t> diag_pos;          // n: A_dd position (E added)
  // Sigma^r: unique target slots, each summing its pattern entries.
  std::vector<int64_t> sr_slot_pos;       // slot -> arena position (subtract)
  std::vector<int> sr_slot_ptr, sr_slot_src;  // CSR slot -> pattern indices
  // Sigma^<: same, into the Sig blocks.
  std::vector<int64_t> sl_slot_pos;
  std::vector<int> sl_slot_ptr, sl_slot_src;
  std::vector<int> sl_cluster;            // per slot: its cluster
  std::vector<int> sl_partner;            // per slot: slot of (c,r) or -1
  std::vector<int> sl_cidx;               // per slot: index into seeded_ids
  std::vector<int> seeded_ids;            // clusters carrying a Sigma^< block
  std::vector<int> cslot_ptr, cslots;     // CSR: seeded cluster index -> its slots
  // Output maps: per dof, position of its diagonal entry in Gd / Pd.
  std::vector<int64_t> out_gr_pos, out_gl_pos;
  bool any_seed = false;

  std::vector<GemmTask> gemm_tasks;
  std::vector<GemmTerm> gemm_terms;
  std::vector<GemmTile> gemm_tiles;
  std::vector<DiagTask> diag_tasks;
  std::vector<GemmTerm> diag_terms;
  std::vector<ScaleTask> scale_tasks;
  std::vector<InvTask> inv_tasks;
  std::vector<BigTask> big_tasks;
  std::vector<SkewTask> skew_tasks;      // RGF path only
  std::vector<CombineTask> comb_tasks;   // RGF path only
  std::vector<SpsiTask> spsi_tasks;      // sparse leaf Psi (K_SPSI)
  std::vector<int> spsi_colptr;          // per task: K + 1 offsets into spsi_row / spsi_val
  std::vector<int> spsi_wcols;           // compact leaves: written Psi columns (S space), H order
  std::vector<MGatherTask> mg_tasks;     // K_MGATHER
  std::vector<MGatherBlock> mg_blocks;
  std::vector<int> spsi_row;             // local row t of the entry
  std::vector<cplx> spsi_val;            // A_{x,S}[t][c] (= -H)
  std::vector<SschurTask> sschur_tasks;  // sparse leaf Schur contributions (K_SSCHUR)
  std::vector<SschurContrib> sschur_contrib;
  std::vector<int> sschur_rc;
  std::vector<LeafDiagTask> ld_tasks;    // K_LEAFDIAG
  std::vector<int> ld_rows;              // T lists
  std::vector<int> ld_optr;              // per task: CSR over its upper-triangle outputs
  std::vector<LeafDiagEntry> ld_entries;
  std::vector<Op> ops;
  std::vector<std::vector<int>> rgf_layers;  // non-empty: an RGF plan (no tree)
  int rgf_gr_ops = 0;                        // ops [0, rgf_gr_ops) = rgf_gr
  // Replay split points (host-buffer solves overlap copies with compute):
  // ops before lesser_op never read the Sigma^< slots; G^r output entries are
  // final once ops [0, gr_done_op) ran.
  int lesser_op = 0, gr_done_op = 0;

  Ledger ref_fold, ref_gless;   // reference ledger per energy (hsc_fold / hsc_gless)
  double exec_cmul = 0.0;       // executed complex MACs per energy (incl. inversions m^3)
  double exec_inv_cmul = 0.0;
  double needed_cmul = 0.0;     // exec_cmul before the real-block weights (0: no real blocks)
  int n_real_clusters = 0;
  int max_block = 0;
};

constexpr int kSmemInvMax = 112;  // largest block inverted by one CTA (registers / shared memory)
// Single-CTA inverse kernel variants by block size (kernels.cu
// launch_inverse, measured with tools/inv_bench.cu): <= 16 and 17..48
// register-resident Gauss-Jordan, 49..64 and 65..kSmemInvMax shared-memory
// blocked Gauss-Jordan (one launch per padded size m8 there, so each launch
// sizes its shared memory for its own blocks).  The plan groups a level's
// inverse tasks by this class, largest first.
inline int inv_size_class(int m) { return m <= 16 ? 0 : m <= 32 ? 1 : m <= 48 ? 2 : m <= 64 ? 3 : 4; }
// CTA tile extents per warp arrangement (see GemmTile::arr).
// arr 3: warp tiles (16 x 16 per warp, fragments from global memory) for small tasks
constexpr int kArrTM[4] = {32, 16, 64, 16};
constexpr int kArrTN[4] = {32, 64, 16, 16};

// Cover an m x n output block with CTA tiles (appended to `out`).  The
// candidates are the three uniform grids and a 32x32 core with its bottom /
// right remainder strips covered by 32x32, 16x64 or 64x16 tiles; the
// cheapest under the measured tile cost model (a fixed part per tile-chunk
// plus a part proportional to the live 8x8 DMMA subtiles; tools/gemm_bench)
// wins.
void tile_task(int task, int m, int n, int ksum, std::vector<GemmTile>& out);
// Upper-triangular 32x32 tiles of a symmetric m x m task (GemmTask::mirror);
// returns the number of output entries the tiles compute.
int64_t tile_task_sym(int task, int m, std::vector<GemmTile>& out);

Plan build_plan(ProblemDesc desc);

// Batched energy-doubling decimation of one dense lead, the restatement of
// surface_self_energy (device.cpp:195-251) as a grouped-kernel program over
// per-energy arenas.  Arena blocks (w x w, row-major):
enum LeadBlock : int {
  LB_H00 = 0, LB_H01, LB_H01CT, LB_ZH,  // constants per energy (ZH = zI - h00)
  LB_ES, LB_E, LB_ALPHA0, LB_ALPHA1, LB_BETA0, LB_BETA1,
  LB_G, LB_M, LB_AM, LB_BM, LB_T1, LB_RHS, LB_FIN, LB_SIG,
  LB_COUNT
};
struct LeadPlan {
  Plan P;          // arena size + task arrays (P.ops holds every op below)
  int w = 0;
  int64_t off[LB_COUNT] = {};
  // op index ranges [begin, end) in P.ops
  int inv_gm[2] = {0, 0};      // g = (z - es)^-1, m = (z - e)^-1 (device.cpp:218, 235)
  int gemm_a[2][2] = {};       // per parity: T1 = h01^H g; AM = alpha m; BM = beta m
  int gemm_b[2] = {0, 0};      // rhs = (z - h00) - T1 h01 (device.cpp:220-221)
  int inv_rhs[2] = {0, 0};     // refined = rhs^-1 (device.cpp:222)
  int gemm_c[2][2] = {};       // per parity: es += ab; e += ab + ba; alpha', beta' (236-243)
  int fin1[2] = {0, 0};        // T1 = h01^H refined
  int fin2[2] = {0, 0};        // sigma = T1 h01 (device.cpp:226-227)
  // decay-criterion variant (devices.sancho_rubio): m only per sweep, and
  // the frozen surface block inverted once at the end (into FIN)
  int inv_m[2] = {0, 0};
  int gemm_a2[2][2] = {};      // per parity: AM = alpha m; BM = beta m
  int inv_fin[2] = {0, 0};
};
LeadPlan build_lead_plan(int w);

// Layered recursive Green's function (rgf_gr / rgf_gless, rgf.cpp:181-380)
// as one replayable op list over per-energy arenas (Plan::rgf_layers set):
// the second, independent GPU path (chain partitions == RGF,
// test_hsc.cpp:648-678) and the paper's comparison baseline.  Every coupling
// is treated as dense.
Plan build_rgf_plan(ProblemDesc desc, std::vector<std::vector<int>> layers);

}  // namespace negfb
