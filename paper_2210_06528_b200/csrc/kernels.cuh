// Kernel launch interface of the B200 MFA encode path (implemented in
// kernels.cu).  Each launcher returns the number of kernels it launched.
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "dev.cuh"

namespace mfb {

// Programmatic dependent launch on the solve's critical chain: each kernel
// of the chain lets its successor launch as soon as it starts
// (griddepcontrol.launch_dependents) and waits for its predecessor's grid to
// complete and flush before touching anything (griddepcontrol.wait), so the
// successor's launch and CTA rasterisation overlap the predecessor's tail.
// Memory semantics are those of plain stream order.  MFADD_NO_PDL disables it.
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
bool pdl_enabled();

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, static_cast<Args&&>(args)...);
}

// Source line of the first failed device bounds check (debug builds), else 0.
int debug_fail_line();
int debug_fail_line_tma();  // stream_tma.cu lines (debug builds)

// K1: per-row find_span + Cox-de Boor basis + window clip
// (knots.cpp:83-129, collocation.cpp:83-111).
struct RowsArgs {
  const AxisProb* probs;
  int nprobs;
  int max_m;
  const double* knots;
  const double* params;  // explicit params (AxisProb::M < 0)
  int* g0;               // local unclipped first column (span - p - col_lo)
  int* first_col;        // BandedCollocation::first_col
  int* count;            // BandedCollocation::count
  double* vals;          // (p+1) per row, clipped entries zero, unclipped positions
  DevStatus* status;
  int prob0;             // the launch covers problems [prob0, prob0 + nprobs)
};
int launch_basis_rows(int degree, const RowsArgs& a, cudaStream_t s);

// K2: banded Gram (collocation.cpp:56-67) + banded Cholesky (lsq.cpp:46-55).
// Writes per column: [1/L(c,c), L(c,c-1..c-p), L(c+1..c+p,c)] (2p+1 doubles).
struct CholArgs {
  const AxisProb* probs;
  const int* prob_ids;  // problems to factor
  int nfactor;
  int max_n;
  int max_m;      // rows of the largest factored problem
  int stage_rows; // 1: the row table is staged in shared memory
  int light;      // 1: one warp per problem, rows read through L1 (runs beside the axis-0 sweep)
  const int* g0;
  const double* vals;
  double* ltab;
  DevStatus* status;
  // Twisted (two-sided) solves of k_solve2d: per problem, the Cholesky factor
  // of the index-reversed Gram matrix ([n][P+1], same row format as the band)
  // followed by the Gram band itself; null when unused.
  double* tw = nullptr;
  std::int64_t tw_stride = 0;
};
// Twisted solve of an extent-n problem: rows [0, a) are eliminated from the
// top, rows [a+P, n) from the bottom, the P rows between last (a dense P x P
// Schur complement).  Needs at least P rows in each outer part.
inline bool tw_ok(int n, int P) { return n >= 4 * P + 2; }
int launch_gram_chol(int degree, const CholArgs& a, cudaStream_t s);
// The solve kernels' right-looking step tables of every factored problem,
// once per solve after the factorizations: rlt + problem id * stride.
int launch_rl_tables(int degree, const CholArgs& a, double* rlt, std::int64_t stride, cudaStream_t s, bool tw = false);
// forward + backward table of an extent-n problem, or its twisted table set
std::int64_t rl_table_doubles(int degree, int n, bool tw = false);

// K3: per-axis fit passes (lsq.cpp:57-61 fused: R^T contraction in row order
// + forward substitution + back substitution).
struct FitArgs {
  int D;
  std::int64_t fs[3];  // field strides
  const double* field;
  const BlockDev* blocks;
  int nblocks;
  const AxisProb* probs;
  const int* g0;
  const double* vals;
  const double* ltab;
  double* t1;
  double* t2;
  double* P;
  double* Y;                         // last-axis forward scratch (|P|)
  unsigned long long* linf_int;      // per block: max |P| over non-shared entries
  const unsigned char* shared_flag;  // per dim concatenated: 1 if the global index is shared
  std::int64_t sflag_off[3];
  int max_lines_strided[3];          // per axis: max lines over blocks
  int max_lines_last;
  std::int64_t pitch_last;           // row pitch (even) of the last-axis input (T1 for D=2, T2 for D=3)
  std::int64_t n_field, n_t1, n_t2, n_P;  // buffer sizes (debug bounds checks)
  const int* segtab;                 // last-axis row segments per axis problem (kSegStride ints)
  std::int64_t zhalf;                // last-axis contraction: Y = [parity 0 | parity 1 | y scratch]
  int defer_back;                    // 1: axis 0 forward-only, 2: contraction only; the rest on P at the end
  int min_n0;                        // smallest axis-0 held extent (partitioned final solve eligibility)
  int fuse2d;                        // D = 2: k_solve2d (CTA per block) replaces k_last_solve + the axis-0 solve
  const double* rlt;                 // right-looking step tables per axis problem (k_rl_tables), or null
  std::int64_t rlt_stride;           // doubles per axis problem in rlt (forward then backward table)
  int max_n0, max_n1, max_zl;        // largest held extents / Z pitch (k_solve2d shared-memory size)
  int tw2d;                          // k_solve2d: twisted passes (rlt holds the twisted table sets)
  int fuse3d;                        // D = 3: every pass a pure contraction, k_solve3d solves axes 2 and 1 (and 0) in smem
  int max_n2, solve3d_threads;       // k_solve3d: largest axis-2 held extent, CTA size
  int s3_slab, s3_nslab, s3_zs;      // k_solve3d: axis-0 indices per slab, slabs per block, tile column pitch
  int s3_nl;                         // k_solve3d: lines per thread (1 or 4)
  int a0_slab, a0_zr;                // k_axis0_slab: axis-1 indices per slab (0: k_axis0_backsub instead), tile row pitch
  void* join_event;                  // cudaEvent_t the last-axis solve waits for (factorizations on a side stream)
};
int launch_fit_strided(int degree, const FitArgs& a, int axis, cudaStream_t s);  // axis < D-1
int launch_fit_last(int degree, const FitArgs& a, cudaStream_t s);
// Shared-memory bytes of k_solve2d for held extents n0 x n1 (0 if it does not fit one CTA).
size_t solve2d_smem(int degree, int n0, int n1, int zl, int kseg, bool tw = false);
// The solve stage after the last-axis contraction (FitArgs::fuse2d / fuse3d; solve_tma.cu); returns its launches.
int launch_solve_stage(int degree, const FitArgs& a, int kseg, cudaStream_t s);
// Shared-memory bytes of k_solve3d for held extents n0 x n1 x n2 and a tile column pitch zs (0 if over the CTA limit).
size_t solve3d_smem(int degree, int n0, int n1, int n2, int zs, int kseg);
// Shared-memory bytes of k_axis0_slab for an axis-0 extent n0 and `lines` lines per slab (0 if over the CTA limit).
size_t axis0_slab_smem(int degree, int n0, int lines);

// D = 1: CTA per block, column-parallel R^T q + serial banded solve (smem: max_n x (2P+2) doubles).
int launch_fit_1d(int degree, const FitArgs& a, int max_n, cudaStream_t s);

// K4: one averaging epoch over every shared control (solver.cpp:112-164 with
// the runtime.cpp:123-158 Jacobi snapshot), jump residuals (solver.cpp:
// 166-193) and the dp numerator/denominator pieces (solver.cpp:402-405).
struct EpochArgs {
  int D;
  int nblocks;
  int B[3];
  std::int64_t N[3];
  const int2* hr;       // holder coordinate ranges, concatenated per dim
  std::int64_t hr_off[3];
  const int* slist;     // shared indices per dim, concatenated
  const int* clist;     // non-shared indices per dim, concatenated
  std::int64_t s_off[3], c_off[3];
  std::int64_t nS[3], nC[3];
  std::int64_t piece[3];  // dof count of each piece
  std::int64_t total;
  const AxisProb* probs;
  int axbase[3];
  const std::int64_t* poff;
  double* P;
  int mode;  // 0 measure only, 1 average n_s == 2 only, 2 average all
  unsigned long long* change;
  unsigned long long* linf_sh;
  EpochAcc* acc;
  // final per-pair jumps (mode 3): pair slot table nblocks*27, per-pair ss/ms
  const int* pair_slot;
  unsigned long long* pair_jumps;
  std::int64_t n_P;  // debug bounds checks
  int max_holders;   // max n_s over all controls (8: <= 2 holders per axis)
};
int launch_epoch(const EpochArgs& a, cudaStream_t s);

// K4 (region form, n_s <= 8): one CTA per tile of a region's box; holder ids
// and offsets are CTA-uniform.  The last CTA to finish computes dp (K5 fused)
// and, inside the epoch-loop graph, sets the WHILE condition.
struct EpochRegionArgs {
  const TileDev* tiles;
  int ntiles;
  int nblocks;
  double* P;
  int mode;  // 0 measure, 3 final pair jumps, -1 loop (1 on iteration 1, 2 after), 4 epoch 0 + iteration 1
  unsigned long long* change;
  unsigned long long* linf_sh;
  const unsigned long long* linf_int;
  EpochState* st;
  double* epoch_out;  // 3 doubles per epoch slot: dp, jump_ss, jump_ms
  unsigned long long* pair_jumps;
  int max_iter;
  double tol;
  unsigned long long cond;  // cudaGraphConditionalHandle (loop mode only)
  int predicated;           // loop mode outside the WHILE node: no-op once converged or past max_iter
  int max_ns;               // largest region n_s (selects the kernel form)
  const double* recv;       // sharded: remote holders' copies (RegionDev::rmask)
  int finalize;             // 1: the last CTA computes dp and writes epoch_out (else k_epoch_finalize)
  int zero_pairs;           // > 0: the finalize also clears pair_jumps[0, zero_pairs) (no memset node in the chain)
  int slot;                 // epoch_out slot when finalize is done separately
  double* snap;             // log_errors: per-epoch snapshots of the shared copies (null: none)
  long long snap_stride;    // doubles per snapshot (= the held lattices' size)
};
int launch_epoch_regions(const EpochRegionArgs& a, cudaStream_t s);
// dp / jumps of the epoch into epoch_out[3*slot] and accumulator reset (one CTA).
int launch_epoch_finalize(const EpochRegionArgs& a, cudaStream_t s);
// Sharded solve: epoch `slot`'s loop bookkeeping on the device (after the dp max-reduction over ranks).
int launch_shard_advance(EpochState* st, const double* epoch_out, int slot, double tol, cudaStream_t s);
// Sharded solve: gather holder copies into the send buffer.
int launch_pack(const PackTile* tiles, int ntiles, const double* P, double* send, cudaStream_t s);

// K9 (log_errors): residual_error (lsq.cpp:66-85) of every local block's held
// lattice over its input box, per epoch (record_epoch, solver.cpp:357-364).
struct BlockResArgs {
  int D;
  int nblocks;                 // local blocks (grid.y)
  const BlockDev* blocks;
  const AxisProb* probs;
  const int* g0;
  const double* vals;
  const double* P;
  const double* field;
  std::int64_t fs[3];
  int ntile;                   // CTAs per block (grid.x)
  double* partial;             // [nblocks][ntile] x {l2^2, linf}
  double* errs;                // [(max_iter + 1)][nglobal] x {l2, linf}
  const EpochState* st;        // slot = st->iter (the epoch just recorded), or `slot` when null
  int slot;
  int expect_iter;             // >= 0: no-op unless st->iter == expect_iter (after a predicated epoch)
  int nglobal, boff;           // all blocks; global id of local block 0
  int max_m0;                  // longest axis-0 row table of a local block (shared-memory staging)
};
int launch_block_residual(int degree, const BlockResArgs& a, cudaStream_t s);

// K9 one-pass form (residual_tma.cu): every recorded epoch's block residuals
// after the loop, from the held lattices P (non-shared controls) and the
// epoch snapshots of the shared copies, Q_loc streamed once per EG epochs.
struct ResTmaArgs {
  int D;
  int nblocks;                       // grid.y (local blocks)
  const BlockDev* blocks;
  const AxisProb* probs;
  const int* g0;
  const double* vals;
  const double* P;
  const double* snap;                // snapshot e at snap + e * snap_stride (same layout as P)
  long long snap_stride;
  const unsigned char* sflag;        // per dim concatenated: 1 if the global control index is shared
  std::int64_t sflag_off[3];
  const EpochState* st;              // epochs recorded = st->iter + 1 (null: 1)
  int W;                             // TMA box inner width (even, one spare column)
  int ntc, nrr;                      // column tiles (D = 3: rows j1) x row ranges per block: grid.x = ntc * nrr
  int lt_cap;                        // window columns per staged plane (>= the widest CTA window)
  int na_cap;                        // staged planes per epoch (>= the most planes a row range touches)
  int eg;                            // epochs per pass (1, 2 or 4; the staged windows scale with it)
  int ng;                            // threads per point (2: each decodes half of the pass's epochs)
  double* partial;                   // [epoch][block][ntc * nrr] x {sum e^2, max |e|}
  double* errs;                      // [(max_iter + 1)][nglobal] x {l2, linf}
  int nglobal, boff;
};
int launch_residual_tma(int degree, const ResTmaArgs& a, const CUtensorMap& map, int threads, cudaStream_t s);
size_t residual_tma_smem(int degree, int W, int eg, int na_cap, int lt_cap);

// K5: dp = max_b change_b / max(1, ||P_b||_inf) and epoch bookkeeping.
struct DpArgs {
  int nblocks;
  unsigned long long* change;
  unsigned long long* linf_sh;
  const unsigned long long* linf_int;
  EpochAcc* acc;
  double* epoch_out;  // 3 doubles: dp, jump_ss, jump_ms
  double* host_mirror;  // optional pinned-mapped copy (nullable)
};
int launch_dp(const DpArgs& a, cudaStream_t s);

// K6: assemble_owned (solver.cpp:281-294).
constexpr long long kAsmOtherRank = -(1ll << 62);
struct AssembleArgs {
  int D;
  int B[3];
  std::int64_t N[3];
  const int* own_coord;  // per dim concatenated: owning block coordinate of each control index
  std::int64_t oc_off[3];
  const AxisProb* probs;
  int axbase[3];
  const std::int64_t* poff;
  const long long* rowbase;  // P offset of each lattice row in each last-dim owner block, minus its col_lo
                             // (kAsmOtherRank: the owner block lives on another rank, entry written as +0.0)
  const double* P;
  double* lattice;
  std::int64_t row0, nrows;  // lattice rows (all dims but the last) to assemble
  std::int64_t col0, ncols;  // last-dim range (a shard's own range when D == 1)
};
int launch_assemble(const AssembleArgs& a, cudaStream_t s);

// K7: decode the global lattice over the input grid (decode.cpp:83-97 as
// called by block_error_slab, solver.cpp:298-328), error field, L2^2/Linf.
struct DecodeArgs {
  int D;
  std::int64_t M[3];  // output (input-grid) extents, padded to 3 with leading 1s
  std::int64_t N[3];  // lattice extents, padded
  int T[3];           // tile extents
  std::int64_t ntiles[3];
  int W[3];           // smem control-box extents bound
  const int* g0[3];   // global rows per (padded) dim
  const double* vals[3];
  int pk[3];          // per padded dim: degree (0 for padding dims)
  const double* lattice;
  const double* field;   // nullable -> pure decode (no error)
  double* out;           // error field (field != null) or decoded values; nullable
  double* partial;       // per tile {l2sq, linf}
};
int launch_decode(int degree, const DecodeArgs& a, cudaStream_t s);
// TMA pipeline geometry: box = (B2 inner, [B1], R rows) per stage, S stages.
struct TmaGeom {
  int B1, B2, R, S;
  int lt_cap;  // doubles of smem reserved for the Cholesky table (0 = use global)
};
// TMA axis-0 fit pass (stream_tma.cu); needs 16-B aligned field row strides.
int launch_fit_axis0_tma(int degree, const FitArgs& a, const CUtensorMap& map, const TmaGeom& g, int ntiles,
                         cudaStream_t s);
// Deferred axis-0 back substitution on the held lattices (+ per-block L-inf).
int launch_axis0_backsub(int degree, const FitArgs& a, int max_n0, std::int64_t max_rest, cudaStream_t s);
// D = 3 middle axis through the T1 tensor map ([rows][pitch]): grid.z = c0.
int launch_fit_mid_tma(int degree, const FitArgs& a, const CUtensorMap& map, const TmaGeom& g, int ntiles, int max_n0,
                       cudaStream_t s);

// TMA last-axis fit pass (D >= 2): 128-B swizzled 16-column boxes of the
// last-axis input, LT lines per CTA.
int launch_fit_last_tma(int degree, const FitArgs& a, const CUtensorMap& map, int LT, int lt_cap, int kseg,
                        cudaStream_t s);

// TMA decode sweep over the whole input grid (D = 2, 3), stream_tma.cu.
struct DecodeSweepArgs {
  int D;
  int M0, M1, M2;   // input grid extents (M2 = 1 for D = 2)
  int N0, N1, N2;   // lattice extents (N2 = 1 for D = 2)
  int ntile1, ntile2, nrange, H;
  int ybeg, yend;   // input rows [ybeg, yend) along axis 0 decoded by this launch
  const int* g0_0;  // global decode rows per dim (row tables, 16-B aligned)
  const double* v_0;
  const int* g0_1;
  const double* v_1;
  const int* g0_2;
  const double* v_2;
  const double* lattice;
  double* err;      // nullable
  double* partial;  // per CTA {l2sq, linf}
  unsigned* ticket; // CTA completion counter (zero between launches)
  double* red2;     // {sum l2sq, max linf}, written by the last CTA
  int win;          // D = 3: every CTA's axis-2 window fits (host-checked): the staged-window kernel form
  int na_cap;       // D = 3 win: staged control planes per row range (host-sized exactly)
};
int launch_decode_tma(int degree, const DecodeSweepArgs& a, const CUtensorMap& map, const TmaGeom& g,
                      cudaStream_t s);

// residual_error (lsq.cpp:66-85) of ONE local problem (the unit sub-boundary,
// lsq.hpp:41): thread per point, decode of the window-clipped rows in the
// reference's axis order with explicit RN operations (bitwise equal pointwise
// errors), per-CTA {sum e^2, max |e|} partials.
struct ResidualArgs {
  int D;
  int m[3], n[3];          // rows / window columns per dim
  const int* g0[3];        // local unclipped first column per row
  const double* vals[3];   // (p+1) per row, out-of-window entries zero
  const double* controls;  // n0 x n1 x n2 row-major
  const double* q;         // m0 x m1 x m2 row-major
  double* pointwise;       // nullable
  double* partial;         // 2 per CTA
  std::int64_t total;
};
int launch_residual_points(int degree, const ResidualArgs& a, int ctas, cudaStream_t s);

// K7b: deterministic reduction of the tile partials.
int launch_reduce_partials(const double* partial, std::int64_t n, double* out2, cudaStream_t s);


// Point evaluation (model.cu): eval_deriv / eval_deriv_sided (decode.cpp:14-80)
// of items against one or more control lattices resident on the device.
struct EvalLattice {
  std::int64_t base;     // offset of the lattice in EvalArgs::ctrl
  std::int64_t ext[3];   // extents
  std::int64_t coff[3];  // col_offset (global index of local column 0)
};
struct EvalItem {
  int lat;       // EvalLattice index
  int side_dim;  // -1: unsided
  int side;      // 0 Below, 1 Above (decode.hpp:24)
  int pad_;
  int ord[3];    // derivative order per dim
  int pad2_;
  double pt[3];  // parameters
};
struct EvalArgs {
  int rank;
  int deg[3];
  const double* knots;
  std::int64_t kn_off[4];
  const double* ctrl;
  const EvalLattice* lats;
  const EvalItem* items;
  std::int64_t n;
  double* out;
  int* err;  // per item: 0, or (code << 8) | dim (1 order > degree, 2 find_span range, 3 lattice window)
};
int launch_eval_points(const EvalArgs& a, cudaStream_t s);
// field.cpp:170-185 on the device: n raw scalars (width 4 or 8, optional byte swap) -> fp64
int launch_raw_to_f64(const unsigned char* raw, std::int64_t n, int width, int swap, double* out, cudaStream_t s);

}  // namespace mfb

#include <vector>
struct mfadd_context;
namespace mfb {
// Host helpers over launch_eval_points (model.cu), shared with engine.cu.
void eval_items_device(mfadd_context* ctx, int rank, const int* degrees, const double* knots,
                       const std::int64_t* kn_off, const double* d_ctrl, const std::vector<EvalLattice>& lats,
                       const std::vector<EvalItem>& items, std::vector<double>& out);
void probe_items(int rank, int dim, double u, int max_order, const std::vector<std::vector<double>>& cross,
                 int lat_below, int lat_above, std::vector<EvalItem>& items);
void probe_reduce(const std::vector<double>& vals, std::size_t first, std::size_t count, int max_order,
                  std::vector<double>& jumps);

}  // namespace mfb
