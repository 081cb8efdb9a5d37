/* include/mfadd_b200.h — C ABI of the B200-native MFA encode library
 * (paper_2210_06528_b200/libmfadd_b200.so).
 *
 * The reference (`mfadd`, /root/reference/proj) has no FFI; its drop-in
 * boundary is the C++ library API `mfadd::core`.  Every entry
 * point below replaces one reference call, cited as file:line under
 * proj/core/include/mfadd/.  Plain pointers and sizes only, no exceptions:
 * each function returns a status code that maps 1:1 onto the reference's
 * exception types (see MFADD_E* below); the C++ and Python host layers turn
 * them back into the same exception classes.
 *
 * Threading: a context owns one CUDA device + stream; calls on one context
 * must be serialised by the caller (the reference's solve() is likewise
 * called from one orchestrating thread, solver.hpp:76).  Results are bitwise
 * reproducible run to run (no floating-point atomics on any summation).
 */
#ifndef MFADD_B200_H
#define MFADD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MFADD_ABI_VERSION 1

/* status codes <-> reference exception types */
#define MFADD_OK 0
#define MFADD_EINVAL 1     /* std::invalid_argument                       */
#define MFADD_ERANGE 2     /* std::out_of_range (find_span, knots.cpp:88) */
#define MFADD_ESINGULAR 3  /* SingularFitError{dim, span} (lsq.hpp:24-28) */
#define MFADD_ERUNTIME 4   /* std::runtime_error                          */
#define MFADD_ELOGIC 5     /* std::logic_error                            */
#define MFADD_ECUDA 6      /* CUDA / NCCL failure (no reference analogue) */
#define MFADD_ENOMEM 7     /* device allocation failure                   */

int mfadd_abi_version(void);
/* Thread-local detail of the last non-zero status. */
const char* mfadd_last_error(void);
int mfadd_last_error_dim(void);      /* SingularFitError::dim  */
int64_t mfadd_last_error_span(void); /* SingularFitError::span */

/* ------------------------------------------------------------------ layout
 * Replaces: Decomposition partition(grid_dims, bounds, blocks_per_dim, degree,
 *           nctrl_per_block, overlap, clamp_interfaces)   layout.hpp:107-111
 * Host-side metadata (integers bit-exact with the reference).  bounds may be
 * NULL ([0,1] per dim; bounds only enter the affine coordinate map). */
typedef struct mfadd_decomposition mfadd_decomposition;

int mfadd_partition(int rank, const int64_t* grid_dims, const double* bounds /* 2*rank */,
                    const int* blocks_per_dim, int degree, const int64_t* nctrl_per_block, int64_t overlap,
                    int clamp_interfaces, mfadd_decomposition** out);
void mfadd_decomposition_free(mfadd_decomposition* dec);
int mfadd_dec_rank(const mfadd_decomposition* dec);
int mfadd_dec_block_count(const mfadd_decomposition* dec);      /* GlobalLayout::block_count */
/* BlockDim (layout.hpp:47-57), 16 int64 per (block, dim), field order:
 * span_lo, span_hi, delta_lo, delta_hi, overlap_lo, overlap_hi,
 * local_span_lo, local_span_hi, dof_lo, dof_hi, own_lo, own_hi,
 * input_lo, input_hi, own_input_lo, own_input_hi */
void mfadd_dec_block_dims(const mfadd_decomposition* dec, int64_t* out);
void mfadd_dec_coords(const mfadd_decomposition* dec, int* out);  /* BlockLayout::coords */
void mfadd_dec_nctrl(const mfadd_decomposition* dec, int64_t* out); /* GlobalLayout::n_ctrl */
int mfadd_dec_knots(const mfadd_decomposition* dec, int dim, double* out /* nullable */); /* kvs[dim].knots */
int mfadd_dec_neighbors(const mfadd_decomposition* dec, int block, int* out, int cap); /* BlockLayout::neighbors */
/* SharedDofMap::holder_span for every control index along dim (layout.hpp:74-76) */
void mfadd_dec_holder_ranges(const mfadd_decomposition* dec, int dim, int* out /* 2*n_ctrl */);
/* exchange_volume (runtime.hpp:78) per block */
void mfadd_dec_exchange_volume(const mfadd_decomposition* dec, int64_t* out);
double mfadd_dec_compression_ratio(const mfadd_decomposition* dec); /* layout.hpp:114 */
int mfadd_dec_any_shared(const mfadd_decomposition* dec);           /* SharedDofMap::any_shared */
/* GlobalLayout::n_input (layout.hpp:86-96): the field extents the decomposition expects */
void mfadd_dec_grid_dims(const mfadd_decomposition* dec, int64_t* out /* rank */);

/* ----------------------------------------------------------------- device */
typedef struct mfadd_context mfadd_context;
/* stream: a cudaStream_t to run on, or NULL for a private stream. */
int mfadd_context_create(int device, void* stream, mfadd_context** out);
void mfadd_context_free(mfadd_context* ctx);
/* Number of kernel launches this context has issued (launch accounting). */
int64_t mfadd_context_launch_count(const mfadd_context* ctx);

/* ------------------------------------------------------------------ solve
 * Replaces: SolveResult solve(const Field&, const Decomposition&,
 *                             const SolverConfig&)                solver.hpp:76
 * A solver is a plan (like a cuFFT plan): the decomposition's device tables
 * and work buffers, created once and executed per field.  Creating it is the
 * analogue of partition() (outside the reference's timed region); executing
 * it is solve(). */
typedef struct {
  int max_outer_iterations; /* SolverConfig::max_outer_iterations (solver.hpp:17) */
  double tolerance;         /* SolverConfig::tolerance                            */
  int workers;              /* accepted, ignored: the GPU replaces the pool       */
  int log_errors;           /* per-epoch block residuals (solver.cpp:357-364)     */
  int enforce_continuity;   /* SolverConfig::enforce_continuity                   */
  int store_error;          /* materialise SolveResult::global_error on device    */
} mfadd_solver_config;

typedef struct {
  int converged, constraint_iterations, n_epochs, n_final_jumps;
  double final_dp, global_l2, global_linf;
  /* PhaseTimings (solver.hpp:48-54), seconds, CUDA-event measured */
  double t_setup, t_local_solve, t_exchange, t_constraint, t_decode;
} mfadd_solve_summary;

typedef struct {
  int iteration; /* EpochStats (solver.hpp:40-46) */
  double dp_max, jump_ss, jump_ms;
} mfadd_epoch_stats;

typedef struct mfadd_solver mfadd_solver;

int mfadd_solver_create(mfadd_context* ctx, const mfadd_decomposition* dec, const mfadd_solver_config* cfg,
                        mfadd_solver** out);
void mfadd_solver_free(mfadd_solver* s);
/* Execute solve() on a field (row-major, last dim fastest, Field::values).
 * field_on_device != 0: `field` is a device pointer on the context's GPU.
 * Otherwise it is host memory and is copied in on the context stream. */
int mfadd_solve(mfadd_solver* s, const double* field, int field_on_device, mfadd_solve_summary* out);
/* End-to-end host call: H2D(field) + solve + D2H(global lattice, and the
 * global_error field when out_error != NULL).  This is the reference-facing
 * drop-in: mfadd::solve with host buffers. */
int mfadd_solve_host(mfadd_solver* s, const double* field_host, double* out_controls_host,
                     double* out_error_host /* nullable */, mfadd_solve_summary* out);

/* A stream of n independent solves with host buffers (e.g. the time steps of
 * a simulation): the H2D copy of field i+1 and the D2H copies of solve i's
 * lattice / error field overlap with the solves (separate copy streams, two
 * device slots).  Per step the copies equal mfadd_solve_host's.  out: n
 * summaries (nullable); the getters below then describe the last solve. */
int mfadd_solve_host_batch(mfadd_solver* s, int n, const double* const* fields_host,
                           double* const* out_controls_host, double* const* out_errors_host /* nullable */,
                           mfadd_solve_summary* out /* nullable */);

/* Results of the last solve (SolveResult members, solver.hpp:56-68). */
int mfadd_solver_epochs(const mfadd_solver* s, mfadd_epoch_stats* out, int cap);
/* InterfaceJump list (solver.hpp:34-38): block_a, block_b, linf_ss, linf_ms */
int mfadd_solver_final_jumps(const mfadd_solver* s, double* out4, int cap);
/* MfaModel::controls — the assembled global lattice, n_ctrl extents */
int mfadd_solver_controls(const mfadd_solver* s, double* out, int out_on_device);
/* SolveResult::global_error (requires cfg.store_error) */
int mfadd_solver_global_error(const mfadd_solver* s, double* out, int out_on_device);
/* BlockState::p of one block (held window, dof_lo..dof_hi extents) */
int mfadd_solver_block_controls(const mfadd_solver* s, int block, double* out, int out_on_device);
/* EpochStats::block_errors {l2, linf} per block of one epoch (log_errors) */
int mfadd_solver_block_errors(const mfadd_solver* s, int epoch, double* out2);
/* Device pointer to the global lattice (valid until the next solve/free). */
const double* mfadd_solver_device_controls(const mfadd_solver* s);
/* Kernel launches issued by the last mfadd_solve (launch accounting). */
int mfadd_solver_last_launches(const mfadd_solver* s);
/* Per-kernel CUDA-event timeline (on the launching stream); clears the record
 * list, which then accumulates over every following solve. */
int mfadd_solver_set_profiling(mfadd_solver* s, int on);
/* (name, milliseconds) of every recorded kernel since set_profiling, in order;
 * names: cap * name_len chars (nullable).  Returns the record count. */
int mfadd_solver_kernel_times(const mfadd_solver* s, char* names, int name_len, double* ms, int cap);

/* ------------------------------------------------------------- multi-GPU
 * The path shards by blocks: rank r of n owns contiguous block
 * ids.  With n <= B0 these are the block rows [r*B0/n, (r+1)*B0/n) along axis
 * 0; with n > B0 (D >= 2, n <= the block count) they are the id ranges
 * [r*nblocks/n, (r+1)*nblocks/n), which may cut a block row (the reference
 * deals any block count to any number of workers, runtime.cpp:115-121).  Each
 * epoch exchanges the copies of the controls shared across ranks
 * (ncclSend/ncclRecv with every rank that holds a copy, the
 * runtime.cpp:123-158 exchange) and max-reduces dp.  Block-row shards send
 * only the lattice halo rows a neighbour's decode reads; finer shards combine
 * the lattice with one all-reduce (u64 sum: every entry has one owner, +0.0
 * elsewhere).  Every rank decodes its own input rows.  Results equal the
 * single-device solve (bitwise for the lattice). */
typedef struct mfadd_comm mfadd_comm;
/* ncclGetUniqueId on one rank; the 128 bytes are then broadcast by the caller. */
int mfadd_nccl_unique_id(unsigned char* out128);
int mfadd_comm_create(mfadd_context* ctx, const unsigned char* id128, int rank, int nranks, mfadd_comm** out);
void mfadd_comm_free(mfadd_comm* comm);
/* A solver for the calling rank's shard; mfadd_solve()/mfadd_solve_host() then
 * run collectively on every rank.  The field argument keeps the global
 * layout, but a host field is read only in the rank's slab (the axis-0 input
 * rows its blocks touch, mfadd_shard_range's box) and a device field must
 * hold valid data there; mfadd_solve_host's out_error receives the input
 * rows the rank decoded ([in_lo, in_hi)) and out_controls the lattice rows
 * the rank owns (mfadd_shard_ctrl_rows): only the halo rows a neighbour's
 * decode reads cross NVLink, never the whole lattice.  Call
 * mfadd_solver_gather_controls (collective) when every rank needs the whole
 * lattice (mfadd_solver_controls / device_controls then hold all of it).  An asynchronous NCCL error, or no progress for
 * MFADD_NCCL_TIMEOUT_S seconds (default 600), aborts the communicator and
 * returns MFADD_ECUDA (later calls on it fail fast). */
int mfadd_solver_create_sharded(mfadd_context* ctx, const mfadd_decomposition* dec, const mfadd_solver_config* cfg,
                                mfadd_comm* comm, mfadd_solver** out);
/* Host-side shard plan: block ids [blo, bhi) and own input rows [in_lo, in_hi)
 * (the rows the rank decodes: its block rows' own inputs, or an even split of
 * the grid's rows when the ranges are finer than block rows). */
int mfadd_shard_range(const mfadd_decomposition* dec, int rank, int nranks, int* blo, int* bhi, int64_t* in_lo,
                      int64_t* in_hi);
/* The lattice rows [own_lo, own_hi) along axis 0 a rank's blocks own entries of
 * (all of them for block-row shards). */
int mfadd_shard_ctrl_rows(const mfadd_decomposition* dec, int rank, int nranks, int64_t* own_lo, int64_t* own_hi);
/* Collective over a sharded solver's communicator: every rank's owned lattice
 * rows to every rank (no-op for a one-device solver). */
int mfadd_solver_gather_controls(mfadd_solver* s);
/* The axis-0 input rows [box_lo, box_hi) a rank's solve reads (its slab: the
 * rows its blocks' fits touch and the rows it decodes). */
int mfadd_shard_box(const mfadd_decomposition* dec, int rank, int nranks, int64_t* box_lo, int64_t* box_hi);
/* Per-epoch exchange layout with one peer (recv=0: what `rank` sends, 1: what it
 * receives): entries (holder block, i0, i1, i2) in buffer order.  Returns the
 * entry count (out may be NULL), or -status on error. */
int mfadd_shard_exchange(const mfadd_decomposition* dec, int rank, int nranks, int peer, int recv, int64_t* out,
                         int64_t cap);
/* All n ranks' shard solvers in one process on the context's device, driven in
 * lockstep with device-to-device copies in place of NCCL (tests). */
int mfadd_solve_loopback(mfadd_context* ctx, const mfadd_decomposition* dec, const mfadd_solver_config* cfg,
                         int nranks, const double* field_host, double* out_controls, double* out_error,
                         mfadd_solve_summary* out, mfadd_epoch_stats* epochs, int epochs_cap, double* final_jumps4,
                         int jumps_cap);

/* ---------------------------------------------------------- fine-grained
 * Unit-parity sub-boundaries.  All buffers are HOST memory;
 * the work runs on the context's GPU. */

/* collocation_matrix(kv, params, col_lo, col_hi)   collocation.hpp:53-58
 * (find_span knots.hpp:36 + basis_funs knots.hpp:53 per row).  Outputs the
 * BandedCollocation packing: first_col, count, values (m x (p+1), clipped
 * row values left-aligned, zero padded). */
int mfadd_collocation(mfadd_context* ctx, const double* knots, int nknots, int degree, const double* params,
                      int64_t m, int64_t col_lo, int64_t col_hi, int64_t* out_first_col, int* out_count,
                      double* out_values);

/* Tensor fit_unconstrained(const LocalProblem&)     lsq.hpp:33
 * Per dim d: knots[kn_off[d]..kn_off[d+1]), params[pm_off[d]..pm_off[d+1]),
 * column window [col_lo[d], col_hi[d]); q has extents m_d (row-major);
 * out_p has extents col_hi[d]-col_lo[d]. */
int mfadd_fit_unconstrained(mfadd_context* ctx, int rank, int degree, const double* knots, const int64_t* kn_off,
                            const double* params, const int64_t* pm_off, const int64_t* col_lo,
                            const int64_t* col_hi, const double* q, double* out_p);

/* ResidualStats residual_error(const LocalProblem&, const Tensor& controls)
 *                                                   lsq.hpp:35-41, lsq.cpp:66-85
 * The local problem as in mfadd_fit_unconstrained; controls has extents
 * col_hi[d]-col_lo[d].  out_pointwise (nullable) = q - decode(controls) with the
 * window-clipped rows, bitwise equal to the reference; l2 = sqrt(sum e^2)
 * (device reduction: equal within rounding), linf = max |e|. */
int mfadd_residual_error(mfadd_context* ctx, int rank, int degree, const double* knots, const int64_t* kn_off,
                         const double* params, const int64_t* pm_off, const int64_t* col_lo, const int64_t* col_hi,
                         const double* q, const double* controls, double* out_pointwise, double* out_l2,
                         double* out_linf);

/* int find_span(const KnotVector&, double)                        knots.hpp:36
 * SpanBasis basis_funs(const KnotVector&, int span, double u)     knots.hpp:53
 * SpanBasis basis_derivs(const KnotVector&, int span, double u, int k)  knots.hpp:56
 * n evaluations on the GPU.  spans == NULL: span = find_span(u) (ERANGE for
 * u outside the evaluable range, the reference's message); else the given
 * spans (one-sided limits), which must satisfy p <= span < nknots - p - 1
 * (EINVAL).  orders = k >= 0 (EINVAL if k > p); out: n x (k+1) x (p+1)
 * values, row 0 = basis_funs, row r = the r-th derivatives (bitwise equal to
 * the reference); out_spans (nullable) receives the spans used. */
int mfadd_basis_funs(mfadd_context* ctx, const double* knots, int nknots, int degree, int64_t n, const double* u,
                     const int* spans, int orders, int* out_spans, double* out);

/* Tensor decode(controls, kvs, params, col_offset)  decode.hpp:20-22 */
int mfadd_decode(mfadd_context* ctx, int rank, int degree, const double* knots, const int64_t* kn_off,
                 const double* params, const int64_t* pm_off, const int64_t* ctrl_ext,
                 const int64_t* col_offset /* nullable */, const double* controls, double* out);

/* ------------------------------------------- MfaModel output path (§8(f))
 * eval_deriv / eval_deriv_sided (decode.hpp:28-40; MfaModel::eval /
 * eval_deriv, model.hpp:29-31) at npts points [npts][rank] on the GPU (one
 * thread per point, bitwise equal to the reference).  degrees[rank]; knots of
 * dim d at knots[kn_off[d] .. kn_off[d+1]); controls row-major with extents
 * ctrl_ext; col_offset (nullable) as in decode(); orders (nullable) the
 * derivative order per dim; side_dim < 0 evaluates unsided, else side 0 =
 * Side::Below, 1 = Side::Above along side_dim.  Errors as the reference:
 * EINVAL (order > degree), ERANGE (find_span, lattice window), for the first
 * failing point. */
#define MFADD_SIDE_BELOW 0
#define MFADD_SIDE_ABOVE 1
int mfadd_eval_points(mfadd_context* ctx, int rank, const int* degrees, const double* knots, const int64_t* kn_off,
                      const int64_t* ctrl_ext, const int64_t* col_offset, const double* controls, int64_t npts,
                      const double* points, const int* orders, int side_dim, int side, double* out);

/* std::vector<double> continuity_jumps(const MfaModel&, int dim, double u,
 * int max_order, int cross_samples)                      solver.hpp:96
 * out: max_order + 1 jumps (probe points evaluated on the GPU). */
int mfadd_continuity_jumps(mfadd_context* ctx, int rank, const int* degrees, const double* knots,
                           const int64_t* kn_off, const int64_t* ctrl_ext, const double* controls, int dim, double u,
                           int max_order, int cross_samples, double* out);

/* The pipeline's continuity probe over every interior interface of a solved
 * decomposition (pipeline.cpp:210-228 over continuity_jumps(BlockState,
 * BlockState, ...), solver.hpp:98), evaluated on the device-resident held
 * lattices of the last solve.  probe_order < 0: degree - 1.  out: probe_order
 * + 1 jumps (max over interfaces); *out_order receives the order used. */
int mfadd_solver_continuity_probe(mfadd_solver* s, int probe_order, int cross_samples, double* out, int* out_order);

/* Tensor MfaModel::decode_grid(const std::vector<int64_t>& res)   model.hpp:34
 * out: prod(res) doubles (GPU decode at u_j = j / (res - 1)). */
int mfadd_decode_grid(mfadd_context* ctx, int rank, int degree, const double* knots, const int64_t* kn_off,
                      const int64_t* ctrl_ext, const double* controls, const int64_t* res, double* out);

/* MfaModel as plain arrays (model.hpp:18-35).  Provenance is nprov key/value
 * strings, written in ascending key order (std::map).  clamp flags and
 * bounds are nullable on write (clamped, [0, 1]). */
typedef struct mfadd_model_view {
  int rank;
  const int* degrees;
  const unsigned char* clamp_left;
  const unsigned char* clamp_right;
  const double* knots;
  const int64_t* kn_off;
  const int64_t* ctrl_ext;
  const double* bounds; /* [rank][2] */
  int nprov;
  const char* const* prov_keys;
  const char* const* prov_values;
  const double* controls;
} mfadd_model_view;

typedef struct mfadd_model mfadd_model; /* a model read from disk; owns its arrays */

/* void write_mfa(const MfaModel&, const std::filesystem::path&)   model.hpp:40
 * MFDD v1 container, bit-exact with the reference writer. */
int mfadd_write_mfa(const char* path, const mfadd_model_view* model);
/* MfaModel read_mfa(const std::filesystem::path&)                 model.hpp:41 */
int mfadd_read_mfa(const char* path, mfadd_model** out);
int mfadd_model_view_of(const mfadd_model* m, mfadd_model_view* out); /* pointers owned by m */
void mfadd_model_free(mfadd_model* m);

/* Field read_raw_grid(path, dims, RawScalar, RawByteOrder)        field.hpp:48-50
 * Raw row-major grid, no header; file size must equal prod(dims) x width.
 * The bytes go to the device and are byte-swapped / widened there; out is
 * prod(dims) doubles in device memory (out_on_device) or host memory. */
#define MFADD_RAW_F32 0
#define MFADD_RAW_F64 1
#define MFADD_RAW_LITTLE 0
#define MFADD_RAW_BIG 1
int mfadd_read_raw_grid(mfadd_context* ctx, const char* path, int rank, const int64_t* dims, int type, int byte_order,
                        double* out, int out_on_device);

#ifdef __cplusplus
}
#endif
#endif /* MFADD_B200_H */
