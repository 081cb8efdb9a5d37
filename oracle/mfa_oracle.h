/* oracle/mfa_oracle.h — plain-C restatement of the reference's domain-
 * decomposed MFA encode path (proj/core/src/{knots,collocation,lsq,decode,
 * layout,solver}.cpp).
 *
 * TEST INFRASTRUCTURE ONLY: the checker for the CUDA product path.  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * liboracle.so.  Parity of this restatement is pinned against the reference
 * itself (oracle/_ref, built from the unmodified sources) and against the
 * committed golden fixtures in tests/golden/.
 *
 * Status codes (mirror the reference exception types):
 *   0 ok, 1 invalid_argument, 2 out_of_range, 3 SingularFitError,
 *   4 runtime_error.
 */
#ifndef MFA_ORACLE_H
#define MFA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

const char* orc_last_error(void);
int orc_last_error_dim(void);
int64_t orc_last_error_span(void);

/* knots.cpp:48-81 */
int orc_make_knot_vector(int degree, int basis_count, double a, double b, int clamp_left, int clamp_right,
                         double* out_knots /* basis_count+degree+1 */);
/* knots.cpp:83-106 */
int orc_find_span(const double* knots, int nknots, int degree, double u, int* out_span);
/* knots.cpp:108-129 */
void orc_basis_funs(const double* knots, int degree, int span, double u, double* out_vals /* p+1 */);
/* collocation.cpp:83-111 */
int orc_collocation(const double* knots, int nknots, int degree, const double* params, int64_t m, int64_t col_lo,
                    int64_t col_hi, int64_t* out_first_col, int* out_count, double* out_values /* m*(p+1) */);
/* lsq.cpp:39-64 (per-dimension knots/params packed with offsets) */
int orc_fit_unconstrained(int rank, int degree, const double* knots, const int64_t* kn_off, const double* params,
                          const int64_t* pm_off, const int64_t* col_lo, const int64_t* col_hi, const double* q,
                          double* out_p);
/* decode.cpp:83-97 */
int orc_decode(int rank, int degree, const double* knots, const int64_t* kn_off, const double* params,
               const int64_t* pm_off, const int64_t* ctrl_ext, const int64_t* col_offset /* nullable */,
               const double* controls, double* out);

/* layout.cpp:217-342 */
typedef struct orc_dec orc_dec;
int orc_partition(int rank, const int64_t* grid_dims, const int* blocks_per_dim, int degree,
                  const int64_t* nctrl_per_block, int64_t overlap, int clamp_interfaces, orc_dec** out);
void orc_dec_free(orc_dec* d);
int orc_dec_nblocks(const orc_dec* d);
/* 16 int64 per (block, dim), same field order as ref_dec_blockdims */
void orc_dec_blockdims(const orc_dec* d, int64_t* out);
void orc_dec_coords(const orc_dec* d, int* out);
void orc_dec_nctrl(const orc_dec* d, int64_t* out);
int orc_dec_knots(const orc_dec* d, int dim, double* out /* nullable: returns count */);
void orc_dec_holder_ranges(const orc_dec* d, int dim, int* out /* 2*n_ctrl */);
int orc_dec_neighbors(const orc_dec* d, int block, int* out, int cap);

/* solver.cpp:332-440 */
typedef struct orc_result orc_result;
int orc_solve(const orc_dec* d, const double* field, int max_outer_iterations, double tolerance, int log_errors,
              int enforce_continuity, orc_result** out);
void orc_result_free(orc_result* r);
/* ints: converged, constraint_iterations, n_epochs, n_final_jumps;
 * dbl: final_dp, global_l2, global_linf */
void orc_result_scalars(const orc_result* r, int* ints4, double* dbl3);
void orc_result_epochs(const orc_result* r, double* out /* 4 per epoch */);
void orc_result_block_errors(const orc_result* r, int epoch, double* out /* 2 per block */);
void orc_result_final_jumps(const orc_result* r, double* out /* 4 per jump */);
void orc_result_controls(const orc_result* r, double* out);
void orc_result_error(const orc_result* r, double* out);
void orc_result_block_p(const orc_result* r, int block, double* out);

#ifdef __cplusplus
}
#endif
#endif
