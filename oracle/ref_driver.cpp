// oracle/ref_driver.cpp — extern "C" driver around the UNMODIFIED reference
// library (/root/reference/proj/core/src/*.cpp), compiled by oracle/Makefile
// into oracle/_ref/libmfadd_ref.so.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's reference / cpu_baseline legs may load this library, and only as
// the checker or the timed CPU baseline — never as the product path.
//
// Every entry point returns a status code and never lets a C++ exception
// escape; the codes mirror the reference's exception types:
//   0 ok, 1 std::invalid_argument, 2 std::out_of_range, 3 SingularFitError,
//   4 std::runtime_error, 5 std::logic_error, 9 anything else.
#include <cstdint>
#include <chrono>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "mfadd/collocation.hpp"
#include "mfadd/decode.hpp"
#include "mfadd/field.hpp"
#include "mfadd/knots.hpp"
#include "mfadd/layout.hpp"
#include "mfadd/lsq.hpp"
#include "mfadd/model.hpp"
#include "mfadd/runtime.hpp"
#include "mfadd/solver.hpp"

using namespace mfadd;

namespace {

thread_local std::string g_err;
thread_local int g_err_dim = -1;
thread_local std::int64_t g_err_span = -1;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const SingularFitError& e) {
    g_err = e.what();
    g_err_dim = e.dim;
    g_err_span = e.span;
    return 3;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return 5;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return 4;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

KnotVector make_kv(const double* knots, int nknots, int degree, int clamp_left, int clamp_right) {
  KnotVector kv;
  kv.degree = degree;
  kv.knots.assign(knots, knots + nknots);
  kv.clamp_left = clamp_left != 0;
  kv.clamp_right = clamp_right != 0;
  return kv;
}

struct RefDec {
  Decomposition dec;
};

struct RefResult {
  SolveResult res;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
int ref_last_error_dim(void) { return g_err_dim; }
long long ref_last_error_span(void) { return g_err_span; }

// ---- knots.hpp ----------------------------------------------------------
int ref_make_knot_vector(int degree, int basis_count, double a, double b, int clamp_left, int clamp_right,
                         double* out_knots, int cap, int* out_n) {
  return guarded([&] {
    const KnotVector kv = make_knot_vector(degree, basis_count, a, b, clamp_left != 0, clamp_right != 0);
    if (static_cast<int>(kv.knots.size()) > cap) throw std::invalid_argument("ref: knot buffer too small");
    std::memcpy(out_knots, kv.knots.data(), kv.knots.size() * sizeof(double));
    *out_n = static_cast<int>(kv.knots.size());
  });
}

int ref_find_span(const double* knots, int nknots, int degree, double u, int* out_span) {
  return guarded([&] { *out_span = find_span(make_kv(knots, nknots, degree, 1, 1), u); });
}

int ref_basis_funs(const double* knots, int nknots, int degree, int span, double u, double* out_vals) {
  return guarded([&] {
    const SpanBasis nb = basis_funs(make_kv(knots, nknots, degree, 1, 1), span, u);
    std::memcpy(out_vals, nb.values.data(), nb.values.size() * sizeof(double));
  });
}

// ---- collocation.hpp ----------------------------------------------------
// out_first_col / out_count: m entries; out_values: m*(p+1) packed like
// BandedCollocation (clipped row values left-aligned, zero padded).
int ref_collocation(const double* knots, int nknots, int degree, const double* params, long long m,
                    long long col_lo, long long col_hi, long long* out_first_col, int* out_count,
                    double* out_values) {
  return guarded([&] {
    const KnotVector kv = make_kv(knots, nknots, degree, 1, 1);
    const BandedCollocation bc =
        collocation_matrix(kv, std::span<const double>(params, static_cast<std::size_t>(m)), col_lo, col_hi);
    for (long long j = 0; j < m; ++j) {
      out_first_col[j] = bc.first_col(j);
      out_count[j] = bc.count(j);
      for (int k = 0; k <= degree; ++k)
        out_values[j * (degree + 1) + k] = (k < bc.count(j)) ? bc.row_values(j)[k] : 0.0;
    }
  });
}

// ---- lsq.hpp: fit_unconstrained / residual_error ------------------------
// Per dimension d: knots (kn_off[d]..kn_off[d+1]) in `knots`, params
// (pm_off[d]..) in `params`, column window [col_lo[d], col_hi[d]).  q has
// extents m_d = pm_off[d+1]-pm_off[d], row-major.  out_p has extents
// n_d = col_hi[d]-col_lo[d].
static LocalProblem build_problem(int rank, int degree, const double* knots, const long long* kn_off,
                                  const double* params, const long long* pm_off, const long long* col_lo,
                                  const long long* col_hi, const double* q) {
  LocalProblem prob;
  std::vector<std::int64_t> ext;
  for (int d = 0; d < rank; ++d) {
    const KnotVector kv = make_kv(knots + kn_off[d], static_cast<int>(kn_off[d + 1] - kn_off[d]), degree, 1, 1);
    const std::int64_t m = pm_off[d + 1] - pm_off[d];
    prob.r.push_back(collocation_matrix(kv, std::span<const double>(params + pm_off[d], static_cast<std::size_t>(m)),
                                        col_lo[d], col_hi[d]));
    ext.push_back(m);
  }
  prob.q = Tensor(ext);
  std::memcpy(prob.q.data(), q, static_cast<std::size_t>(prob.q.size()) * sizeof(double));
  return prob;
}

int ref_fit_unconstrained(int rank, int degree, const double* knots, const long long* kn_off, const double* params,
                          const long long* pm_off, const long long* col_lo, const long long* col_hi, const double* q,
                          double* out_p) {
  return guarded([&] {
    const LocalProblem prob = build_problem(rank, degree, knots, kn_off, params, pm_off, col_lo, col_hi, q);
    const Tensor p = fit_unconstrained(prob);
    std::memcpy(out_p, p.data(), static_cast<std::size_t>(p.size()) * sizeof(double));
  });
}

int ref_residual_error(int rank, int degree, const double* knots, const long long* kn_off, const double* params,
                       const long long* pm_off, const long long* col_lo, const long long* col_hi, const double* q,
                       const double* p, double* out_l2, double* out_linf, double* out_pointwise) {
  return guarded([&] {
    const LocalProblem prob = build_problem(rank, degree, knots, kn_off, params, pm_off, col_lo, col_hi, q);
    std::vector<std::int64_t> ext;
    for (int d = 0; d < rank; ++d) ext.push_back(col_hi[d] - col_lo[d]);
    Tensor pt(ext);
    std::memcpy(pt.data(), p, static_cast<std::size_t>(pt.size()) * sizeof(double));
    const ResidualStats r = residual_error(prob, pt);
    *out_l2 = r.l2;
    *out_linf = r.linf;
    if (out_pointwise)
      std::memcpy(out_pointwise, r.pointwise.data(), static_cast<std::size_t>(r.pointwise.size()) * sizeof(double));
  });
}

// ---- decode.hpp ---------------------------------------------------------
// controls extents ctrl_ext[d]; col_offset may be NULL.
int ref_decode(int rank, int degree, const double* knots, const long long* kn_off, const double* params,
               const long long* pm_off, const long long* ctrl_ext, const long long* col_offset,
               const double* controls, double* out) {
  return guarded([&] {
    std::vector<KnotVector> kvs;
    std::vector<std::vector<double>> ps;
    std::vector<std::int64_t> ext, off;
    for (int d = 0; d < rank; ++d) {
      kvs.push_back(make_kv(knots + kn_off[d], static_cast<int>(kn_off[d + 1] - kn_off[d]), degree, 1, 1));
      ps.emplace_back(params + pm_off[d], params + pm_off[d + 1]);
      ext.push_back(ctrl_ext[d]);
      if (col_offset) off.push_back(col_offset[d]);
    }
    Tensor c(ext);
    std::memcpy(c.data(), controls, static_cast<std::size_t>(c.size()) * sizeof(double));
    const Tensor outt = decode(c, kvs, ps, off);
    std::memcpy(out, outt.data(), static_cast<std::size_t>(outt.size()) * sizeof(double));
  });
}

// ---- field.hpp: reference generators (used only to re-express tests) ----
int ref_gen_field(const char* generator, int rank, const long long* npts, double* out_values) {
  return guarded([&] {
    std::vector<std::int64_t> n(npts, npts + rank);
    const Field f = make_field(generator, n);
    std::memcpy(out_values, f.values.data(), static_cast<std::size_t>(f.values.size()) * sizeof(double));
  });
}

// ---- layout.hpp: partition ----------------------------------------------
int ref_partition(int rank, const long long* grid_dims, const double* bounds, const int* blocks_per_dim, int degree,
                  const long long* nctrl_per_block, long long overlap, int clamp_interfaces, void** out_handle) {
  return guarded([&] {
    std::vector<std::int64_t> g(grid_dims, grid_dims + rank), nc(nctrl_per_block, nctrl_per_block + rank);
    std::vector<std::array<double, 2>> b;
    for (int d = 0; d < rank; ++d) b.push_back({bounds ? bounds[2 * d] : 0.0, bounds ? bounds[2 * d + 1] : 1.0});
    std::vector<int> bp(blocks_per_dim, blocks_per_dim + rank);
    auto h = std::make_unique<RefDec>();
    h->dec = partition(g, b, bp, degree, nc, overlap, clamp_interfaces != 0);
    *out_handle = h.release();
  });
}

void ref_dec_free(void* h) { delete static_cast<RefDec*>(h); }

int ref_dec_nblocks(void* h) { return static_cast<int>(static_cast<RefDec*>(h)->dec.blocks.size()); }

int ref_dec_rank(void* h) { return static_cast<RefDec*>(h)->dec.global.rank(); }

// 16 int64 per (block, dim): span_lo, span_hi, delta_lo, delta_hi,
// overlap_lo, overlap_hi, local_span_lo, local_span_hi, dof_lo, dof_hi,
// own_lo, own_hi, input_lo, input_hi, own_input_lo, own_input_hi.
void ref_dec_blockdims(void* h, long long* out) {
  const Decomposition& dec = static_cast<RefDec*>(h)->dec;
  std::size_t o = 0;
  for (const BlockLayout& blk : dec.blocks)
    for (const BlockDim& bd : blk.dims) {
      const std::int64_t v[16] = {bd.span_lo,       bd.span_hi,       bd.delta_lo,   bd.delta_hi,
                                  bd.overlap_lo,    bd.overlap_hi,    bd.local_span_lo, bd.local_span_hi,
                                  bd.dof_lo,        bd.dof_hi,        bd.own_lo,     bd.own_hi,
                                  bd.input_lo,      bd.input_hi,      bd.own_input_lo, bd.own_input_hi};
      for (int k = 0; k < 16; ++k) out[o++] = v[k];
    }
}

void ref_dec_coords(void* h, int* out) {
  const Decomposition& dec = static_cast<RefDec*>(h)->dec;
  std::size_t o = 0;
  for (const BlockLayout& blk : dec.blocks)
    for (int c : blk.coords) out[o++] = c;
}

int ref_dec_neighbors(void* h, int block, int* out, int cap) {
  const auto& nb = static_cast<RefDec*>(h)->dec.blocks[static_cast<std::size_t>(block)].neighbors;
  for (std::size_t i = 0; i < nb.size() && static_cast<int>(i) < cap; ++i) out[i] = nb[i];
  return static_cast<int>(nb.size());
}

void ref_dec_nctrl(void* h, long long* out) {
  const auto& g = static_cast<RefDec*>(h)->dec.global;
  for (int d = 0; d < g.rank(); ++d) out[d] = g.n_ctrl[static_cast<std::size_t>(d)];
}

int ref_dec_knots(void* h, int dim, double* out, int cap) {
  const auto& kv = static_cast<RefDec*>(h)->dec.global.kvs[static_cast<std::size_t>(dim)];
  for (std::size_t i = 0; i < kv.knots.size() && static_cast<int>(i) < cap; ++i) out[i] = kv.knots[i];
  return static_cast<int>(kv.knots.size());
}

// holder_span pairs for every control index along dim: out[2*i], out[2*i+1].
void ref_dec_holder_ranges(void* h, int dim, int* out) {
  const Decomposition& dec = static_cast<RefDec*>(h)->dec;
  const std::int64_t n = dec.global.n_ctrl[static_cast<std::size_t>(dim)];
  for (std::int64_t i = 0; i < n; ++i) {
    const auto r = dec.shared.holder_span(dim, i);
    out[2 * i] = r.first;
    out[2 * i + 1] = r.second;
  }
}

int ref_dec_n_s(void* h, const long long* dof) {
  const Decomposition& dec = static_cast<RefDec*>(h)->dec;
  std::vector<std::int64_t> d(dof, dof + dec.global.rank());
  return dec.shared.n_s(d);
}

int ref_dec_holders(void* h, const long long* dof, int* out, int cap) {
  const Decomposition& dec = static_cast<RefDec*>(h)->dec;
  std::vector<std::int64_t> d(dof, dof + dec.global.rank());
  const auto ids = dec.shared.holders(d);
  for (std::size_t i = 0; i < ids.size() && static_cast<int>(i) < cap; ++i) out[i] = ids[i];
  return static_cast<int>(ids.size());
}

void ref_dec_exchange_volume(void* h, long long* out) {
  const auto v = exchange_volume(static_cast<RefDec*>(h)->dec);
  for (std::size_t i = 0; i < v.size(); ++i) out[i] = v[i];
}

double ref_dec_compression_ratio(void* h) { return compression_ratio(static_cast<RefDec*>(h)->dec.global); }

int ref_dec_any_shared(void* h) { return static_cast<RefDec*>(h)->dec.shared.any_shared() ? 1 : 0; }

// ---- solver.hpp: solve --------------------------------------------------
static double g_last_solve_s = 0.0;

int ref_solve(void* dec_handle, const double* field_values, const double* bounds, int max_outer_iterations,
              double tolerance, int workers, int log_errors, int enforce_continuity, void** out_result) {
  return guarded([&] {
    const Decomposition& dec = static_cast<RefDec*>(dec_handle)->dec;
    Field f;
    f.dims = dec.global.n_input;
    for (int d = 0; d < dec.global.rank(); ++d)
      f.bounds.push_back({bounds ? bounds[2 * d] : 0.0, bounds ? bounds[2 * d + 1] : 1.0});
    f.values = Tensor(f.dims);
    std::memcpy(f.values.data(), field_values, static_cast<std::size_t>(f.values.size()) * sizeof(double));
    SolverConfig cfg;
    cfg.max_outer_iterations = max_outer_iterations;
    cfg.tolerance = tolerance;
    cfg.workers = workers;
    cfg.log_errors = log_errors != 0;
    cfg.enforce_continuity = enforce_continuity != 0;
    auto r = std::make_unique<RefResult>();
    // the timed region is mfadd::solve() only (the Field
    // build above and the result copies afterwards are outside it)
    const auto t0 = std::chrono::steady_clock::now();
    r->res = solve(f, dec, cfg);
    g_last_solve_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out_result = r.release();
  });
}

// Wall seconds of the last ref_solve's solve() call (steady_clock).
double ref_last_solve_seconds(void) { return g_last_solve_s; }

void ref_result_free(void* h) { delete static_cast<RefResult*>(h); }

// scalars: converged, constraint_iterations, n_epochs, n_final_jumps;
// doubles: final_dp, global_l2, global_linf, t_setup, t_local, t_exchange,
// t_constraint, t_decode.
void ref_result_scalars(void* h, int* ints4, double* dbl8) {
  const SolveResult& r = static_cast<RefResult*>(h)->res;
  ints4[0] = r.converged ? 1 : 0;
  ints4[1] = r.constraint_iterations;
  ints4[2] = static_cast<int>(r.epochs.size());
  ints4[3] = static_cast<int>(r.final_jumps.size());
  dbl8[0] = r.final_dp;
  dbl8[1] = r.global_l2;
  dbl8[2] = r.global_linf;
  dbl8[3] = r.timings.setup;
  dbl8[4] = r.timings.local_solve;
  dbl8[5] = r.timings.exchange;
  dbl8[6] = r.timings.constraint;
  dbl8[7] = r.timings.decode;
}

// per epoch: iteration, dp_max, jump_ss, jump_ms  (4 doubles)
void ref_result_epochs(void* h, double* out) {
  const SolveResult& r = static_cast<RefResult*>(h)->res;
  for (std::size_t e = 0; e < r.epochs.size(); ++e) {
    out[4 * e + 0] = r.epochs[e].iteration;
    out[4 * e + 1] = r.epochs[e].dp_max;
    out[4 * e + 2] = r.epochs[e].jump_ss;
    out[4 * e + 3] = r.epochs[e].jump_ms;
  }
}

// per epoch per block {l2, linf} when log_errors (nblocks*2 doubles per epoch)
int ref_result_block_errors(void* h, int epoch, double* out) {
  const SolveResult& r = static_cast<RefResult*>(h)->res;
  const auto& be = r.epochs[static_cast<std::size_t>(epoch)].block_errors;
  for (std::size_t b = 0; b < be.size(); ++b) {
    out[2 * b] = be[b][0];
    out[2 * b + 1] = be[b][1];
  }
  return static_cast<int>(be.size());
}

// per final jump: block_a, block_b, linf_ss, linf_ms
void ref_result_final_jumps(void* h, double* out) {
  const SolveResult& r = static_cast<RefResult*>(h)->res;
  for (std::size_t i = 0; i < r.final_jumps.size(); ++i) {
    out[4 * i + 0] = r.final_jumps[i].block_a;
    out[4 * i + 1] = r.final_jumps[i].block_b;
    out[4 * i + 2] = r.final_jumps[i].linf_ss;
    out[4 * i + 3] = r.final_jumps[i].linf_ms;
  }
}

void ref_result_controls(void* h, double* out) {
  const Tensor& t = static_cast<RefResult*>(h)->res.model.controls;
  std::memcpy(out, t.data(), static_cast<std::size_t>(t.size()) * sizeof(double));
}

void ref_result_error(void* h, double* out) {
  const Tensor& t = static_cast<RefResult*>(h)->res.global_error;
  std::memcpy(out, t.data(), static_cast<std::size_t>(t.size()) * sizeof(double));
}

long long ref_result_block_size(void* h, int block) {
  return static_cast<RefResult*>(h)->res.blocks[static_cast<std::size_t>(block)].p.size();
}

void ref_result_block_p(void* h, int block, double* out) {
  const Tensor& t = static_cast<RefResult*>(h)->res.blocks[static_cast<std::size_t>(block)].p;
  std::memcpy(out, t.data(), static_cast<std::size_t>(t.size()) * sizeof(double));
}

// ---- model.hpp / decode.hpp: §8(f) rows (MfaModel output path, probe) ----
namespace {
// A model from flat arrays: per-dim degree and clamp flags, knots of dim d at
// knots[kn_off[d] .. kn_off[d+1]), bounds [rank][2] (NULL: [0,1]).
MfaModel make_model(int rank, const int* degrees, const int* clamp_l, const int* clamp_r, const double* knots,
                    const long long* kn_off, const long long* ctrl_ext, const double* bounds, const double* controls) {
  MfaModel m;
  std::vector<std::int64_t> ext;
  for (int d = 0; d < rank; ++d) {
    m.degrees.push_back(degrees[d]);
    m.kvs.push_back(make_kv(knots + kn_off[d], static_cast<int>(kn_off[d + 1] - kn_off[d]), degrees[d],
                            clamp_l ? clamp_l[d] : 1, clamp_r ? clamp_r[d] : 1));
    m.bounds.push_back({bounds ? bounds[2 * d] : 0.0, bounds ? bounds[2 * d + 1] : 1.0});
    ext.push_back(ctrl_ext[d]);
  }
  m.controls = Tensor(ext);
  std::memcpy(m.controls.data(), controls, static_cast<std::size_t>(m.controls.size()) * sizeof(double));
  return m;
}
}  // namespace

// eval_deriv / eval_deriv_sided (decode.hpp:28-40) at npts points [npts][rank];
// orders may be NULL (values); side_dim < 0: unsided; side 0 Below, 1 Above.
int ref_eval_points(int rank, const int* degrees, const double* knots, const long long* kn_off,
                    const long long* ctrl_ext, const long long* col_offset, const double* controls, long long npts,
                    const double* points, const int* orders, int side_dim, int side, double* out) {
  return guarded([&] {
    const MfaModel m = make_model(rank, degrees, nullptr, nullptr, knots, kn_off, ctrl_ext, nullptr, controls);
    std::vector<std::int64_t> off;
    if (col_offset)
      for (int d = 0; d < rank; ++d) off.push_back(col_offset[d]);
    std::vector<int> ord;
    if (orders)
      for (int d = 0; d < rank; ++d) ord.push_back(orders[d]);
    for (long long i = 0; i < npts; ++i) {
      std::span<const double> pt(points + i * rank, static_cast<std::size_t>(rank));
      out[i] = side_dim < 0 ? eval_deriv(m.controls, m.kvs, pt, ord, off)
                            : eval_deriv_sided(m.controls, m.kvs, pt, ord, side_dim, side ? Side::Above : Side::Below, off);
    }
  });
}

// MfaModel::decode_grid (model.cpp:39-49)
int ref_decode_grid(int rank, const int* degrees, const double* knots, const long long* kn_off,
                    const long long* ctrl_ext, const double* controls, const long long* res, double* out) {
  return guarded([&] {
    const MfaModel m = make_model(rank, degrees, nullptr, nullptr, knots, kn_off, ctrl_ext, nullptr, controls);
    const Tensor t = m.decode_grid(std::vector<std::int64_t>(res, res + rank));
    std::memcpy(out, t.data(), static_cast<std::size_t>(t.size()) * sizeof(double));
  });
}

// write_mfa (model.cpp:93-118); provenance as nprov key/value C strings.
int ref_write_mfa(const char* path, int rank, const int* degrees, const int* clamp_l, const int* clamp_r,
                  const double* knots, const long long* kn_off, const long long* ctrl_ext, const double* bounds,
                  int nprov, const char* const* keys, const char* const* values, const double* controls) {
  return guarded([&] {
    MfaModel m = make_model(rank, degrees, clamp_l, clamp_r, knots, kn_off, ctrl_ext, bounds, controls);
    for (int i = 0; i < nprov; ++i) m.provenance[keys[i]] = values[i];
    write_mfa(m, path);
  });
}

// read_mfa (model.cpp:120-167): status only (used for the error-path checks)
int ref_read_mfa_check(const char* path) {
  return guarded([&] { (void)read_mfa(path); });
}

// read_raw_grid (field.cpp:149-191): type 0 f32 / 1 f64, order 0 little / 1 big
int ref_read_raw_grid(const char* path, int rank, const long long* dims, int type, int order, double* out) {
  return guarded([&] {
    const Field f = read_raw_grid(path, std::vector<std::int64_t>(dims, dims + rank),
                                  type ? RawScalar::Float64 : RawScalar::Float32,
                                  order ? RawByteOrder::Big : RawByteOrder::Little, {});
    std::memcpy(out, f.values.data(), static_cast<std::size_t>(f.values.size()) * sizeof(double));
  });
}

// continuity_jumps on an assembled model (solver.hpp:96)
int ref_continuity_jumps_model(int rank, const int* degrees, const double* knots, const long long* kn_off,
                               const long long* ctrl_ext, const double* controls, int dim, double u, int max_order,
                               int cross_samples, double* out) {
  return guarded([&] {
    const MfaModel m = make_model(rank, degrees, nullptr, nullptr, knots, kn_off, ctrl_ext, nullptr, controls);
    const auto j = continuity_jumps(m, dim, u, max_order, cross_samples);
    std::memcpy(out, j.data(), j.size() * sizeof(double));
  });
}

// continuity_jumps between two solved blocks (solver.hpp:98), as used by the
// pipeline's probe (pipeline.cpp:210-228)
int ref_continuity_jumps_blocks(void* dec_handle, void* result, int below, int above, int dim, double u,
                                int max_order, int cross_samples, double* out) {
  return guarded([&] {
    const Decomposition& dec = static_cast<RefDec*>(dec_handle)->dec;
    const SolveResult& r = static_cast<RefResult*>(result)->res;
    const auto j = continuity_jumps(r.blocks[static_cast<std::size_t>(below)], r.blocks[static_cast<std::size_t>(above)],
                                    dec, dim, u, max_order, cross_samples);
    std::memcpy(out, j.data(), j.size() * sizeof(double));
  });
}

// GlobalLayout::span_param (layout.cpp:22-27)
double ref_dec_span_param(void* h, int dim, long long t) { return static_cast<RefDec*>(h)->dec.global.span_param(dim, t); }

}  // extern "C"
