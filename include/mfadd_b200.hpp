// include/mfadd_b200.hpp — C++ drop-in shim over the C ABI (mfadd_b200.h).
//
// Re-states the reference's `mfadd::core` encode API (proj/core/include/mfadd/)
// with the same type names, member names, defaults and exception types, so a
// caller of the reference (pipeline.cpp:195 `solve(field, dec, config)`, the
// doctest suites) switches by including this header and linking
// libmfadd_b200.so instead of mfadd_core:
//
//     #include "mfadd_b200.hpp"
//     namespace mfadd = mfadd_b200;   // the one-line switch
//
// Header-only, C++17.  Value semantics like the reference: Tensor owns a
// std::vector<double>, row-major, last dim fastest (tensor.hpp:10-73).  Every
// status code of the ABI is rethrown as the reference's exception type
// (SURVEY.md §8b): invalid_argument / out_of_range / SingularFitError /
// runtime_error / logic_error.  The GPU work runs on a per-thread default
// context (device 0) unless a Context is passed explicitly.
#ifndef MFADD_B200_HPP
#define MFADD_B200_HPP

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mfadd_b200.h"

namespace mfadd_b200 {

// ------------------------------------------------------------------ errors
// SingularFitError (lsq.hpp:24-28)
struct SingularFitError : std::runtime_error {
  int dim;
  std::int64_t span;
  SingularFitError(int dim_, std::int64_t span_, const std::string& what)
      : std::runtime_error(what), dim(dim_), span(span_) {}
};

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

inline void check(int status) {
  if (status == MFADD_OK) return;
  const std::string msg = mfadd_last_error();
  switch (status) {
    case MFADD_EINVAL: throw std::invalid_argument(msg);
    case MFADD_ERANGE: throw std::out_of_range(msg);
    case MFADD_ESINGULAR: throw SingularFitError(mfadd_last_error_dim(), mfadd_last_error_span(), msg);
    case MFADD_ERUNTIME: throw std::runtime_error(msg);
    case MFADD_ELOGIC: throw std::logic_error(msg);
    case MFADD_ENOMEM: throw std::bad_alloc();
    default: throw CudaError(msg);
  }
}

// ------------------------------------------------------------------ tensor
// Tensor (tensor.hpp:10-73): extents + row-major values.
class Tensor {
 public:
  Tensor() = default;
  explicit Tensor(std::vector<std::int64_t> extents)
      : extents_(std::move(extents)), data_(static_cast<std::size_t>(count(extents_)), 0.0) {}
  Tensor(std::vector<std::int64_t> extents, std::vector<double> data)
      : extents_(std::move(extents)), data_(std::move(data)) {
    if (static_cast<std::int64_t>(data_.size()) != count(extents_))
      throw std::invalid_argument("Tensor: data size does not match extents");
  }
  int rank() const { return static_cast<int>(extents_.size()); }
  const std::vector<std::int64_t>& extents() const { return extents_; }
  std::int64_t extent(int d) const { return extents_[static_cast<std::size_t>(d)]; }
  std::int64_t size() const { return static_cast<std::int64_t>(data_.size()); }
  double* data() { return data_.data(); }
  const double* data() const { return data_.data(); }
  std::vector<double>& values() { return data_; }
  const std::vector<double>& values() const { return data_; }
  double& operator[](std::int64_t i) { return data_[static_cast<std::size_t>(i)]; }
  double operator[](std::int64_t i) const { return data_[static_cast<std::size_t>(i)]; }

  static std::int64_t count(const std::vector<std::int64_t>& e) {
    std::int64_t n = 1;
    for (const auto v : e) n *= v;
    return n;
  }

 private:
  std::vector<std::int64_t> extents_;
  std::vector<double> data_;
};

// ----------------------------------------------------------------- context
// One CUDA device + stream (no reference analogue: the reference's thread
// pool, SolverConfig::workers, is replaced by the GPU).
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr) {
    mfadd_context* c = nullptr;
    check(mfadd_context_create(device, stream, &c));
    h_.reset(c);
  }
  mfadd_context* get() const { return h_.get(); }
  std::int64_t launch_count() const { return mfadd_context_launch_count(h_.get()); }

 private:
  struct Del {
    void operator()(mfadd_context* c) const { mfadd_context_free(c); }
  };
  std::unique_ptr<mfadd_context, Del> h_;
};

inline Context& default_context() {
  thread_local Context ctx(0);
  return ctx;
}

// ------------------------------------------------------------------ layout
// KnotVector (knots.hpp:11-29); the encode path only uses clamped knots.
struct KnotVector {
  int degree = 0;
  std::vector<double> knots;
  bool clamp_left = true;
  bool clamp_right = true;
  int basis_count() const { return static_cast<int>(knots.size()) - degree - 1; }
  double domain_min() const { return knots[static_cast<std::size_t>(degree)]; }
  double domain_max() const { return knots[static_cast<std::size_t>(basis_count())]; }
};

// BlockDim (layout.hpp:47-57), same members and order.
struct BlockDim {
  std::int64_t span_lo = 0, span_hi = 0;
  std::int64_t delta_lo = 0, delta_hi = 0;
  std::int64_t overlap_lo = 0, overlap_hi = 0;
  std::int64_t local_span_lo = 0, local_span_hi = 0;
  std::int64_t dof_lo = 0, dof_hi = 0;
  std::int64_t own_lo = 0, own_hi = 0;
  std::int64_t input_lo = 0, input_hi = 0;
  std::int64_t own_input_lo = 0, own_input_hi = 0;
};

// BlockLayout (layout.hpp:59-66)
struct BlockLayout {
  int id = 0;
  std::vector<int> coords;
  std::vector<BlockDim> dims;
  std::vector<int> neighbors;
};

// Decomposition (layout.hpp:98-105) as a handle plus the reference's
// metadata views (global knots/extents, per-block layouts, holder ranges).
class Decomposition {
 public:
  Decomposition() = default;
  explicit Decomposition(mfadd_decomposition* h) : h_(h, &mfadd_decomposition_free) { load(); }
  const mfadd_decomposition* get() const { return h_.get(); }
  int rank() const { return rank_; }
  std::int64_t block_count() const { return static_cast<std::int64_t>(blocks.size()); }
  double compression_ratio() const { return mfadd_dec_compression_ratio(h_.get()); }
  bool any_shared() const { return mfadd_dec_any_shared(h_.get()) != 0; }
  // SharedDofMap::holder_span(dim, i) (layout.hpp:74-76)
  std::pair<int, int> holder_span(int dim, std::int64_t i) const {
    const auto& r = holder_ranges_[static_cast<std::size_t>(dim)];
    return {r[static_cast<std::size_t>(2 * i)], r[static_cast<std::size_t>(2 * i + 1)]};
  }
  // exchange_volume (runtime.hpp) per block
  std::vector<std::int64_t> exchange_volume() const {
    std::vector<std::int64_t> v(blocks.size());
    mfadd_dec_exchange_volume(h_.get(), v.data());
    return v;
  }

  std::vector<KnotVector> kvs;          // GlobalLayout::kvs
  std::vector<std::int64_t> n_ctrl;     // GlobalLayout::n_ctrl
  std::vector<std::int64_t> n_input;    // GlobalLayout::n_input (field extents)
  std::vector<BlockLayout> blocks;      // Decomposition::blocks

 private:
  void load() {
    const mfadd_decomposition* d = h_.get();
    rank_ = mfadd_dec_rank(d);
    const int nb = mfadd_dec_block_count(d);
    n_ctrl.assign(static_cast<std::size_t>(rank_), 0);
    mfadd_dec_nctrl(d, n_ctrl.data());
    n_input.assign(static_cast<std::size_t>(rank_), 0);
    mfadd_dec_grid_dims(d, n_input.data());
    int degree = 0;
    for (int k = 0; k < rank_; ++k) {
      KnotVector kv;
      kv.knots.resize(static_cast<std::size_t>(mfadd_dec_knots(d, k, nullptr)));
      mfadd_dec_knots(d, k, kv.knots.data());
      kvs.push_back(std::move(kv));
    }
    std::vector<std::int64_t> bd(static_cast<std::size_t>(nb) * rank_ * 16);
    mfadd_dec_block_dims(d, bd.data());
    std::vector<int> coords(static_cast<std::size_t>(nb) * rank_);
    mfadd_dec_coords(d, coords.data());
    blocks.resize(static_cast<std::size_t>(nb));
    for (int b = 0; b < nb; ++b) {
      BlockLayout& bl = blocks[static_cast<std::size_t>(b)];
      bl.id = b;
      for (int k = 0; k < rank_; ++k) {
        bl.coords.push_back(coords[static_cast<std::size_t>(b * rank_ + k)]);
        const std::int64_t* f = bd.data() + (static_cast<std::size_t>(b) * rank_ + k) * 16;
        bl.dims.push_back(BlockDim{f[0], f[1], f[2], f[3], f[4], f[5], f[6], f[7], f[8], f[9], f[10], f[11], f[12],
                                   f[13], f[14], f[15]});
      }
      std::vector<int> nbr(static_cast<std::size_t>(nb));
      const int nn = mfadd_dec_neighbors(d, b, nbr.data(), nb);
      bl.neighbors.assign(nbr.begin(), nbr.begin() + nn);
    }
    // degree = (#knots - n_ctrl - 1): the clamped global knot vector
    if (rank_ > 0) degree = static_cast<int>(kvs[0].knots.size() - static_cast<std::size_t>(n_ctrl[0]) - 1);
    for (auto& kv : kvs) kv.degree = degree;
    holder_ranges_.resize(static_cast<std::size_t>(rank_));
    for (int k = 0; k < rank_; ++k) {
      holder_ranges_[static_cast<std::size_t>(k)].resize(static_cast<std::size_t>(2 * n_ctrl[static_cast<std::size_t>(k)]));
      mfadd_dec_holder_ranges(d, k, holder_ranges_[static_cast<std::size_t>(k)].data());
    }
  }
  std::shared_ptr<mfadd_decomposition> h_;
  int rank_ = 0;
  std::vector<std::vector<int>> holder_ranges_;
};

// partition (layout.hpp:107-111); bounds enter only the coordinate map.
inline Decomposition partition(const std::vector<std::int64_t>& grid_dims,
                               const std::vector<std::array<double, 2>>& bounds,
                               const std::vector<int>& blocks_per_dim, int degree,
                               const std::vector<std::int64_t>& nctrl_per_block, std::int64_t overlap,
                               bool clamp_interfaces) {
  const int rank = static_cast<int>(grid_dims.size());
  if (blocks_per_dim.size() != grid_dims.size() || nctrl_per_block.size() != grid_dims.size())
    throw std::invalid_argument("partition: rank mismatch");
  std::vector<double> b;
  for (const auto& x : bounds) {
    b.push_back(x[0]);
    b.push_back(x[1]);
  }
  mfadd_decomposition* h = nullptr;
  check(mfadd_partition(rank, grid_dims.data(), bounds.empty() ? nullptr : b.data(), blocks_per_dim.data(), degree,
                        nctrl_per_block.data(), overlap, clamp_interfaces ? 1 : 0, &h));
  return Decomposition(h);
}

// ------------------------------------------------------------------- field
// Field (field.hpp:14-24)
struct Field {
  std::vector<std::int64_t> dims;
  std::vector<std::array<double, 2>> bounds;
  Tensor values;
  std::string name;
  int rank() const { return static_cast<int>(dims.size()); }
};

// read_raw_grid (field.hpp:43-50): the bytes are converted on the GPU
enum class RawScalar { Float32, Float64 };
enum class RawByteOrder { Little, Big };
inline Field read_raw_grid(const std::string& path, const std::vector<std::int64_t>& dims, RawScalar type,
                           RawByteOrder order = RawByteOrder::Little,
                           const std::vector<std::array<double, 2>>& bounds = {}, Context& ctx = default_context()) {
  Field f;
  f.dims = dims;
  f.bounds = bounds.empty() ? std::vector<std::array<double, 2>>(dims.size(), {0.0, 1.0}) : bounds;
  if (f.bounds.size() != dims.size()) throw std::invalid_argument("read_raw_grid: bounds/dims mismatch");
  f.values = Tensor(dims);
  check(mfadd_read_raw_grid(ctx.get(), path.c_str(), static_cast<int>(dims.size()), dims.data(),
                            type == RawScalar::Float32 ? MFADD_RAW_F32 : MFADD_RAW_F64,
                            order == RawByteOrder::Big ? MFADD_RAW_BIG : MFADD_RAW_LITTLE, f.values.data(), 0));
  const auto slash = path.find_last_of('/');
  f.name = slash == std::string::npos ? path : path.substr(slash + 1);
  return f;
}

// ------------------------------------------------------------------- solve
// SolverConfig (solver.hpp:16-22), same defaults.
struct SolverConfig {
  int max_outer_iterations = 10;
  double tolerance = 1e-10;
  int workers = 1;
  bool log_errors = true;
  bool enforce_continuity = true;
};

// InterfaceJump / EpochStats / PhaseTimings (solver.hpp:34-54)
struct InterfaceJump {
  int block_a = -1, block_b = -1;
  double linf_ss = 0.0;
  double linf_ms = 0.0;
};
struct EpochStats {
  int iteration = 0;
  double dp_max = 0.0;
  double jump_ss = 0.0;
  double jump_ms = 0.0;
  std::vector<std::array<double, 2>> block_errors;
};
struct PhaseTimings {
  double setup = 0.0, local_solve = 0.0, exchange = 0.0, constraint = 0.0, decode = 0.0;
};

// decode.hpp:24
enum class Side { Below, Above };

namespace detail {
inline void pack_knots(const std::vector<KnotVector>& kvs, std::vector<double>& kn, std::vector<std::int64_t>& ko,
                       std::vector<int>& deg) {
  ko.assign(1, 0);
  for (const auto& kv : kvs) {
    kn.insert(kn.end(), kv.knots.begin(), kv.knots.end());
    ko.push_back(static_cast<std::int64_t>(kn.size()));
    deg.push_back(kv.degree);
  }
}
}  // namespace detail

// eval_deriv_sided (decode.hpp:35-38); side_dim < 0: eval_deriv (decode.hpp:28-30)
inline double eval_deriv_sided(const Tensor& controls, const std::vector<KnotVector>& kvs,
                               const std::vector<double>& point, const std::vector<int>& orders, int side_dim,
                               Side side, const std::vector<std::int64_t>& col_offset = {},
                               Context& ctx = default_context()) {
  std::vector<double> kn;
  std::vector<std::int64_t> ko;
  std::vector<int> deg;
  detail::pack_knots(kvs, kn, ko, deg);
  if (point.size() != kvs.size() || controls.rank() != static_cast<int>(kvs.size()))
    throw std::invalid_argument("decode: dimension mismatch between lattice, knot vectors and parameters");
  double out = 0.0;
  check(mfadd_eval_points(ctx.get(), controls.rank(), deg.data(), kn.data(), ko.data(), controls.extents().data(),
                          col_offset.empty() ? nullptr : col_offset.data(), controls.data(), 1, point.data(),
                          orders.empty() ? nullptr : orders.data(), side_dim, side == Side::Above ? 1 : 0, &out));
  return out;
}
inline double eval_deriv(const Tensor& controls, const std::vector<KnotVector>& kvs, const std::vector<double>& point,
                         const std::vector<int>& orders, const std::vector<std::int64_t>& col_offset = {},
                         Context& ctx = default_context()) {
  return eval_deriv_sided(controls, kvs, point, orders, -1, Side::Above, col_offset, ctx);
}

// MfaModel (model.hpp:18-35)
struct MfaModel {
  std::vector<int> degrees;
  std::vector<KnotVector> kvs;
  Tensor controls;
  std::vector<std::array<double, 2>> bounds;
  std::map<std::string, std::string> provenance;
  int rank() const { return static_cast<int>(kvs.size()); }
  double param_of(int dim, double x) const {
    const auto& b = bounds[static_cast<std::size_t>(dim)];
    return (x - b[0]) / (b[1] - b[0]);
  }
  double eval(const std::vector<double>& params) const { return mfadd_b200::eval_deriv(controls, kvs, params, {}); }
  double eval_deriv(const std::vector<double>& params, const std::vector<int>& orders) const {
    return mfadd_b200::eval_deriv(controls, kvs, params, orders);
  }
  // model.cpp:39-49 (GPU decode at u_j = j / (res - 1))
  Tensor decode_grid(const std::vector<std::int64_t>& res, Context& ctx = default_context()) const {
    if (static_cast<int>(res.size()) != rank()) throw std::invalid_argument("decode_grid: resolution rank mismatch");
    std::vector<double> kn;
    std::vector<std::int64_t> ko;
    std::vector<int> deg;
    detail::pack_knots(kvs, kn, ko, deg);
    std::vector<std::int64_t> ext;
    for (auto r : res) ext.push_back(r < 1 ? 1 : r);
    Tensor out(ext);
    check(mfadd_decode_grid(ctx.get(), rank(), deg[0], kn.data(), ko.data(), controls.extents().data(),
                            controls.data(), res.data(), out.data()));
    return out;
  }
};

// continuity_jumps(const MfaModel&, ...) (solver.hpp:96)
inline std::vector<double> continuity_jumps(const MfaModel& model, int dim, double u_interface, int max_order,
                                            int cross_samples = 5, Context& ctx = default_context()) {
  std::vector<double> kn;
  std::vector<std::int64_t> ko;
  std::vector<int> deg;
  detail::pack_knots(model.kvs, kn, ko, deg);
  std::vector<double> out(static_cast<std::size_t>(max_order < 0 ? 1 : max_order + 1), 0.0);
  check(mfadd_continuity_jumps(ctx.get(), model.rank(), deg.data(), kn.data(), ko.data(),
                               model.controls.extents().data(), model.controls.data(), dim, u_interface, max_order,
                               cross_samples, out.data()));
  return out;
}

// write_mfa / read_mfa (model.hpp:40-41): MFDD v1, byte-identical with the reference
inline void write_mfa(const MfaModel& model, const std::string& path) {
  std::vector<double> kn, bnd;
  std::vector<std::int64_t> ko;
  std::vector<int> deg;
  detail::pack_knots(model.kvs, kn, ko, deg);
  std::vector<unsigned char> cl, cr;
  for (const auto& kv : model.kvs) {
    cl.push_back(kv.clamp_left ? 1 : 0);
    cr.push_back(kv.clamp_right ? 1 : 0);
  }
  for (const auto& b : model.bounds) {
    bnd.push_back(b[0]);
    bnd.push_back(b[1]);
  }
  std::vector<const char*> keys, vals;
  for (const auto& [k, v] : model.provenance) {
    keys.push_back(k.c_str());
    vals.push_back(v.c_str());
  }
  mfadd_model_view v{};
  v.rank = model.rank();
  v.degrees = model.degrees.data();
  v.clamp_left = cl.data();
  v.clamp_right = cr.data();
  v.knots = kn.data();
  v.kn_off = ko.data();
  v.ctrl_ext = model.controls.extents().data();
  v.bounds = bnd.data();
  v.nprov = static_cast<int>(keys.size());
  v.prov_keys = keys.data();
  v.prov_values = vals.data();
  v.controls = model.controls.data();
  check(mfadd_write_mfa(path.c_str(), &v));
}

inline MfaModel read_mfa(const std::string& path) {
  mfadd_model* h = nullptr;
  check(mfadd_read_mfa(path.c_str(), &h));
  std::unique_ptr<mfadd_model, void (*)(mfadd_model*)> hold(h, mfadd_model_free);
  mfadd_model_view v{};
  check(mfadd_model_view_of(h, &v));
  MfaModel m;
  std::vector<std::int64_t> ext(v.ctrl_ext, v.ctrl_ext + v.rank);
  for (int d = 0; d < v.rank; ++d) {
    KnotVector kv;
    kv.degree = v.degrees[d];
    kv.knots.assign(v.knots + v.kn_off[d], v.knots + v.kn_off[d + 1]);
    kv.clamp_left = v.clamp_left[d] != 0;
    kv.clamp_right = v.clamp_right[d] != 0;
    m.degrees.push_back(kv.degree);
    m.kvs.push_back(std::move(kv));
    m.bounds.push_back({v.bounds[2 * d], v.bounds[2 * d + 1]});
  }
  for (int i = 0; i < v.nprov; ++i) m.provenance[v.prov_keys[i]] = v.prov_values[i];
  m.controls = Tensor(ext, std::vector<double>(v.controls, v.controls + Tensor::count(ext)));
  return m;
}

// BlockState (solver.hpp:26-32): the held lattice of one block.
struct BlockState {
  int id = 0;
  std::vector<std::int64_t> col_offset;
  Tensor p;
};

// SolveResult (solver.hpp:56-68)
struct SolveResult {
  MfaModel model;
  bool converged = false;
  int constraint_iterations = 0;
  double final_dp = 0.0;
  std::vector<EpochStats> epochs;
  std::vector<InterfaceJump> final_jumps;
  PhaseTimings timings;
  std::vector<BlockState> blocks;
  double global_l2 = 0.0;
  double global_linf = 0.0;
  Tensor global_error;
};

// A reusable plan: the decomposition's device tables and work buffers.
// solve() below builds one per call like the reference; keep a Solver to
// amortise creation across fields with the same layout.
class Solver {
 public:
  Solver(const Decomposition& dec, const SolverConfig& cfg, Context& ctx = default_context()) : dec_(dec) {
    mfadd_solver_config c{cfg.max_outer_iterations, cfg.tolerance, cfg.workers, cfg.log_errors ? 1 : 0,
                          cfg.enforce_continuity ? 1 : 0, 1};
    mfadd_solver* s = nullptr;
    check(mfadd_solver_create(ctx.get(), dec.get(), &c, &s));
    h_.reset(s);
  }
  // Host field in, host results out (H2D + solve + D2H).
  SolveResult run(const Field& field, bool want_blocks = true) {
    check_field(field);
    SolveResult r;
    r.model.controls = Tensor(dec_.n_ctrl);
    r.global_error = Tensor(field.dims);
    mfadd_solve_summary sm{};
    check(mfadd_solve_host(h_.get(), field.values.data(), r.model.controls.data(), r.global_error.data(), &sm));
    fill(r, sm, field, want_blocks);
    return r;
  }
  // Device-resident field (a device pointer on the context's GPU).
  SolveResult run_device(const double* field_dev, const Field& meta, bool want_blocks = false) {
    if (meta.dims != dec_.n_input) throw std::invalid_argument("solve: field extents disagree with the decomposition");
    SolveResult r;
    mfadd_solve_summary sm{};
    check(mfadd_solve(h_.get(), field_dev, 1, &sm));
    r.model.controls = Tensor(dec_.n_ctrl);
    check(mfadd_solver_controls(h_.get(), r.model.controls.data(), 0));
    r.global_error = Tensor(meta.dims);
    check(mfadd_solver_global_error(h_.get(), r.global_error.data(), 0));
    fill(r, sm, meta, want_blocks);
    return r;
  }
  mfadd_solver* get() const { return h_.get(); }

 private:
  // solver.cpp:333-338: the field must match the decomposition's input extents
  void check_field(const Field& field) const {
    if (field.dims != dec_.n_input) throw std::invalid_argument("solve: field extents disagree with the decomposition");
    if (field.values.size() != Tensor::count(field.dims))
      throw std::invalid_argument("solve: field values do not match dims");
  }
  void fill(SolveResult& r, const mfadd_solve_summary& sm, const Field& field, bool want_blocks) const {
    r.converged = sm.converged != 0;
    r.constraint_iterations = sm.constraint_iterations;
    r.final_dp = sm.final_dp;
    r.global_l2 = sm.global_l2;
    r.global_linf = sm.global_linf;
    r.timings = PhaseTimings{sm.t_setup, sm.t_local_solve, sm.t_exchange, sm.t_constraint, sm.t_decode};
    std::vector<mfadd_epoch_stats> ep(static_cast<std::size_t>(sm.n_epochs));
    mfadd_solver_epochs(h_.get(), ep.data(), sm.n_epochs);
    for (int e = 0; e < sm.n_epochs; ++e) {
      EpochStats s;
      s.iteration = ep[static_cast<std::size_t>(e)].iteration;
      s.dp_max = ep[static_cast<std::size_t>(e)].dp_max;
      s.jump_ss = ep[static_cast<std::size_t>(e)].jump_ss;
      s.jump_ms = ep[static_cast<std::size_t>(e)].jump_ms;
      std::vector<double> be(2 * dec_.blocks.size());
      if (mfadd_solver_block_errors(h_.get(), e, be.data()) == MFADD_OK)
        for (std::size_t b = 0; b < dec_.blocks.size(); ++b) s.block_errors.push_back({be[2 * b], be[2 * b + 1]});
      r.epochs.push_back(std::move(s));
    }
    std::vector<double> j4(4 * static_cast<std::size_t>(sm.n_final_jumps));
    mfadd_solver_final_jumps(h_.get(), j4.data(), sm.n_final_jumps);
    for (int j = 0; j < sm.n_final_jumps; ++j)
      r.final_jumps.push_back(InterfaceJump{static_cast<int>(j4[4 * j]), static_cast<int>(j4[4 * j + 1]),
                                            j4[4 * j + 2], j4[4 * j + 3]});
    r.model.kvs = dec_.kvs;
    r.model.bounds = field.bounds;
    for (const auto& kv : dec_.kvs) r.model.degrees.push_back(kv.degree);
    if (want_blocks)
      for (const auto& bl : dec_.blocks) {
        BlockState st;
        st.id = bl.id;
        std::vector<std::int64_t> ext;
        for (const auto& d : bl.dims) {
          st.col_offset.push_back(d.dof_lo);
          ext.push_back(d.dof_hi - d.dof_lo);
        }
        st.p = Tensor(ext);
        check(mfadd_solver_block_controls(h_.get(), bl.id, st.p.data(), 0));
        r.blocks.push_back(std::move(st));
      }
  }
  struct Del {
    void operator()(mfadd_solver* s) const { mfadd_solver_free(s); }
  };
  Decomposition dec_;
  std::unique_ptr<mfadd_solver, Del> h_;
};

// solve (solver.hpp:76)
inline SolveResult solve(const Field& field, const Decomposition& dec, const SolverConfig& config) {
  Solver s(dec, config);
  return s.run(field);
}

// ------------------------------------------------------ unit sub-boundaries
// BandedCollocation (collocation.hpp:15-49) packing, plus the knots/params it
// was built from (the device path recomputes rows from them).
struct BandedCollocation {
  std::int64_t rows = 0, cols = 0;
  int band = 0;
  std::vector<std::int64_t> first_col;
  std::vector<int> count;
  std::vector<double> values;  // rows x band
  KnotVector kv;
  std::vector<double> params;
  std::int64_t col_lo = 0, col_hi = 0;
};

// collocation_matrix (collocation.hpp:53-58)
inline BandedCollocation collocation_matrix(const KnotVector& kv, const std::vector<double>& params,
                                            std::int64_t col_lo, std::int64_t col_hi,
                                            Context& ctx = default_context()) {
  BandedCollocation r;
  r.rows = static_cast<std::int64_t>(params.size());
  r.cols = col_hi - col_lo;
  r.band = kv.degree + 1;
  r.first_col.resize(params.size());
  r.count.resize(params.size());
  r.values.resize(params.size() * static_cast<std::size_t>(r.band));
  check(mfadd_collocation(ctx.get(), kv.knots.data(), static_cast<int>(kv.knots.size()), kv.degree, params.data(),
                          r.rows, col_lo, col_hi, r.first_col.data(), r.count.data(), r.values.data()));
  r.kv = kv;
  r.params = params;
  r.col_lo = col_lo;
  r.col_hi = col_hi;
  return r;
}
inline BandedCollocation collocation_matrix(const KnotVector& kv, const std::vector<double>& params) {
  return collocation_matrix(kv, params, 0, kv.basis_count());
}

// LocalProblem (lsq.hpp:15-21)
struct LocalProblem {
  std::vector<BandedCollocation> r;
  Tensor q;
};

// fit_unconstrained (lsq.hpp:33)
inline Tensor fit_unconstrained(const LocalProblem& problem, Context& ctx = default_context()) {
  const int rank = static_cast<int>(problem.r.size());
  if (rank == 0 || problem.q.rank() != rank) throw std::invalid_argument("fit_unconstrained: rank mismatch");
  std::vector<double> knots, params;
  std::vector<std::int64_t> kn_off{0}, pm_off{0}, lo, hi, ext;
  for (const auto& c : problem.r) {
    knots.insert(knots.end(), c.kv.knots.begin(), c.kv.knots.end());
    params.insert(params.end(), c.params.begin(), c.params.end());
    kn_off.push_back(static_cast<std::int64_t>(knots.size()));
    pm_off.push_back(static_cast<std::int64_t>(params.size()));
    lo.push_back(c.col_lo);
    hi.push_back(c.col_hi);
    ext.push_back(c.col_hi - c.col_lo);
  }
  Tensor out(ext);
  check(mfadd_fit_unconstrained(ctx.get(), rank, problem.r[0].kv.degree, knots.data(), kn_off.data(), params.data(),
                                pm_off.data(), lo.data(), hi.data(), problem.q.data(), out.data()));
  return out;
}

// ResidualStats / residual_error (lsq.hpp:35-41)
struct ResidualStats {
  double l2 = 0.0;
  double linf = 0.0;
  Tensor pointwise;
};

inline ResidualStats residual_error(const LocalProblem& problem, const Tensor& controls,
                                    Context& ctx = default_context()) {
  const int rank = static_cast<int>(problem.r.size());
  if (rank == 0 || problem.q.rank() != rank || controls.rank() != rank)
    throw std::invalid_argument("residual_error: rank mismatch");
  std::vector<double> knots, params;
  std::vector<std::int64_t> kn_off{0}, pm_off{0}, lo, hi;
  for (int d = 0; d < rank; ++d) {
    const auto& c = problem.r[static_cast<std::size_t>(d)];
    if (controls.extent(d) != c.col_hi - c.col_lo) throw std::invalid_argument("residual_error: control extents");
    knots.insert(knots.end(), c.kv.knots.begin(), c.kv.knots.end());
    params.insert(params.end(), c.params.begin(), c.params.end());
    kn_off.push_back(static_cast<std::int64_t>(knots.size()));
    pm_off.push_back(static_cast<std::int64_t>(params.size()));
    lo.push_back(c.col_lo);
    hi.push_back(c.col_hi);
  }
  ResidualStats st;
  st.pointwise = Tensor(problem.q.extents());
  check(mfadd_residual_error(ctx.get(), rank, problem.r[0].kv.degree, knots.data(), kn_off.data(), params.data(),
                             pm_off.data(), lo.data(), hi.data(), problem.q.data(), controls.data(),
                             st.pointwise.data(), &st.l2, &st.linf));
  return st;
}

// SpanBasis (knots.hpp:39-50)
struct SpanBasis {
  int span = 0;
  int orders = 0;
  std::vector<double> values;       // p+1 values, N_{span-p..span}
  std::vector<double> derivatives;  // (orders+1) x (p+1), row 0 = values
  double deriv(int k, int j) const {
    return derivatives[static_cast<std::size_t>(k * static_cast<int>(values.size()) + j)];
  }
};

// find_span (knots.hpp:36)
inline int find_span(const KnotVector& kv, double u, Context& ctx = default_context()) {
  std::vector<double> v(static_cast<std::size_t>(kv.degree + 1));
  int span = 0;
  check(mfadd_basis_funs(ctx.get(), kv.knots.data(), static_cast<int>(kv.knots.size()), kv.degree, 1, &u, nullptr, 0,
                         &span, v.data()));
  return span;
}

// basis_derivs (knots.hpp:56); basis_funs (knots.hpp:53) is its k = 0 row
inline SpanBasis basis_derivs(const KnotVector& kv, int span, double u, int k, Context& ctx = default_context()) {
  SpanBasis b;
  b.span = span;
  b.orders = k;
  const std::size_t w = static_cast<std::size_t>(kv.degree + 1);
  b.derivatives.resize(w * static_cast<std::size_t>(k + 1));
  int sp = span;
  check(mfadd_basis_funs(ctx.get(), kv.knots.data(), static_cast<int>(kv.knots.size()), kv.degree, 1, &u, &span, k,
                         &sp, b.derivatives.data()));
  b.values.assign(b.derivatives.begin(), b.derivatives.begin() + static_cast<std::ptrdiff_t>(w));
  return b;
}
inline SpanBasis basis_funs(const KnotVector& kv, int span, double u, Context& ctx = default_context()) {
  return basis_derivs(kv, span, u, 0, ctx);
}

// decode (decode.hpp:20-22)
inline Tensor decode(const Tensor& controls, const std::vector<KnotVector>& kvs,
                     const std::vector<std::vector<double>>& params, const std::vector<std::int64_t>& col_offset = {},
                     Context& ctx = default_context()) {
  const int rank = controls.rank();
  if (static_cast<int>(kvs.size()) != rank || static_cast<int>(params.size()) != rank)
    throw std::invalid_argument("decode: rank mismatch");
  std::vector<double> knots, pr;
  std::vector<std::int64_t> kn_off{0}, pm_off{0}, ext;
  for (int d = 0; d < rank; ++d) {
    knots.insert(knots.end(), kvs[static_cast<std::size_t>(d)].knots.begin(), kvs[static_cast<std::size_t>(d)].knots.end());
    pr.insert(pr.end(), params[static_cast<std::size_t>(d)].begin(), params[static_cast<std::size_t>(d)].end());
    kn_off.push_back(static_cast<std::int64_t>(knots.size()));
    pm_off.push_back(static_cast<std::int64_t>(pr.size()));
    ext.push_back(static_cast<std::int64_t>(params[static_cast<std::size_t>(d)].size()));
  }
  Tensor out(ext);
  check(mfadd_decode(ctx.get(), rank, kvs[0].degree, knots.data(), kn_off.data(), pr.data(), pm_off.data(),
                     controls.extents().data(), col_offset.empty() ? nullptr : col_offset.data(), controls.data(),
                     out.data()));
  return out;
}

}  // namespace mfadd_b200

#endif  // MFADD_B200_HPP
