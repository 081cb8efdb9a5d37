// C++ drop-in check: the reference's own test cases written against the
// mfadd:: names, compiled against include/mfadd_b200.hpp and linked to
// libmfadd_b200.so.  `cpu` mode touches host-side layout only; `gpu` mode runs
// solve / fit_unconstrained / decode on device 0.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "mfadd_b200.hpp"
namespace mfadd = mfadd_b200;  // the one-line switch a reference caller makes

static int failures = 0;
#define EXPECT(c)                                                 \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
      ++failures;                                                 \
    }                                                             \
  } while (0)

static void cpu_cases() {
  // test_layout.cpp:32-68: two blocks of 8 controls, p=3, overlap 1
  auto d = mfadd::partition({64}, {{0.0, 1.0}}, {2}, 3, {8}, 1, false);
  EXPECT(d.rank() == 1 && d.block_count() == 2);
  const auto& b0 = d.blocks[0].dims[0];
  const auto& b1 = d.blocks[1].dims[0];
  EXPECT(b0.own_lo == 0 && b0.own_hi == 8 && b1.own_lo == 8 && b1.own_hi == 16);
  EXPECT(b0.dof_lo == 0 && b0.dof_hi == 10 && b1.dof_lo == 6 && b1.dof_hi == 16);
  EXPECT(d.blocks[0].neighbors.size() == 1 && d.blocks[0].neighbors[0] == 1);
  EXPECT(d.holder_span(0, 7).first == 0 && d.holder_span(0, 7).second == 1);
  // test_layout.cpp:123-139: compression ratio 4.0
  EXPECT(mfadd::partition({200, 200}, {{0, 1}, {0, 1}}, {5, 5}, 3, {20, 20}, 0, false).compression_ratio() == 4.0);
  // test_runtime.cpp:137-145: exchange volume {4, 4}
  const auto ev = mfadd::partition({64}, {{0, 1}}, {2}, 3, {8}, 1, false).exchange_volume();
  EXPECT(ev.size() == 2 && ev[0] == 4 && ev[1] == 4);
  // knots (test_knots.cpp:13-35): clamped, p+1 zeros/ones
  EXPECT(d.kvs[0].degree == 3 && d.kvs[0].knots.front() == 0.0 && d.kvs[0].knots.back() == 1.0);
  // precondition failures are std::invalid_argument (layout.cpp:222-267)
  bool threw = false;
  try {
    mfadd::partition({64}, {{0, 1}}, {2}, 3, {1}, 0, false);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  EXPECT(threw);
}

static mfadd::Field sinc2d(std::int64_t nx, std::int64_t ny) {
  mfadd::Field f;
  f.dims = {nx, ny};
  f.bounds = {{-4.0, 4.0}, {-4.0, 4.0}};
  f.values = mfadd::Tensor({nx, ny});
  for (std::int64_t i = 0; i < nx; ++i)
    for (std::int64_t j = 0; j < ny; ++j) {
      const double x = -4.0 + 8.0 * static_cast<double>(i) / static_cast<double>(nx - 1);
      const double y = -4.0 + 8.0 * static_cast<double>(j) / static_cast<double>(ny - 1);
      const double r = std::sqrt(x * x + y * y);
      f.values[i * ny + j] = r == 0.0 ? 1.0 : std::sin(r) / r;
    }
  return f;
}

static void gpu_cases() {
  // test_solver.cpp:189-205: 2x2 blocks need two constraint iterations, 4 epochs
  const auto f = sinc2d(64, 64);
  const auto dec = mfadd::partition(f.dims, f.bounds, {2, 2}, 3, {12, 12}, 0, false);
  mfadd::SolverConfig cfg;
  cfg.log_errors = false;
  const auto r = mfadd::solve(f, dec, cfg);
  EXPECT(r.converged && r.constraint_iterations == 2 && r.epochs.size() == 4);
  EXPECT(r.epochs[1].jump_ms > 1e-12 && r.epochs[2].jump_ss < 1e-12 && r.epochs[2].jump_ms < 1e-12);
  EXPECT(r.model.controls.size() == 24 * 24 && r.global_error.size() == 64 * 64);
  EXPECT(r.blocks.size() == 4);
  // L2 / L-inf are the norms of the returned pointwise error field
  double l2 = 0.0, li = 0.0;
  for (std::int64_t i = 0; i < r.global_error.size(); ++i) {
    l2 += r.global_error[i] * r.global_error[i];
    li = std::fmax(li, std::fabs(r.global_error[i]));
  }
  EXPECT(r.global_linf > 0.0 && li == r.global_linf);
  EXPECT(std::fabs(std::sqrt(l2) - r.global_l2) <= 1e-12 * r.global_l2);
  // the reference defaults (log_errors = true): per-epoch block residuals
  const auto rl = mfadd::solve(f, dec, mfadd::SolverConfig{});
  EXPECT(rl.epochs.size() == r.epochs.size() && rl.epochs[0].block_errors.size() == 4);
  EXPECT(rl.epochs.back().block_errors[0][0] > 0.0 && rl.epochs.back().block_errors[0][1] > 0.0);
  EXPECT(rl.model.controls.values() == r.model.controls.values());
  // the error field is q - decode(controls) at the grid params
  std::vector<std::vector<double>> u(2);
  for (int d = 0; d < 2; ++d)
    for (std::int64_t j = 0; j < 64; ++j) u[static_cast<std::size_t>(d)].push_back(static_cast<double>(j) / 63.0);
  const auto dec_vals = mfadd::decode(r.model.controls, r.model.kvs, u);
  double mx = 0.0;
  for (std::int64_t i = 0; i < dec_vals.size(); ++i)
    mx = std::fmax(mx, std::fabs((f.values[i] - dec_vals[i]) - r.global_error[i]));
  EXPECT(mx < 1e-12);
  // lsq.cpp: polynomial reproduction through fit_unconstrained (test_lsq.cpp:80-101)
  mfadd::KnotVector kv = r.model.kvs[0];
  mfadd::LocalProblem lp;
  lp.r.push_back(mfadd::collocation_matrix(kv, u[0]));
  lp.r.push_back(mfadd::collocation_matrix(kv, u[1]));
  lp.q = mfadd::Tensor({64, 64});
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j < 64; ++j) lp.q[i * 64 + j] = 1.0 + u[0][i] - 2.0 * u[1][j] + u[0][i] * u[1][j] * u[1][j];
  const auto P = mfadd::fit_unconstrained(lp);
  const auto back = mfadd::decode(P, r.model.kvs, u);
  double e = 0.0;
  for (std::int64_t i = 0; i < back.size(); ++i) e = std::fmax(e, std::fabs(back[i] - lp.q[i]));
  EXPECT(e < 1e-9);
  // residual_error (lsq.hpp:41) of the fit: pointwise = q - decode(P)
  const auto rs = mfadd::residual_error(lp, P);
  double rl2 = 0.0, rli = 0.0, rmx = 0.0;
  for (std::int64_t i = 0; i < rs.pointwise.size(); ++i) {
    rl2 += rs.pointwise[i] * rs.pointwise[i];
    rli = std::fmax(rli, std::fabs(rs.pointwise[i]));
    rmx = std::fmax(rmx, std::fabs(rs.pointwise[i] - (lp.q[i] - back[i])));
  }
  EXPECT(rmx < 1e-13 && rli == rs.linf && std::fabs(std::sqrt(rl2) - rs.l2) <= 1e-12 * std::fmax(rs.l2, 1e-300));
  // find_span / basis_funs / basis_derivs (knots.hpp:36-56)
  const int sp = mfadd::find_span(kv, 0.5);
  EXPECT(kv.knots[static_cast<std::size_t>(sp)] <= 0.5 && 0.5 < kv.knots[static_cast<std::size_t>(sp) + 1]);
  const auto bf = mfadd::basis_funs(kv, sp, 0.5);
  double pu = 0.0;
  for (double v : bf.values) pu += v;
  EXPECT(bf.values.size() == 4 && std::fabs(pu - 1.0) < 1e-14);
  const auto bd = mfadd::basis_derivs(kv, sp, 0.5, 2);
  double d1 = 0.0;
  for (int j = 0; j < 4; ++j) d1 += bd.deriv(1, j);
  EXPECT(bd.values == bf.values && std::fabs(d1) < 1e-9);
  bool range = false;
  try {
    mfadd::find_span(kv, 1.5);
  } catch (const std::out_of_range&) {
    range = true;
  }
  EXPECT(range);
  // solver.cpp:335-338: a field whose extents disagree with the decomposition
  bool extents = false;
  try {
    mfadd::Field ft = sinc2d(64, 64);
    ft.dims = {32, 128};
    mfadd::solve(ft, dec, cfg);
  } catch (const std::invalid_argument&) {
    extents = true;
  }
  EXPECT(extents);
  // SingularFitError{dim, span} through the shim (lsq.cpp:46-55)
  bool singular = false;
  try {
    mfadd::LocalProblem bad;
    // 40 samples crowded into the first knot span: enough rows, but columns
    // past the data have no support (uncovered_column, lsq.cpp:25-35)
    std::vector<double> few;
    for (int i = 0; i < 40; ++i) few.push_back(0.001 * i);
    bad.r.push_back(mfadd::collocation_matrix(kv, few));
    bad.q = mfadd::Tensor({40});
    mfadd::fit_unconstrained(bad);
  } catch (const mfadd::SingularFitError& ex) {
    singular = ex.dim == 0 && ex.span == 4;  // columns 0..3 supported (one knot span of data)
  }
  EXPECT(singular);
  // MfaModel output path (model.hpp): MFDD round trip, decode_grid, eval and
  // the continuity probe on the converged model (floating interfaces: the
  // value and first p-1 derivatives agree across an interior knot).
  mfadd::MfaModel mm = r.model;
  mm.provenance["source"] = "sinc";
  const std::string path = "/tmp/mfadd_shim_model.mfa";
  mfadd::write_mfa(mm, path);
  const auto back_m = mfadd::read_mfa(path);
  EXPECT(back_m.controls.values() == mm.controls.values() && back_m.provenance == mm.provenance);
  EXPECT(back_m.kvs[1].knots == mm.kvs[1].knots && back_m.bounds == mm.bounds);
  const auto grid = mm.decode_grid({64, 64});
  double gmx = 0.0;
  for (std::int64_t i = 0; i < grid.size(); ++i) gmx = std::fmax(gmx, std::fabs(grid[i] - dec_vals[i]));
  EXPECT(gmx < 1e-12);
  EXPECT(std::fabs(mm.eval({u[0][5], u[1][7]}) - dec_vals[5 * 64 + 7]) < 1e-12);
  const auto jumps = mfadd::continuity_jumps(mm, 0, mm.kvs[0].knots[3 + 5], 2);
  EXPECT(jumps.size() == 3 && jumps[0] < 1e-12 && jumps[1] < 1e-9);
  std::remove(path.c_str());
}

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  try {
    cpu_cases();
    if (gpu) gpu_cases();
  } catch (const std::exception& ex) {
    std::printf("FAIL exception: %s\n", ex.what());
    return 2;
  }
  std::printf("%s: %d failures\n", gpu ? "gpu" : "cpu", failures);
  return failures == 0 ? 0 : 1;
}
