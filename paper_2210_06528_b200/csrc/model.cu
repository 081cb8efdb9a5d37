// model.cu — the MfaModel side of the encode path:
//
//   k_eval_points    batched point evaluation of one or more control lattices
//                    with derivatives and one-sided spans (eval_deriv /
//                    eval_deriv_sided, decode.cpp:14-80; basis_derivs,
//                    knots.cpp:131-203), thread per evaluation
//   k_raw_to_f64     raw grid conversion on the device (byte swap + widening,
//                    field.cpp:149-191)
//
// and the C ABI entry points built on them: mfadd_eval_points,
// mfadd_continuity_jumps (solver.cpp:197-261), mfadd_decode_grid
// (model.cpp:39-49), mfadd_read_raw_grid, and the MFDD v1 container
// (mfadd_write_mfa / mfadd_read_mfa, model.cpp:53-167; host file I/O).
//
// Point values are bitwise equal to the reference: explicit round-to-nearest
// operations in the reference's order (its build has no FMA contraction).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <array>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "abi.hpp"
#include "kernels.cuh"

using namespace mfb_abi;

#define CK(x) cuda_check((x), #x)

namespace mfb {
namespace {

constexpr int kEvalThreads = 128;
constexpr int kMaxP1 = kMaxDegree + 1;

// knots.cpp:83-106 (the caller has range-checked u)
__device__ int dev_find_span(const double* kn, int p, int nb, double u) {
  if (u >= kn[nb]) {
    int s = nb - 1;
    while (s > p && kn[s] == kn[s + 1]) --s;
    return s;
  }
  int low = p, high = nb, mid = (low + high) / 2;
  while (u < kn[mid] || u >= kn[mid + 1]) {
    if (u < kn[mid])
      high = mid;
    else
      low = mid;
    mid = (low + high) / 2;
  }
  return mid;
}

// knots.cpp:108-129 (basis_funs), explicit RN ops
__device__ void dev_basis_funs(const double* kn, int p, int span, double u, double* N) {
  double left[kMaxP1], right[kMaxP1];
  N[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = __dsub_rn(u, kn[span + 1 - j]);
    right[j] = __dsub_rn(kn[span + j], u);
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double denom = __dadd_rn(right[r + 1], left[j - r]);
      const double temp = __ddiv_rn(N[r], denom);
      N[r] = __dadd_rn(saved, __dmul_rn(right[r + 1], temp));
      saved = __dmul_rn(left[j - r], temp);
    }
    N[j] = saved;
  }
}

// knots.cpp:131-203 (basis_derivs, The NURBS Book A2.3): row k of the
// derivative table into D, explicit RN ops in the reference's order.
__device__ void dev_basis_deriv_row(const double* kn, int p, int span, double u, int k, double* D) {
  double ndu[kMaxP1][kMaxP1], left[kMaxP1], right[kMaxP1], a[2][kMaxP1];
  ndu[0][0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = __dsub_rn(u, kn[span + 1 - j]);
    right[j] = __dsub_rn(kn[span + j], u);
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      ndu[j][r] = __dadd_rn(right[r + 1], left[j - r]);
      const double temp = __ddiv_rn(ndu[r][j - 1], ndu[j][r]);
      ndu[r][j] = __dadd_rn(saved, __dmul_rn(right[r + 1], temp));
      saved = __dmul_rn(left[j - r], temp);
    }
    ndu[j][j] = saved;
  }
  for (int r = 0; r <= p; ++r) {
    int s1 = 0, s2 = 1;
    a[0][0] = 1.0;
    double dk = 0.0;
    for (int kk = 1; kk <= k; ++kk) {
      double d = 0.0;
      const int rk = r - kk, pk = p - kk;
      if (r >= kk) {
        a[s2][0] = __ddiv_rn(a[s1][0], ndu[pk + 1][rk]);
        d = __dmul_rn(a[s2][0], ndu[rk][pk]);
      }
      const int j1 = rk >= -1 ? 1 : -rk;
      const int j2 = (r - 1 <= pk) ? kk - 1 : p - r;
      for (int j = j1; j <= j2; ++j) {
        a[s2][j] = __ddiv_rn(__dsub_rn(a[s1][j], a[s1][j - 1]), ndu[pk + 1][rk + j]);
        d = __dadd_rn(d, __dmul_rn(a[s2][j], ndu[rk + j][pk]));
      }
      if (r <= pk) {
        a[s2][kk] = __ddiv_rn(-a[s1][kk - 1], ndu[pk + 1][r]);
        d = __dadd_rn(d, __dmul_rn(a[s2][kk], ndu[r][pk]));
      }
      dk = d;
      const int t = s1;
      s1 = s2;
      s2 = t;
    }
    D[r] = dk;
  }
  // DER(kk, j) *= factor, factor = p (p-1) ... : applied row by row in turn
  double factor = static_cast<double>(p);
  for (int kk = 1; kk <= k; ++kk) {
    if (kk == k)
      for (int j = 0; j <= p; ++j) D[j] = __dmul_rn(D[j], factor);
    factor = __dmul_rn(factor, static_cast<double>(p - kk));
  }
}

__global__ void __launch_bounds__(kEvalThreads) k_eval_points(EvalArgs a) {
  const std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= a.n) return;
  const EvalItem it = a.items[i];
  const EvalLattice L = a.lats[it.lat];
  double B[3][kMaxP1];
  std::int64_t base[3];
  for (int k = 0; k < a.rank; ++k) {  // decode.cpp:63-79
    const int p = a.deg[k];
    const double* kn = a.knots + a.kn_off[k];
    const int nb = static_cast<int>(a.kn_off[k + 1] - a.kn_off[k]) - p - 1;
    const int order = it.ord[k];
    if (order < 0 || order > p) {
      a.err[i] = (1 << 8) | k;
      a.out[i] = 0.0;
      return;
    }
    const double u = it.pt[k];
    if (u < kn[p] || u > kn[nb]) {
      a.err[i] = (2 << 8) | k;
      a.out[i] = 0.0;
      return;
    }
    int s = dev_find_span(kn, p, nb, u);
    if (k == it.side_dim && it.side == 0 && u == kn[s] && u > kn[p]) {  // sided_span, decode.cpp:18-25
      --s;
      while (s > p && kn[s] == kn[s + 1]) --s;
    }
    if (order == 0)
      dev_basis_funs(kn, p, s, u, B[k]);
    else
      dev_basis_deriv_row(kn, p, s, u, order, B[k]);
    base[k] = static_cast<std::int64_t>(s) - p - L.coff[k];
  }
  for (int k = 0; k < a.rank; ++k)  // decode.cpp:31-39
    if (base[k] < 0 || base[k] + a.deg[k] >= L.ext[k]) {
      a.err[i] = (3 << 8) | k;
      a.out[i] = 0.0;
      return;
    }
  // decode.cpp:40-57: odometer over the active bases, last dim fastest
  std::int64_t stride[3];
  {
    std::int64_t st = 1;
    for (int k = a.rank - 1; k >= 0; --k) {
      stride[k] = st;
      st *= L.ext[k];
    }
  }
  int idx[3] = {0, 0, 0};
  double acc = 0.0;
  const double* c = a.ctrl + L.base;
  while (true) {
    double w = 1.0;
    std::int64_t off = 0;
    for (int k = 0; k < a.rank; ++k) {
      w = __dmul_rn(w, B[k][idx[k]]);
      off += (base[k] + idx[k]) * stride[k];
    }
    acc = __dadd_rn(acc, __dmul_rn(w, c[off]));
    int k = a.rank - 1;
    for (; k >= 0; --k) {
      if (++idx[k] <= a.deg[k]) break;
      idx[k] = 0;
    }
    if (k < 0) break;
  }
  a.out[i] = acc;
  a.err[i] = 0;
}

// find_span / basis_funs / basis_derivs (knots.cpp:83-203) per parameter:
// out row 0 = basis_funs, rows 1..k = basis_derivs rows; err per item (1: u
// outside the evaluable range).
__global__ void __launch_bounds__(kEvalThreads) k_basis_points(const double* kn, int p, int nb, std::int64_t n,
                                                               const double* u, const int* spans, int k,
                                                               int* out_spans, double* out, int* err) {
  const std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double x = u[i];
  int s;
  if (spans) {
    s = spans[i];
  } else {
    if (x < kn[p] || x > kn[nb]) {
      err[i] = 1;
      return;
    }
    s = dev_find_span(kn, p, nb, x);
  }
  err[i] = 0;
  out_spans[i] = s;
  double* o = out + i * static_cast<std::int64_t>(k + 1) * (p + 1);
  dev_basis_funs(kn, p, s, x, o);
  for (int r = 1; r <= k; ++r) dev_basis_deriv_row(kn, p, s, x, r, o + r * (p + 1));
}

// field.cpp:170-185: float32 / float64, optional byte swap, widened to fp64
__global__ void k_raw_to_f64(const unsigned char* raw, std::int64_t n, int width, int swap, double* out) {
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (width == 4) {
      unsigned v = reinterpret_cast<const unsigned*>(raw)[i];
      if (swap) v = __byte_perm(v, 0, 0x0123);
      out[i] = static_cast<double>(__uint_as_float(v));
    } else {
      unsigned long long v = reinterpret_cast<const unsigned long long*>(raw)[i];
      if (swap) {
        const unsigned lo = static_cast<unsigned>(v), hi = static_cast<unsigned>(v >> 32);
        v = (static_cast<unsigned long long>(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
      }
      out[i] = __longlong_as_double(static_cast<long long>(v));
    }
  }
}

}  // namespace

int launch_raw_to_f64(const unsigned char* raw, std::int64_t n, int width, int swap, double* out, cudaStream_t s) {
  if (n <= 0) return 0;
  const std::int64_t blocks = std::min<std::int64_t>((n + 255) / 256, 148 * 16);
  k_raw_to_f64<<<static_cast<unsigned>(blocks), 256, 0, s>>>(raw, n, width, swap, out);
  return 1;
}

int launch_eval_points(const EvalArgs& a, cudaStream_t s) {
  if (a.n <= 0) return 0;
  k_eval_points<<<static_cast<unsigned>((a.n + kEvalThreads - 1) / kEvalThreads), kEvalThreads, 0, s>>>(a);
  return 1;
}

}  // namespace mfb

// ===================================================================== host
namespace {

template <class T>
struct DevVec {  // owning device array
  T* p = nullptr;
  DevVec() = default;
  DevVec(const DevVec&) = delete;
  DevVec& operator=(const DevVec&) = delete;
  explicit DevVec(std::size_t n) {
    if (n) CK(cudaMalloc(&p, n * sizeof(T)));
  }
  ~DevVec() {
    if (p) cudaFree(p);
  }
};

template <class T>
void h2d(T* d, const T* h, std::size_t n, cudaStream_t s) {
  if (n) CK(cudaMemcpyAsync(d, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
}

// The first failing evaluation (lowest index, like the reference's caller
// loop) as the reference's exception (decode.cpp:34-36,69-71; knots.cpp:88-90).
void raise_eval_error(const std::vector<int>& err, const std::vector<mfb::EvalItem>& items, const int* deg,
                      const double* knots, const std::int64_t* kn_off) {
  for (std::size_t i = 0; i < err.size(); ++i) {
    if (!err[i]) continue;
    const int code = err[i] >> 8, k = err[i] & 0xff;
    if (code == 1)
      throw std::invalid_argument("eval_deriv: order " + std::to_string(items[i].ord[k]) +
                                  " exceeds degree in dimension " + std::to_string(k));
    if (code == 2) {
      const double* kn = knots + kn_off[k];
      const int nb = static_cast<int>(kn_off[k + 1] - kn_off[k]) - deg[k] - 1;
      throw std::out_of_range("find_span: parameter " + std::to_string(items[i].pt[k]) + " outside evaluable range [" +
                              std::to_string(kn[deg[k]]) + ", " + std::to_string(kn[nb]) + "]");
    }
    throw std::out_of_range("eval: active basis range falls outside the control lattice window");
  }
}

void check_knots(int rank, const int* degrees, const std::int64_t* kn_off) {
  if (rank < 1 || rank > 3) throw std::invalid_argument("decode: dimension mismatch between lattice, knot vectors and parameters");
  for (int k = 0; k < rank; ++k) {
    if (degrees[k] < 1 || degrees[k] > mfb::kMaxDegree)
      throw std::invalid_argument("eval: degree must be in [1, " + std::to_string(mfb::kMaxDegree) + "]");
    if (kn_off[k + 1] - kn_off[k] < 2 * (degrees[k] + 1)) throw std::invalid_argument("KnotVector: too few knots");
  }
}

}  // namespace

namespace mfb {

// Evaluate `items` against lattices already on the device; results and
// per-item error words to the host.  Shared by the C ABI below and the
// solver's continuity probe (engine.cu).
void eval_items_device(mfadd_context* ctx, int rank, const int* degrees, const double* knots,
                       const std::int64_t* kn_off, const double* d_ctrl, const std::vector<EvalLattice>& lats,
                       const std::vector<EvalItem>& items, std::vector<double>& out) {
  cudaStream_t st = ctx->stream;
  const std::size_t n = items.size();
  out.assign(n, 0.0);
  if (n == 0) return;
  DevVec<double> dk(static_cast<std::size_t>(kn_off[rank]));
  DevVec<EvalLattice> dl(lats.size());
  DevVec<EvalItem> di(n);
  DevVec<double> dout(n);
  DevVec<int> derr(n);
  h2d(dk.p, knots, static_cast<std::size_t>(kn_off[rank]), st);
  h2d(dl.p, lats.data(), lats.size(), st);
  h2d(di.p, items.data(), n, st);
  EvalArgs a{};
  a.rank = rank;
  for (int k = 0; k < rank; ++k) a.deg[k] = degrees[k];
  for (int k = 0; k <= rank; ++k) a.kn_off[k] = kn_off[k];
  a.knots = dk.p;
  a.ctrl = d_ctrl;
  a.lats = dl.p;
  a.items = di.p;
  a.n = static_cast<std::int64_t>(n);
  a.out = dout.p;
  a.err = derr.p;
  ctx->launches += launch_eval_points(a, st);
  CK(cudaGetLastError());
  std::vector<int> err(n);
  CK(cudaMemcpyAsync(out.data(), dout.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(err.data(), derr.p, n * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  raise_eval_error(err, items, degrees, knots, kn_off);
}

// probe_jumps (solver.cpp:212-241): the probe points of one interface in the
// reference's enumeration order (cross dims odometer, last fastest), each at
// orders 0..max_order on both sides; items [point][order][below, above].
void probe_items(int rank, int dim, double u, int max_order, const std::vector<std::vector<double>>& cross,
                 int lat_below, int lat_above, std::vector<EvalItem>& items) {
  std::vector<std::size_t> sel(cross.size(), 0);
  while (true) {
    double pt[3] = {0.0, 0.0, 0.0};
    pt[dim] = u;
    int c = 0;
    for (int k = 0; k < rank; ++k) {
      if (k == dim) continue;
      pt[k] = cross[static_cast<std::size_t>(c)][sel[static_cast<std::size_t>(c)]];
      ++c;
    }
    for (int r = 0; r <= max_order; ++r)
      for (int side = 0; side < 2; ++side) {
        EvalItem it{};
        it.lat = side == 0 ? lat_below : lat_above;
        it.side_dim = dim;
        it.side = side;  // 0 Below, 1 Above
        it.ord[dim] = r;
        for (int k = 0; k < 3; ++k) it.pt[k] = pt[k];
        items.push_back(it);
      }
    int k = static_cast<int>(cross.size()) - 1;
    for (; k >= 0; --k) {
      if (++sel[static_cast<std::size_t>(k)] < cross[static_cast<std::size_t>(k)].size()) break;
      sel[static_cast<std::size_t>(k)] = 0;
    }
    if (k < 0 || cross.empty()) break;
  }
}

// jumps[r] = max |above - below| over the interface's items (solver.cpp:229-231)
void probe_reduce(const std::vector<double>& vals, std::size_t first, std::size_t count, int max_order,
                  std::vector<double>& jumps) {
  for (std::size_t q = 0; q < count; q += 2) {
    const int r = static_cast<int>((q / 2) % static_cast<std::size_t>(max_order + 1));
    const double d = std::abs(vals[first + q + 1] - vals[first + q]);
    jumps[static_cast<std::size_t>(r)] = std::max(jumps[static_cast<std::size_t>(r)], d);
  }
}

}  // namespace mfb

// ===================================================================== MFDD
struct mfadd_model {
  std::vector<int> degrees;
  std::vector<unsigned char> clamp_left, clamp_right;
  std::vector<double> knots;
  std::vector<std::int64_t> kn_off, ext;
  std::vector<double> bounds;
  std::vector<std::string> keys, values;
  std::vector<const char*> key_ptrs, value_ptrs;
  std::vector<double> controls;
};

namespace {

constexpr char kMagic[4] = {'M', 'F', 'D', 'D'};
constexpr std::uint32_t kVersion = 1;

// MfaModel::validate (model.cpp:11-24)
void validate_model(const mfadd_model_view& m) {
  if (m.rank < 1) throw std::invalid_argument("MfaModel: inconsistent dimension counts");
  for (int d = 0; d < m.rank; ++d) {
    const std::int64_t nk = m.kn_off[d + 1] - m.kn_off[d];
    if (nk - m.degrees[d] - 1 != m.ctrl_ext[d])
      throw std::invalid_argument("MfaModel: control extent must equal #knots - p - 1 in dimension " +
                                  std::to_string(d));
  }
}

// Little-endian scalar writers/readers (model.cpp:56-91; this host is LE).
struct Out {
  std::ofstream f;
  template <class T>
  void put(T v) {
    f.write(reinterpret_cast<const char*>(&v), sizeof(T));
  }
  void str(const std::string& s) {
    put<std::uint32_t>(static_cast<std::uint32_t>(s.size()));
    f.write(s.data(), static_cast<std::streamsize>(s.size()));
  }
};

struct In {
  std::ifstream f;
  template <class T>
  T get() {
    T v{};
    f.read(reinterpret_cast<char*>(&v), sizeof(T));
    if (!f) throw std::runtime_error("read_mfa: truncated payload");
    return v;
  }
  std::string str() {
    const std::uint32_t n = get<std::uint32_t>();
    std::string s(n, '\0');
    f.read(s.data(), n);
    if (!f) throw std::runtime_error("read_mfa: truncated payload");
    return s;
  }
};

void fill_view(const mfadd_model& m, mfadd_model_view& v) {
  v.rank = static_cast<int>(m.degrees.size());
  v.degrees = m.degrees.data();
  v.clamp_left = m.clamp_left.data();
  v.clamp_right = m.clamp_right.data();
  v.knots = m.knots.data();
  v.kn_off = m.kn_off.data();
  v.ctrl_ext = m.ext.data();
  v.bounds = m.bounds.data();
  v.nprov = static_cast<int>(m.keys.size());
  v.prov_keys = m.key_ptrs.data();
  v.prov_values = m.value_ptrs.data();
  v.controls = m.controls.data();
}

}  // namespace

// ===================================================================== C ABI
MFB_API int mfadd_eval_points(mfadd_context* ctx, int rank, const int* degrees, const double* knots,
                              const int64_t* kn_off, const int64_t* ctrl_ext, const int64_t* col_offset,
                              const double* controls, int64_t npts, const double* points, const int* orders,
                              int side_dim, int side, double* out) {
  return guarded([&] {
    ContextScope scope(ctx);
    check_knots(rank, degrees, kn_off);
    if (side_dim >= rank) throw std::invalid_argument("eval_deriv_sided: side dimension out of range");
    std::int64_t nctl = 1;
    mfb::EvalLattice L{};
    for (int k = 0; k < rank; ++k) {
      L.ext[k] = ctrl_ext[k];
      L.coff[k] = col_offset ? col_offset[k] : 0;
      nctl *= ctrl_ext[k];
    }
    std::vector<mfb::EvalItem> items(static_cast<std::size_t>(npts));
    for (std::int64_t i = 0; i < npts; ++i) {
      mfb::EvalItem& it = items[static_cast<std::size_t>(i)];
      it.lat = 0;
      it.side_dim = side_dim;
      it.side = side ? 1 : 0;
      for (int k = 0; k < rank; ++k) {
        it.pt[k] = points[i * rank + k];
        it.ord[k] = orders ? orders[k] : 0;
      }
    }
    DevVec<double> dc(static_cast<std::size_t>(nctl));
    h2d(dc.p, controls, static_cast<std::size_t>(nctl), ctx->stream);
    std::vector<double> vals;
    mfb::eval_items_device(ctx, rank, degrees, knots, kn_off, dc.p, {L}, items, vals);
    std::memcpy(out, vals.data(), vals.size() * sizeof(double));
  });
}

MFB_API int mfadd_basis_funs(mfadd_context* ctx, const double* knots, int nknots, int degree, int64_t n,
                             const double* u, const int* spans, int orders, int* out_spans, double* out) {
  return guarded([&] {
    ContextScope scope(ctx);
    if (degree < 1 || degree > mfb::kMaxDegree)
      throw std::invalid_argument("basis_funs: degree must be in [1, " + std::to_string(mfb::kMaxDegree) + "]");
    if (nknots < 2 * (degree + 1)) throw std::invalid_argument("KnotVector: too few knots");
    if (orders < 0 || orders > degree)  // knots.cpp:133-134
      throw std::invalid_argument("basis_derivs: order must satisfy 0 <= k <= p (got " + std::to_string(orders) + ")");
    const int nb = nknots - degree - 1;
    if (spans)
      for (std::int64_t i = 0; i < n; ++i)
        if (spans[i] < degree || spans[i] >= nb)
          throw std::invalid_argument("basis_funs: span " + std::to_string(spans[i]) + " outside [" +
                                      std::to_string(degree) + ", " + std::to_string(nb) + ")");
    if (n <= 0) return;
    cudaStream_t st = ctx->stream;
    const std::size_t nv = static_cast<std::size_t>(n) * (orders + 1) * (degree + 1);
    DevVec<double> dk(static_cast<std::size_t>(nknots)), du(static_cast<std::size_t>(n)), dout(nv);
    DevVec<int> dsp(static_cast<std::size_t>(n)), dspo(static_cast<std::size_t>(n)), derr(static_cast<std::size_t>(n));
    h2d(dk.p, knots, static_cast<std::size_t>(nknots), st);
    h2d(du.p, u, static_cast<std::size_t>(n), st);
    if (spans) h2d(dsp.p, spans, static_cast<std::size_t>(n), st);
    mfb::k_basis_points<<<static_cast<unsigned>((n + mfb::kEvalThreads - 1) / mfb::kEvalThreads), mfb::kEvalThreads,
                          0, st>>>(dk.p, degree, nb, n, du.p, spans ? dsp.p : nullptr, orders, dspo.p, dout.p, derr.p);
    ctx->launches += 1;
    CK(cudaGetLastError());
    std::vector<int> err(static_cast<std::size_t>(n));
    CK(cudaMemcpyAsync(err.data(), derr.p, err.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out, dout.p, nv * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (out_spans) CK(cudaMemcpyAsync(out_spans, dspo.p, err.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (std::int64_t i = 0; i < n; ++i)  // first failing parameter (knots.cpp:88-90)
      if (err[static_cast<std::size_t>(i)])
        throw std::out_of_range("find_span: parameter " + std::to_string(u[i]) + " outside evaluable range [" +
                                std::to_string(knots[degree]) + ", " + std::to_string(knots[nb]) + "]");
  });
}

MFB_API int mfadd_continuity_jumps(mfadd_context* ctx, int rank, const int* degrees, const double* knots,
                                   const int64_t* kn_off, const int64_t* ctrl_ext, const double* controls, int dim,
                                   double u, int max_order, int cross_samples, double* out) {
  return guarded([&] {
    ContextScope scope(ctx);
    check_knots(rank, degrees, kn_off);
    if (dim < 0 || dim >= rank) throw std::invalid_argument("continuity_jumps: dimension out of range");
    if (max_order >= degrees[dim] + 1) throw std::invalid_argument("continuity_jumps: order exceeds degree");
    if (max_order < 0) throw std::invalid_argument("continuity_jumps: negative order");
    std::vector<std::vector<double>> cross;  // solver.cpp:247-254
    for (int k = 0; k < rank; ++k) {
      if (k == dim) continue;
      std::vector<double> pts;
      for (int s = 0; s < cross_samples; ++s)
        pts.push_back(cross_samples == 1 ? 0.5
                                         : 0.1 + 0.8 * static_cast<double>(s) / static_cast<double>(cross_samples - 1));
      cross.push_back(std::move(pts));
    }
    mfb::EvalLattice L{};
    std::int64_t nctl = 1;
    for (int k = 0; k < rank; ++k) {
      L.ext[k] = ctrl_ext[k];
      nctl *= ctrl_ext[k];
    }
    std::vector<mfb::EvalItem> items;
    mfb::probe_items(rank, dim, u, max_order, cross, 0, 0, items);
    DevVec<double> dc(static_cast<std::size_t>(nctl));
    h2d(dc.p, controls, static_cast<std::size_t>(nctl), ctx->stream);
    std::vector<double> vals;
    mfb::eval_items_device(ctx, rank, degrees, knots, kn_off, dc.p, {L}, items, vals);
    std::vector<double> jumps(static_cast<std::size_t>(max_order) + 1, 0.0);
    mfb::probe_reduce(vals, 0, vals.size(), max_order, jumps);
    std::memcpy(out, jumps.data(), jumps.size() * sizeof(double));
  });
}

MFB_API int mfadd_decode_grid(mfadd_context* ctx, int rank, int degree, const double* knots, const int64_t* kn_off,
                              const int64_t* ctrl_ext, const double* controls, const int64_t* res, double* out) {
  std::vector<double> params;
  std::vector<int64_t> pm_off(1, 0);
  const int rc = guarded([&] {  // model.cpp:39-49
    if (rank < 1 || rank > 3) throw std::invalid_argument("decode_grid: resolution rank mismatch");
    for (int d = 0; d < rank; ++d) {
      if (res[d] < 2) throw std::invalid_argument("decode_grid: need at least 2 points per dimension");
      for (std::int64_t j = 0; j < res[d]; ++j)
        params.push_back(static_cast<double>(j) / static_cast<double>(res[d] - 1));
      pm_off.push_back(static_cast<int64_t>(params.size()));
    }
  });
  if (rc != MFADD_OK) return rc;
  return mfadd_decode(ctx, rank, degree, knots, kn_off, params.data(), pm_off.data(), ctrl_ext, nullptr, controls, out);
}

MFB_API int mfadd_read_raw_grid(mfadd_context* ctx, const char* path, int rank, const int64_t* dims, int type,
                                int byte_order, double* out, int out_on_device) {
  return guarded([&] {  // field.cpp:149-191
    ContextScope scope(ctx);
    if (rank < 1) throw std::invalid_argument("read_raw_grid: dims required");
    std::int64_t count = 1;
    for (int d = 0; d < rank; ++d) {
      if (dims[d] < 1) throw std::invalid_argument("read_raw_grid: dims must be positive");
      count *= dims[d];
    }
    const int width = type == MFADD_RAW_F32 ? 4 : 8;
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error(std::string("read_raw_grid: cannot open ") + path);
    in.seekg(0, std::ios::end);
    const std::int64_t actual = static_cast<std::int64_t>(in.tellg());
    const std::int64_t expected = count * width;
    if (actual != expected)
      throw std::runtime_error(std::string("read_raw_grid: size mismatch for ") + path + ": expected " +
                               std::to_string(expected) + " bytes (" + std::to_string(count) + " values), found " +
                               std::to_string(actual));
    in.seekg(0);
    cudaStream_t st = ctx->stream;
    unsigned char* host = nullptr;
    CK(cudaMallocHost(&host, static_cast<std::size_t>(expected)));
    std::unique_ptr<unsigned char, cudaError_t (*)(void*)> hold(host, cudaFreeHost);
    in.read(reinterpret_cast<char*>(host), expected);
    if (!in) throw std::runtime_error(std::string("read_raw_grid: short read from ") + path);
    DevVec<unsigned char> raw(static_cast<std::size_t>(expected));
    CK(cudaMemcpyAsync(raw.p, host, static_cast<std::size_t>(expected), cudaMemcpyHostToDevice, st));
    std::unique_ptr<DevVec<double>> tmp;
    double* dst = out;
    if (!out_on_device) {
      tmp = std::make_unique<DevVec<double>>(static_cast<std::size_t>(count));
      dst = tmp->p;
    }
    const int swap = (byte_order == MFADD_RAW_BIG) ? 1 : 0;  // this host is little-endian
    ctx->launches += mfb::launch_raw_to_f64(raw.p, count, width, swap, dst, st);
    CK(cudaGetLastError());
    if (!out_on_device)
      CK(cudaMemcpyAsync(out, dst, static_cast<std::size_t>(count) * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

MFB_API int mfadd_write_mfa(const char* path, const mfadd_model_view* m) {
  return guarded([&] {  // model.cpp:93-118
    if (!m) throw std::invalid_argument("write_mfa: null model");
    validate_model(*m);
    std::map<std::string, std::string> prov;  // std::map order, last assignment wins
    for (int i = 0; i < m->nprov; ++i) prov[m->prov_keys[i]] = m->prov_values[i];
    Out o;
    o.f.open(path, std::ios::binary | std::ios::trunc);
    if (!o.f) throw std::runtime_error(std::string("write_mfa: cannot open ") + path);
    o.f.write(kMagic, 4);
    o.put<std::uint32_t>(kVersion);
    o.put<std::uint32_t>(static_cast<std::uint32_t>(m->rank));
    for (int d = 0; d < m->rank; ++d) {
      o.put<std::uint32_t>(static_cast<std::uint32_t>(m->degrees[d]));
      o.put<std::uint8_t>(m->clamp_left ? (m->clamp_left[d] ? 1 : 0) : 1);
      o.put<std::uint8_t>(m->clamp_right ? (m->clamp_right[d] ? 1 : 0) : 1);
      o.put<std::uint64_t>(static_cast<std::uint64_t>(m->kn_off[d + 1] - m->kn_off[d]));
      o.put<std::uint64_t>(static_cast<std::uint64_t>(m->ctrl_ext[d]));
      o.put<double>(m->bounds ? m->bounds[2 * d] : 0.0);
      o.put<double>(m->bounds ? m->bounds[2 * d + 1] : 1.0);
    }
    o.put<std::uint32_t>(static_cast<std::uint32_t>(prov.size()));
    for (const auto& [k, v] : prov) {
      o.str(k);
      o.str(v);
    }
    o.f.write(reinterpret_cast<const char*>(m->knots), static_cast<std::streamsize>(m->kn_off[m->rank] * 8));
    std::int64_t n = 1;
    for (int d = 0; d < m->rank; ++d) n *= m->ctrl_ext[d];
    o.f.write(reinterpret_cast<const char*>(m->controls), static_cast<std::streamsize>(n * 8));
    if (!o.f) throw std::runtime_error(std::string("write_mfa: write failed for ") + path);
  });
}

MFB_API int mfadd_read_mfa(const char* path, mfadd_model** out) {
  return guarded([&] {  // model.cpp:120-167
    In in;
    in.f.open(path, std::ios::binary);
    if (!in.f) throw std::runtime_error(std::string("read_mfa: cannot open ") + path);
    char magic[4];
    in.f.read(magic, 4);
    if (!in.f || std::memcmp(magic, kMagic, 4) != 0) throw std::runtime_error(std::string("read_mfa: bad magic in ") + path);
    const std::uint32_t version = in.get<std::uint32_t>();
    if (version != kVersion)
      throw std::runtime_error("read_mfa: unsupported format version " + std::to_string(version) + " (expected " +
                               std::to_string(kVersion) + ")");
    auto m = std::make_unique<mfadd_model>();
    const std::uint32_t d = in.get<std::uint32_t>();
    if (d < 1 || d > 3) throw std::runtime_error("read_mfa: unsupported dimension count");
    std::vector<std::uint64_t> nk(d);
    for (std::uint32_t k = 0; k < d; ++k) {
      m->degrees.push_back(static_cast<int>(in.get<std::uint32_t>()));
      m->clamp_left.push_back(in.get<std::uint8_t>() != 0 ? 1 : 0);
      m->clamp_right.push_back(in.get<std::uint8_t>() != 0 ? 1 : 0);
      nk[k] = in.get<std::uint64_t>();
      m->ext.push_back(static_cast<std::int64_t>(in.get<std::uint64_t>()));
      const double b0 = in.get<double>();
      const double b1 = in.get<double>();
      m->bounds.push_back(b0);
      m->bounds.push_back(b1);
    }
    const std::uint32_t nprov = in.get<std::uint32_t>();
    std::map<std::string, std::string> prov;
    for (std::uint32_t i = 0; i < nprov; ++i) {
      std::string key = in.str();
      prov[key] = in.str();
    }
    for (auto& [k, v] : prov) {
      m->keys.push_back(k);
      m->values.push_back(v);
    }
    m->kn_off.push_back(0);
    for (std::uint32_t k = 0; k < d; ++k) {
      for (std::uint64_t i = 0; i < nk[k]; ++i) m->knots.push_back(in.get<double>());
      m->kn_off.push_back(static_cast<std::int64_t>(m->knots.size()));
    }
    std::int64_t n = 1;
    for (std::int64_t e : m->ext) n *= e;
    m->controls.resize(static_cast<std::size_t>(n));
    for (std::int64_t i = 0; i < n; ++i) m->controls[static_cast<std::size_t>(i)] = in.get<double>();
    for (auto& k : m->keys) m->key_ptrs.push_back(k.c_str());
    for (auto& v : m->values) m->value_ptrs.push_back(v.c_str());
    mfadd_model_view v{};
    fill_view(*m, v);
    validate_model(v);
    *out = m.release();
  });
}

MFB_API int mfadd_model_view_of(const mfadd_model* m, mfadd_model_view* out) {
  return guarded([&] {
    if (!m || !out) throw std::invalid_argument("mfadd_model_view_of: null argument");
    fill_view(*m, *out);
  });
}

MFB_API void mfadd_model_free(mfadd_model* m) { delete m; }
