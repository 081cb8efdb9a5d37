// engine.cu — C ABI (include/mfadd_b200.h) of the B200-native MFA encode
// path: plan construction (device tables from the host decomposition) and
// the solve() orchestration (solver.cpp:332-440) over the sm_100a kernels in
// kernels.cu.  No CPU fallback: every value of SolveResult is produced on the
// GPU; the host only builds integer metadata tables at plan time and reads
// back scalars.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <thread>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/mfadd_b200.h"
#include "dev.cuh"
#include "kernels.cuh"
#include "layout.hpp"

using mfb::AxisProb;
using mfb::BlockDev;
using mfb::Decomp;

#include "abi.hpp"

using namespace mfb_abi;

namespace mfb_abi {
thread_local std::string g_err;
thread_local int g_err_dim = -1;
thread_local std::int64_t g_err_span = -1;
}  // namespace mfb_abi

namespace {

#define CK(x) cuda_check((x), #x)
#define NCK(x)                                                                                   \
  do {                                                                                           \
    const ncclResult_t r_ = (x);                                                                 \
    if (r_ != ncclSuccess) throw ApiError(MFADD_ECUDA, std::string(#x) + ": " + ncclGetErrorString(r_)); \
  } while (0)

// Owning device buffer.
template <class T>
struct DBuf {
  T* p = nullptr;
  std::size_t n = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() {
    if (p) cudaFree(p);
  }
  void alloc(std::size_t count) {
    if (p) cudaFree(p);
    p = nullptr;
    n = count;
    if (count == 0) return;
    const cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
      p = nullptr;
      throw ApiError(MFADD_ENOMEM, "cudaMalloc(" + std::to_string(count * sizeof(T)) + " bytes) failed: " +
                                       cudaGetErrorString(e));
    }
  }
  void upload(const std::vector<T>& h, cudaStream_t s) {
    alloc(h.size());
    if (!h.empty()) CK(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
  }
};

// Host binary search with the find_span rule (knots.cpp:83-106) — used only
// to size the decode kernel's shared-memory control box at plan time.
int host_find_span(const std::vector<double>& kn, int p, double u) {
  const int n = static_cast<int>(kn.size()) - p - 1;
  if (u >= kn[static_cast<std::size_t>(n)]) {
    int s = n - 1;
    while (s > p && kn[static_cast<std::size_t>(s)] == kn[static_cast<std::size_t>(s) + 1]) --s;
    return s;
  }
  if (u <= kn[static_cast<std::size_t>(p)]) return p;
  int low = p, high = n, mid = (low + high) / 2;
  while (u < kn[static_cast<std::size_t>(mid)] || u >= kn[static_cast<std::size_t>(mid) + 1]) {
    if (u < kn[static_cast<std::size_t>(mid)])
      high = mid;
    else
      low = mid;
    mid = (low + high) / 2;
  }
  return mid;
}

constexpr int kRowPad = 64;  // rows of slack after every row table (bulk copies read whole chunks)

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      throw ApiError(MFADD_ECUDA, "cuTensorMapEncodeTiled entry point unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// Tiled fp64 tensor map over a row-major array; dims/box innermost first.
CUtensorMap make_tmap(const double* base, int rank, const std::uint64_t* dims, const std::uint32_t* box,
                      CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_NONE) {
  CUtensorMap m;
  std::uint64_t strides[3] = {0, 0, 0};
  std::uint64_t st = 8;
  for (int i = 0; i + 1 < rank; ++i) {
    st *= dims[i];
    strides[i] = st;
  }
  const std::uint32_t estr[3] = {1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, static_cast<cuuint32_t>(rank),
                                 const_cast<double*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw ApiError(MFADD_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

int round_up(int x, int a) { return (x + a - 1) / a * a; }

}  // namespace

// ===================================================================== types
struct mfadd_decomposition {
  Decomp d;
};


namespace {


// Optional per-kernel CUDA-event timeline (bench roofline / phase evidence).
struct Timeline {
  struct Rec {
    std::string name;
    cudaEvent_t a = nullptr, b = nullptr;
  };
  bool on = false;
  std::vector<Rec> recs;
  std::size_t used = 0;
  cudaStream_t st = nullptr;
  ~Timeline() {
    for (auto& r : recs) {
      if (r.a) cudaEventDestroy(r.a);
      if (r.b) cudaEventDestroy(r.b);
    }
  }
  void reset(cudaStream_t s) {
    used = 0;
    st = s;
  }
  // MFADD_SYNC_CHECK=1: synchronise after every kernel and name the failing one.
  const char* cur = "";
  bool sync_check = std::getenv("MFADD_SYNC_CHECK") != nullptr;
  void begin(const char* name) {
    cur = name;
    if (!on) return;
    if (used == recs.size()) {
      recs.emplace_back();
      CK(cudaEventCreate(&recs.back().a));
      CK(cudaEventCreate(&recs.back().b));
    }
    recs[used].name = name;
    CK(cudaEventRecord(recs[used].a, st));
  }
  void end() {
    if (sync_check) {
      const cudaError_t e = cudaStreamSynchronize(st);
      if (e != cudaSuccess) throw ApiError(MFADD_ECUDA, std::string("kernel ") + cur + ": " + cudaGetErrorString(e));
      if (const int line = mfb::debug_fail_line())
        throw ApiError(MFADD_ECUDA, std::string("kernel ") + cur + ": bounds check failed at kernels.cu:" + std::to_string(line));
      if (const int line = mfb::debug_fail_line_tma())
        throw ApiError(MFADD_ECUDA, std::string("kernel ") + cur + ": check failed at stream_tma.cu:" + std::to_string(line));
    }
    if (!on) return;
    CK(cudaEventRecord(recs[used].b, st));
    ++used;
  }
};

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// Device tables for a batch of local problems sharing one degree: the fit
// machinery of both solve() and fit_unconstrained().
struct Workload {
  int D = 0, p = 0;
  std::vector<AxisProb> probs;
  std::vector<BlockDev> blocks;
  std::vector<int> factor_ids;
  std::int64_t total_rows = 0, total_cols = 0, total_p = 0, total_t1 = 0, total_t2 = 0;
  std::int64_t fs[3] = {0, 0, 0};
  std::int64_t field_n = 0;  // elements of the field buffer the fit reads
  int max_m = 0, max_n_factor = 0;
  int max_lines_strided[3] = {0, 0, 0};
  int max_lines_last = 0;
  std::int64_t pitch_last = 1;

  DBuf<double> knots, params;
  DBuf<AxisProb> d_probs;
  DBuf<BlockDev> d_blocks;
  DBuf<int> d_factor, g0, first_col, count;
  DBuf<double> vals, ltab, t1, t2, P, Y, rlt, twf;
  std::int64_t rlt_stride = 0, twf_stride = 0;
  bool tw2d = false;  // k_solve2d runs the twisted (two-sided) passes
  // D = 3: every pass a pure contraction and one CTA per block solves all three axes (k_solve3d)
  bool fuse3d = false;
  int s3_n[3] = {0, 0, 0}, s3_zs = 0, s3_threads = 0, s3_slab = 0, s3_nslab = 0, s3_nl = 1, a0_slab = 0, a0_zr = 0;
  DBuf<unsigned long long> linf_int;
  DBuf<unsigned char> sflag;
  std::int64_t sflag_off[3] = {0, 0, 0};
  // TMA axis-0 pass (field row strides must be 16-B multiples)
  bool tma_axis0 = false;
  mfb::TmaGeom axis0_geo{1, 1, 16, 4, 0};
  int axis0_tiles = 0;
  // TMA last-axis pass (D >= 2)
  // axis-0 sweep as a pure contraction (defer 2): Gram/Cholesky on a side
  // stream, overlapping the sweep (fork after the basis rows, join before the
  // first pass that needs a factor)
  int defer_mode = 0;
  cudaStream_t side = nullptr;
  cudaEvent_t ev_rows = nullptr, ev_rows2 = nullptr, ev_chol = nullptr;
  bool rows_split = false;  // the non-axis-0 rows are built on the side stream (joined before the last axis)
  ~Workload() {
    if (ev_rows) cudaEventDestroy(ev_rows);
    if (ev_chol) cudaEventDestroy(ev_chol);
    if (ev_rows2) cudaEventDestroy(ev_rows2);
    if (side) cudaStreamDestroy(side);
  }
  bool tma_mid = false;  // D = 3 middle axis through a T1 tensor map
  mfb::TmaGeom mid_geo{1, 1, 8, 4, 0};
  int mid_tiles = 0, mid_n0 = 0;
  bool tma_last = false;
  int last_LT = 128, last_ltcap = 0, last_kseg = 1;
  std::vector<int> segtab;  // kSegStride ints per axis problem (last-axis problems filled)
  DBuf<int> d_segtab;
  std::int64_t zhalf = 0;  // one parity half of the last-axis contraction buffer
  std::array<std::int64_t, 3> field_dims{1, 1, 1};  // global field extents (solver) for the tensor map

  void plan_tma(bool enable) {
    tma_axis0 = false;
    if (!enable || D < 2 || std::getenv("MFADD_NO_TMA")) return;
    int mx1 = 0, mx2 = 0;
    for (const auto& b : blocks) {
      mx1 = std::max(mx1, probs[static_cast<std::size_t>(b.ax[1])].m);
      if (D == 3) mx2 = std::max(mx2, probs[static_cast<std::size_t>(b.ax[2])].m);
    }
    if (field_dims[static_cast<std::size_t>(D - 1)] % 2 != 0) return;  // row stride not 16-B aligned
    // B2 is the TMA box width W (even); it includes one spare column so the
    // box can start on an even (16-B aligned) column (stream_tma.cu).
    if (D == 2) {
      // columns per CTA (threads = cols + 2): 144 -> four tiles of a C5 block,
      // seven CTAs per SM with a 3-stage ring (one wave for 256 blocks)
      const int wmax = env_int("MFADD_AX0_COLS", 144);
      const int nt = (mx1 + wmax - 1) / wmax;
      const int cols = round_up((mx1 + nt - 1) / nt, 2);
      axis0_geo.B2 = cols + 2;
      axis0_geo.B1 = 1;
      axis0_tiles = (mx1 + cols - 1) / cols;
    } else {
      if (mx2 + 1 > 256) return;
      axis0_geo.B2 = round_up(mx2 + 1, 2);
      axis0_geo.B1 = std::max(1, env_int("MFADD_AX0_B1", 256 / axis0_geo.B2));
      axis0_tiles = (mx1 + axis0_geo.B1 - 1) / axis0_geo.B1;
    }
    axis0_geo.R = 8;
    axis0_geo.S = env_int("MFADD_FIT_S", 3);
    int mxn = 0;
    for (const auto& b : blocks) mxn = std::max(mxn, probs[static_cast<std::size_t>(b.ax[0])].n);
    const int need = (mxn + 2 * (p + 1)) * (2 * p + 1);  // padded Cholesky table in smem
    if (need > 6144) return;                             // > 48 KB: generic kernel
    axis0_geo.lt_cap = need;
    tma_axis0 = true;
    // last axis: LT lines per CTA (<= 256, multiple of 32), padded L table in smem
    int mxnl = 0;
    for (const auto& b : blocks) mxnl = std::max(mxnl, probs[static_cast<std::size_t>(b.ax[D - 1])].n);
    const int needl = (mxnl + 2 * (p + 1)) * (2 * p + 1);
    if (needl <= 6144 && max_lines_last > 0 && !std::getenv("MFADD_NO_TMA_LAST")) {
      const int ncta = std::max((max_lines_last + 255) / 256, env_int("MFADD_LAST_LSPLIT", 1));  // CTAs per block-segment
      last_LT = round_up((max_lines_last + ncta - 1) / ncta, 32);  // whole warps
      last_ltcap = needl;
      tma_last = true;
      plan_segments();
    }
    // Axis-0 solve deferred to the held lattices (stream_tma.cu k_axis0_backsub):
    // 2 = the sweep only contracts (Gram/Cholesky overlap it), 1 = only the
    // back substitution is deferred, 0 = fused (MFADD_DEFER overrides).
    if (tma_last) defer_mode = std::getenv("MFADD_DEFER") ? std::atoi(std::getenv("MFADD_DEFER")) : 2;
    // D = 3 middle axis: per (block, c0) slice of T1 = [m1 rows][pitch]
    if (D == 3 && !std::getenv("MFADD_NO_TMA_MID")) {
      int mx = 0, mxn1 = 0, mxn0 = 0;
      for (const auto& b : blocks) {
        mx = std::max(mx, probs[static_cast<std::size_t>(b.ax[2])].m);
        mxn1 = std::max(mxn1, probs[static_cast<std::size_t>(b.ax[1])].n);
        mxn0 = std::max(mxn0, probs[static_cast<std::size_t>(b.ax[0])].n);
      }
      const int needm = (mxn1 + 2 * (p + 1)) * (2 * p + 1);
      if (needm <= 6144) {
        const int nt = (mx + 253) / 254;
        const int cols = round_up((mx + nt - 1) / nt, 2);
        mid_geo = mfb::TmaGeom{1, cols + 2, 8, 4, needm};
        mid_tiles = (mx + cols - 1) / cols;
        mid_n0 = mxn0;
        tma_mid = true;
      }
    }
  }

  // Row segments of the last-axis problems: about 2 contraction threads per
  // SM thread slot over all lines, segments of >= 64 rows on 16-row chunk
  // boundaries; carries sized per block.
  void plan_segments() {
    std::int64_t lines = 0;
    for (const auto& b : blocks) {
      std::int64_t Ll = 1;
      for (int k = 0; k + 1 < D; ++k) Ll *= probs[static_cast<std::size_t>(b.ax[k])].n;
      lines += round_up(static_cast<int>(Ll), last_LT);
    }
    // ~2 contraction threads per SM thread slot over all lines (C5: two
    // segments; more segments add carries and a partial second wave)
    const int want = static_cast<int>(std::lround(2.0 * 148 * 256 / static_cast<double>(std::max<std::int64_t>(lines, 1))));
    segtab.assign(probs.size() * mfb::kSegStride, 0);
    last_kseg = 1;
    for (const auto& b : blocks) {
      const int pid = b.ax[D - 1];
      const AxisProb& pr = probs[static_cast<std::size_t>(pid)];
      static const int kforce = env_int("MFADD_LAST_SEGS", 0);  // measurement aid
      int K = std::max(1, std::min({kforce > 0 ? kforce : want, mfb::kMaxSeg, pr.m / 64}));
      // a segment must span more than P+1 columns so that carry ranges of
      // consecutive boundaries never overlap
      while (K > 1 && static_cast<std::int64_t>(pr.n) < static_cast<std::int64_t>(K) * 4 * (p + 1)) --K;
      int* t = segtab.data() + static_cast<std::size_t>(pid) * mfb::kSegStride;
      t[0] = K;
      for (int sgi = 0; sgi <= K; ++sgi)
        t[1 + sgi] = sgi == K ? pr.m : std::min(pr.m, (static_cast<int>(static_cast<std::int64_t>(pr.m) * sgi / K) + 8) / 16 * 16);
      last_kseg = std::max(last_kseg, K);
    }
    zhalf = 0;
    for (auto& b : blocks) {
      std::int64_t Ll = 1;
      for (int k = 0; k + 1 < D; ++k) Ll *= probs[static_cast<std::size_t>(b.ax[k])].n;
      // column pitch: even (16-B aligned bulk copies of columns) and = 2 mod 4
      // (k_solve2d's column-parallel phase then has at most 2-way conflicts)
      b.zl = static_cast<int>((Ll + 1) / 4 * 4 + 2);
      b.zoff = zhalf;
      zhalf += (probs[static_cast<std::size_t>(b.ax[D - 1])].n + 2 * (p + 1)) * b.zl;
    }
  }

  // Derive offsets/sizes from probs + blocks (row/col offsets, intermediates).
  void layout_tables() {
    total_rows = 0;
    total_cols = 0;
    max_m = 0;
    for (auto& pr : probs) {  // 4-row aligned (16-B bulk copies of g0 / vals)
      pr.row_off = total_rows;
      total_rows = (total_rows + pr.m + 3) / 4 * 4;
      max_m = std::max(max_m, pr.m);
    }
    total_rows += kRowPad;
    std::vector<char> is_factor(probs.size(), 0);
    for (int id : factor_ids) is_factor[static_cast<std::size_t>(id)] = 1;
    max_n_factor = 0;
    for (std::size_t i = 0; i < probs.size(); ++i) {
      probs[i].col_off = total_cols;
      if (is_factor[i]) {
        total_cols += probs[i].n;
        max_n_factor = std::max(max_n_factor, probs[i].n);
      }
    }
    total_p = total_t1 = total_t2 = 0;
    for (auto& mx : max_lines_strided) mx = 0;
    max_lines_last = 0;
    pitch_last = 1;
    if (D >= 2)
      for (const auto& b : blocks)
        pitch_last = std::max<std::int64_t>(pitch_last, probs[static_cast<std::size_t>(b.ax[D - 1])].m);
    pitch_last = (pitch_last + 1) / 2 * 2;  // even: 16-B aligned rows (TMA)
    for (auto& b : blocks) {
      std::int64_t np = 1;
      std::array<std::int64_t, 3> m{1, 1, 1}, n{1, 1, 1};
      for (int k = 0; k < D; ++k) {
        m[k] = probs[static_cast<std::size_t>(b.ax[k])].m;
        n[k] = probs[static_cast<std::size_t>(b.ax[k])].n;
        np *= n[k];
      }
      b.poff = total_p;
      total_p += np;
      b.t1off = total_t1;
      b.t2off = total_t2;
      if (D == 2) total_t1 += n[0] * pitch_last;
      if (D == 3) total_t1 += n[0] * m[1] * pitch_last;  // [n0][m1][pitch]
      if (D == 3) total_t2 += n[0] * n[1] * pitch_last;
      for (int d = 0; d + 1 < D; ++d) {
        std::int64_t L = 1, Tr = 1;
        for (int k = 0; k < D; ++k) {
          if (k < d) L *= n[k];
          if (k > d) Tr *= m[k];
        }
        max_lines_strided[d] = static_cast<int>(std::max<std::int64_t>(max_lines_strided[d], L * Tr));
      }
      std::int64_t Ll = 1;
      for (int k = 0; k + 1 < D; ++k) Ll *= n[k];
      max_lines_last = static_cast<int>(std::max<std::int64_t>(max_lines_last, Ll));
    }
  }

  void allocate(cudaStream_t s) {
    d_probs.upload(probs, s);
    d_blocks.upload(blocks, s);
    d_factor.upload(factor_ids, s);
    g0.alloc(static_cast<std::size_t>(total_rows));
    first_col.alloc(static_cast<std::size_t>(total_rows));
    count.alloc(static_cast<std::size_t>(total_rows));
    vals.alloc(static_cast<std::size_t>(total_rows * (p + 1)));
    ltab.alloc(static_cast<std::size_t>(std::max<std::int64_t>(total_cols, 1) * (2 * p + 1)));
    // k_solve2d's twisted passes (MFADD_TWIST=1; measured slower than the plain
    // passes on C5, see k_solve2d_tw): every factored extent long enough and
    // the CTA's tile + side buffers within shared memory
    tw2d = false;
    if (D == 2 && tma_last && std::getenv("MFADD_TWIST") && !std::getenv("MFADD_NO_FUSE2D")) {
      int mn0 = 0, mn1 = 0, mzl = 0;
      bool ok = !blocks.empty();
      for (const auto& b : blocks) {
        mn0 = std::max(mn0, probs[static_cast<std::size_t>(b.ax[0])].n);
        mn1 = std::max(mn1, probs[static_cast<std::size_t>(b.ax[1])].n);
        mzl = std::max(mzl, b.zl);
      }
      for (int id : factor_ids) ok = ok && mfb::tw_ok(probs[static_cast<std::size_t>(id)].n, p);
      tw2d = ok && mfb::solve2d_smem(p, mn0, mn1, mzl, last_kseg, true) > 0;
    }
    fuse3d = false;
    if (D == 3 && defer_mode == 2 && tma_last && tma_mid && tma_axis0 && !blocks.empty() &&
        !std::getenv("MFADD_NO_FUSE3D")) {
      s3_n[0] = s3_n[1] = s3_n[2] = 0;
      bool n1_odd = false;
      for (const auto& b : blocks)
        for (int k = 0; k < 3; ++k) {
          const int nk = probs[static_cast<std::size_t>(b.ax[k])].n;
          s3_n[k] = std::max(s3_n[k], nk);
          if (k == 1 && (nk & 1)) n1_odd = true;
        }
      // slab = axis-0 indices per CTA: the whole block when it fits one CTA,
      // else ~224 lines (column runs start 16-B aligned: an even line count)
      auto pitch = [&](int slab) { return (slab * s3_n[1] + 1) / 4 * 4 + 2; };
      auto fits = [&](int slab, std::size_t cap) {
        const std::size_t b = mfb::solve3d_smem(p, s3_n[0], s3_n[1], s3_n[2], pitch(slab), last_kseg);
        return b > 0 && b <= cap;
      };
      int slab = s3_n[0];
      if (!fits(slab, 227 * 1024) || std::getenv("MFADD_S3_SLAB")) {
        slab = std::max(1, env_int("MFADD_S3_SLAB", std::max(1, 224 / s3_n[1])));
        if (n1_odd) slab = std::max(2, slab & ~1);
        while (slab > (n1_odd ? 2 : 1) && !fits(slab, static_cast<std::size_t>(env_int("MFADD_S3_KB", 75)) * 1024))
          slab -= n1_odd ? 2 : 1;
      }
      slab = std::min(slab, s3_n[0]);
      fuse3d = fits(slab, 227 * 1024) && (slab == s3_n[0] || !n1_odd || slab % 2 == 0);
      s3_slab = slab;
      s3_nslab = (s3_n[0] + slab - 1) / slab;
      s3_zs = pitch(slab);
      const int lines = std::max({slab * s3_n[1], slab * s3_n[2], s3_nslab == 1 ? s3_n[1] * s3_n[2] : 1});
      s3_threads = std::min(640, std::max(128, (lines + 31) / 32 * 32));
      // four lines per thread where the slabs fill the GPU many times over
      std::int64_t all_lines = 0;
      for (const auto& b : blocks)
        all_lines += static_cast<std::int64_t>(probs[static_cast<std::size_t>(b.ax[0])].n) * probs[static_cast<std::size_t>(b.ax[1])].n;
      s3_nl = env_int("MFADD_S3_NL", all_lines >= 2048 * 148 ? 4 : 1);
      // the axis-0 solve on i1 slabs of ~224 lines in place of the strided
      // walkers (C4: last-axis group 440 -> 402 us, C3 95.9 -> 91.2 us);
      // MFADD_A0_SLAB sets the slab, MFADD_NO_A0_SLAB keeps the walkers
      a0_slab = 0;
      if (fuse3d && s3_nslab > 1 && !std::getenv("MFADD_NO_A0_SLAB")) {
        int sl = std::min(s3_n[1], std::max(1, env_int("MFADD_A0_SLAB", std::max(1, 224 / s3_n[2]))));
        while (sl > 1 && (mfb::axis0_slab_smem(p, s3_n[0], sl * s3_n[2]) == 0 ||
                          mfb::axis0_slab_smem(p, s3_n[0], sl * s3_n[2]) > static_cast<std::size_t>(env_int("MFADD_S3_KB", 75)) * 1024))
          --sl;
        if (mfb::axis0_slab_smem(p, s3_n[0], sl * s3_n[2]) > 0) {
          a0_slab = sl;
          a0_zr = (sl * s3_n[2] + 1) & ~1;
        }
      }
    }
    rlt_stride = (mfb::rl_table_doubles(p, max_n_factor, tw2d) + 1) / 2 * 2;  // even: 16-B aligned per problem
    rlt.alloc(static_cast<std::size_t>(probs.size() * rlt_stride));
    if (tw2d) {
      twf_stride = 2 * static_cast<std::int64_t>(max_n_factor) * (p + 1);
      twf.alloc(static_cast<std::size_t>(probs.size() * twf_stride));
    }
    t1.alloc(static_cast<std::size_t>(total_t1));
    t2.alloc(static_cast<std::size_t>(total_t2));
    P.alloc(static_cast<std::size_t>(total_p));
    Y.alloc(static_cast<std::size_t>(tma_last ? 2 * zhalf + total_p : total_p));
    linf_int.alloc(blocks.size());
    if (tma_last) d_segtab.upload(segtab, s);
  }

  // K1 + K2
  int setup(mfadd_context* ctx, Timeline* tl = nullptr) {
    Timeline dummy;
    dummy.st = ctx->stream;
    if (!tl) tl = &dummy;
    static const bool chol_inline = std::getenv("MFADD_CHOL_INLINE") != nullptr;  // measurement aid
    const bool fork = defer_mode == 2 && !chol_inline;
    // With the side stream, only the axis-0 problems' rows (the first ones:
    // what the axis-0 sweep reads) are built before the sweep; the rest are
    // built on the side stream ahead of the factorizations and joined before
    // the last-axis contraction.
    int n0p = 0;
    rows_split = false;
    if (fork && D >= 2) {
      int lo_other = 1 << 30;
      for (const auto& b : blocks) {
        n0p = std::max(n0p, b.ax[0] + 1);
        for (int k = 1; k < D; ++k) lo_other = std::min(lo_other, b.ax[k]);
      }
      rows_split = n0p < static_cast<int>(probs.size()) && lo_other >= n0p;
    }
    auto rows_args = [&](int lo, int hi) {
      int mm = 0;
      for (int i = lo; i < hi; ++i) mm = std::max(mm, probs[static_cast<std::size_t>(i)].m);
      return mfb::RowsArgs{d_probs.p, hi - lo, mm, knots.p, params.p, g0.p, first_col.p, count.p, vals.p,
                           ctx->d_status, lo};
    };
    tl->begin("basis_rows");
    int l = mfb::launch_basis_rows(p, rows_split ? rows_args(0, n0p) : rows_args(0, static_cast<int>(probs.size())),
                                   ctx->stream);
    tl->end();
    int max_m_factor = 0;
    for (int id : factor_ids) max_m_factor = std::max(max_m_factor, probs[static_cast<std::size_t>(id)].m);
    mfb::CholArgs ca{d_probs.p, d_factor.p, static_cast<int>(factor_ids.size()), max_n_factor, max_m_factor, 0, 0,
                     g0.p, vals.p, ltab.p, ctx->d_status};
    if (tw2d) {
      ca.tw = twf.p;
      ca.tw_stride = twf_stride;
    }
    if (fork) {  // the factorizations run beside the axis-0 sweep
      if (!side) {
        CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&ev_rows, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_rows2, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_chol, cudaEventDisableTiming));
      }
      CK(cudaEventRecord(ev_rows, ctx->stream));
      CK(cudaStreamWaitEvent(side, ev_rows, 0));
      cudaStream_t main_st = tl->st;
      tl->st = side;
      static const bool heavy = std::getenv("MFADD_CHOL_HEAVY") != nullptr;  // measurement aid
      ca.light = heavy ? 0 : 1;
      tl->begin("gram_chol");
      if (rows_split) {
        l += mfb::launch_basis_rows(p, rows_args(n0p, static_cast<int>(probs.size())), side);
        CK(cudaEventRecord(ev_rows2, side));
      }
      l += mfb::launch_gram_chol(p, ca, side);
      if ((D == 2 && tma_last) || fuse3d) l += mfb::launch_rl_tables(p, ca, rlt.p, rlt_stride, side, tw2d);
      tl->end();
      tl->st = main_st;
      CK(cudaEventRecord(ev_chol, side));
    } else {
      tl->begin("gram_chol");
      l += mfb::launch_gram_chol(p, ca, ctx->stream);
      if ((D == 2 && tma_last) || fuse3d) l += mfb::launch_rl_tables(p, ca, rlt.p, rlt_stride, ctx->stream, tw2d);
      tl->end();
    }
    CK(cudaGetLastError());
    return l;
  }

  // K3
  int fit(mfadd_context* ctx, const double* field, Timeline* tl = nullptr) {
    Timeline dummy;
    dummy.st = ctx->stream;
    if (!tl) tl = &dummy;
    CK(cudaMemsetAsync(linf_int.p, 0, blocks.size() * sizeof(unsigned long long), ctx->stream));
    mfb::FitArgs fa{};
    fa.D = D;
    for (int k = 0; k < 3; ++k) fa.fs[k] = fs[k];
    fa.field = field;
    fa.blocks = d_blocks.p;
    fa.nblocks = static_cast<int>(blocks.size());
    fa.probs = d_probs.p;
    fa.g0 = g0.p;
    fa.vals = vals.p;
    fa.ltab = ltab.p;
    fa.t1 = t1.p;
    fa.t2 = t2.p;
    fa.P = P.p;
    fa.Y = Y.p;
    fa.linf_int = linf_int.p;
    fa.shared_flag = sflag.p;
    for (int k = 0; k < 3; ++k) {
      fa.sflag_off[k] = sflag_off[k];
      fa.max_lines_strided[k] = max_lines_strided[k];
    }
    fa.max_lines_last = max_lines_last;
    fa.pitch_last = pitch_last;
    fa.segtab = d_segtab.p;
    fa.zhalf = zhalf;
    // axis 0 forward-only, L0^-T on the held lattices at the end (stream_tma.cu)
    fa.defer_back = defer_mode;
    fa.n_field = field_n;
    fa.n_t1 = total_t1;
    fa.n_t2 = total_t2;
    fa.n_P = total_p;
    static const char* kNames[2] = {"fit_axis0", "fit_axis1"};
    int l = 0;
    if (fuse3d) {
      fa.fuse3d = 1;
      fa.max_n0 = s3_n[0];
      fa.max_n1 = s3_n[1];
      fa.max_n2 = s3_n[2];
      fa.s3_slab = s3_slab;
      fa.s3_nslab = s3_nslab;
      fa.s3_zs = s3_zs;
      fa.s3_nl = s3_nl;
      fa.a0_slab = a0_slab;
      fa.a0_zr = a0_zr;
      fa.solve3d_threads = s3_threads;
    }
    for (int d = 0; d + 1 < D; ++d) {
      tl->begin(kNames[d]);
      if (d == 0 && tma_axis0) {
        std::uint64_t dims[3];
        std::uint32_t box[3];
        for (int k = 0; k < D; ++k) dims[k] = static_cast<std::uint64_t>(field_dims[static_cast<std::size_t>(D - 1 - k)]);
        box[0] = static_cast<std::uint32_t>(axis0_geo.B2);
        if (D == 2) {
          box[1] = static_cast<std::uint32_t>(axis0_geo.R);
        } else {
          box[1] = static_cast<std::uint32_t>(axis0_geo.B1);
          box[2] = static_cast<std::uint32_t>(axis0_geo.R);
        }
        const CUtensorMap map = make_tmap(field, D, dims, box);
        l += mfb::launch_fit_axis0_tma(p, fa, map, axis0_geo, axis0_tiles, ctx->stream);
      } else if (d == 1 && tma_mid) {
        const std::uint64_t dims[2] = {static_cast<std::uint64_t>(pitch_last),
                                       static_cast<std::uint64_t>(total_t1 / pitch_last)};
        const std::uint32_t box[2] = {static_cast<std::uint32_t>(mid_geo.B2), static_cast<std::uint32_t>(mid_geo.R)};
        const CUtensorMap map = make_tmap(t1.p, 2, dims, box);
        l += mfb::launch_fit_mid_tma(p, fa, map, mid_geo, mid_tiles, mid_n0, ctx->stream);
      } else {
        l += mfb::launch_fit_strided(p, fa, d, ctx->stream);
      }
      tl->end();
      // join the factorizations (D = 2 with the TMA last axis: inside the
      // last-axis launch, after its contraction, which needs no factor)
      // (D = 3 fused solve: the contractions need only the basis rows; the
      // factors join inside the last-axis launch as well)
      if (d == 0 && defer_mode == 2 && fuse3d) {
        if (rows_split) CK(cudaStreamWaitEvent(ctx->stream, ev_rows2, 0));
      } else if (d == 0 && defer_mode == 2 && !(D == 2 && tma_last)) {
        CK(cudaStreamWaitEvent(ctx->stream, ev_chol, 0));
      }
    }
    if (D == 1 && defer_mode == 2) CK(cudaStreamWaitEvent(ctx->stream, ev_chol, 0));
    if (D == 2 && defer_mode == 2 && tma_last && !std::getenv("MFADD_NO_FUSE2D")) {
      for (const auto& b : blocks) {
        fa.max_n0 = std::max(fa.max_n0, probs[static_cast<std::size_t>(b.ax[0])].n);
        fa.max_n1 = std::max(fa.max_n1, probs[static_cast<std::size_t>(b.ax[1])].n);
        fa.max_zl = std::max(fa.max_zl, b.zl);
      }
      fa.fuse2d = mfb::solve2d_smem(p, fa.max_n0, fa.max_n1, fa.max_zl, last_kseg, tw2d) > 0 ? 1 : 0;
      fa.tw2d = fa.fuse2d && tw2d ? 1 : 0;
    }
    if (rows_split && D == 2) CK(cudaStreamWaitEvent(ctx->stream, ev_rows2, 0));  // last-axis + decode rows
    if ((D == 2 && defer_mode == 2 && tma_last) || fuse3d) fa.join_event = ev_chol;
    if ((D == 2 && tma_last) || fuse3d) {
      fa.rlt = rlt.p;
      fa.rlt_stride = rlt_stride;
    }
    tl->begin("fit_last");
    if (tma_last) {
      const double* src = D == 2 ? t1.p : t2.p;
      const std::int64_t rows = (D == 2 ? total_t1 : total_t2) / pitch_last;
      const std::uint64_t dims[2] = {static_cast<std::uint64_t>(pitch_last), static_cast<std::uint64_t>(rows)};
      const std::uint32_t box[2] = {16u, static_cast<std::uint32_t>(last_LT)};
      const CUtensorMap map = make_tmap(src, 2, dims, box, CU_TENSOR_MAP_SWIZZLE_128B);
      l += mfb::launch_fit_last_tma(p, fa, map, last_LT, last_ltcap, last_kseg, ctx->stream);
    } else if (D == 1 && max_n_factor * (2 * p + 2) <= 24576) {  // z + factor in <= 192 KB smem
      l += mfb::launch_fit_1d(p, fa, max_n_factor, ctx->stream);
    } else {
      l += mfb::launch_fit_last(p, fa, ctx->stream);
    }
    tl->end();
    if (fa.defer_back && !fa.fuse2d && !(fa.fuse3d && (fa.s3_nslab == 1 || fa.a0_slab > 0))) {
      int mxn0 = 0;
      std::int64_t mxr = 1;
      fa.min_n0 = 1 << 30;
      for (const auto& b : blocks) {
        fa.min_n0 = std::min(fa.min_n0, probs[static_cast<std::size_t>(b.ax[0])].n);
        mxn0 = std::max(mxn0, probs[static_cast<std::size_t>(b.ax[0])].n);
        std::int64_t r = 1;
        for (int k = 1; k < D; ++k) r *= probs[static_cast<std::size_t>(b.ax[k])].n;
        mxr = std::max(mxr, r);
      }
      tl->begin("fit_backsub0");
      l += mfb::launch_axis0_backsub(p, fa, mxn0, mxr, ctx->stream);
      tl->end();
    }
    CK(cudaGetLastError());
    return l;
  }

  // Map a device status word onto the reference's exceptions.
  void raise_status(const mfb::DevStatus& st, const char* who) {
    if (st.code == 0) return;
    const AxisProb& pr = probs[static_cast<std::size_t>(st.axis_prob)];
    if (st.code == 1)
      throw std::invalid_argument(std::string(who) + "collocation_matrix: param row " + std::to_string(st.row) +
                                  " has no active basis inside the column window");
    if (st.code == 2)
      throw std::out_of_range(std::string(who) + "find_span: parameter outside evaluable range (row " +
                              std::to_string(st.row) + ")");
    // singular: lsq.cpp:25-35 uncovered column from the rows of that problem
    std::vector<int> fc(static_cast<std::size_t>(pr.m)), cnt(static_cast<std::size_t>(pr.m));
    std::vector<double> v(static_cast<std::size_t>(pr.m) * (p + 1));
    std::vector<int> gg(static_cast<std::size_t>(pr.m));
    CK(cudaMemcpy(fc.data(), first_col.p + pr.row_off, fc.size() * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(cnt.data(), count.p + pr.row_off, cnt.size() * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(gg.data(), g0.p + pr.row_off, gg.size() * sizeof(int), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(v.data(), vals.p + pr.row_off * (p + 1), v.size() * sizeof(double), cudaMemcpyDeviceToHost));
    std::vector<char> cov(static_cast<std::size_t>(pr.n), 0);
    for (int j = 0; j < pr.m; ++j)
      for (int k = 0; k < cnt[static_cast<std::size_t>(j)]; ++k) {
        const int col = fc[static_cast<std::size_t>(j)] + k;
        if (v[static_cast<std::size_t>(j) * (p + 1) + (col - gg[static_cast<std::size_t>(j)])] != 0.0)
          cov[static_cast<std::size_t>(col)] = 1;
      }
    std::int64_t col = -1;
    for (int c = 0; c < pr.n; ++c)
      if (!cov[static_cast<std::size_t>(c)]) {
        col = c;
        break;
      }
    throw mfb::SingularFit(pr.dim, col,
                           std::string(who) + "fit_unconstrained: singular normal matrix in dimension " +
                               std::to_string(pr.dim) +
                               (col >= 0 ? " (no input data supports local basis " + std::to_string(col) + ")"
                                         : " (ill-conditioned collocation)"));
  }
};

constexpr int kTiles3[3] = {4, 8, 32};
constexpr int kTiles2[3] = {1, 16, 64};
constexpr int kTiles1[3] = {1, 1, 1024};

// Decode-over-a-grid plan (K7): padded to 3 dims.
struct DecodePlan {
  int D = 0;
  std::int64_t M[3] = {1, 1, 1}, N[3] = {1, 1, 1}, ntiles[3] = {1, 1, 1};
  int T[3] = {1, 1, 1}, W[3] = {1, 1, 1}, pk[3] = {0, 0, 0};
  int prob_of[3] = {-1, -1, -1};  // padded dim -> AxisProb id (or -1 = unit)

  void init(int rank, int p, const std::int64_t* Mi, const std::int64_t* Ni) {
    D = rank;
    const int* t = rank == 3 ? kTiles3 : (rank == 2 ? kTiles2 : kTiles1);
    for (int k = 0; k < 3; ++k) {
      const int src = k - (3 - rank);
      M[k] = src >= 0 ? Mi[src] : 1;
      N[k] = src >= 0 ? Ni[src] : 1;
      T[k] = t[k];
      pk[k] = src >= 0 ? p : 0;
      ntiles[k] = (M[k] + T[k] - 1) / T[k];
    }
  }
  // W[k] = max over tiles of the control window width (exact, host knots).
  void size_windows(int k, const std::vector<double>& kn, const std::vector<double>& params, int p,
                    std::int64_t col_lo) {
    int w = 1;
    for (std::int64_t t = 0; t < ntiles[k]; ++t) {
      const std::int64_t a = t * T[k], b = std::min<std::int64_t>(M[k], a + T[k]) - 1;
      const int s0 = host_find_span(kn, p, params[static_cast<std::size_t>(a)]);
      const int s1 = host_find_span(kn, p, params[static_cast<std::size_t>(b)]);
      w = std::max(w, s1 - s0 + p + 1);
    }
    (void)col_lo;
    W[k] = w;
  }
};

}  // namespace

struct mfadd_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  bool aborted = false;  // after an NCCL error or a timeout: every later call fails fast
};

struct ShardPeer {
  int rank = -1;
  std::int64_t send_off = 0, send_count = 0, recv_off = 0, recv_count = 0;
};

struct mfadd_solver {
  mfadd_context* ctx = nullptr;
  Decomp dec;
  mfadd_solver_config cfg{};
  Workload wl;
  int axbase[3] = {0, 0, 0};
  int dec_prob[3] = {-1, -1, -1};
  DecodePlan dp;
  // TMA decode sweep (D >= 2, even last extent)
  bool tma_decode = false;
  mfb::TmaGeom dgeo{1, 1, 16, 4, 0};
  int dnt1 = 1, dnt2 = 1, dnrange = 1, dH = 1;
  bool dwin = false;  // D = 3: staged-window decode kernel form
  int dna_cap = 0;    // its staged planes per row range

  DBuf<int2> hr;
  DBuf<int> slist, clist, own_coord, pair_slot, unit_g0;
  DBuf<long long> rowbase;  // k_assemble: P offset per (lattice row, last-dim owner block)
  DBuf<double> unit_vals;
  DBuf<std::int64_t> poff;
  std::int64_t hr_off[3] = {0, 0, 0}, s_off[3] = {0, 0, 0}, c_off[3] = {0, 0, 0}, oc_off[3] = {0, 0, 0};
  std::int64_t nS[3] = {0, 0, 0}, nC[3] = {0, 0, 0}, piece[3] = {0, 0, 0}, total_shared = 0;
  DBuf<unsigned long long> change, linf_sh, pair_jumps;
  DBuf<mfb::EpochAcc> acc;
  DBuf<double> epoch_out, lattice, error, partial, red2, field_buf;
  DBuf<unsigned> ticket;  // decode CTA completion counter
  int npairs = 0;
  std::vector<std::array<int, 2>> pair_ids;
  // Non-empty when some shared control has a holder that is not a neighbour of
  // another holder: the reference throws this runtime_error from
  // enforce_constraints in the first exchange epoch (solver.cpp:134-141).
  std::string holder_fault;
  int max_holders = 1;
  // log_errors: per-epoch block residuals
  DBuf<double> res_partial, block_errs;
  int res_ntile = 0, res_max_m0 = 0;
  // one-pass form (residual_tma.cu): epoch snapshots of the shared copies,
  // every epoch's residuals after the loop
  bool res_snap = false;
  DBuf<double> snap, res_part2;
  int res_W = 0, res_ntc = 0, res_nrr = 1, res_threads = 0, res_ltcap = 0, res_nacap = 0, res_eg = 1, res_ng = 1;
  std::vector<double> h_block_errs;
  // shard: rank of nranks owns blocks [srange.blo, srange.bhi)
  int rank = 0, nranks = 1;
  // lattice rows (axis 0) this rank's decode reads: its own rows plus a halo
  // of at most P rows per side from the neighbouring ranks
  std::int64_t need_lo = 0, need_hi = 0;
  mfb::ShardRange srange;
  bool lattice_complete = false;  // partial ranges: the lattice has been summed over the ranks since the last assembly
  std::vector<int> local_of;  // global block id -> local index (-1: other rank)
  mfadd_comm* comm = nullptr;
  std::vector<ShardPeer> peers;
  std::int64_t send_total = 0, recv_total = 0;
  DBuf<double> sendbuf, recvbuf;
  DBuf<mfb::PackTile> pack_tiles;
  int npack = 0;
  DBuf<mfb::TileDev> xtiles;  // cross-rank region tiles
  int nxtiles = 0;
  // region-form epochs (max_holders <= 8): tables + the epoch-loop graph
  DBuf<mfb::TileDev> tiles;
  int ntiles = 0;
  DBuf<mfb::EpochState> est;
  cudaGraph_t loop_graph = nullptr;
  cudaGraphExec_t loop_exec = nullptr;
  const double* loop_field = nullptr;  // field the loop graph's residual kernels read (log_errors)
  // whole-solve graphs keyed by (field buffer, output slot): the first solve of
  // a key runs direct launches (one-time attribute setup), the second captures
  struct SolveGraph {
    const double* field = nullptr;
    const double* lattice = nullptr;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
  };
  std::vector<SolveGraph> graphs;
  cudaStream_t aux_stream = nullptr;  // captures conditional-node bodies
  // log_errors: the one-pass residual kernel (FP64 / latency-bound) runs on its
  // own stream beside the assembly and the decode (HBM-bound)
  cudaStream_t res_stream = nullptr;
  cudaEvent_t ev_res_fork = nullptr, ev_res_join = nullptr;
  // mfadd_solve_host_batch: second field / output slot, copy streams, events
  DBuf<double> field_buf2, lattice_alt, error_alt;
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t bev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // h2d[2], comp[2], d2h[2]
  // pinned result block: red2[2] | DevStatus | epoch_out | EpochState | pair_jumps
  double* hres = nullptr;
  std::size_t hres_eo = 0, hres_es = 0, hres_pj = 0, hres_n = 0;

  // results
  std::vector<mfadd_epoch_stats> epochs;
  std::vector<double> final_jumps;
  mfadd_solve_summary summary{};
  bool have_result = false;
  int last_launches = 0;
  Timeline tl;
  cudaEvent_t ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};

  ~mfadd_solver() {
    // graphs first: the solve graph holds event-record nodes on ev[]
    for (auto& gr : graphs)
      if (gr.exec) cudaGraphExecDestroy(gr.exec);
    if (loop_exec) cudaGraphExecDestroy(loop_exec);
    if (loop_graph) cudaGraphDestroy(loop_graph);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (auto& e : bev)
      if (e) cudaEventDestroy(e);
    if (aux_stream) cudaStreamDestroy(aux_stream);
    if (res_stream) cudaStreamDestroy(res_stream);
    if (ev_res_fork) cudaEventDestroy(ev_res_fork);
    if (ev_res_join) cudaEventDestroy(ev_res_join);
    if (h2d_stream) cudaStreamDestroy(h2d_stream);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    if (hres) cudaFreeHost(hres);
  }
};

// ===================================================================== API
MFB_API int mfadd_abi_version(void) { return MFADD_ABI_VERSION; }
MFB_API const char* mfadd_last_error(void) { return g_err.c_str(); }
MFB_API int mfadd_last_error_dim(void) { return g_err_dim; }
MFB_API int64_t mfadd_last_error_span(void) { return g_err_span; }

// ---------------------------------------------------------------- layout
MFB_API int mfadd_partition(int rank, const int64_t* grid_dims, const double* bounds, const int* blocks_per_dim,
                            int degree, const int64_t* nctrl_per_block, int64_t overlap, int clamp_interfaces,
                            mfadd_decomposition** out) {
  return guarded([&] {
    auto h = std::make_unique<mfadd_decomposition>();
    h->d = mfb::partition(rank, grid_dims, bounds, blocks_per_dim, degree, nctrl_per_block, overlap,
                          clamp_interfaces != 0);
    *out = h.release();
  });
}
MFB_API void mfadd_decomposition_free(mfadd_decomposition* dec) { delete dec; }
MFB_API int mfadd_dec_rank(const mfadd_decomposition* dec) { return dec->d.rank; }
MFB_API int mfadd_dec_block_count(const mfadd_decomposition* dec) { return dec->d.nblocks; }
MFB_API void mfadd_dec_block_dims(const mfadd_decomposition* dec, int64_t* out) {
  std::memcpy(out, dec->d.bd.data(), dec->d.bd.size() * sizeof(int64_t));
}
MFB_API void mfadd_dec_coords(const mfadd_decomposition* dec, int* out) {
  for (int b = 0; b < dec->d.nblocks; ++b)
    for (int k = 0; k < dec->d.rank; ++k) out[b * dec->d.rank + k] = dec->d.coords[static_cast<std::size_t>(b)][k];
}
MFB_API void mfadd_dec_nctrl(const mfadd_decomposition* dec, int64_t* out) {
  for (int k = 0; k < dec->d.rank; ++k) out[k] = dec->d.n_ctrl[k];
}
MFB_API int mfadd_dec_knots(const mfadd_decomposition* dec, int dim, double* out) {
  const auto& kn = dec->d.knots[dim];
  if (out) std::memcpy(out, kn.data(), kn.size() * sizeof(double));
  return static_cast<int>(kn.size());
}
MFB_API int mfadd_dec_neighbors(const mfadd_decomposition* dec, int block, int* out, int cap) {
  const auto& nb = dec->d.neighbors[static_cast<std::size_t>(block)];
  for (std::size_t i = 0; i < nb.size() && static_cast<int>(i) < cap; ++i) out[i] = nb[i];
  return static_cast<int>(nb.size());
}
MFB_API void mfadd_dec_holder_ranges(const mfadd_decomposition* dec, int dim, int* out) {
  const auto& h = dec->d.holder[dim];
  for (std::size_t i = 0; i < h.size(); ++i) {
    out[2 * i] = h[i][0];
    out[2 * i + 1] = h[i][1];
  }
}
MFB_API void mfadd_dec_exchange_volume(const mfadd_decomposition* dec, int64_t* out) {
  const auto v = mfb::exchange_volume(dec->d);
  std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
}
MFB_API double mfadd_dec_compression_ratio(const mfadd_decomposition* dec) {
  return static_cast<double>(dec->d.total_inputs()) / static_cast<double>(dec->d.total_ctrl());
}
MFB_API int mfadd_dec_any_shared(const mfadd_decomposition* dec) { return dec->d.any_shared ? 1 : 0; }
MFB_API void mfadd_dec_grid_dims(const mfadd_decomposition* dec, int64_t* out) {
  for (int k = 0; k < dec->d.rank; ++k) out[k] = dec->d.grid[k];
}

// ---------------------------------------------------------------- context
MFB_API int mfadd_context_create(int device, void* stream, mfadd_context** out) {
  return guarded([&] {
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) throw ApiError(MFADD_ECUDA, "mfadd_context_create: no CUDA device " + std::to_string(device));
    auto c = std::make_unique<mfadd_context>();
    c->device = device;
    ContextScope scope(c.get());
    if (stream) {
      c->stream = static_cast<cudaStream_t>(stream);
    } else {
      CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    CK(cudaMalloc(&c->d_status, sizeof(mfb::DevStatus)));
    CK(cudaMemset(c->d_status, 0, sizeof(mfb::DevStatus)));
    CK(cudaMallocHost(&c->h_pinned, 64 * sizeof(double)));
    *out = c.release();
  });
}

MFB_API void mfadd_context_free(mfadd_context* ctx) {
  if (!ctx) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->d_status) cudaFree(ctx->d_status);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  if (prev >= 0) cudaSetDevice(prev);
}

MFB_API int64_t mfadd_context_launch_count(const mfadd_context* ctx) { return ctx->launches; }

namespace {

mfb::DevStatus read_status(mfadd_context* ctx) {
  mfb::DevStatus st{};
  CK(cudaMemcpyAsync(&st, ctx->d_status, sizeof st, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (st.code) CK(cudaMemsetAsync(ctx->d_status, 0, sizeof(mfb::DevStatus), ctx->stream));
  return st;
}

void check_config(const mfadd_solver_config& c) {  // solver.cpp:333-335
  if (c.max_outer_iterations < 1) throw std::invalid_argument("SolverConfig: max iterations must be >= 1");
  if (!(c.tolerance > 0.0)) throw std::invalid_argument("SolverConfig: tolerance must be > 0");
}

double bits_to_double(unsigned long long u) {
  double d;
  std::memcpy(&d, &u, sizeof d);
  return d;
}

mfb::EpochRegionArgs region_args(mfadd_solver* s, int mode) {
  mfb::EpochRegionArgs a{};
  a.tiles = s->tiles.p;
  a.ntiles = s->ntiles;
  a.nblocks = static_cast<int>(s->wl.blocks.size());  // local blocks
  a.P = s->wl.P.p;
  a.mode = mode;
  a.change = s->change.p;
  a.linf_sh = s->linf_sh.p;
  a.linf_int = s->wl.linf_int.p;
  a.st = s->est.p;
  a.epoch_out = s->epoch_out.p;
  a.pair_jumps = s->pair_jumps.p;
  a.max_iter = s->cfg.max_outer_iterations;
  a.tol = s->cfg.tolerance;
  a.max_ns = s->max_holders;
  a.finalize = 1;  // the last CTA computes dp (and ends the graph loop)
  a.snap = s->res_snap ? s->snap.p : nullptr;
  a.snap_stride = s->wl.total_p;
  return a;
}

mfb::BlockResArgs res_args(mfadd_solver* s, const double* dfield, const mfb::EpochState* st, int slot) {
  mfb::BlockResArgs a{};
  a.D = s->dec.rank;
  a.nblocks = static_cast<int>(s->wl.blocks.size());
  a.blocks = s->wl.d_blocks.p;
  a.probs = s->wl.d_probs.p;
  a.g0 = s->wl.g0.p;
  a.vals = s->wl.vals.p;
  a.P = s->wl.P.p;
  a.field = dfield;
  for (int k = 0; k < 3; ++k) a.fs[k] = s->wl.fs[k];
  a.ntile = s->res_ntile;
  a.partial = s->res_partial.p;
  a.errs = s->block_errs.p;
  a.st = st;
  a.slot = slot;
  a.nglobal = s->dec.nblocks;
  a.boff = s->srange.blo;
  a.expect_iter = -1;
  a.max_m0 = s->res_max_m0;
  return a;
}

// record_epoch's block residuals (solver.cpp:357-364) of every recorded
// epoch in one pass after the loop (snapshot form; st->iter + 1 epochs).
int launch_residuals_all(mfadd_solver* s, const double* dfield, cudaStream_t cs) {
  const Decomp& d = s->dec;
  const Workload& wl = s->wl;
  mfb::ResTmaArgs a{};
  a.D = d.rank;
  a.nblocks = static_cast<int>(wl.blocks.size());
  a.blocks = wl.d_blocks.p;
  a.probs = wl.d_probs.p;
  a.g0 = wl.g0.p;
  a.vals = wl.vals.p;
  a.P = wl.P.p;
  a.snap = s->snap.p;
  a.snap_stride = wl.total_p;
  a.sflag = wl.sflag.p;
  for (int k = 0; k < 3; ++k) a.sflag_off[k] = wl.sflag_off[k];
  a.st = s->est.p;
  a.W = s->res_W;
  a.ntc = s->res_ntc;
  a.nrr = s->res_nrr;
  a.lt_cap = s->res_ltcap;
  a.na_cap = s->res_nacap;
  a.eg = s->res_eg;
  a.ng = s->res_ng;
  a.partial = s->res_part2.p;
  a.errs = s->block_errs.p;
  a.nglobal = d.nblocks;
  a.boff = s->srange.blo;
  std::uint64_t dims[3];
  std::uint32_t box[3];
  for (int k = 0; k < d.rank; ++k) dims[k] = static_cast<std::uint64_t>(d.grid[d.rank - 1 - k]);
  box[0] = static_cast<std::uint32_t>(s->res_W);
  if (d.rank == 2) {
    box[1] = 8u;
  } else {
    box[1] = 1u;
    box[2] = 8u;
  }
  const CUtensorMap map = make_tmap(dfield, d.rank, dims, box);
  s->tl.begin("residual");
  const int l = mfb::launch_residual_tma(wl.p, a, map, s->res_threads, cs);
  s->tl.end();
  return l;
}

// record_epoch's block residuals (solver.cpp:357-364) when log_errors.
int launch_residuals(mfadd_solver* s, const double* dfield, const mfb::EpochState* st, int slot, cudaStream_t cs) {
  if (!s->cfg.log_errors || s->res_snap) return 0;
  s->tl.begin("residual");
  const int l = mfb::launch_block_residual(s->wl.p, res_args(s, dfield, st, slot), cs);
  s->tl.end();
  return l;
}

// Shared controls as regions (mfb::enumerate_regions), each cut into tiles of
// at most kTile controls.  Regions whose holders are all local become local
// tiles; on a sharded solver, regions that also have holders on other ranks
// become cross tiles whose remote holders read the receive buffer (rmask),
// plus pack tiles that gather this rank's copies for each peer.
void build_regions(mfadd_solver* s, const std::vector<int>& pair_slot) {
  // 256 threads x 4 controls per pass (n_s = 2); several passes per tile
  // amortise the per-tile reduction
  static const int kTile = std::getenv("MFADD_EPOCH_TILE") ? std::atoi(std::getenv("MFADD_EPOCH_TILE")) : 4096;
  const Decomp& d = s->dec;
  const int D = d.rank, sh = 3 - D;  // box dims are right-aligned in the kernel's 3-D view
  const std::vector<mfb::Region> regs = mfb::enumerate_regions(d);
  const std::vector<mfb::PeerLayout> peers = mfb::shard_peers(d, regs, s->rank, s->nranks);
  // receive-buffer offset of (region, holder) and the peer segments
  std::vector<std::int64_t> rbase(regs.size() * 8, -1);
  s->peers.clear();
  std::int64_t soff = 0, roff = 0;
  std::vector<mfb::PackTile> packs;
  for (const auto& pl : peers) {
    ShardPeer sp;
    sp.rank = pl.peer;
    sp.send_off = soff;
    sp.send_count = pl.send_count;
    sp.recv_off = roff;
    sp.recv_count = pl.recv_count;
    for (const auto& e : pl.recv) {
      rbase[static_cast<std::size_t>(e.first) * 8 + e.second] = roff;
      roff += regs[static_cast<std::size_t>(e.first)].size();
    }
    for (const auto& e : pl.send) {  // pack this rank's copy of (region, holder) at soff
      const mfb::Region& R = regs[static_cast<std::size_t>(e.first)];
      const int b = R.ids[static_cast<std::size_t>(e.second)];
      const int lb = s->local_of[static_cast<std::size_t>(b)];
      std::int64_t stride = 1, base = 0;
      mfb::PackTile pt{};
      for (int k = D - 1; k >= 0; --k) {
        const AxisProb& pk = s->wl.probs[static_cast<std::size_t>(s->axbase[k] + R.coords[static_cast<std::size_t>(e.second)][static_cast<std::size_t>(k)])];
        base += (R.lo[static_cast<std::size_t>(k)] - pk.col_lo) * stride;
        pt.str[sh + k] = static_cast<int>(stride);
        stride *= pk.n;
      }
      pt.base = s->wl.blocks[static_cast<std::size_t>(lb)].poff + base;
      int ext[3] = {1, 1, 1};
      for (int k = 0; k < D; ++k) ext[sh + k] = static_cast<int>(R.ext[static_cast<std::size_t>(k)]);
      pt.ext1 = ext[1];
      pt.ext2 = ext[2];
      const int total = static_cast<int>(R.size());
      for (int st0 = 0; st0 < total; st0 += kTile) {
        mfb::PackTile t = pt;
        t.dst = soff;
        t.start = st0;
        t.count = std::min(kTile, total - st0);
        packs.push_back(t);
      }
      soff += R.size();
    }
    s->peers.push_back(sp);
  }
  s->send_total = soff;
  s->recv_total = roff;
  std::vector<mfb::TileDev> local_tiles, cross_tiles;
  for (std::size_t ri = 0; ri < regs.size(); ++ri) {
    const mfb::Region& G = regs[ri];
    bool any_local = false;
    for (int h = 0; h < G.ns; ++h) any_local = any_local || s->local_of[static_cast<std::size_t>(G.ids[static_cast<std::size_t>(h)])] >= 0;
    if (!any_local) continue;
    const std::int64_t total64 = G.size();
    if (total64 >= (std::int64_t{1} << 24))  // fast_divmod range (kernels.cu)
      throw std::invalid_argument("mfadd_b200: a shared-control region exceeds 2^24 controls");
    mfb::RegionDev R{};
    R.ns = G.ns;
    for (int k = 0; k < 3; ++k) R.ext[k] = 1;
    for (int k = 0; k < D; ++k) R.ext[sh + k] = static_cast<int>(G.ext[static_cast<std::size_t>(k)]);
    for (int h = 0; h < G.ns; ++h) {
      const int id = G.ids[static_cast<std::size_t>(h)];
      const int lb = s->local_of[static_cast<std::size_t>(id)];
      if (lb >= 0) {
        std::int64_t stride = 1, base = 0;
        for (int k = D - 1; k >= 0; --k) {
          const AxisProb& pk = s->wl.probs[static_cast<std::size_t>(s->axbase[k] + G.coords[static_cast<std::size_t>(h)][static_cast<std::size_t>(k)])];
          base += (G.lo[static_cast<std::size_t>(k)] - pk.col_lo) * stride;
          R.str[h][sh + k] = static_cast<int>(stride);
          stride *= pk.n;
        }
        R.ids[h] = lb;
        R.base[h] = s->wl.blocks[static_cast<std::size_t>(lb)].poff + base;
      } else {  // remote holder: linear index into its receive-buffer copy
        R.rmask |= 1 << h;
        R.ids[h] = -1;
        R.base[h] = rbase[ri * 8 + static_cast<std::size_t>(h)];
        if (R.base[h] < 0) throw std::logic_error("build_regions: remote holder without a receive slot");
        R.str[h][0] = R.ext[1] * R.ext[2];
        R.str[h][1] = R.ext[2];
        R.str[h][2] = 1;
      }
    }
    int q = 0;
    for (int h1 = 0; h1 < G.ns; ++h1)
      for (int h2 = h1 + 1; h2 < G.ns; ++h2, ++q) {
        int code = 0, mul = 1;
        for (int k = D - 1; k >= 0; --k) {
          code += (G.coords[static_cast<std::size_t>(h2)][static_cast<std::size_t>(k)] -
                   G.coords[static_cast<std::size_t>(h1)][static_cast<std::size_t>(k)] + 1) * mul;
          mul *= 3;
        }
        R.pslot[q] = pair_slot[static_cast<std::size_t>(G.ids[static_cast<std::size_t>(h1)]) * 27 + code];
      }
    const int total = static_cast<int>(total64);
    auto& dst = R.rmask ? cross_tiles : local_tiles;
    for (int st0 = 0; st0 < total; st0 += kTile) dst.push_back({R, st0, std::min(kTile, total - st0)});
  }
  // region_tile_local (kernels.cu) addresses the held lattices with 32-bit offsets
  if (s->wl.total_p >= (std::int64_t{1} << 31))
    throw std::invalid_argument("mfadd_b200: held lattices exceed 2^31 controls on one device");
  s->ntiles = static_cast<int>(local_tiles.size());
  s->nxtiles = static_cast<int>(cross_tiles.size());
  s->npack = static_cast<int>(packs.size());
  if (s->ntiles > 0) s->tiles.upload(local_tiles, s->ctx->stream);
  if (s->nxtiles > 0) s->xtiles.upload(cross_tiles, s->ctx->stream);
  if (s->npack > 0) s->pack_tiles.upload(packs, s->ctx->stream);
  s->sendbuf.alloc(static_cast<std::size_t>(std::max<std::int64_t>(s->send_total, 1)));
  s->recvbuf.alloc(static_cast<std::size_t>(std::max<std::int64_t>(s->recv_total, 1)));
}

// The epoch loop (solver.cpp:394-413) as a CUDA graph: a conditional WHILE
// node whose body is one region-form epoch; the epoch's last CTA computes dp
// and sets the condition, so the loop runs with no host round trips.
void build_loop_graph(mfadd_solver* s, const double* dfield) {
  if (s->loop_exec) {
    CK(cudaGraphExecDestroy(s->loop_exec));
    s->loop_exec = nullptr;
  }
  if (s->loop_graph) {
    CK(cudaGraphDestroy(s->loop_graph));
    s->loop_graph = nullptr;
  }
  s->loop_field = dfield;
  CK(cudaGraphCreate(&s->loop_graph, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, s->loop_graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, s->loop_graph, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaStream_t cs = s->aux_stream;
  CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  mfb::EpochRegionArgs a = region_args(s, -1);
  a.cond = static_cast<unsigned long long>(h);
  mfb::launch_epoch_regions(a, cs);
  if (s->cfg.log_errors && !s->res_snap) mfb::launch_block_residual(s->wl.p, res_args(s, dfield, s->est.p, 0), cs);
  CK(cudaStreamEndCapture(cs, &body));
  CK(cudaGraphInstantiate(&s->loop_exec, s->loop_graph, 0));
}

// The WHILE condition of the epoch loop in the graph being captured on `st`
// (default 1 at every launch of the graph; the epochs set it).
cudaGraphConditionalHandle make_loop_handle(cudaStream_t st) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, nullptr, nullptr));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  return h;
}

// The epoch loop as a conditional WHILE node appended to the graph being
// captured on `st` (whole-solve graph), on condition `h`.
void add_loop_node(mfadd_solver* s, cudaStream_t st, const double* dfield, cudaGraphConditionalHandle h) {
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t ndeps = 0;
  CK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &ndeps));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  CK(cudaGraphAddNode(&node, g, deps, ndeps, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  cudaStream_t bs = s->aux_stream;
  CK(cudaStreamBeginCaptureToGraph(bs, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  mfb::EpochRegionArgs a = region_args(s, -1);
  a.cond = static_cast<unsigned long long>(h);
  mfb::launch_epoch_regions(a, bs);
  if (s->cfg.log_errors && !s->res_snap) mfb::launch_block_residual(s->wl.p, res_args(s, dfield, s->est.p, 0), bs);
  CK(cudaStreamEndCapture(bs, &body));
  CK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
}

}  // namespace

// ---------------------------------------------------------------- solver
namespace {

// Geometry of the one-pass residual kernel (residual_tma.cu): column tiles
// (D = 2) or rows j1 (D = 3) x row ranges per block, and the exact sizes of
// the staged windows (planes per row range, window columns per CTA) computed
// from the same spans the device row tables hold.  Picks the most epochs per
// pass (4, 2, 1) whose staging fits the shared-memory budget.
void plan_residual_tma(mfadd_solver* s) {
  const Decomp& d = s->dec;
  Workload& wl = s->wl;
  const int D = d.rank, p = d.degree;
  auto g0_of = [&](const AxisProb& pr, int j) {  // the device row table's g0 (span - p - col_lo)
    const double u = static_cast<double>(pr.in_lo + j) / static_cast<double>(pr.M - 1);
    return host_find_span(d.knots[static_cast<std::size_t>(pr.dim)], p, u) - p - static_cast<int>(pr.col_lo);
  };
  int mxm1 = 0, mxm2 = 0, mnm0 = 1 << 30;
  for (const auto& b : wl.blocks) {
    mnm0 = std::min(mnm0, wl.probs[static_cast<std::size_t>(b.ax[0])].m);
    mxm1 = std::max(mxm1, wl.probs[static_cast<std::size_t>(b.ax[1])].m);
    if (D == 3) mxm2 = std::max(mxm2, wl.probs[static_cast<std::size_t>(b.ax[2])].m);
  }
  int cols = 0;
  if (D == 2) {  // column tiles of W - 2 columns (W <= 256: the TMA box limit)
    const int nt = (mxm1 + 253) / 254;
    cols = round_up((mxm1 + nt - 1) / nt, 2);
    s->res_W = cols + 2;
    s->res_ntc = (mxm1 + cols - 1) / cols;
  } else {  // one row j1 per CTA, the block's whole axis-2 extent in one box
    s->res_W = round_up(mxm2 + 1, 2);
    s->res_ntc = mxm1;
    if (s->res_W > 256) return;
  }
  // widest lattice window of a CTA (distinct axis problems only)
  int ltc = 1;
  std::vector<char> seen(wl.probs.size(), 0);
  for (const auto& b : wl.blocks) {
    const int pid = b.ax[D == 2 ? 1 : 2];
    if (seen[static_cast<std::size_t>(pid)]) continue;
    seen[static_cast<std::size_t>(pid)] = 1;
    const AxisProb& pr = wl.probs[static_cast<std::size_t>(pid)];
    if (D == 2) {
      for (int jf = 0; jf < pr.m; jf += cols)
        ltc = std::max(ltc, g0_of(pr, std::min(pr.m - 1, jf + cols - 1)) - g0_of(pr, jf) + p + 1);
    } else {
      ltc = std::max(ltc, g0_of(pr, pr.m - 1) - g0_of(pr, 0) + p + 1);
    }
  }
  s->res_ltcap = ltc;
  s->res_threads = round_up(s->res_W, 32);
  // planes touched by one row range (distinct axis-0 problems), per nrr
  auto na_for = [&](int nrr) {
    int na = 1;
    std::vector<char> seen0(wl.probs.size(), 0);
    for (const auto& b : wl.blocks) {
      const int pid = b.ax[0];
      if (seen0[static_cast<std::size_t>(pid)]) continue;
      seen0[static_cast<std::size_t>(pid)] = 1;
      const AxisProb& pr = wl.probs[static_cast<std::size_t>(pid)];
      const int nch = (pr.m + 7) / 8, cpr = (nch + nrr - 1) / nrr;
      for (int c0 = 0; c0 < nch; c0 += cpr) {
        const int y0 = c0 * 8, y1 = std::min(pr.m, (c0 + cpr) * 8);
        const int lo = std::min(std::max(g0_of(pr, y0), 0), pr.n - 1);
        const int hi = std::min(std::max(g0_of(pr, y1 - 1) + p, 0), pr.n - 1);
        na = std::max(na, hi - lo + 1);
      }
    }
    return na;
  };
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->ctx->device);
  const std::int64_t ctas = static_cast<std::int64_t>(s->res_ntc) * static_cast<std::int64_t>(wl.blocks.size());
  const int want = static_cast<int>((6LL * sms + ctas - 1) / ctas);  // ~6 CTAs of work per SM
  const int maxr = std::max(1, (mnm0 / 8) / 4);                     // >= 4 chunks per row range
  const std::size_t budget = static_cast<std::size_t>(env_int("MFADD_RES_SMEM_KB", 110)) * 1024;
  const int eg_force = env_int("MFADD_RES_EG", 0), nrr_force = env_int("MFADD_RES_NRR", 0);
  bool ok = false;
  for (int eg : {4, 2, 1}) {
    if (eg_force && eg != eg_force) continue;
    for (int nrr = std::max(1, std::min(want, maxr)); nrr <= std::max(maxr, 1) && !ok; ++nrr) {
      if (nrr_force && nrr != nrr_force) continue;
      const int na = na_for(nrr);
      if (mfb::residual_tma_smem(p, s->res_W, eg, na, s->res_ltcap) <= budget) {
        s->res_eg = eg;
        s->res_nrr = nrr;
        s->res_nacap = na;
        ok = true;
      }
    }
    if (ok) break;
  }
  if (!ok) return;  // the per-epoch kernels stay
  s->res_ng = (s->res_eg == 4 && s->res_threads * 2 <= 512) ? env_int("MFADD_RES_NG", 1) : 1;
  s->res_snap = true;
  s->snap.alloc(static_cast<std::size_t>(s->cfg.max_outer_iterations + 1) * static_cast<std::size_t>(wl.total_p));
  s->res_part2.alloc(static_cast<std::size_t>(s->cfg.max_outer_iterations + 1) * wl.blocks.size() *
                     static_cast<std::size_t>(s->res_ntc) * s->res_nrr * 2);
}

// Solver construction for rank `rank` of `nranks` (1: the whole decomposition).
std::unique_ptr<mfadd_solver> create_solver(mfadd_context* ctx, const mfadd_decomposition* dech,
                                            const mfadd_solver_config* cfg, int rank, int nranks, mfadd_comm* comm) {
    ContextScope scope(ctx);
    auto s = std::make_unique<mfadd_solver>();
    s->ctx = ctx;
    s->dec = dech->d;
    s->cfg = *cfg;
    const Decomp& d = s->dec;
    const int D = d.rank, p = d.degree;
    s->rank = rank;
    s->nranks = nranks;
    s->comm = comm;
    s->srange = mfb::shard_range(d, rank, nranks);
    s->local_of.assign(static_cast<std::size_t>(d.nblocks), -1);
    for (int b = s->srange.blo; b < s->srange.bhi; ++b) s->local_of[static_cast<std::size_t>(b)] = b - s->srange.blo;
    if (p > mfb::kMaxDegree)
      throw std::invalid_argument("mfadd_b200: degree " + std::to_string(p) + " exceeds the compiled maximum " +
                                  std::to_string(mfb::kMaxDegree));
    for (int k = 0; k < D; ++k)
      if (d.blocks[k] > 256)
        throw std::invalid_argument("mfadd_b200: at most 256 blocks per dimension are supported (dimension " +
                                    std::to_string(k) + " has " + std::to_string(d.blocks[k]) + ")");
    Workload& wl = s->wl;
    wl.D = D;
    wl.p = p;
    // knots (one vector per dim) and field strides
    std::vector<double> kn;
    std::int64_t knot_off[3] = {0, 0, 0};
    for (int k = 0; k < D; ++k) {
      knot_off[k] = static_cast<std::int64_t>(kn.size());
      kn.insert(kn.end(), d.knots[k].begin(), d.knots[k].end());
    }
    {
      std::int64_t st = 1;
      for (int k = D - 1; k >= 0; --k) {
        wl.fs[k] = st;
        st *= d.grid[k];
      }
      wl.field_n = st;
    }
    // axis problems: one per (dim, block coordinate) — solver.cpp:59-66,83-88
    for (int k = 0; k < D; ++k) {
      s->axbase[k] = static_cast<int>(wl.probs.size());
      for (int c = 0; c < d.blocks[k]; ++c) {
        AxisProb pr{};
        pr.dim = k;
        pr.m = static_cast<int>(d.dim_field(k, c, mfb::IN_HI) - d.dim_field(k, c, mfb::IN_LO));
        pr.n = static_cast<int>(d.dim_field(k, c, mfb::DOF_HI) - d.dim_field(k, c, mfb::DOF_LO));
        pr.col_lo = d.dim_field(k, c, mfb::DOF_LO);
        pr.in_lo = d.dim_field(k, c, mfb::IN_LO);
        pr.M = d.grid[k];
        pr.knot_off = knot_off[k];
        pr.nknots = static_cast<int>(d.knots[k].size());
        wl.factor_ids.push_back(static_cast<int>(wl.probs.size()));
        wl.probs.push_back(pr);
      }
    }
    // LocalProblem::validate (lsq.cpp:9-20) for every block, lowest id first
    for (int b = 0; b < d.nblocks; ++b)
      for (int k = 0; k < D; ++k) {
        const AxisProb& pr = wl.probs[static_cast<std::size_t>(s->axbase[k] + d.coords[static_cast<std::size_t>(b)][k])];
        if (pr.m < pr.n)
          throw std::invalid_argument("block " + std::to_string(b) + ": LocalProblem: underdetermined in dimension " +
                                      std::to_string(k) + " (" + std::to_string(pr.m) + " rows < " +
                                      std::to_string(pr.n) + " cols)");
      }
    // global decode rows (decode.cpp:83-97 on the full lattice window)
    for (int k = 0; k < D; ++k) {
      AxisProb pr{};
      pr.dim = k;
      pr.m = static_cast<int>(d.grid[k]);
      pr.n = static_cast<int>(d.n_ctrl[k]);
      pr.col_lo = 0;
      pr.in_lo = 0;
      pr.M = d.grid[k];
      pr.knot_off = knot_off[k];
      pr.nknots = static_cast<int>(d.knots[k].size());
      s->dec_prob[k] = static_cast<int>(wl.probs.size());
      wl.probs.push_back(pr);
    }
    // blocks (this rank's)
    for (int b = s->srange.blo; b < s->srange.bhi; ++b) {
      BlockDev bd{};
      std::int64_t fb = 0;
      for (int k = 0; k < D; ++k) {
        bd.ax[k] = s->axbase[k] + d.coords[static_cast<std::size_t>(b)][k];
        fb += d.at(b, k, mfb::IN_LO) * wl.fs[k];
      }
      bd.fbase = fb;
      wl.blocks.push_back(bd);
    }
    wl.layout_tables();
    for (int k = 0; k < D; ++k) wl.field_dims[static_cast<std::size_t>(k)] = d.grid[k];
    wl.plan_tma(true);
    cudaStream_t st = ctx->stream;
    wl.allocate(st);
    wl.knots.upload(kn, st);
    // shared flags, holder ranges, S/C lists, owner coords
    std::vector<unsigned char> sflag;
    std::vector<int2> hr;
    std::vector<int> sl, cl, oc;
    for (int k = 0; k < D; ++k) {
      wl.sflag_off[k] = static_cast<std::int64_t>(sflag.size());
      s->hr_off[k] = static_cast<std::int64_t>(hr.size());
      s->s_off[k] = static_cast<std::int64_t>(sl.size());
      s->c_off[k] = static_cast<std::int64_t>(cl.size());
      s->oc_off[k] = static_cast<std::int64_t>(oc.size());
      for (std::int64_t i = 0; i < d.n_ctrl[k]; ++i) {
        const auto r = d.holder[k][static_cast<std::size_t>(i)];
        hr.push_back(make_int2(r[0], r[1]));
        const bool sh = r[1] > r[0];
        sflag.push_back(sh ? 1 : 0);
        (sh ? sl : cl).push_back(static_cast<int>(i));
        int owner = -1;
        for (int c = 0; c < d.blocks[k]; ++c)
          if (i >= d.dim_field(k, c, mfb::OWN_LO) && i < d.dim_field(k, c, mfb::OWN_HI)) owner = c;
        if (owner < 0) throw std::logic_error("partition: control index without an owner");
        oc.push_back(owner);
      }
      s->nS[k] = static_cast<std::int64_t>(sl.size()) - s->s_off[k];
      s->nC[k] = static_cast<std::int64_t>(cl.size()) - s->c_off[k];
    }
    s->max_holders = 1;
    for (int k = 0; k < D; ++k) {
      int mx = 1;
      for (const auto& r : d.holder[k]) mx = std::max(mx, r[1] - r[0] + 1);
      s->max_holders *= mx;
    }
    if (s->max_holders > 27) throw std::logic_error("partition: a control has more than 3 holders along one axis");
    if (s->max_holders > 8) s->max_holders = 27;
    s->total_shared = 0;
    for (int pc = 0; pc < D; ++pc) {
      std::int64_t cnt = 1;
      for (int k = 0; k < D; ++k) cnt *= k < pc ? s->nC[k] : (k == pc ? s->nS[k] : d.n_ctrl[k]);
      s->piece[pc] = cnt;
      s->total_shared += cnt;
    }
    wl.sflag.upload(sflag, st);
    s->hr.upload(hr, st);
    s->slist.upload(sl.empty() ? std::vector<int>{0} : sl, st);
    s->clist.upload(cl.empty() ? std::vector<int>{0} : cl, st);
    s->own_coord.upload(oc, st);
    std::vector<std::int64_t> po(static_cast<std::size_t>(d.nblocks), -1);  // by global id (-1: another rank's block)
    for (int b = s->srange.blo; b < s->srange.bhi; ++b)
      po[static_cast<std::size_t>(b)] = wl.blocks[static_cast<std::size_t>(b - s->srange.blo)].poff;
    s->poff.upload(po, st);
    {  // assemble_owned's P offset of every lattice row in each last-dim owner block (k_assemble)
      const int dl = D - 1;
      std::int64_t rows = 1;
      for (int k = 0; k < dl; ++k) rows *= d.n_ctrl[k];
      const int Bl = d.blocks[dl];
      std::vector<long long> rb(static_cast<std::size_t>(rows * Bl), 0);
      for (std::int64_t r = 0; r < rows; ++r) {
        std::int64_t rr = r, il[3] = {0, 0, 0};
        int cl[3] = {0, 0, 0};
        for (int k = dl - 1; k >= 0; --k) {
          il[k] = rr % d.n_ctrl[k];
          rr /= d.n_ctrl[k];
          cl[k] = oc[static_cast<std::size_t>(s->oc_off[k] + il[k])];
        }
        int lead = 0;
        for (int k = 0; k < dl; ++k) lead = lead * d.blocks[k] + cl[k];
        for (int c = 0; c < Bl; ++c) {
          std::int64_t o = 0;
          for (int k = 0; k < dl; ++k) {
            const AxisProb& pk = wl.probs[static_cast<std::size_t>(s->axbase[k] + cl[k])];
            o = o * pk.n + (il[k] - pk.col_lo);
          }
          const AxisProb& pl = wl.probs[static_cast<std::size_t>(s->axbase[dl] + c)];
          const std::int64_t pb = po[static_cast<std::size_t>(lead * Bl + c)];
          rb[static_cast<std::size_t>(r * Bl + c)] = pb < 0 ? mfb::kAsmOtherRank : pb + o * pl.n - pl.col_lo;
        }
      }
      s->rowbase.upload(rb, st);
    }
    // final-jump pair slots in the reference's order (solver.cpp:170-174)
    std::vector<int> ps(static_cast<std::size_t>(d.nblocks) * 27, -1);
    for (int a = 0; a < d.nblocks; ++a)
      for (int j : d.neighbors[static_cast<std::size_t>(a)]) {
        if (j < a) continue;
        int code = 0, mul = 1;
        for (int k = D - 1; k >= 0; --k) {
          code += (d.coords[static_cast<std::size_t>(j)][k] - d.coords[static_cast<std::size_t>(a)][k] + 1) * mul;
          mul *= 3;
        }
        ps[static_cast<std::size_t>(a) * 27 + code] = static_cast<int>(s->pair_ids.size());
        s->pair_ids.push_back({a, j});
      }
    s->npairs = static_cast<int>(s->pair_ids.size());
    // solver.cpp:134-141 + runtime.cpp:17-21: a block only hears from its
    // neighbours (coordinate distance <= 1).  Find, for the lowest block id,
    // the first held control (row-major) with a holder two coordinates away.
    for (int b = 0; b < d.nblocks && s->holder_fault.empty(); ++b) {
      const auto& cb = d.coords[static_cast<std::size_t>(b)];
      std::array<std::int64_t, 3> lo{0, 0, 0}, hi{1, 1, 1}, fmin{-1, -1, -1};
      for (int k = 0; k < D; ++k) {
        lo[k] = d.at(b, k, mfb::DOF_LO);
        hi[k] = d.at(b, k, mfb::DOF_HI);
        for (std::int64_t i = lo[k]; i < hi[k]; ++i) {
          const auto r = d.holder[k][static_cast<std::size_t>(i)];
          if (r[0] < cb[k] - 1 || r[1] > cb[k] + 1) {
            fmin[k] = i;
            break;
          }
        }
      }
      bool found = false;
      std::array<std::int64_t, 3> best{0, 0, 0};
      for (int k = 0; k < D; ++k) {
        if (fmin[k] < 0) continue;
        std::array<std::int64_t, 3> cand = lo;
        cand[k] = fmin[k];
        if (!found || std::lexicographical_compare(cand.begin(), cand.begin() + D, best.begin(), best.begin() + D))
          best = cand;
        found = true;
      }
      if (!found) continue;
      int ns = 1, near = 1;
      for (int k = 0; k < D; ++k) {
        const auto r = d.holder[k][static_cast<std::size_t>(best[k])];
        ns *= r[1] - r[0] + 1;
        near *= std::min(r[1], cb[k] + 1) - std::max(r[0], cb[k] - 1) + 1;
      }
      s->holder_fault = "enforce_constraints: block " + std::to_string(b) + " received " + std::to_string(near - 1) +
                        " contributions for a control shared by " + std::to_string(ns) + " blocks";
    }
    s->pair_slot.upload(ps, st);
    if (s->max_holders <= 8 && d.any_shared) build_regions(s.get(), ps);
    s->pair_jumps.alloc(static_cast<std::size_t>(std::max(1, s->npairs)) * 2);
    s->change.alloc(wl.blocks.size());  // by local block index
    s->linf_sh.alloc(wl.blocks.size());
    s->acc.alloc(1);
    s->est.alloc(1);
    s->epoch_out.alloc(static_cast<std::size_t>(cfg->max_outer_iterations + 1) * 3 + 3);
    s->lattice.alloc(static_cast<std::size_t>(d.total_ctrl()));
    if (cfg->store_error) s->error.alloc(static_cast<std::size_t>(d.total_inputs()));
    // decode plan
    s->dp.init(D, p, d.grid.data(), d.n_ctrl.data());
    for (int k = 0; k < 3; ++k) {
      const int src = k - (3 - D);
      if (src < 0) continue;
      std::vector<double> u(static_cast<std::size_t>(d.grid[src]));
      for (std::int64_t j = 0; j < d.grid[src]; ++j)
        u[static_cast<std::size_t>(j)] = static_cast<double>(j) / static_cast<double>(d.grid[src] - 1);
      s->dp.size_windows(k, d.knots[src], u, p, 0);
      s->dp.prob_of[k] = s->dec_prob[src];
    }
    std::size_t npart = static_cast<std::size_t>(s->dp.ntiles[0] * s->dp.ntiles[1] * s->dp.ntiles[2]);
    if (D >= 2 && d.grid[D - 1] % 2 == 0 && !std::getenv("MFADD_NO_TMA")) {
      const int M1 = static_cast<int>(d.grid[1]), M2 = D == 3 ? static_cast<int>(d.grid[2]) : 1;
      const int inner = D == 2 ? M1 : M2;
      const int nt = (inner + 255) / 256;
      s->dgeo.B2 = round_up((inner + nt - 1) / nt, 2);
      s->dgeo.B1 = D == 2 ? 1 : std::max(1, 256 / s->dgeo.B2);
      s->dgeo.R = 8;
      s->dgeo.S = env_int("MFADD_DEC_S", 3);
      // D = 3: shared axis-2 window of each control plane (k_decode_tma), up to B2 + p + 2 columns
      s->dgeo.lt_cap = (D == 3 && !std::getenv("MFADD_NO_DEC_WINDOW")) ? s->dgeo.B2 + p + 2 : 0;
      s->dnt2 = (inner + s->dgeo.B2 - 1) / s->dgeo.B2;
      s->dnt1 = D == 2 ? 1 : (M1 + s->dgeo.B1 - 1) / s->dgeo.B1;
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
      const int M0 = static_cast<int>(s->srange.in_hi - s->srange.in_lo);  // this rank's input rows
      auto plan_rows = [&](int per_sm) {  // per_sm: CTAs per SM the row ranges aim at
        const int want = std::max(1, (per_sm * sms + s->dnt1 * s->dnt2 - 1) / (s->dnt1 * s->dnt2));
        const int nr = std::max(1, std::min(want, (M0 + s->dgeo.R - 1) / s->dgeo.R));
        s->dH = round_up((M0 + nr - 1) / nr, s->dgeo.R);
        s->dnrange = (M0 + s->dH - 1) / s->dH;
      };
      // (D = 2: 12 measured best on C5, 0.569 vs 0.577 ms per solve at 8; flat for D = 3)
      plan_rows(env_int("MFADD_DEC_CTAS", D == 2 ? 12 : 8));
      s->tma_decode = true;
      npart = std::max(npart, static_cast<std::size_t>(s->dnt1) * s->dnt2 * s->dnrange);
      if (D == 3 && s->dgeo.B1 == 1 && s->dgeo.lt_cap > 0) {  // every tile's axis-2 window fits: window-only kernel
        const std::vector<double>& kn2 = d.knots[2];
        auto g0 = [&](int j) { return host_find_span(kn2, p, static_cast<double>(j) / static_cast<double>(M2 - 1)) - p; };
        int mrw = 0;
        for (int tx = 0; tx < s->dnt2; ++tx) {
          const int jf = tx * s->dgeo.B2, jl = std::min(M2 - 1, jf + s->dgeo.B2 - 1);
          mrw = std::max(mrw, g0(jl) - g0(jf) + p + 1);
        }
        s->dwin = mrw <= s->dgeo.lt_cap && mrw <= s->dgeo.B2;
        if (s->dwin) {  // staged windows: row ranges short enough that their planes fit the budget
          s->dgeo.lt_cap = mrw;
          const std::vector<double>& kn0 = d.knots[0];
          auto g00 = [&](std::int64_t j) {
            return host_find_span(kn0, p, static_cast<double>(j) / static_cast<double>(d.grid[0] - 1)) - p;
          };
          const std::int64_t ybeg = s->srange.in_lo, yend = s->srange.in_hi;
          auto na_for = [&](int H) {
            int na = 1;
            for (std::int64_t y0 = ybeg; y0 < yend; y0 += H) {
              const std::int64_t y1 = std::min<std::int64_t>(yend, y0 + H);
              const int hi = static_cast<int>(std::min<std::int64_t>(g00(y1 - 1) + p, d.n_ctrl[0] - 1));
              na = std::max(na, hi - g00(y0) + 1);
            }
            return na;
          };
          // wide windows (C3: ~135 columns per CTA against C4's ~70): longer row
          // ranges amortise the staging, 48 KB of windows and ~4 CTAs per SM
          // (C3 decode 92.7 -> 78.3 us; C4 is fastest at 24 KB / 8: 693 vs 784 us)
          const bool wide = static_cast<std::size_t>(mrw) * 8 * 48 > 36 * 1024;
          if (wide) plan_rows(env_int("MFADD_DEC_CTAS", 4));
          const std::size_t budget = static_cast<std::size_t>(env_int("MFADD_DEC_STAGE_KB", wide ? 48 : 24)) * 1024;
          int H = s->dH;
          while (H > 8 && static_cast<std::size_t>(na_for(H)) * mrw * 8 > budget) H -= 8;
          s->dH = H;
          s->dnrange = static_cast<int>((M0 + H - 1) / H);
          s->dna_cap = na_for(H);
          npart = std::max(npart, static_cast<std::size_t>(s->dnt1) * s->dnt2 * s->dnrange);
        }
      }
    }
    s->partial.alloc(npart * 2);
    s->red2.alloc(2);
    s->need_lo = 0;
    s->need_hi = d.n_ctrl[0];
    if (nranks > 1 && s->tma_decode) {  // spans of the rank's first / last own input row (decode.cpp:63-79)
      const std::vector<double>& kn0 = d.knots[0];
      auto span = [&](std::int64_t j) {
        return host_find_span(kn0, p, static_cast<double>(j) / static_cast<double>(d.grid[0] - 1));
      };
      s->need_lo = std::max<std::int64_t>(0, span(s->srange.in_lo) - p);
      s->need_hi = std::min<std::int64_t>(d.n_ctrl[0], span(s->srange.in_hi - 1) + 1);
    }
    s->ticket.alloc(1);
    CK(cudaMemsetAsync(s->ticket.p, 0, sizeof(unsigned), st));
    s->unit_g0.upload(std::vector<int>{0}, st);
    s->unit_vals.upload(std::vector<double>{1.0}, st);
    for (auto& e : s->ev) CK(cudaEventCreate(&e));
    CK(cudaMemsetAsync(s->change.p, 0, s->change.n * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(s->linf_sh.p, 0, s->linf_sh.n * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(s->acc.p, 0, sizeof(mfb::EpochAcc), st));
    CK(cudaMemsetAsync(s->est.p, 0, sizeof(mfb::EpochState), st));
    CK(cudaStreamCreateWithFlags(&s->aux_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&s->res_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&s->ev_res_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&s->ev_res_join, cudaEventDisableTiming));
    if (nranks > 1) {
      if (s->max_holders > 8)
        throw std::invalid_argument("mfadd_b200: a sharded solve needs at most two holders per axis");
    }
    s->hres_eo = 4;
    s->hres_es = s->hres_eo + s->epoch_out.n;
    s->hres_pj = s->hres_es + (sizeof(mfb::EpochState) + 7) / 8;
    s->hres_n = s->hres_pj + s->pair_jumps.n;
    CK(cudaMallocHost(&s->hres, s->hres_n * sizeof(double)));
    if (cfg->log_errors) {
      int mx = 1;
      for (const auto& b : wl.blocks) {
        const int m0 = wl.probs[static_cast<std::size_t>(b.ax[0])].m;
        s->res_max_m0 = std::max(s->res_max_m0, m0);
        int tr = 1;
        for (int k = 1; k < D; ++k) tr *= wl.probs[static_cast<std::size_t>(b.ax[k])].m;
        mx = std::max(mx, D == 1 ? m0 : tr);
      }
      s->res_ntile = (mx + 127) / 128;  // one thread per trailing point (no cap: every point is counted)
      s->res_partial.alloc(wl.blocks.size() * static_cast<std::size_t>(s->res_ntile) * 2);
      s->block_errs.alloc(static_cast<std::size_t>(cfg->max_outer_iterations + 1) * d.nblocks * 2);
      // one-pass snapshot form (residual_tma.cu) where the epochs run as
      // region kernels on one device and the field rows are 16-B aligned
      const bool regions_ok = s->ntiles > 0 || !d.any_shared;
      if (D >= 2 && nranks == 1 && regions_ok && d.grid[D - 1] % 2 == 0 && !std::getenv("MFADD_RES_LEGACY"))
        plan_residual_tma(s.get());
    }
    // (after the log_errors plan: the loop body writes the epoch snapshots)
    if (nranks == 1 && s->ntiles > 0 && cfg->enforce_continuity) build_loop_graph(s.get(), nullptr);
    CK(cudaStreamSynchronize(st));
    return s;
}

}  // namespace

MFB_API int mfadd_solver_create(mfadd_context* ctx, const mfadd_decomposition* dech, const mfadd_solver_config* cfg,
                                mfadd_solver** out) {
  return guarded([&] { *out = create_solver(ctx, dech, cfg, 0, 1, nullptr).release(); });
}

MFB_API int mfadd_solver_create_sharded(mfadd_context* ctx, const mfadd_decomposition* dech,
                                        const mfadd_solver_config* cfg, mfadd_comm* comm, mfadd_solver** out) {
  return guarded([&] {
    if (!comm) throw std::invalid_argument("mfadd_solver_create_sharded: null communicator");
    *out = create_solver(ctx, dech, cfg, comm->rank, comm->nranks, comm).release();
  });
}

MFB_API void mfadd_solver_free(mfadd_solver* s) {
  if (!s) return;
  int prev = -1;
  cudaGetDevice(&prev);
  cudaSetDevice(s->ctx->device);
  cudaStreamSynchronize(s->ctx->stream);
  delete s;
  (void)cudaGetLastError();  // teardown errors must not surface in a later call
  if (prev >= 0) cudaSetDevice(prev);
}

namespace {

mfb::EpochArgs epoch_args(mfadd_solver* s, int mode) {
  mfb::EpochArgs a{};
  const Decomp& d = s->dec;
  a.D = d.rank;
  a.nblocks = d.nblocks;
  for (int k = 0; k < 3; ++k) {
    a.B[k] = d.blocks[k];
    a.N[k] = d.n_ctrl[k];
    a.hr_off[k] = s->hr_off[k];
    a.s_off[k] = s->s_off[k];
    a.c_off[k] = s->c_off[k];
    a.nS[k] = s->nS[k];
    a.nC[k] = s->nC[k];
    a.piece[k] = s->piece[k];
    a.axbase[k] = s->axbase[k];
  }
  a.hr = s->hr.p;
  a.slist = s->slist.p;
  a.clist = s->clist.p;
  a.total = s->total_shared;
  a.probs = s->wl.d_probs.p;
  a.poff = s->poff.p;
  a.P = s->wl.P.p;
  a.mode = mode;
  a.change = s->change.p;
  a.linf_sh = s->linf_sh.p;
  a.acc = s->acc.p;
  a.pair_slot = s->pair_slot.p;
  a.pair_jumps = s->pair_jumps.p;
  a.n_P = s->wl.total_p;
  a.max_holders = s->max_holders;
  return a;
}

// One epoch: K4 + K5; returns launches.  Result lands in epoch_out[3*slot].
int run_epoch(mfadd_solver* s, int mode, int slot) {
  s->tl.begin("epoch");
  int l = mfb::launch_epoch(epoch_args(s, mode), s->ctx->stream);
  s->tl.end();
  mfb::DpArgs da{s->dec.nblocks, s->change.p, s->linf_sh.p, s->wl.linf_int.p, s->acc.p, s->epoch_out.p + 3 * slot,
                 nullptr};
  s->tl.begin("dp");
  l += mfb::launch_dp(da, s->ctx->stream);
  s->tl.end();
  CK(cudaGetLastError());
  return l;
}

float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// The lattice part this rank assembles: its owned control rows along axis 0
// (for D == 1 the single lattice row, restricted to the owned columns).
void set_assemble_range(const mfadd_solver* s, mfb::AssembleArgs& aa) {
  const Decomp& d = s->dec;
  if (d.rank == 1) {
    aa.row0 = 0;
    aa.nrows = 1;
    aa.col0 = s->srange.own_lo;
    aa.ncols = s->srange.own_hi - s->srange.own_lo;
    return;
  }
  std::int64_t rest = 1;
  for (int k = 1; k + 1 < d.rank; ++k) rest *= d.n_ctrl[k];
  aa.row0 = s->srange.own_lo * rest;
  aa.nrows = (s->srange.own_hi - s->srange.own_lo) * rest;
  aa.col0 = 0;
  aa.ncols = d.n_ctrl[d.rank - 1];
}

// Decode of the lattice at this rank's own input rows (all rows on one rank) +
// the deterministic partial reduction into red2 (solver.cpp:425-438).
int enqueue_decode(mfadd_solver* s, const double* dfield) {
  mfadd_context* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const Decomp& d = s->dec;
  Workload& wl = s->wl;
  int launches = 0;
  // ---- block_error_slab over every block == global decode (solver.cpp:425-438)
  mfb::DecodeArgs da{};
  const DecodePlan& dp = s->dp;
  da.D = d.rank;
  for (int k = 0; k < 3; ++k) {
    da.M[k] = dp.M[k];
    da.N[k] = dp.N[k];
    da.T[k] = dp.T[k];
    da.ntiles[k] = dp.ntiles[k];
    da.W[k] = dp.W[k];
    da.pk[k] = dp.pk[k];
    if (dp.prob_of[k] >= 0) {
      const AxisProb& pr = wl.probs[static_cast<std::size_t>(dp.prob_of[k])];
      da.g0[k] = wl.g0.p + pr.row_off;
      da.vals[k] = wl.vals.p + pr.row_off * (wl.p + 1);
    } else {
      da.g0[k] = s->unit_g0.p;
      da.vals[k] = s->unit_vals.p;
    }
  }
  da.lattice = s->lattice.p;
  da.field = dfield;
  da.out = s->cfg.store_error ? s->error.p : nullptr;
  da.partial = s->partial.p;
  std::int64_t nparts = static_cast<std::int64_t>(s->partial.n / 2);
  s->tl.begin("decode");
  if (s->tma_decode) {
    mfb::DecodeSweepArgs ds{};
    ds.D = d.rank;
    ds.M0 = static_cast<int>(d.grid[0]);
    ds.M1 = static_cast<int>(d.grid[1]);
    ds.M2 = d.rank == 3 ? static_cast<int>(d.grid[2]) : 1;
    ds.N0 = static_cast<int>(d.n_ctrl[0]);
    ds.N1 = static_cast<int>(d.n_ctrl[1]);
    ds.N2 = d.rank == 3 ? static_cast<int>(d.n_ctrl[2]) : 1;
    ds.ntile1 = s->dnt1;
    ds.ntile2 = s->dnt2;
    ds.nrange = s->dnrange;
    ds.H = s->dH;
    ds.ybeg = static_cast<int>(s->srange.in_lo);
    ds.yend = static_cast<int>(s->srange.in_hi);
    auto rows = [&](int k, const int** g, const double** v) {
      const AxisProb& pr = wl.probs[static_cast<std::size_t>(s->dec_prob[k])];
      *g = wl.g0.p + pr.row_off;
      *v = wl.vals.p + pr.row_off * (wl.p + 1);
    };
    rows(0, &ds.g0_0, &ds.v_0);
    rows(1, &ds.g0_1, &ds.v_1);
    if (d.rank == 3) rows(2, &ds.g0_2, &ds.v_2);
    ds.lattice = s->lattice.p;
    ds.err = s->cfg.store_error ? s->error.p : nullptr;
    ds.partial = s->partial.p;
    std::uint64_t dims[3];
    std::uint32_t box[3];
    for (int k = 0; k < d.rank; ++k) dims[k] = static_cast<std::uint64_t>(d.grid[d.rank - 1 - k]);
    box[0] = static_cast<std::uint32_t>(s->dgeo.B2);
    if (d.rank == 2) {
      box[1] = static_cast<std::uint32_t>(s->dgeo.R);
    } else {
      box[1] = static_cast<std::uint32_t>(s->dgeo.B1);
      box[2] = static_cast<std::uint32_t>(s->dgeo.R);
    }
    ds.ticket = s->ticket.p;
    ds.red2 = s->red2.p;
    ds.win = s->dwin ? 1 : 0;
    ds.na_cap = s->dna_cap;
    const CUtensorMap map = make_tmap(dfield, d.rank, dims, box);
    launches += mfb::launch_decode_tma(wl.p, ds, map, s->dgeo, st);
    nparts = 0;  // reduced by the decode's last CTA
  } else {
    launches += mfb::launch_decode(wl.p, da, st);
    nparts = s->dp.ntiles[0] * s->dp.ntiles[1] * s->dp.ntiles[2];
  }
  s->tl.end();
  if (nparts > 0) {
    s->tl.begin("reduce");
    launches += mfb::launch_reduce_partials(s->partial.p, nparts, s->red2.p, st);
    s->tl.end();
  }
  return launches;
}

// Issue every device operation of one solve on the context stream (kernels,
// the epoch-loop conditional node, result copies into pinned memory); no
// host synchronisation, so the sequence can be captured into a graph.
int enqueue_solve(mfadd_solver* s, const double* dfield) {
  mfadd_context* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const Decomp& d = s->dec;
  Workload& wl = s->wl;
  int launches = 0;
  s->tl.st = st;
  (void)cudaGetLastError();  // report only this solve's launch errors
  CK(cudaEventRecord(s->ev[0], st));
  // ---- setup: basis rows + Gram/Cholesky (solver.cpp:346 make_block_state)
  launches += wl.setup(ctx, &s->tl);
  CK(cudaEventRecord(s->ev[1], st));
  // ---- decoupled local fits (solver.cpp:369-373)
  launches += wl.fit(ctx, dfield, &s->tl);
  CK(cudaEventRecord(s->ev[2], st));
  // ---- record_epoch(0, 0.0)
  const bool regions = s->ntiles > 0;
  const bool loop = s->cfg.enforce_continuity && d.any_shared;
  if (loop && !s->holder_fault.empty()) {
    // the reference fails in the fit first if it is singular, then in the
    // first exchange epoch (solver.cpp:134-141)
    wl.raise_status(read_status(ctx), "");
    throw std::runtime_error(s->holder_fault);
  }
  CK(cudaMemsetAsync(s->est.p, 0, sizeof(mfb::EpochState), st));
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(st, &cs));
  const bool captured = cs == cudaStreamCaptureStatusActive;
  // In the whole-solve graph, record_epoch(0) and iteration 1 share one pass
  // over the shared controls (mode 4): iteration 1 reads exactly the state
  // epoch 0 measures, and its update leaves the n_s > 2 copies untouched.
  const bool fuse01 = captured && loop && regions && s->nranks == 1;
  if (fuse01) {
    launches += launch_residuals(s, dfield, nullptr, 0, st);  // record_epoch(0) block errors, before the update
    const cudaGraphConditionalHandle h = make_loop_handle(st);
    mfb::EpochRegionArgs a = region_args(s, 4);
    a.cond = static_cast<unsigned long long>(h);
    a.zero_pairs = static_cast<int>(s->pair_jumps.n);  // cleared here instead of by a memset node
    s->tl.begin("epoch");
    launches += mfb::launch_epoch_regions(a, st);
    s->tl.end();
    launches += launch_residuals(s, dfield, s->est.p, 0, st);  // record_epoch(1) block errors
    // the next iterations as plain (predicated) kernel nodes: a conditional
    // node costs more than a kernel that exits at once
    static const int unroll = env_int("MFADD_UNROLL_EPOCHS", 3);
    for (int u = 0; u < unroll; ++u) {
      mfb::EpochRegionArgs b = region_args(s, -1);
      b.cond = static_cast<unsigned long long>(h);
      b.predicated = 1;
      s->tl.begin("epoch");
      launches += mfb::launch_epoch_regions(b, st);
      s->tl.end();
      if (s->cfg.log_errors && !s->res_snap) {
        mfb::BlockResArgs ra = res_args(s, dfield, s->est.p, 0);
        ra.expect_iter = 2 + u;  // skipped with its epoch
        launches += mfb::launch_block_residual(s->wl.p, ra, st);
      }
    }
    s->tl.begin("epoch");
    add_loop_node(s, st, dfield, h);
    s->tl.end();
  } else {
  if (regions) {
    s->tl.begin("epoch");
    launches += mfb::launch_epoch_regions(region_args(s, 0), st);
    s->tl.end();
  } else {
    launches += run_epoch(s, 0, 0);
  }
  launches += launch_residuals(s, dfield, nullptr, 0, st);  // record_epoch(0, ...) block errors
  }
  // ---- outer iterations (solver.cpp:394-413), entirely on the device
  if (loop && !fuse01) {
    s->tl.begin("epoch");
    if (captured)
      add_loop_node(s, st, dfield, make_loop_handle(st));
    else {
      if (!s->loop_exec || (s->cfg.log_errors && !s->res_snap && s->loop_field != dfield)) build_loop_graph(s, dfield);
      CK(cudaGraphLaunch(s->loop_exec, st));
    }
    s->tl.end();
  }
  // ---- every epoch's block residuals in one pass (log_errors, snapshot form)
  // (beside the assembly and the decode on res_stream, joined before the
  // results are read back; on the solve's own stream when kernels are timed)
  static const bool res_inline = std::getenv("MFADD_RES_INLINE") != nullptr;
  const bool res_side = s->cfg.log_errors && s->res_snap && !s->tl.on && !s->tl.sync_check && !res_inline;
  if (res_side) {
    CK(cudaEventRecord(s->ev_res_fork, st));
    CK(cudaStreamWaitEvent(s->res_stream, s->ev_res_fork, 0));
    launches += launch_residuals_all(s, dfield, s->res_stream);
    CK(cudaEventRecord(s->ev_res_join, s->res_stream));
  } else if (s->cfg.log_errors && s->res_snap) {
    launches += launch_residuals_all(s, dfield, st);
  }
  CK(cudaEventRecord(s->ev[3], st));
  // ---- final jumps per neighbour pair (solver.cpp:416).  After a mode-2
  // epoch all copies of each control are bit-identical and every per-pair
  // jump is exactly 0 (the kernel checks the last iteration on the device).
  if (s->npairs > 0) {
    if (!fuse01)  // (the fused epoch's finalize cleared them)
      CK(cudaMemsetAsync(s->pair_jumps.p, 0, s->pair_jumps.n * sizeof(unsigned long long), st));
    s->tl.begin("pair_jumps");
    launches += regions ? mfb::launch_epoch_regions(region_args(s, 3), st)
                        : mfb::launch_epoch(epoch_args(s, 3), st);
    s->tl.end();
  }
  // ---- assemble_owned (solver.cpp:418-423)
  mfb::AssembleArgs aa{};
  aa.D = d.rank;
  for (int k = 0; k < 3; ++k) {
    aa.B[k] = d.blocks[k];
    aa.N[k] = d.n_ctrl[k];
    aa.oc_off[k] = s->oc_off[k];
    aa.axbase[k] = s->axbase[k];
  }
  aa.own_coord = s->own_coord.p;
  aa.rowbase = s->rowbase.p;
  aa.probs = wl.d_probs.p;
  aa.poff = s->poff.p;
  aa.P = wl.P.p;
  aa.lattice = s->lattice.p;
  set_assemble_range(s, aa);
  s->tl.begin("assemble");
  launches += mfb::launch_assemble(aa, st);
  s->tl.end();
  // ---- block_error_slab over every block == global decode (solver.cpp:425-438)
  launches += enqueue_decode(s, dfield);
  if (res_side) CK(cudaStreamWaitEvent(st, s->ev_res_join, 0));
  CK(cudaGetLastError());
  double* hr = s->hres;
  CK(cudaMemcpyAsync(hr, s->red2.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hr + 2, ctx->d_status, sizeof(mfb::DevStatus), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hr + s->hres_eo, s->epoch_out.p, s->epoch_out.n * sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(hr + s->hres_es, s->est.p, sizeof(mfb::EpochState), cudaMemcpyDeviceToHost, st));
  if (s->npairs > 0)
    CK(cudaMemcpyAsync(hr + s->hres_pj, s->pair_jumps.p, s->pair_jumps.n * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost, st));
  CK(cudaEventRecord(s->ev[4], st));
  return launches;
}

// Wait for an enqueued solve and unpack its results (the only host sync).
void finish_solve(mfadd_solver* s, int launches) {
  mfadd_context* ctx = s->ctx;
  cudaStream_t st = ctx->stream;
  const Decomp& d = s->dec;
  CK(cudaStreamSynchronize(st));
  const double* hr = s->hres;
  mfb::DevStatus stt{};
  std::memcpy(&stt, hr + 2, sizeof stt);
  if (stt.code) {
    CK(cudaMemsetAsync(ctx->d_status, 0, sizeof(mfb::DevStatus), st));
    CK(cudaStreamSynchronize(st));
    s->wl.raise_status(stt, "");
  }
  const double* eo = hr + s->hres_eo;
  mfb::EpochState es{};
  std::memcpy(&es, hr + s->hres_es, sizeof es);
  s->epochs.clear();
  mfadd_solve_summary& sum = s->summary;
  sum = mfadd_solve_summary{};
  s->epochs.push_back({0, 0.0, eo[1], eo[2]});
  sum.converged = 1;
  if (s->cfg.enforce_continuity && d.any_shared) {
    const int last = es.iter;
    for (int it = 1; it <= last; ++it)
      s->epochs.push_back({it, eo[3 * it], eo[3 * it + 1], eo[3 * it + 2]});
    sum.final_dp = eo[3 * last];
    sum.converged = es.converged;
    sum.constraint_iterations = es.converged ? last - 1 : last;  // solver.cpp:406-412
    launches += last;  // one epoch kernel per loop iteration
  }
  sum.global_l2 = std::sqrt(hr[0]);
  sum.global_linf = hr[1];
  const auto* pj = reinterpret_cast<const unsigned long long*>(hr + s->hres_pj);
  s->final_jumps.assign(static_cast<std::size_t>(s->npairs) * 4, 0.0);
  for (int i = 0; i < s->npairs; ++i) {
    s->final_jumps[4 * static_cast<std::size_t>(i)] = s->pair_ids[static_cast<std::size_t>(i)][0];
    s->final_jumps[4 * static_cast<std::size_t>(i) + 1] = s->pair_ids[static_cast<std::size_t>(i)][1];
    s->final_jumps[4 * static_cast<std::size_t>(i) + 2] = bits_to_double(pj[2 * static_cast<std::size_t>(i)]);
    s->final_jumps[4 * static_cast<std::size_t>(i) + 3] = bits_to_double(pj[2 * static_cast<std::size_t>(i) + 1]);
  }
  sum.n_epochs = static_cast<int>(s->epochs.size());
  sum.n_final_jumps = s->npairs;
  if (s->cfg.log_errors) {
    s->h_block_errs.resize(static_cast<std::size_t>(sum.n_epochs) * d.nblocks * 2);
    CK(cudaMemcpy(s->h_block_errs.data(), s->block_errs.p, s->h_block_errs.size() * sizeof(double),
                  cudaMemcpyDeviceToHost));
  }
  static const bool no_timings = std::getenv("MFADD_NO_TIMINGS") != nullptr;  // measurement aid
  if (!no_timings) {
    sum.t_setup = ev_ms(s->ev[0], s->ev[1]) * 1e-3;
    sum.t_local_solve = ev_ms(s->ev[1], s->ev[2]) * 1e-3;
    sum.t_exchange = 0.0;  // single device: the exchange is fused into K4
    sum.t_constraint = ev_ms(s->ev[2], s->ev[3]) * 1e-3;
    sum.t_decode = ev_ms(s->ev[3], s->ev[4]) * 1e-3;
  }
  s->last_launches = launches;
  ctx->launches += launches;
  s->have_result = true;
}

// ---------------------------------------------------------------- sharded
// A group of shard solvers driven in lockstep (one per process with NCCL, or
// all ranks in one process with the loopback transport).  Per epoch: pack the
// cross-rank holder copies, exchange, average (local tiles + cross tiles; both
// ranks of a cross region form the identical ascending-holder sum, so every
// copy stays bitwise equal to the single-device solve), dp/jumps max-reduced
// across ranks (solver.cpp:394-413 with the runtime.cpp exchange over NCCL).
struct Transport {
  virtual ~Transport() = default;
  virtual void exchange(std::vector<mfadd_solver*>& g) = 0;               // send -> recv buffers
  virtual void max_u64(std::vector<mfadd_solver*>& g, std::size_t off, std::size_t n, bool pairs) = 0;
  // owned lattice rows to the ranks whose decode reads them (full: to every rank)
  virtual void gather_lattice(std::vector<mfadd_solver*>& g, bool full) = 0;
  // elementwise sum of a device array that every rank filled at its own entries
  using ArrayOf = std::pair<double*, std::size_t> (*)(mfadd_solver*);
  virtual void sum_f64(std::vector<mfadd_solver*>& g, ArrayOf arr) = 0;
  // red2: sum l2^2 over ranks (each decoded its own rows), or max when every
  // rank decoded all rows (generic decode path: identical values), max linf
  virtual void reduce_err(std::vector<mfadd_solver*>& g, bool sum_l2) = 0;
};

// The lattice rows rank q's decode reads (mfadd_solver::need_lo/need_hi of q).
void lattice_need(const mfadd_solver* s, int q, std::int64_t& lo, std::int64_t& hi) {
  const Decomp& d = s->dec;
  lo = 0;
  hi = d.n_ctrl[0];
  if (!s->tma_decode) return;
  const mfb::ShardRange r = mfb::shard_range(d, q, s->nranks);
  const int p = d.degree;
  auto span = [&](std::int64_t j) {
    return host_find_span(d.knots[0], p, static_cast<double>(j) / static_cast<double>(d.grid[0] - 1));
  };
  lo = std::max<std::int64_t>(0, span(r.in_lo) - p);
  hi = std::min<std::int64_t>(d.n_ctrl[0], span(r.in_hi - 1) + 1);
}

std::int64_t lattice_row_elems(const Decomp& d) {
  std::int64_t r = 1;
  for (int k = 1; k < d.rank; ++k) r *= d.n_ctrl[k];
  return r;
}

struct NcclTransport : Transport {
  void exchange(std::vector<mfadd_solver*>& g) override {
    mfadd_solver* s = g[0];
    if (s->peers.empty()) return;
    cudaStream_t st = s->ctx->stream;
    NCK(ncclGroupStart());
    for (const auto& pr : s->peers) {
      if (pr.send_count) NCK(ncclSend(s->sendbuf.p + pr.send_off, pr.send_count, ncclFloat64, pr.rank, s->comm->comm, st));
      if (pr.recv_count) NCK(ncclRecv(s->recvbuf.p + pr.recv_off, pr.recv_count, ncclFloat64, pr.rank, s->comm->comm, st));
    }
    NCK(ncclGroupEnd());
  }
  void max_u64(std::vector<mfadd_solver*>& g, std::size_t off, std::size_t n, bool pairs) override {
    mfadd_solver* s = g[0];
    auto* p = pairs ? s->pair_jumps.p + off : reinterpret_cast<unsigned long long*>(s->epoch_out.p + off);
    NCK(ncclAllReduce(p, p, n, ncclUint64, ncclMax, s->comm->comm, s->ctx->stream));
  }
  void sum_f64(std::vector<mfadd_solver*>& g, ArrayOf arr) override {
    const auto a = arr(g[0]);
    NCK(ncclAllReduce(a.first, a.first, a.second, ncclFloat64, ncclSum, g[0]->comm->comm, g[0]->ctx->stream));
  }
  void gather_lattice(std::vector<mfadd_solver*>& g, bool full) override {
    mfadd_solver* s = g[0];
    const Decomp& d = s->dec;
    if (s->srange.partial) {
      // every entry is owned by exactly one rank and +0.0 elsewhere: the sum
      // of the 64-bit patterns is the owner's value, bit for bit
      if (!s->lattice_complete)
        NCK(ncclAllReduce(s->lattice.p, s->lattice.p, s->lattice.n, ncclUint64, ncclSum, s->comm->comm, s->ctx->stream));
      s->lattice_complete = true;
      return;
    }
    const std::int64_t row = lattice_row_elems(d);
    NCK(ncclGroupStart());
    for (int q = 0; q < s->nranks; ++q) {
      if (q == s->rank) continue;
      const mfb::ShardRange mine = s->srange, theirs = mfb::shard_range(d, q, s->nranks);
      std::int64_t qlo = 0, qhi = d.n_ctrl[0];  // rows q's decode reads (full: all)
      if (!full) lattice_need(s, q, qlo, qhi);
      const std::int64_t s0 = std::max(mine.own_lo, qlo), s1 = std::min(mine.own_hi, qhi);
      const std::int64_t r0 = std::max(theirs.own_lo, full ? std::int64_t{0} : s->need_lo),
                         r1 = std::min(theirs.own_hi, full ? d.n_ctrl[0] : s->need_hi);
      if (s1 > s0)
        NCK(ncclSend(s->lattice.p + s0 * row, (s1 - s0) * row, ncclFloat64, q, s->comm->comm, s->ctx->stream));
      if (r1 > r0)
        NCK(ncclRecv(s->lattice.p + r0 * row, (r1 - r0) * row, ncclFloat64, q, s->comm->comm, s->ctx->stream));
    }
    NCK(ncclGroupEnd());
  }
  void reduce_err(std::vector<mfadd_solver*>& g, bool sum_l2) override {
    mfadd_solver* s = g[0];
    NCK(ncclAllReduce(s->red2.p, s->red2.p, 1, ncclFloat64, sum_l2 ? ncclSum : ncclMax, s->comm->comm,
                      s->ctx->stream));
    NCK(ncclAllReduce(s->red2.p + 1, s->red2.p + 1, 1, ncclFloat64, ncclMax, s->comm->comm, s->ctx->stream));
  }
};

// All ranks' shard solvers in one process on one device (tests): the host
// orders every step, so no kernel waits on another.
struct LoopbackTransport : Transport {
  void exchange(std::vector<mfadd_solver*>& g) override {
    for (mfadd_solver* r : g)
      for (const auto& pr : r->peers) {
        mfadd_solver* q = g[static_cast<std::size_t>(pr.rank)];
        const ShardPeer* back = nullptr;
        for (const auto& pq : q->peers)
          if (pq.rank == r->rank) back = &pq;
        if (!back || back->send_count != pr.recv_count) throw std::logic_error("loopback: asymmetric exchange plan");
        if (pr.recv_count)
          CK(cudaMemcpyAsync(r->recvbuf.p + pr.recv_off, q->sendbuf.p + back->send_off, pr.recv_count * sizeof(double),
                             cudaMemcpyDeviceToDevice, r->ctx->stream));
      }
  }
  void max_u64(std::vector<mfadd_solver*>& g, std::size_t off, std::size_t n, bool pairs) override {
    std::vector<unsigned long long> acc(n, 0ull), v(n);
    for (mfadd_solver* s : g) {
      const void* p = pairs ? static_cast<const void*>(s->pair_jumps.p + off) : static_cast<const void*>(s->epoch_out.p + off);
      CK(cudaMemcpyAsync(v.data(), p, n * 8, cudaMemcpyDeviceToHost, s->ctx->stream));
      CK(cudaStreamSynchronize(s->ctx->stream));
      for (std::size_t i = 0; i < n; ++i) acc[i] = std::max(acc[i], v[i]);
    }
    for (mfadd_solver* s : g) {
      void* p = pairs ? static_cast<void*>(s->pair_jumps.p + off) : static_cast<void*>(s->epoch_out.p + off);
      CK(cudaMemcpyAsync(p, acc.data(), n * 8, cudaMemcpyHostToDevice, s->ctx->stream));
      CK(cudaStreamSynchronize(s->ctx->stream));
    }
  }
  void sum_f64(std::vector<mfadd_solver*>& g, ArrayOf arr) override {
    const std::size_t n = arr(g[0]).second;
    std::vector<double> acc(n, 0.0), v(n);
    for (mfadd_solver* s : g) {  // rank order
      CK(cudaMemcpy(v.data(), arr(s).first, n * sizeof(double), cudaMemcpyDeviceToHost));
      for (std::size_t i = 0; i < n; ++i) acc[i] += v[i];
    }
    for (mfadd_solver* s : g) CK(cudaMemcpy(arr(s).first, acc.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  }
  void gather_lattice(std::vector<mfadd_solver*>& g, bool full) override {
    const Decomp& d = g[0]->dec;
    if (g[0]->srange.partial) {  // the u64 sum of NcclTransport, on the host
      if (g[0]->lattice_complete) return;
      const std::size_t n = g[0]->lattice.n;
      std::vector<unsigned long long> acc(n, 0ull), v(n);
      for (mfadd_solver* s : g) {
        CK(cudaMemcpyAsync(v.data(), s->lattice.p, n * 8, cudaMemcpyDeviceToHost, s->ctx->stream));
        CK(cudaStreamSynchronize(s->ctx->stream));
        for (std::size_t i = 0; i < n; ++i) acc[i] += v[i];
      }
      for (mfadd_solver* s : g) {
        CK(cudaMemcpyAsync(s->lattice.p, acc.data(), n * 8, cudaMemcpyHostToDevice, s->ctx->stream));
        CK(cudaStreamSynchronize(s->ctx->stream));
        s->lattice_complete = true;
      }
      return;
    }
    const std::int64_t row = lattice_row_elems(d);
    for (mfadd_solver* q : g)
      for (mfadd_solver* r : g) {
        if (q == r) continue;
        const std::int64_t r0 = std::max(q->srange.own_lo, full ? std::int64_t{0} : r->need_lo),
                           r1 = std::min(q->srange.own_hi, full ? d.n_ctrl[0] : r->need_hi);
        if (r1 > r0)
          CK(cudaMemcpyAsync(r->lattice.p + r0 * row, q->lattice.p + r0 * row, (r1 - r0) * row * sizeof(double),
                             cudaMemcpyDeviceToDevice, r->ctx->stream));
      }
  }
  void reduce_err(std::vector<mfadd_solver*>& g, bool sum_l2) override {
    double l2 = 0.0, li = 0.0, v[2];
    for (mfadd_solver* s : g) {  // rank order
      CK(cudaMemcpyAsync(v, s->red2.p, sizeof v, cudaMemcpyDeviceToHost, s->ctx->stream));
      CK(cudaStreamSynchronize(s->ctx->stream));
      l2 = sum_l2 ? l2 + v[0] : std::max(l2, v[0]);
      li = std::max(li, v[1]);
    }
    v[0] = l2;
    v[1] = li;
    for (mfadd_solver* s : g) {
      CK(cudaMemcpyAsync(s->red2.p, v, sizeof v, cudaMemcpyHostToDevice, s->ctx->stream));
      CK(cudaStreamSynchronize(s->ctx->stream));
    }
  }
};

int shard_pack(mfadd_solver* s) {
  return mfb::launch_pack(s->pack_tiles.p, s->npack, s->wl.P.p, s->sendbuf.p, s->ctx->stream);
}

// One epoch's averaging/measurement on this rank after the exchange.
int shard_compute(mfadd_solver* s, int mode, int slot, bool predicated = false) {
  cudaStream_t st = s->ctx->stream;
  int l = 0;
  mfb::EpochRegionArgs a = region_args(s, mode);
  a.predicated = predicated ? 1 : 0;  // no-op once an earlier epoch of the chunk converged
  a.finalize = 0;
  a.recv = s->recvbuf.p;
  a.slot = slot;
  l += mfb::launch_epoch_regions(a, st);
  a.tiles = s->xtiles.p;
  a.ntiles = s->nxtiles;
  l += mfb::launch_epoch_regions(a, st);
  if (mode != 3) {
    a.tiles = s->tiles.p;
    a.ntiles = s->ntiles;
    l += mfb::launch_epoch_finalize(a, st);
  }
  return l;
}

// Wait for the context stream of a sharded solver while polling the
// communicator: an asynchronous NCCL error (a lost peer, a failed
// connection) or no progress within MFADD_NCCL_TIMEOUT_S seconds (default
// 600) aborts the communicator and raises MFADD_ECUDA instead of hanging
// (the reference's workers are threads of one process and cannot be lost).
void sync_sharded(mfadd_solver* s) {
  cudaStream_t st = s->ctx->stream;
  mfadd_comm* c = s->comm;
  if (!c) {
    CK(cudaStreamSynchronize(st));
    return;
  }
  if (c->aborted) throw ApiError(MFADD_ECUDA, "mfadd: the NCCL communicator was aborted by an earlier failure");
  static const double limit = std::getenv("MFADD_NCCL_TIMEOUT_S") ? std::atof(std::getenv("MFADD_NCCL_TIMEOUT_S")) : 600.0;
  const auto t0 = std::chrono::steady_clock::now();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) CK(e);
    ncclResult_t ae = ncclSuccess;
    ncclCommGetAsyncError(c->comm, &ae);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (ae != ncclSuccess && ae != ncclInProgress) {
      ncclCommAbort(c->comm);
      c->aborted = true;
      throw ApiError(MFADD_ECUDA, std::string("NCCL asynchronous error on rank ") + std::to_string(c->rank) + ": " +
                                      ncclGetErrorString(ae) + " (communicator aborted)");
    }
    if (el > limit) {
      ncclCommAbort(c->comm);
      c->aborted = true;
      throw ApiError(MFADD_ECUDA, "NCCL: no progress for " + std::to_string(static_cast<int>(limit)) + " s on rank " +
                                      std::to_string(c->rank) + " (communicator aborted; MFADD_NCCL_TIMEOUT_S)");
    }
    std::this_thread::yield();
  }
}

int shard_assemble_decode(mfadd_solver* s, const double* dfield) {
  const Decomp& d = s->dec;
  Workload& wl = s->wl;
  cudaStream_t st = s->ctx->stream;
  int l = 0;
  mfb::AssembleArgs aa{};
  aa.D = d.rank;
  for (int k = 0; k < 3; ++k) {
    aa.B[k] = d.blocks[k];
    aa.N[k] = d.n_ctrl[k];
    aa.oc_off[k] = s->oc_off[k];
    aa.axbase[k] = s->axbase[k];
  }
  aa.own_coord = s->own_coord.p;
  aa.rowbase = s->rowbase.p;
  aa.probs = wl.d_probs.p;
  aa.poff = s->poff.p;
  aa.P = wl.P.p;
  aa.lattice = s->lattice.p;
  set_assemble_range(s, aa);
  // block-id ranges finer than block rows: the lattice is combined by a sum
  // over ranks of bit patterns, so every entry this rank does not own is +0.0
  if (s->srange.partial) {
    CK(cudaMemsetAsync(s->lattice.p, 0, s->lattice.n * sizeof(double), st));
    s->lattice_complete = false;
  }
  l += mfb::launch_assemble(aa, st);
  return l;
}

int shard_decode(mfadd_solver* s, const double* dfield) { return enqueue_decode(s, dfield); }

void solve_group(std::vector<mfadd_solver*>& g, const std::vector<const double*>& fields, Transport& tr) {
  static const bool trace = std::getenv("MFADD_TRACE") != nullptr;
  auto tmark = [&](const char* what, int it) {
    if (!trace) return;
    for (mfadd_solver* s : g) CK(cudaStreamSynchronize(s->ctx->stream));
    std::fprintf(stderr, "[mfadd shard] %s %d\n", what, it);
  };
  mfadd_solver* s0 = g[0];
  const Decomp& d = s0->dec;
  const bool loop = s0->cfg.enforce_continuity && d.any_shared;
  std::vector<int> launches(g.size(), 0);
  for (std::size_t r = 0; r < g.size(); ++r) {
    mfadd_solver* s = g[r];
    s->have_result = false;
    s->tl.st = s->ctx->stream;
    (void)cudaGetLastError();
    if (loop && !s->holder_fault.empty()) {
      s->wl.setup(s->ctx, &s->tl);
      s->wl.fit(s->ctx, fields[r], &s->tl);
      s->wl.raise_status(read_status(s->ctx), "");
      throw std::runtime_error(s->holder_fault);
    }
    CK(cudaEventRecord(s->ev[0], s->ctx->stream));
    launches[r] += s->wl.setup(s->ctx, &s->tl);
    CK(cudaEventRecord(s->ev[1], s->ctx->stream));
    launches[r] += s->wl.fit(s->ctx, fields[r], &s->tl);
    CK(cudaEventRecord(s->ev[2], s->ctx->stream));
    CK(cudaMemsetAsync(s->est.p, 0, sizeof(mfb::EpochState), s->ctx->stream));
  }
  // One epoch on every rank.  The loop bookkeeping runs on the device
  // (k_shard_advance, after dp is max-reduced over the ranks), and an
  // iteration enqueued behind an unread one is predicated on st->converged, so
  // the host reads the loop state once per chunk of iterations, not per epoch.
  auto epoch = [&](int mode, int slot, bool predicated) {
    for (std::size_t r = 0; r < g.size(); ++r) launches[r] += shard_pack(g[r]);
    tr.exchange(g);
    for (std::size_t r = 0; r < g.size(); ++r) launches[r] += shard_compute(g[r], mode, slot, predicated);
    tr.max_u64(g, static_cast<std::size_t>(3 * slot), 3, false);
    for (std::size_t r = 0; r < g.size(); ++r) {
      mfadd_solver* s = g[r];
      launches[r] += mfb::launch_shard_advance(s->est.p, s->epoch_out.p, slot, s->cfg.tolerance, s->ctx->stream);
      if (s->cfg.log_errors && !s->res_snap) {  // record_epoch's block errors, skipped with a skipped epoch
        s->tl.begin("residual");
        mfb::BlockResArgs ra = res_args(s, fields[r], s->est.p, slot);
        ra.expect_iter = slot;
        launches[r] += mfb::launch_block_residual(s->wl.p, ra, s->ctx->stream);
        s->tl.end();
      }
    }
  };
  auto read_state = [&](mfadd_solver* s) {  // identical on every rank after the max
    mfb::EpochState es{};
    CK(cudaMemcpyAsync(&es, s->est.p, sizeof es, cudaMemcpyDeviceToHost, s->ctx->stream));
    sync_sharded(s);
    return es;
  };
  if (s0->cfg.log_errors)
    for (mfadd_solver* s : g)
      CK(cudaMemsetAsync(s->block_errs.p, 0, s->block_errs.n * sizeof(double), s->ctx->stream));
  tmark("fit done", 0);
  epoch(0, 0, false);  // record_epoch(0, 0.0)
  tmark("epoch", 0);
  int last = 0;
  bool converged = true;
  if (loop) {
    converged = false;
    const int chunk = std::max(1, env_int("MFADD_SHARD_CHUNK", 3));  // iterations per host sync
    for (int it = 1; it <= s0->cfg.max_outer_iterations && !converged;) {
      const int hi = std::min(s0->cfg.max_outer_iterations, it + chunk - 1);
      for (int j = it; j <= hi; ++j) {
        epoch(j >= 2 ? 2 : 1, j, j > it);
        tmark("epoch", j);
      }
      mfb::EpochState es{};
      for (mfadd_solver* s : g) es = read_state(s);
      last = es.last_iter;
      converged = es.converged != 0;
      it = hi + 1;
    }
  }
  for (mfadd_solver* s : g) CK(cudaEventRecord(s->ev[3], s->ctx->stream));
  if (s0->npairs > 0) {  // final jumps (solver.cpp:416); exactly zero after a mode-2 epoch
    for (mfadd_solver* s : g)
      CK(cudaMemsetAsync(s->pair_jumps.p, 0, s->pair_jumps.n * sizeof(unsigned long long), s->ctx->stream));
    if (last < 2) {
      for (std::size_t r = 0; r < g.size(); ++r) launches[r] += shard_pack(g[r]);
      tr.exchange(g);
      for (std::size_t r = 0; r < g.size(); ++r) launches[r] += shard_compute(g[r], 3, 0);
      tr.max_u64(g, 0, s0->pair_jumps.n, true);
    }
  }
  tmark("jumps", 0);
  if (s0->cfg.log_errors && s0->res_snap && g.size() == 1) {  // the host-driven loop of one device
    mfb::EpochState es{};
    es.iter = last;
    CK(cudaMemcpyAsync(s0->est.p, &es, sizeof es, cudaMemcpyHostToDevice, s0->ctx->stream));
    launches[0] += launch_residuals_all(s0, fields[0], s0->ctx->stream);
  }
  for (std::size_t r = 0; r < g.size(); ++r) launches[r] += shard_assemble_decode(g[r], fields[r]);
  tr.gather_lattice(g, false);  // the halo rows each rank's decode reads (no all-gather)
  tmark("assembled", 0);
  for (std::size_t r = 0; r < g.size(); ++r) launches[r] += shard_decode(g[r], fields[r]);
  tr.reduce_err(g, s0->tma_decode);
  if (s0->cfg.log_errors) tr.sum_f64(g, [](mfadd_solver* s) { return std::make_pair(s->block_errs.p, s->block_errs.n); });
  tmark("decoded", 0);
  // results (identical on every rank after the reductions)
  for (std::size_t r = 0; r < g.size(); ++r) {
    mfadd_solver* s = g[r];
    cudaStream_t st = s->ctx->stream;
    double* hr = s->hres;
    CK(cudaMemcpyAsync(hr, s->red2.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hr + 2, s->ctx->d_status, sizeof(mfb::DevStatus), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hr + s->hres_eo, s->epoch_out.p, s->epoch_out.n * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (s->npairs > 0)
      CK(cudaMemcpyAsync(hr + s->hres_pj, s->pair_jumps.p, s->pair_jumps.n * sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(s->ev[4], st));
    mfb::EpochState es{};
    es.iter = last;
    es.last_iter = last;
    es.converged = converged ? 1 : 0;
    sync_sharded(s);
    std::memcpy(hr + s->hres_es, &es, sizeof es);
    finish_solve(s, launches[r] - (loop ? last : 0));  // finish_solve adds one launch per iteration
  }
}

// Enqueue one solve on the context stream without waiting: replay the cached
// whole-solve graph of (field, output slot) when possible (no per-kernel
// profiling, no debug sync checks, no holder fault), else direct launches.
int enqueue_cached(mfadd_solver* s, const double* dfield) {
  const bool graphable = !s->tl.on && !s->tl.sync_check && s->holder_fault.empty() && !std::getenv("MFADD_NO_GRAPH");
  if (!graphable) return enqueue_solve(s, dfield);
  cudaStream_t st = s->ctx->stream;
  mfadd_solver::SolveGraph* gr = nullptr;
  for (auto& e : s->graphs)
    if (e.field == dfield && e.lattice == s->lattice.p) gr = &e;
  if (!gr) {  // first solve of this key: direct launches (one-time attribute setup outside capture)
    if (s->graphs.size() >= 4) {
      if (s->graphs.front().exec) CK(cudaGraphExecDestroy(s->graphs.front().exec));
      s->graphs.erase(s->graphs.begin());
    }
    s->graphs.push_back({dfield, s->lattice.p, nullptr, 0});
    return enqueue_solve(s, dfield);
  }
  if (!gr->exec) {
    cudaGraph_t g = nullptr;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
    int launches = 0;
    try {
      launches = enqueue_solve(s, dfield);
    } catch (...) {
      cudaStreamEndCapture(st, &g);
      if (g) cudaGraphDestroy(g);
      throw;
    }
    CK(cudaStreamEndCapture(st, &g));
    const cudaError_t e = cudaGraphInstantiate(&gr->exec, g, 0);
    cudaGraphDestroy(g);
    CK(e);
    gr->launches = launches;
  }
  CK(cudaGraphLaunch(gr->exec, st));
  return gr->launches;
}

// solve(): replay the cached whole-solve graph when possible (no per-kernel
// profiling, no debug sync checks, no holder fault), else launch directly.
void solve_impl(mfadd_solver* s, const double* dfield) {
  s->have_result = false;
  if (s->nranks > 1) {  // sharded: host-driven epochs with NCCL exchanges
    std::vector<mfadd_solver*> g{s};
    NcclTransport tr;
    solve_group(g, {dfield}, tr);
    return;
  }
  static const bool host_loop = std::getenv("MFADD_HOST_LOOP") != nullptr;
  if (host_loop && s->holder_fault.empty() && (s->ntiles > 0 || !s->dec.any_shared)) {
    // profiling aid: every kernel as a direct launch (host-driven epoch loop)
    std::vector<mfadd_solver*> g{s};
    LoopbackTransport tr;
    solve_group(g, {dfield}, tr);
    return;
  }
  finish_solve(s, enqueue_cached(s, dfield));
}

}  // namespace

namespace {
// Host field -> device for one solve.  A sharded solver reads only its slab:
// the axis-0 input rows [box_lo, box_hi) its blocks' fits (and its own decode
// rows, a subset) touch, at their global offsets (each GPU
// uploads the union of its blocks' input boxes).  Returns the bytes copied.
std::size_t upload_field(mfadd_solver* s, const double* host, double* dev, cudaStream_t st) {
  const Decomp& d = s->dec;
  std::int64_t row = 1;
  for (int k = 1; k < d.rank; ++k) row *= d.grid[k];
  std::int64_t lo = 0, hi = d.grid[0];
  if (s->nranks > 1 && s->tma_decode) {  // (the generic decode path decodes every row on every rank)
    lo = s->srange.box_lo;
    hi = s->srange.box_hi;
  }
  const std::size_t n = static_cast<std::size_t>((hi - lo) * row);
  CK(cudaMemcpyAsync(dev + lo * row, host + lo * row, n * sizeof(double), cudaMemcpyHostToDevice, st));
  return n * sizeof(double);
}
// Lattice -> host: a sharded solver returns the lattice rows it owns (its
// blocks' owned controls; mfadd_solver_gather_controls assembles the rest).
void download_controls(mfadd_solver* s, double* host, cudaStream_t st) {
  const Decomp& d = s->dec;
  std::int64_t row = 1;
  for (int k = 1; k < d.rank; ++k) row *= d.n_ctrl[k];
  std::int64_t lo = 0, hi = d.n_ctrl[0];
  if (s->nranks > 1) {
    lo = s->srange.own_lo;
    hi = s->srange.own_hi;
  }
  CK(cudaMemcpyAsync(host + lo * row, s->lattice.p + lo * row, static_cast<std::size_t>((hi - lo) * row) * sizeof(double),
                     cudaMemcpyDeviceToHost, st));
}
// Error field -> host: a sharded solver returns the input rows it decoded.
void download_error(mfadd_solver* s, double* host, cudaStream_t st) {
  const Decomp& d = s->dec;
  std::int64_t row = 1;
  for (int k = 1; k < d.rank; ++k) row *= d.grid[k];
  std::int64_t lo = 0, hi = d.grid[0];
  if (s->nranks > 1 && s->tma_decode) {  // (the generic decode path decodes every row on every rank)
    lo = s->srange.in_lo;
    hi = s->srange.in_hi;
  }
  CK(cudaMemcpyAsync(host + lo * row, s->error.p + lo * row, static_cast<std::size_t>((hi - lo) * row) * sizeof(double),
                     cudaMemcpyDeviceToHost, st));
}
}  // namespace

MFB_API int mfadd_solve(mfadd_solver* s, const double* field, int field_on_device, mfadd_solve_summary* out) {
  return guarded([&] {
    ContextScope scope(s->ctx);
    check_config(s->cfg);
    const double* df = field;
    if (!field_on_device) {
      const std::size_t n = static_cast<std::size_t>(s->dec.total_inputs());
      if (s->field_buf.n != n) s->field_buf.alloc(n);
      upload_field(s, field, s->field_buf.p, s->ctx->stream);
      df = s->field_buf.p;
    }
    solve_impl(s, df);
    if (out) *out = s->summary;
  });
}

// Measurement aid (not part of the boundary): the cached whole-solve graph of
// one device field n times back to back, one host read-back at the end: what
// a solve costs on the device without the host round trip between solves.
extern "C" __attribute__((visibility("default"))) int mfadd_debug_solve_repeat(mfadd_solver* s, const double* dfield, int n) {
  return guarded([&] {
    ContextScope scope(s->ctx);
    int launches = 0;
    for (int i = 0; i < n; ++i) launches = enqueue_cached(s, dfield);
    finish_solve(s, launches);
  });
}

MFB_API int mfadd_solve_host(mfadd_solver* s, const double* field_host, double* out_controls_host,
                             double* out_error_host, mfadd_solve_summary* out) {
  return guarded([&] {
    ContextScope scope(s->ctx);
    check_config(s->cfg);
    if (out_error_host && !s->cfg.store_error)
      throw std::invalid_argument("mfadd_solve_host: out_error requires store_error in the solver config");
    const std::size_t n = static_cast<std::size_t>(s->dec.total_inputs());
    if (s->field_buf.n != n) s->field_buf.alloc(n);
    cudaStream_t st = s->ctx->stream;
    upload_field(s, field_host, s->field_buf.p, st);
    solve_impl(s, s->field_buf.p);
    if (out_controls_host) download_controls(s, out_controls_host, st);
    if (out_error_host) download_error(s, out_error_host, st);
    CK(cudaStreamSynchronize(st));
    if (out) *out = s->summary;
  });
}

// A stream of independent solves (e.g. the time steps of a simulation) with
// host buffers: field i+1 is copied in while solve i computes and while the
// results of solve i are copied out (separate H2D / D2H streams, two device
// field and output slots).  Per step the copies are exactly those of
// mfadd_solve_host; only their overlap differs.
MFB_API int mfadd_solve_host_batch(mfadd_solver* s, int n, const double* const* fields_host,
                                   double* const* out_controls_host, double* const* out_errors_host,
                                   mfadd_solve_summary* out) {
  return guarded([&] {
    ContextScope scope(s->ctx);
    check_config(s->cfg);
    const std::size_t nf = static_cast<std::size_t>(s->dec.total_inputs());
    if (n <= 0) return;
    for (int i = 0; i < n; ++i)
      if (out_errors_host && out_errors_host[i] && !s->cfg.store_error)
        throw std::invalid_argument("mfadd_solve_host_batch: out_errors requires store_error in the solver config");
    if (s->nranks > 1 || s->tl.on || s->tl.sync_check) {  // no overlap: one call per step
      for (int i = 0; i < n; ++i) {
        if (s->field_buf.n != nf) s->field_buf.alloc(nf);
        upload_field(s, fields_host[i], s->field_buf.p, s->ctx->stream);
        solve_impl(s, s->field_buf.p);
        if (out_controls_host && out_controls_host[i]) download_controls(s, out_controls_host[i], s->ctx->stream);
        if (out_errors_host && out_errors_host[i]) download_error(s, out_errors_host[i], s->ctx->stream);
        CK(cudaStreamSynchronize(s->ctx->stream));
        if (out) out[i] = s->summary;
      }
      return;
    }
    // one-time resources
    if (s->field_buf.n != nf) s->field_buf.alloc(nf);
    if (s->field_buf2.n != nf) s->field_buf2.alloc(nf);
    if (s->lattice_alt.n != s->lattice.n) s->lattice_alt.alloc(s->lattice.n);
    if (s->cfg.store_error && s->error_alt.n != s->error.n) s->error_alt.alloc(s->error.n);
    if (!s->h2d_stream) CK(cudaStreamCreateWithFlags(&s->h2d_stream, cudaStreamNonBlocking));
    if (!s->d2h_stream) CK(cudaStreamCreateWithFlags(&s->d2h_stream, cudaStreamNonBlocking));
    for (auto& e : s->bev)
      if (!e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    cudaEvent_t* ev_h2d = s->bev;
    cudaEvent_t* ev_comp = s->bev + 2;
    cudaEvent_t* ev_d2h = s->bev + 4;
    cudaStream_t cs = s->ctx->stream;
    double* fbuf[2] = {s->field_buf.p, s->field_buf2.p};
    int cur_slot = 0;  // which output buffers s->lattice / s->error hold
    auto use_slot = [&](int slot) {
      if (slot != cur_slot) {
        s->lattice.swap(s->lattice_alt);
        if (s->cfg.store_error) s->error.swap(s->error_alt);
        cur_slot = slot;
      }
    };
    auto h2d = [&](int i) {
      const int slot = i & 1;
      if (i >= 2) CK(cudaStreamWaitEvent(s->h2d_stream, ev_comp[slot], 0));  // solve i-2 done reading
      CK(cudaMemcpyAsync(fbuf[slot], fields_host[i], nf * sizeof(double), cudaMemcpyHostToDevice, s->h2d_stream));
      CK(cudaEventRecord(ev_h2d[slot], s->h2d_stream));
    };
    try {
      h2d(0);
      if (n > 1) h2d(1);
      for (int i = 0; i < n; ++i) {
        const int slot = i & 1;
        use_slot(slot);
        CK(cudaStreamWaitEvent(cs, ev_h2d[slot], 0));
        if (i >= 2) CK(cudaStreamWaitEvent(cs, ev_d2h[slot], 0));  // outputs of solve i-2 copied out
        s->have_result = false;
        const int launches = enqueue_cached(s, fbuf[slot]);
        CK(cudaEventRecord(ev_comp[slot], cs));
        CK(cudaStreamWaitEvent(s->d2h_stream, ev_comp[slot], 0));
        if (out_controls_host && out_controls_host[i])
          CK(cudaMemcpyAsync(out_controls_host[i], s->lattice.p, s->lattice.n * sizeof(double),
                             cudaMemcpyDeviceToHost, s->d2h_stream));
        if (out_errors_host && out_errors_host[i])
          CK(cudaMemcpyAsync(out_errors_host[i], s->error.p, s->error.n * sizeof(double), cudaMemcpyDeviceToHost,
                             s->d2h_stream));
        CK(cudaEventRecord(ev_d2h[slot], s->d2h_stream));
        if (i + 2 < n) h2d(i + 2);
        finish_solve(s, launches);  // waits for solve i only; the copies keep running
        if (out) out[i] = s->summary;
      }
      CK(cudaStreamSynchronize(s->d2h_stream));
      CK(cudaStreamSynchronize(s->h2d_stream));
    } catch (...) {
      cudaStreamSynchronize(s->d2h_stream);
      cudaStreamSynchronize(s->h2d_stream);
      throw;
    }
    // s->lattice / s->error now hold the last solve's outputs (read by the getters)
  });
}

MFB_API int mfadd_solver_epochs(const mfadd_solver* s, mfadd_epoch_stats* out, int cap) {
  const int n = static_cast<int>(s->epochs.size());
  for (int i = 0; i < n && i < cap; ++i) out[i] = s->epochs[static_cast<std::size_t>(i)];
  return n;
}

MFB_API int mfadd_solver_final_jumps(const mfadd_solver* s, double* out4, int cap) {
  const int n = static_cast<int>(s->final_jumps.size() / 4);
  for (int i = 0; i < n && i < cap; ++i)
    for (int k = 0; k < 4; ++k) out4[4 * i + k] = s->final_jumps[4 * static_cast<std::size_t>(i) + k];
  return n;
}

MFB_API int mfadd_solver_controls(const mfadd_solver* s, double* out, int out_on_device) {
  return guarded([&] {
    if (!s->have_result) throw std::logic_error("mfadd_solver_controls: no solve result");
    ContextScope scope(s->ctx);
    CK(cudaMemcpyAsync(out, s->lattice.p, s->lattice.n * sizeof(double),
                       out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s->ctx->stream));
    CK(cudaStreamSynchronize(s->ctx->stream));
  });
}

MFB_API int mfadd_solver_global_error(const mfadd_solver* s, double* out, int out_on_device) {
  return guarded([&] {
    if (!s->have_result) throw std::logic_error("mfadd_solver_global_error: no solve result");
    if (!s->cfg.store_error) throw std::invalid_argument("mfadd_solver_global_error: solver built without store_error");
    ContextScope scope(s->ctx);
    CK(cudaMemcpyAsync(out, s->error.p, s->error.n * sizeof(double),
                       out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s->ctx->stream));
    CK(cudaStreamSynchronize(s->ctx->stream));
  });
}

MFB_API int mfadd_solver_block_controls(const mfadd_solver* s, int block, double* out, int out_on_device) {
  return guarded([&] {
    if (!s->have_result) throw std::logic_error("mfadd_solver_block_controls: no solve result");
    if (block < 0 || block >= s->dec.nblocks) throw std::out_of_range("mfadd_solver_block_controls: block id");
    const int lb = s->local_of[static_cast<std::size_t>(block)];
    if (lb < 0) throw std::out_of_range("mfadd_solver_block_controls: block " + std::to_string(block) + " is on rank " +
                                        std::to_string(mfb::shard_of_block(s->dec, s->nranks, block)));
    ContextScope scope(s->ctx);
    const BlockDev& b = s->wl.blocks[static_cast<std::size_t>(lb)];
    std::int64_t np = 1;
    for (int k = 0; k < s->dec.rank; ++k) np *= s->wl.probs[static_cast<std::size_t>(b.ax[k])].n;
    CK(cudaMemcpyAsync(out, s->wl.P.p + b.poff, static_cast<std::size_t>(np) * sizeof(double),
                       out_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s->ctx->stream));
    CK(cudaStreamSynchronize(s->ctx->stream));
  });
}

// The pipeline's continuity probe (pipeline.cpp:210-228): for every block and
// every dim with an upper neighbour, continuity_jumps(below, above, dec, dim,
// u = span_param(dim, span_hi), order) (solver.cpp:263-277) on the held
// lattices of the last solve, all probe points of all interfaces in one
// batched GPU evaluation (model.cu); max over interfaces per order.
MFB_API int mfadd_solver_continuity_probe(mfadd_solver* s, int probe_order, int cross_samples, double* out,
                                          int* out_order) {
  return guarded([&] {
    if (!s->have_result) throw std::logic_error("mfadd_solver_continuity_probe: no solve result");
    if (s->nranks != 1) throw std::logic_error("mfadd_solver_continuity_probe: needs every block on this rank");
    ContextScope scope(s->ctx);
    const Decomp& d = s->dec;
    const int rank = d.rank;
    const int order = probe_order >= 0 ? probe_order : d.degree - 1;
    auto span_param = [&](int k, std::int64_t t) {  // layout.cpp:22-27
      const auto& sk = d.span_knot[static_cast<std::size_t>(k)];
      const auto& kn = d.knots[static_cast<std::size_t>(k)];
      if (t == static_cast<std::int64_t>(sk.size())) return kn[kn.size() - static_cast<std::size_t>(d.degree) - 1];
      return kn[static_cast<std::size_t>(sk[static_cast<std::size_t>(t)])];
    };
    std::vector<mfb::EvalLattice> lats(static_cast<std::size_t>(d.nblocks));
    for (int b = 0; b < d.nblocks; ++b) {
      const BlockDev& bd = s->wl.blocks[static_cast<std::size_t>(b)];
      mfb::EvalLattice& L = lats[static_cast<std::size_t>(b)];
      L.base = bd.poff;
      for (int k = 0; k < rank; ++k) {
        L.ext[k] = s->wl.probs[static_cast<std::size_t>(bd.ax[k])].n;
        L.coff[k] = s->wl.probs[static_cast<std::size_t>(bd.ax[k])].col_lo;
      }
    }
    std::vector<mfb::EvalItem> items;
    std::vector<std::size_t> firsts;
    for (int b = 0; b < d.nblocks; ++b)
      for (int dim = 0; dim < rank; ++dim) {
        const auto& c = d.coords[static_cast<std::size_t>(b)];
        if (c[static_cast<std::size_t>(dim)] + 1 >= d.blocks[static_cast<std::size_t>(dim)]) continue;
        int ac[3] = {c[0], c[1], c[2]};
        ++ac[dim];
        const int above = d.block_id(ac);
        const double u = span_param(dim, d.at(b, dim, mfb::SPAN_HI));
        std::vector<std::vector<double>> cross;  // probe_cross_params, solver.cpp:197-209
        for (int k = 0; k < rank; ++k) {
          if (k == dim) continue;
          const double lo = span_param(k, d.at(b, k, mfb::SPAN_LO)), hi = span_param(k, d.at(b, k, mfb::SPAN_HI));
          std::vector<double> pts;
          for (int q = 0; q < cross_samples; ++q) {
            const double t = cross_samples == 1
                                 ? 0.5
                                 : 0.1 + 0.8 * static_cast<double>(q) / static_cast<double>(cross_samples - 1);
            pts.push_back(lo + t * (hi - lo));
          }
          cross.push_back(std::move(pts));
        }
        firsts.push_back(items.size());
        mfb::probe_items(rank, dim, u, order, cross, b, above, items);
      }
    firsts.push_back(items.size());
    std::vector<int> degs(static_cast<std::size_t>(rank), d.degree);
    std::vector<double> kn;
    std::vector<std::int64_t> ko(1, 0);
    for (int k = 0; k < rank; ++k) {
      kn.insert(kn.end(), d.knots[static_cast<std::size_t>(k)].begin(), d.knots[static_cast<std::size_t>(k)].end());
      ko.push_back(static_cast<std::int64_t>(kn.size()));
    }
    std::vector<double> vals;
    mfb::eval_items_device(s->ctx, rank, degs.data(), kn.data(), ko.data(), s->wl.P.p, lats, items, vals);
    std::vector<double> jumps(static_cast<std::size_t>(order) + 1, 0.0);
    for (std::size_t f = 0; f + 1 < firsts.size(); ++f)
      mfb::probe_reduce(vals, firsts[f], firsts[f + 1] - firsts[f], order, jumps);
    std::memcpy(out, jumps.data(), jumps.size() * sizeof(double));
    if (out_order) *out_order = order;
  });
}

MFB_API int mfadd_solver_block_errors(const mfadd_solver* s, int epoch, double* out2) {
  return guarded([&] {
    if (!s->have_result) throw std::logic_error("mfadd_solver_block_errors: no solve result");
    if (!s->cfg.log_errors) throw std::invalid_argument("mfadd_solver_block_errors: solver built without log_errors");
    const int nb = s->dec.nblocks;
    if (epoch < 0 || static_cast<std::size_t>(epoch + 1) * nb * 2 > s->h_block_errs.size())
      throw std::out_of_range("mfadd_solver_block_errors: epoch");
    std::memcpy(out2, s->h_block_errs.data() + static_cast<std::size_t>(epoch) * nb * 2, nb * 2 * sizeof(double));
  });
}

MFB_API const double* mfadd_solver_device_controls(const mfadd_solver* s) { return s->lattice.p; }

MFB_API int mfadd_solver_gather_controls(mfadd_solver* s) {
  return guarded([&] {
    if (s->nranks <= 1) return;
    ContextScope scope(s->ctx);
    std::vector<mfadd_solver*> g{s};
    NcclTransport tr;
    tr.gather_lattice(g, true);
    sync_sharded(s);
  });
}

MFB_API int mfadd_solver_set_profiling(mfadd_solver* s, int on) {
  s->tl.on = on != 0;
  s->tl.reset(s->ctx->stream);  // records accumulate across solves until the next call
  return MFADD_OK;
}

MFB_API int mfadd_solver_kernel_times(const mfadd_solver* s, char* names, int name_len, double* ms, int cap) {
  const int n = static_cast<int>(s->tl.used);
  for (int i = 0; i < n && i < cap; ++i) {
    const auto& r = s->tl.recs[static_cast<std::size_t>(i)];
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    ms[i] = t;
    if (names) {
      std::strncpy(names + static_cast<std::size_t>(i) * name_len, r.name.c_str(), static_cast<std::size_t>(name_len) - 1);
      names[static_cast<std::size_t>(i) * name_len + name_len - 1] = 0;
    }
  }
  return n;
}
MFB_API int mfadd_solver_last_launches(const mfadd_solver* s) { return s->last_launches; }

// ---------------------------------------------------------------- fine-grained
namespace {

void check_params_ascending(const double* p, std::int64_t m) {  // collocation.cpp:89-93
  if (m <= 0) throw std::invalid_argument("collocation_matrix: empty parameter list");
  for (std::int64_t j = 1; j < m; ++j)
    if (p[j] < p[j - 1]) throw std::invalid_argument("collocation_matrix: params must be ascending");
}

void check_window(int nknots, int degree, std::int64_t lo, std::int64_t hi) {
  const std::int64_t nb = nknots - degree - 1;
  if (lo < 0 || hi > nb || lo >= hi) throw std::invalid_argument("collocation_matrix: bad column window");
}

}  // namespace

MFB_API int mfadd_collocation(mfadd_context* ctx, const double* knots, int nknots, int degree, const double* params,
                              int64_t m, int64_t col_lo, int64_t col_hi, int64_t* out_first_col, int* out_count,
                              double* out_values) {
  return guarded([&] {
    ContextScope scope(ctx);
    if (degree < 1 || degree > mfb::kMaxDegree) throw std::invalid_argument("mfadd_collocation: unsupported degree");
    check_params_ascending(params, m);
    check_window(nknots, degree, col_lo, col_hi);
    Workload wl;
    wl.D = 1;
    wl.p = degree;
    AxisProb pr{};
    pr.dim = 0;
    pr.m = static_cast<int>(m);
    pr.n = static_cast<int>(col_hi - col_lo);
    pr.col_lo = col_lo;
    pr.M = -1;
    pr.param_off = 0;
    pr.knot_off = 0;
    pr.nknots = nknots;
    wl.probs.push_back(pr);
    wl.layout_tables();
    cudaStream_t st = ctx->stream;
    wl.d_probs.upload(wl.probs, st);
    wl.knots.upload(std::vector<double>(knots, knots + nknots), st);
    wl.params.upload(std::vector<double>(params, params + m), st);
    wl.g0.alloc(static_cast<std::size_t>(m));
    wl.first_col.alloc(static_cast<std::size_t>(m));
    wl.count.alloc(static_cast<std::size_t>(m));
    wl.vals.alloc(static_cast<std::size_t>(m) * (degree + 1));
    mfb::RowsArgs ra{wl.d_probs.p, 1, pr.m, wl.knots.p, wl.params.p, wl.g0.p, wl.first_col.p, wl.count.p, wl.vals.p,
                     ctx->d_status};
    ctx->launches += mfb::launch_basis_rows(degree, ra, st);
    CK(cudaGetLastError());
    std::vector<int> g0(static_cast<std::size_t>(m)), fc(static_cast<std::size_t>(m));
    std::vector<double> v(static_cast<std::size_t>(m) * (degree + 1));
    CK(cudaMemcpyAsync(g0.data(), wl.g0.p, g0.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fc.data(), wl.first_col.p, fc.size() * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(out_count, wl.count.p, static_cast<std::size_t>(m) * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(v.data(), wl.vals.p, v.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    const mfb::DevStatus stt = read_status(ctx);
    wl.raise_status(stt, "");
    // repack to BandedCollocation layout (clipped values left-aligned)
    for (std::int64_t j = 0; j < m; ++j) {
      out_first_col[j] = fc[static_cast<std::size_t>(j)];
      const int shift = fc[static_cast<std::size_t>(j)] - g0[static_cast<std::size_t>(j)];
      for (int k = 0; k <= degree; ++k) {
        const int src = k + shift;
        out_values[j * (degree + 1) + k] =
            (k < out_count[j] && src <= degree) ? v[static_cast<std::size_t>(j) * (degree + 1) + src] : 0.0;
      }
    }
  });
}

MFB_API int mfadd_fit_unconstrained(mfadd_context* ctx, int rank, int degree, const double* knots,
                                    const int64_t* kn_off, const double* params, const int64_t* pm_off,
                                    const int64_t* col_lo, const int64_t* col_hi, const double* q, double* out_p) {
  return guarded([&] {
    ContextScope scope(ctx);
    if (rank < 1 || rank > 3) throw std::invalid_argument("fit_unconstrained: rank must be 1..3");
    if (degree < 1 || degree > mfb::kMaxDegree) throw std::invalid_argument("fit_unconstrained: unsupported degree");
    Workload wl;
    wl.D = rank;
    wl.p = degree;
    BlockDev bd{};
    std::int64_t qn = 1;
    for (int k = 0; k < rank; ++k) {
      const std::int64_t m = pm_off[k + 1] - pm_off[k];
      check_params_ascending(params + pm_off[k], m);
      check_window(static_cast<int>(kn_off[k + 1] - kn_off[k]), degree, col_lo[k], col_hi[k]);
      AxisProb pr{};
      pr.dim = k;
      pr.m = static_cast<int>(m);
      pr.n = static_cast<int>(col_hi[k] - col_lo[k]);
      pr.col_lo = col_lo[k];
      pr.M = -1;
      pr.param_off = pm_off[k];
      pr.knot_off = kn_off[k];
      pr.nknots = static_cast<int>(kn_off[k + 1] - kn_off[k]);
      bd.ax[k] = k;
      wl.factor_ids.push_back(k);
      wl.probs.push_back(pr);
      qn *= m;
    }
    for (int k = 0; k < rank; ++k)  // lsq.cpp:14-18
      if (wl.probs[static_cast<std::size_t>(k)].m < wl.probs[static_cast<std::size_t>(k)].n)
        throw std::invalid_argument("LocalProblem: underdetermined in dimension " + std::to_string(k) + " (" +
                                    std::to_string(wl.probs[static_cast<std::size_t>(k)].m) + " rows < " +
                                    std::to_string(wl.probs[static_cast<std::size_t>(k)].n) + " cols)");
    {
      std::int64_t stv = 1;
      for (int k = rank - 1; k >= 0; --k) {
        wl.fs[k] = stv;
        stv *= wl.probs[static_cast<std::size_t>(k)].m;
      }
      wl.field_n = stv;
    }
    wl.blocks.push_back(bd);
    wl.layout_tables();
    cudaStream_t st = ctx->stream;
    wl.allocate(st);
    wl.knots.upload(std::vector<double>(knots, knots + kn_off[rank]), st);
    wl.params.upload(std::vector<double>(params, params + pm_off[rank]), st);
    std::vector<unsigned char> sf;
    for (int k = 0; k < rank; ++k) {
      wl.sflag_off[k] = static_cast<std::int64_t>(sf.size());
      sf.resize(sf.size() + static_cast<std::size_t>(col_hi[k]), 0);
    }
    wl.sflag.upload(sf, st);
    DBuf<double> dq;
    dq.upload(std::vector<double>(q, q + qn), st);
    ctx->launches += wl.setup(ctx);
    ctx->launches += wl.fit(ctx, dq.p);
    const mfb::DevStatus stt = read_status(ctx);
    wl.raise_status(stt, "");
    CK(cudaMemcpyAsync(out_p, wl.P.p, static_cast<std::size_t>(wl.total_p) * sizeof(double), cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
  });
}

MFB_API int mfadd_residual_error(mfadd_context* ctx, int rank, int degree, const double* knots, const int64_t* kn_off,
                                 const double* params, const int64_t* pm_off, const int64_t* col_lo,
                                 const int64_t* col_hi, const double* q, const double* controls,
                                 double* out_pointwise, double* out_l2, double* out_linf) {
  return guarded([&] {
    ContextScope scope(ctx);
    if (rank < 1 || rank > 3) throw std::invalid_argument("residual_error: rank must be 1..3");
    if (degree < 1 || degree > mfb::kMaxDegree) throw std::invalid_argument("residual_error: unsupported degree");
    Workload wl;
    wl.D = rank;
    wl.p = degree;
    std::int64_t qn = 1, pn = 1;
    for (int k = 0; k < rank; ++k) {
      const std::int64_t m = pm_off[k + 1] - pm_off[k];
      check_params_ascending(params + pm_off[k], m);
      check_window(static_cast<int>(kn_off[k + 1] - kn_off[k]), degree, col_lo[k], col_hi[k]);
      AxisProb pr{};
      pr.dim = k;
      pr.m = static_cast<int>(m);
      pr.n = static_cast<int>(col_hi[k] - col_lo[k]);
      pr.col_lo = col_lo[k];
      pr.M = -1;
      pr.param_off = pm_off[k];
      pr.knot_off = kn_off[k];
      pr.nknots = static_cast<int>(kn_off[k + 1] - kn_off[k]);
      wl.probs.push_back(pr);
      qn *= m;
      pn *= pr.n;
    }
    wl.layout_tables();
    cudaStream_t st = ctx->stream;
    wl.d_probs.upload(wl.probs, st);
    wl.knots.upload(std::vector<double>(knots, knots + kn_off[rank]), st);
    wl.params.upload(std::vector<double>(params, params + pm_off[rank]), st);
    wl.g0.alloc(static_cast<std::size_t>(wl.total_rows));
    wl.first_col.alloc(static_cast<std::size_t>(wl.total_rows));
    wl.count.alloc(static_cast<std::size_t>(wl.total_rows));
    wl.vals.alloc(static_cast<std::size_t>(wl.total_rows) * (degree + 1));
    mfb::RowsArgs ra{wl.d_probs.p, rank, wl.max_m, wl.knots.p, wl.params.p, wl.g0.p, wl.first_col.p, wl.count.p,
                     wl.vals.p, ctx->d_status};
    ctx->launches += mfb::launch_basis_rows(degree, ra, st);
    DBuf<double> dq, dp, dout, dpart, dred;
    dq.upload(std::vector<double>(q, q + qn), st);
    dp.upload(std::vector<double>(controls, controls + pn), st);
    if (out_pointwise) dout.alloc(static_cast<std::size_t>(qn));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    const int ctas = static_cast<int>(std::max<std::int64_t>(1, std::min<std::int64_t>((qn + 255) / 256, 8 * sms)));
    dpart.alloc(static_cast<std::size_t>(ctas) * 2);
    dred.alloc(2);
    mfb::ResidualArgs a{};
    a.D = rank;
    for (int k = 0; k < 3; ++k) {
      const int kk = k < rank ? k : 0;
      const AxisProb& pr = wl.probs[static_cast<std::size_t>(kk)];
      a.m[k] = k < rank ? pr.m : 1;
      a.n[k] = k < rank ? pr.n : 1;
      a.g0[k] = wl.g0.p + pr.row_off;
      a.vals[k] = wl.vals.p + pr.row_off * (degree + 1);
    }
    a.controls = dp.p;
    a.q = dq.p;
    a.pointwise = out_pointwise ? dout.p : nullptr;
    a.partial = dpart.p;
    a.total = qn;
    ctx->launches += mfb::launch_residual_points(degree, a, ctas, st);
    ctx->launches += mfb::launch_reduce_partials(dpart.p, ctas, dred.p, st);
    CK(cudaGetLastError());
    const mfb::DevStatus stt = read_status(ctx);
    wl.raise_status(stt, "");
    double red[2] = {0.0, 0.0};
    CK(cudaMemcpyAsync(red, dred.p, sizeof red, cudaMemcpyDeviceToHost, st));
    if (out_pointwise)
      CK(cudaMemcpyAsync(out_pointwise, dout.p, static_cast<std::size_t>(qn) * sizeof(double), cudaMemcpyDeviceToHost,
                         st));
    CK(cudaStreamSynchronize(st));
    if (out_l2) *out_l2 = std::sqrt(red[0]);
    if (out_linf) *out_linf = red[1];
  });
}

MFB_API int mfadd_decode(mfadd_context* ctx, int rank, int degree, const double* knots, const int64_t* kn_off,
                         const double* params, const int64_t* pm_off, const int64_t* ctrl_ext,
                         const int64_t* col_offset, const double* controls, double* out) {
  return guarded([&] {
    ContextScope scope(ctx);
    if (rank < 1 || rank > 3) throw std::invalid_argument("decode: dimension mismatch between lattice, knot vectors and parameters");
    if (degree < 1 || degree > mfb::kMaxDegree) throw std::invalid_argument("decode: unsupported degree");
    Workload wl;
    wl.D = rank;
    wl.p = degree;
    std::int64_t Mi[3], Ni[3], nctl = 1, nout = 1;
    std::vector<std::vector<double>> kv(static_cast<std::size_t>(rank)), pv(static_cast<std::size_t>(rank));
    for (int k = 0; k < rank; ++k) {
      const std::int64_t m = pm_off[k + 1] - pm_off[k];
      const std::int64_t off = col_offset ? col_offset[k] : 0;
      check_params_ascending(params + pm_off[k], m);
      check_window(static_cast<int>(kn_off[k + 1] - kn_off[k]), degree, off, off + ctrl_ext[k]);
      AxisProb pr{};
      pr.dim = k;
      pr.m = static_cast<int>(m);
      pr.n = static_cast<int>(ctrl_ext[k]);
      pr.col_lo = off;
      pr.M = -1;
      pr.param_off = pm_off[k];
      pr.knot_off = kn_off[k];
      pr.nknots = static_cast<int>(kn_off[k + 1] - kn_off[k]);
      wl.probs.push_back(pr);
      Mi[k] = m;
      Ni[k] = ctrl_ext[k];
      nctl *= ctrl_ext[k];
      nout *= m;
      kv[static_cast<std::size_t>(k)].assign(knots + kn_off[k], knots + kn_off[k + 1]);
      pv[static_cast<std::size_t>(k)].assign(params + pm_off[k], params + pm_off[k + 1]);
    }
    wl.layout_tables();
    cudaStream_t st = ctx->stream;
    wl.d_probs.upload(wl.probs, st);
    wl.knots.upload(std::vector<double>(knots, knots + kn_off[rank]), st);
    wl.params.upload(std::vector<double>(params, params + pm_off[rank]), st);
    wl.g0.alloc(static_cast<std::size_t>(wl.total_rows));
    wl.first_col.alloc(static_cast<std::size_t>(wl.total_rows));
    wl.count.alloc(static_cast<std::size_t>(wl.total_rows));
    wl.vals.alloc(static_cast<std::size_t>(wl.total_rows) * (degree + 1));
    mfb::RowsArgs ra{wl.d_probs.p, rank, wl.max_m, wl.knots.p, wl.params.p, wl.g0.p, wl.first_col.p, wl.count.p,
                     wl.vals.p, ctx->d_status};
    ctx->launches += mfb::launch_basis_rows(degree, ra, st);
    DecodePlan dp;
    dp.init(rank, degree, Mi, Ni);
    for (int k = 0; k < 3; ++k) {
      const int src = k - (3 - rank);
      if (src < 0) continue;
      // window widths in local columns: spans relative to the same knots
      dp.size_windows(k, kv[static_cast<std::size_t>(src)], pv[static_cast<std::size_t>(src)], degree, 0);
      dp.prob_of[k] = src;
    }
    DBuf<double> dctl, dout, dpart;
    DBuf<int> ug0;
    DBuf<double> uval;
    dctl.upload(std::vector<double>(controls, controls + nctl), st);
    dout.alloc(static_cast<std::size_t>(nout));
    ug0.upload(std::vector<int>{0}, st);
    uval.upload(std::vector<double>{1.0}, st);
    mfb::DecodeArgs da{};
    da.D = rank;
    for (int k = 0; k < 3; ++k) {
      da.M[k] = dp.M[k];
      da.N[k] = dp.N[k];
      da.T[k] = dp.T[k];
      da.ntiles[k] = dp.ntiles[k];
      da.W[k] = dp.W[k];
      da.pk[k] = dp.pk[k];
      if (dp.prob_of[k] >= 0) {
        const AxisProb& pr = wl.probs[static_cast<std::size_t>(dp.prob_of[k])];
        da.g0[k] = wl.g0.p + pr.row_off;
        da.vals[k] = wl.vals.p + pr.row_off * (degree + 1);
      } else {
        da.g0[k] = ug0.p;
        da.vals[k] = uval.p;
      }
    }
    da.lattice = dctl.p;
    da.field = nullptr;
    da.out = dout.p;
    da.partial = nullptr;
    ctx->launches += mfb::launch_decode(degree, da, st);
    CK(cudaGetLastError());
    const mfb::DevStatus stt = read_status(ctx);
    wl.raise_status(stt, "");
    CK(cudaMemcpyAsync(out, dout.p, static_cast<std::size_t>(nout) * sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

// ---------------------------------------------------------------- multi-GPU
MFB_API int mfadd_nccl_unique_id(unsigned char* out128) {
  return guarded([&] {
    ncclUniqueId id;
    NCK(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId size");
    std::memcpy(out128, &id, sizeof id);
  });
}

MFB_API int mfadd_comm_create(mfadd_context* ctx, const unsigned char* id128, int rank, int nranks, mfadd_comm** out) {
  return guarded([&] {
    ContextScope scope(ctx);
    auto c = std::make_unique<mfadd_comm>();
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof id);
    NCK(ncclCommInitRank(&c->comm, nranks, id, rank));
    c->rank = rank;
    c->nranks = nranks;
    *out = c.release();
  });
}

MFB_API void mfadd_comm_free(mfadd_comm* c) {
  if (!c) return;
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
}

MFB_API int mfadd_shard_range(const mfadd_decomposition* dec, int rank, int nranks, int* blo, int* bhi,
                              int64_t* in_lo, int64_t* in_hi) {
  return guarded([&] {
    const mfb::ShardRange r = mfb::shard_range(dec->d, rank, nranks);
    *blo = r.blo;
    *bhi = r.bhi;
    if (in_lo) *in_lo = r.in_lo;
    if (in_hi) *in_hi = r.in_hi;
  });
}

MFB_API int mfadd_shard_ctrl_rows(const mfadd_decomposition* dec, int rank, int nranks, int64_t* own_lo,
                                  int64_t* own_hi) {
  return guarded([&] {
    const mfb::ShardRange r = mfb::shard_range(dec->d, rank, nranks);
    *own_lo = r.own_lo;
    *own_hi = r.own_hi;
  });
}

MFB_API int mfadd_shard_box(const mfadd_decomposition* dec, int rank, int nranks, int64_t* box_lo, int64_t* box_hi) {
  return guarded([&] {
    const mfb::ShardRange r = mfb::shard_range(dec->d, rank, nranks);
    *box_lo = r.box_lo;
    *box_hi = r.box_hi;
  });
}

MFB_API int mfadd_shard_exchange(const mfadd_decomposition* dec, int rank, int nranks, int peer, int recv,
                                 int64_t* out, int64_t cap) {
  int64_t count = -1;
  const int rc = guarded([&] {
    const mfb::Decomp& d = dec->d;
    const auto regs = mfb::enumerate_regions(d);
    count = 0;
    for (const auto& pl : mfb::shard_peers(d, regs, rank, nranks)) {
      if (pl.peer != peer) continue;
      for (const auto& e : recv ? pl.recv : pl.send) {
        const mfb::Region& R = regs[static_cast<std::size_t>(e.first)];
        for (std::int64_t i0 = 0; i0 < R.ext[0]; ++i0)
          for (std::int64_t i1 = 0; i1 < R.ext[1]; ++i1)
            for (std::int64_t i2 = 0; i2 < R.ext[2]; ++i2) {
              if (out && count < cap) {  // (holder block, global control indices)
                out[4 * count] = R.ids[static_cast<std::size_t>(e.second)];
                out[4 * count + 1] = R.lo[0] + i0;
                out[4 * count + 2] = R.lo[1] + i1;
                out[4 * count + 3] = R.lo[2] + i2;
              }
              ++count;
            }
      }
    }
  });
  return rc == MFADD_OK ? static_cast<int>(count) : -rc;
}

MFB_API int mfadd_solve_loopback(mfadd_context* ctx, const mfadd_decomposition* dec, const mfadd_solver_config* cfg,
                                 int nranks, const double* field_host, double* out_controls, double* out_error,
                                 mfadd_solve_summary* out, mfadd_epoch_stats* epochs, int epochs_cap,
                                 double* final_jumps4, int jumps_cap) {
  return guarded([&] {
    ContextScope scope(ctx);
    std::vector<std::unique_ptr<mfadd_solver>> own;
    std::vector<mfadd_solver*> g;
    for (int r = 0; r < nranks; ++r) {
      own.push_back(create_solver(ctx, dec, cfg, r, nranks, nullptr));
      g.push_back(own.back().get());
    }
    // one field buffer per rank, NaN outside the rank's slab (upload_field):
    // any read outside the slab would show in the results
    const std::size_t n = static_cast<std::size_t>(dec->d.total_inputs());
    std::vector<DBuf<double>> fb(g.size());
    std::vector<const double*> fields;
    for (std::size_t r = 0; r < g.size(); ++r) {
      fb[r].alloc(n);
      CK(cudaMemsetAsync(fb[r].p, 0xff, n * sizeof(double), ctx->stream));
      upload_field(g[r], field_host, fb[r].p, ctx->stream);
      fields.push_back(fb[r].p);
    }
    LoopbackTransport tr;
    solve_group(g, fields, tr);
    mfadd_solver* s0 = g[0];
    if (out_controls)  // each rank's owned lattice rows
      for (mfadd_solver* s : g) download_controls(s, out_controls, s->ctx->stream);
    CK(cudaStreamSynchronize(ctx->stream));
    if (out_error) {  // each rank's own input rows
      const mfb::Decomp& d = dec->d;
      std::int64_t row = 1;
      for (int k = 1; k < d.rank; ++k) row *= d.grid[k];
      for (mfadd_solver* s : g)
        CK(cudaMemcpy(out_error + s->srange.in_lo * row, s->error.p + s->srange.in_lo * row,
                      (s->srange.in_hi - s->srange.in_lo) * row * sizeof(double), cudaMemcpyDeviceToHost));
    }
    if (out) *out = s0->summary;
    for (int i = 0; i < static_cast<int>(s0->epochs.size()) && i < epochs_cap; ++i) epochs[i] = s0->epochs[static_cast<std::size_t>(i)];
    for (int i = 0; i < s0->npairs && i < jumps_cap; ++i)
      for (int k = 0; k < 4; ++k) final_jumps4[4 * i + k] = s0->final_jumps[4 * static_cast<std::size_t>(i) + k];
  });
}
