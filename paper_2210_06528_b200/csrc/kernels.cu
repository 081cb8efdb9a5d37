// sm_100a kernels of the B200-native domain-decomposed MFA encode path.
//
// Kernel map (reference routine each one replaces; paths under
// /root/reference/proj/core/src):
//   K1 k_basis_rows   find_span + basis_funs + collocation window clip
//                     (knots.cpp:83-129, collocation.cpp:83-111)
//   K2 k_gram_chol    BandedCollocation::gram + Eigen LLT
//                     (collocation.cpp:56-67, lsq.cpp:46-55)
//   K3 k_fit_strided  fit_unconstrained axis pass on a non-contiguous axis
//      k_fit_last     ... on the contiguous (last) axis
//                     (lsq.cpp:57-61, collocation.cpp:46-54, tensor.hpp:78-106)
//   K4 k_epoch        one exchange/averaging epoch over all shared controls
//                     (solver.cpp:112-164,381-398; runtime.cpp:123-158) +
//                     jump_residuals (solver.cpp:166-193)
//   K5 k_dp           dp = max_b change_b / max(1, ||P_b||) (solver.cpp:402-405)
//   K6 k_assemble     assemble_owned (solver.cpp:281-294)
//   K7 k_decode       decode + error + L2^2/Linf partials (decode.cpp:83-97,
//                     solver.cpp:298-328)
// Bitwise-exact pieces: spans, first_col/count (integers), basis values and
// Gram entries (explicit round-to-nearest ops, no FMA contraction, same
// operation order as the reference).  The contractions and triangular solves
// use FMA; they agree with the reference at rounding level (tolerance parity).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"

#include <cstdio>

// Debug builds (-DMFB_DEBUG, libmfadd_b200_debug.so) range-check global
// indices; a failed check records its source line in a device word and makes
// the thread return (no trap, so the host can still read the record).
#ifdef MFB_DEBUG
__device__ int g_mfb_debug_line = 0;
#define MFB_ASSERT(c, tag)                        \
  do {                                            \
    if (!(c)) {                                   \
      atomicCAS(&g_mfb_debug_line, 0, __LINE__);  \
      return;                                     \
    }                                             \
  } while (0)
#else
#define MFB_ASSERT(c, tag) \
  do {                     \
  } while (0)
#endif

namespace mfb {

bool pdl_enabled() {
  static const bool on = std::getenv("MFADD_NO_PDL") == nullptr;
  return on;
}

namespace {

constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ void set_status(DevStatus* st, int code, int prob, int row) {
  if (atomicCAS(&st->code, 0, code) == 0) {
    st->axis_prob = prob;
    st->row = row;
  }
}

__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

__device__ __forceinline__ unsigned long long umax(unsigned long long a, unsigned long long b) { return a > b ? a : b; }

__device__ __forceinline__ unsigned long long warp_umax(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = umax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// Block-wide max of a u64, result valid in thread 0.  `red` >= 32 entries.
__device__ __forceinline__ unsigned long long block_umax(unsigned long long v, unsigned long long* red) {
  v = warp_umax(v);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = lane < nw ? red[lane] : 0ull;
    v = warp_umax(v);
  }
  return v;
}

// ------------------------------------------------------------------- K1
template <int P>
__global__ void __launch_bounds__(256) k_basis_rows(RowsArgs a) {
  pdl_enter();
  const int pid = a.prob0 + static_cast<int>(blockIdx.y);
  const AxisProb pr = a.probs[pid];
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= pr.m) return;
  const double* kn = a.knots + pr.knot_off;
  // solver.cpp:64: u = (double)(input_lo + j) / (double)(M - 1), IEEE division
  const double u = pr.M >= 0 ? __ddiv_rn(static_cast<double>(pr.in_lo + j), static_cast<double>(pr.M - 1))
                             : a.params[pr.param_off + j];
  const int nb = pr.nknots - P - 1;
  const double lo = kn[P], hi = kn[nb];
  const std::int64_t row = pr.row_off + j;
  if (u < lo || u > hi) {  // knots.cpp:88-90
    set_status(a.status, 2, pid, j);
    a.g0[row] = 0;
    a.first_col[row] = 0;
    a.count[row] = 0;
#pragma unroll
    for (int k = 0; k <= P; ++k) a.vals[row * (P + 1) + k] = 0.0;
    return;
  }
  int span;
  if (u >= hi) {  // knots.cpp:91-95: right endpoint -> last nonempty span
    int s = nb - 1;
    while (s > P && kn[s] == kn[s + 1]) --s;
    span = s;
  } else {  // knots.cpp:96-105: the unique s in [P, nb) with kn[s] <= u < kn[s+1]
    // a guess from uniform spacing plus a short walk (the decomposition's
    // knots are uniform: two loads instead of the ~11 of the binary search);
    // the binary search of the reference when the walk does not settle
    int g = P + static_cast<int>((u - lo) / (hi - lo) * static_cast<double>(nb - P));
    g = g < P ? P : (g > nb - 1 ? nb - 1 : g);
    int steps = 0;
    while (steps < 4 && u < kn[g]) --g, ++steps;
    while (steps < 4 && u >= kn[g + 1]) ++g, ++steps;
    if (kn[g] <= u && u < kn[g + 1]) {
      span = g;
    } else {
      int low = P, high = nb, mid = (low + high) / 2;
      while (u < kn[mid] || u >= kn[mid + 1]) {
        if (u < kn[mid])
          high = mid;
        else
          low = mid;
        mid = (low + high) / 2;
      }
      span = mid;
    }
  }
  // knots.cpp:108-129 Cox-de Boor, explicit RN ops (no contraction)
  double N[P + 1], left[P + 1], right[P + 1];
  N[0] = 1.0;
#pragma unroll
  for (int jj = 1; jj <= P; ++jj) {
    left[jj] = __dsub_rn(u, kn[span + 1 - jj]);
    right[jj] = __dsub_rn(kn[span + jj], u);
    double saved = 0.0;
#pragma unroll
    for (int r = 0; r < jj; ++r) {
      const double denom = __dadd_rn(right[r + 1], left[jj - r]);
      const double temp = __ddiv_rn(N[r], denom);
      N[r] = __dadd_rn(saved, __dmul_rn(right[r + 1], temp));
      saved = __dmul_rn(left[jj - r], temp);
    }
    N[jj] = saved;
  }
  // collocation.cpp:97-108: clip to the column window
  const std::int64_t g0 = static_cast<std::int64_t>(span) - P;
  const std::int64_t clo = pr.col_lo, chi = pr.col_lo + pr.n;
  const std::int64_t lc = g0 > clo ? g0 : clo;
  const std::int64_t hc = (g0 + P + 1) < chi ? (g0 + P + 1) : chi;
  if (lc >= hc) set_status(a.status, 1, pid, j);
  a.g0[row] = static_cast<int>(g0 - clo);
  a.first_col[row] = static_cast<int>(lc - clo);
  a.count[row] = hc > lc ? static_cast<int>(hc - lc) : 0;
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    const std::int64_t g = g0 + k;
    a.vals[row * (P + 1) + k] = (g >= lc && g < hc) ? N[k] : 0.0;
  }
}

// Banded Cholesky (the Eigen LLT of lsq.cpp:46-49 restricted to the band: L
// has no fill outside it) by one thread, right-looking within each row: as
// soon as L(c,c-k) is known it is applied to the pending sums of the entries
// left of it and to the diagonal, so the dependent chain per entry is one
// multiply and one FMA.  The last P rows sit in a register ring with
// compile-time slots (row j in slot j mod P; the column loop is unrolled by
// P), so the next row's first entries overlap this row's rsqrt.  src row c
// holds [G(c,c), G(c,c-1), .., G(c,c-P)] (zero where c-k < 0); row c of dst
// becomes [1/L(c,c), L(c,c-1), .., L(c,c-P)] (dst may be src).  FLIP: the
// factor of the index-reversed matrix, G'(c,c-k) = G(n-1-c+k, n-1-c) read from
// src.  Rows [0, rows) are factored.  Returns the first non-positive pivot's
// row (Eigen LLT NumericalIssue -> SingularFitError) or -1.
template <int P, bool FLIP>
__device__ __forceinline__ int banded_chol(const double* src, double* dst, const int n, const int rows) {
  double R[P][P + 1];  // R[j mod P] = [1/L(j,j), L(j,j-1), .., L(j,j-P)]
#pragma unroll
  for (int r = 0; r < P; ++r)
#pragma unroll
    for (int k = 0; k <= P; ++k) R[r][k] = 0.0;
  // Branch-free body (the tail past `rows` reads row 0 and is not stored), so
  // the compiler can overlap a row's first entries with the previous row's
  // reciprocal square root.
  int bad = -1;
  for (int c0 = 0; c0 < rows; c0 += P) {
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int c = c0 + u;
      const bool in = c < rows;
      double g[P + 1];
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        if (FLIP) {
          const bool ok = in && k <= c;  // row n-1-c+k < n
          const double gv = src[(ok ? n - 1 - c + k : 0) * (P + 1) + k];
          g[k] = ok ? gv : (in ? 0.0 : 1.0);
        } else {
          g[k] = in ? src[c * (P + 1) + k] : 1.0;
        }
      }
      double Lc[P + 1];
#pragma unroll
      for (int k = P; k >= 1; --k) {
        const int sj = (u - k + P) % P;  // row c-k
        const double lk = g[k] * R[sj][0];
        Lc[k] = lk;
#pragma unroll
        for (int k2 = k - 1; k2 >= 1; --k2) g[k2] = fma(-lk, R[(u - k2 + P) % P][k - k2], g[k2]);
        g[0] = fma(-lk, lk, g[0]);
      }
      double dg = g[0];
      const bool sing = !(dg > 0.0);
      bad = (sing && in && bad < 0) ? c : bad;
      dg = sing ? 1.0 : dg;
      // 1/sqrt(dg): fp32 estimate + two Newton steps (no slow-path branch)
      double y = static_cast<double>(rsqrtf(static_cast<float>(dg)));
      y = y * fma(-0.5 * dg, y * y, 1.5);
      y = y * fma(-0.5 * dg, y * y, 1.5);
      Lc[0] = y;
      double* Gc = dst + (in ? c : 0) * (P + 1);
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        if (in) Gc[k] = Lc[k];
        R[u % P][k] = Lc[k];
      }
    }
  }
  return bad;
}

// ------------------------------------------------------------------- K2
template <int P>
__global__ void __launch_bounds__(256) k_gram_chol(CholArgs a) {
  extern __shared__ double sm[];  // n*(P+1): sm[c*(P+1)+k] = G(c, c-k) -> L(c, c-k)
  const int pid = a.prob_ids[blockIdx.x];
  const AxisProb pr = a.probs[pid];
  const int n = pr.n, m = pr.m;
  const int* g0 = a.g0 + pr.row_off;
  const double* v = a.vals + pr.row_off * (P + 1);
  double* band = a.ltab + pr.col_off * (2 * P + 1);  // light mode: the Gram band between the two launches
  // twisted solves: a pristine copy of the band (sm2) and the factor of the
  // index-reversed matrix (sm3), behind everything else in shared memory
  double* sm2 = a.tw ? sm + a.max_n * (P + 1) + (a.stage_rows ? a.max_m * (P + 1) + (a.max_m + 1) / 2 : 0) : nullptr;
  double* sm3 = a.tw ? sm2 + a.max_n * (P + 1) : nullptr;
  if (a.light == 2) {  // Cholesky-only launch: the band written by the Gram-only launch
    constexpr int B = 8;  // independent loads in flight per thread (one warp)
    const int nv = n * (P + 1), nt = static_cast<int>(blockDim.x);
    for (int e0 = threadIdx.x; e0 < nv; e0 += B * nt) {
      double t[B];
#pragma unroll
      for (int u = 0; u < B; ++u) t[u] = e0 + u * nt < nv ? band[e0 + u * nt] : 0.0;
#pragma unroll
      for (int u = 0; u < B; ++u)
        if (e0 + u * nt < nv) {
          sm[e0 + u * nt] = t[u];
          if (sm2) sm2[e0 + u * nt] = t[u];
        }
    }
    __syncthreads();
  } else {
  if (a.stage_rows) {  // row table -> smem (coalesced), then the Gram reads are smem hits
    double* sv = sm + a.max_n * (P + 1);
    int* sg = reinterpret_cast<int*>(sv + a.max_m * (P + 1));
    {  // 8 independent loads in flight per thread (the copy is latency-bound otherwise)
      constexpr int B = 8;
      const int nv = m * (P + 1), nt = static_cast<int>(blockDim.x);
      for (int i0 = threadIdx.x; i0 < nv; i0 += B * nt) {
        double t[B];
#pragma unroll
        for (int u = 0; u < B; ++u) t[u] = i0 + u * nt < nv ? __ldg(v + i0 + u * nt) : 0.0;
#pragma unroll
        for (int u = 0; u < B; ++u)
          if (i0 + u * nt < nv) sv[i0 + u * nt] = t[u];
      }
      for (int i0 = threadIdx.x; i0 < m; i0 += B * nt) {
        int t[B];
#pragma unroll
        for (int u = 0; u < B; ++u) t[u] = i0 + u * nt < m ? __ldg(g0 + i0 + u * nt) : 0;
#pragma unroll
        for (int u = 0; u < B; ++u)
          if (i0 + u * nt < m) sg[i0 + u * nt] = t[u];
      }
    }
    __syncthreads();
    v = sv;
    g0 = sg;
  }
  // collocation.cpp:56-67: each entry accumulated over rows in row order
  for (int e = threadIdx.x; e < n * (P + 1); e += blockDim.x) {
    const int c = e / (P + 1), k = e - c * (P + 1);
    double s = 0.0;
    if (c - k >= 0) {
      int lo = 0, hi = m;  // first row with g0 >= c - P
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (g0[mid] < c - P)
          lo = mid + 1;
        else
          hi = mid;
      }
      for (int j = lo; j < m; ++j) {
        const int gj = g0[j];
        if (gj > c - k) break;
        s = __dadd_rn(s, __dmul_rn(v[j * (P + 1) + (c - gj)], v[j * (P + 1) + (c - k - gj)]));
      }
    }
    sm[e] = s;
    if (sm2) sm2[e] = s;
  }
  if (a.light == 1) {  // Gram-only launch
    for (int e = threadIdx.x; e < n * (P + 1); e += blockDim.x) band[e] = sm[e];
    return;
  }
  __syncthreads();
  }
  // Banded Cholesky by thread 0; twisted solves: the first thread of warp 1
  // factors the index-reversed matrix beside it (its own warp: neither
  // instruction stream waits for the other), only as far as the bottom half
  // of the twisted solve reaches.
  if (threadIdx.x == 0) {
    const int bad = banded_chol<P, false>(sm, sm, n, n);
    if (bad >= 0) set_status(a.status, 3, pid, bad);
  } else if (a.tw && threadIdx.x == 32) {
    banded_chol<P, true>(sm2, sm3, n, n - (n - P) / 2);  // nb + P rows (tw_bot)
  }
  __syncthreads();
  // table per column: [1/L(c,c), L(c,c-k) k=1..P, L(c+k,c) k=1..P]
  double* out = a.ltab + pr.col_off * (2 * P + 1);
  for (int e = threadIdx.x; e < n * (2 * P + 1); e += blockDim.x) {
    const int c = e / (2 * P + 1), q = e - c * (2 * P + 1);
    double val;
    if (q == 0) {
      val = sm[c * (P + 1)];
    } else if (q <= P) {
      val = (c - q >= 0) ? sm[c * (P + 1) + q] : 0.0;
    } else {
      const int k = q - P;
      val = (c + k < n) ? sm[(c + k) * (P + 1) + k] : 0.0;
    }
    out[e] = val;
  }
  if (a.tw) {  // reversed factor, then the Gram band
    double* tw = a.tw + static_cast<std::int64_t>(pid) * a.tw_stride;
    const int fr = (n - (n - P) / 2) * (P + 1);  // factored rows of the reversed matrix
    for (int e = threadIdx.x; e < n * (P + 1); e += blockDim.x) {
      tw[e] = e < fr ? sm3[e] : 0.0;
      tw[n * (P + 1) + e] = sm2[e];
    }
  }
}

// ------------------------------------------------------------------- K3
constexpr int kRowChunk = 64;  // rows staged per smem chunk (strided pass)
constexpr int kPrefetch = 4;   // input rows in flight per thread
constexpr int kStridedThreads = 256;

// Flush the window column `cbase`: forward substitution of column c
// (y_c = (b_c - sum_k L(c,c-k) y_{c-k}) / L(c,c)), then shift the window.
#define MFB_FLUSH_FWD(STORE)                                      \
  {                                                               \
    const int c_ = cbase;                                         \
    if (c_ >= 0 && c_ < n) {                                      \
      const double* Lc_ = lt + static_cast<std::int64_t>(c_) * (2 * P + 1); \
      double s_ = acc[0];                                         \
      _Pragma("unroll") for (int k_ = 1; k_ <= P; ++k_) s_ = fma(-Lc_[k_], yw[k_ - 1], s_); \
      const double y_ = s_ * Lc_[0];                              \
      STORE;                                                      \
      _Pragma("unroll") for (int k_ = P - 1; k_ >= 1; --k_) yw[k_] = yw[k_ - 1]; \
      yw[0] = y_;                                                 \
    }                                                             \
    _Pragma("unroll") for (int k_ = 0; k_ < P; ++k_) acc[k_] = acc[k_ + 1]; \
    acc[P] = 0.0;                                                 \
    ++cbase;                                                      \
  }

template <int P>
__global__ void __launch_bounds__(kStridedThreads) k_fit_strided(FitArgs a, int d) {
  __shared__ int s_g0[kRowChunk];
  __shared__ double s_v[kRowChunk * (P + 1)];
  const int b = blockIdx.y;
  const BlockDev blk = a.blocks[b];
  const AxisProb pr = a.probs[blk.ax[d]];
  const int m = pr.m, n = pr.n;
  std::int64_t L = 1, Tr = 1;
  for (int k = 0; k < a.D; ++k) {
    if (k < d) L *= a.probs[blk.ax[k]].n;
    if (k > d) Tr *= a.probs[blk.ax[k]].m;
  }
  const std::int64_t nlines = L * Tr;
  const std::int64_t line0 = static_cast<std::int64_t>(blockIdx.x) * blockDim.x;
  if (line0 >= nlines) return;
  const std::int64_t line = line0 + threadIdx.x;
  const bool active = line < nlines;
  const std::int64_t l = active ? line / Tr : 0, t = active ? line - (line / Tr) * Tr : 0;
  const double* src;
  std::int64_t sst;
  if (d == 0) {
    std::int64_t off = blk.fbase, r = t;
    for (int k = a.D - 1; k >= 1; --k) {
      const std::int64_t mk = a.probs[blk.ax[k]].m;
      off += (r % mk) * a.fs[k];
      r /= mk;
    }
    src = a.field + off;
    sst = a.fs[0];
  } else {  // d == 1 of D = 3: T1[c0][j1][pitch]
    src = a.t1 + blk.t1off + l * (static_cast<std::int64_t>(m) * a.pitch_last) + t;
    sst = a.pitch_last;
  }
  // Outputs use the common even pitch on their last axis: T1 (D = 3) is
  // [n0][m1][pitch], the last-axis input (pass D-2) is [..][pitch].
  std::int64_t Tro = Tr, tpos = t;
  if (d == a.D - 2) {
    Tro = a.pitch_last;
  } else if (a.D == 3 && d == 0) {
    const std::int64_t m2 = a.probs[blk.ax[2]].m;
    Tro = a.probs[blk.ax[1]].m * a.pitch_last;
    tpos = (t / m2) * a.pitch_last + (t - (t / m2) * m2);
  }
  double* dst = (d == 0 ? a.t1 + blk.t1off : a.t2 + blk.t2off) + (l * n) * Tro + tpos;
  const std::int64_t dstr = Tro;
#ifdef MFB_DEBUG
  if (active) {
    const double* sb = d == 0 ? a.field : a.t1;
    const std::int64_t sn = d == 0 ? a.n_field : a.n_t1;
    MFB_ASSERT(src - sb >= 0 && (src - sb) + static_cast<std::int64_t>(m - 1) * sst < sn, "strided src");
    const double* db = d == 0 ? a.t1 : a.t2;
    const std::int64_t dn = d == 0 ? a.n_t1 : a.n_t2;
    MFB_ASSERT(dst - db >= 0 && (dst - db) + static_cast<std::int64_t>(n - 1) * dstr < dn, "strided dst");
  }
#endif
  const int* g0g = a.g0 + pr.row_off;
  const double* vg = a.vals + pr.row_off * (P + 1);
  const double* lt = a.ltab + pr.col_off * (2 * P + 1);

  double acc[P + 1], yw[P];
#pragma unroll
  for (int k = 0; k <= P; ++k) acc[k] = 0.0;
#pragma unroll
  for (int k = 0; k < P; ++k) yw[k] = 0.0;
  int cbase = g0g[0] < 0 ? g0g[0] : 0;
  double qr[kPrefetch];
#pragma unroll
  for (int u = 0; u < kPrefetch; ++u) qr[u] = (active && u < m) ? src[static_cast<std::int64_t>(u) * sst] : 0.0;

  for (int j0 = 0; j0 < m; j0 += kRowChunk) {
    const int jn = (m - j0) < kRowChunk ? (m - j0) : kRowChunk;
    __syncthreads();
    for (int e = threadIdx.x; e < jn; e += blockDim.x) s_g0[e] = g0g[j0 + e];
    for (int e = threadIdx.x; e < jn * (P + 1); e += blockDim.x) s_v[e] = vg[static_cast<std::int64_t>(j0) * (P + 1) + e];
    __syncthreads();
    for (int jj = 0; jj < jn; jj += kPrefetch) {
#pragma unroll
      for (int u = 0; u < kPrefetch; ++u) {
        if (jj + u < jn) {
          const double q = qr[u];
          const int jg = j0 + jj + u + kPrefetch;
          qr[u] = (active && jg < m) ? src[static_cast<std::int64_t>(jg) * sst] : 0.0;
          const int g = s_g0[jj + u];
          while (cbase < g) MFB_FLUSH_FWD(if (active) dst[static_cast<std::int64_t>(c_) * dstr] = y_)
          const double* vr = s_v + (jj + u) * (P + 1);
#pragma unroll
          for (int k = 0; k <= P; ++k) acc[k] = fma(vr[k], q, acc[k]);
        }
      }
    }
  }
  while (cbase < n) MFB_FLUSH_FWD(if (active) dst[static_cast<std::int64_t>(c_) * dstr] = y_)

  // Back substitution x_c = (y_c - sum_k L(c+k,c) x_{c+k}) / L(c,c), in place.
  double xw[P];
#pragma unroll
  for (int k = 0; k < P; ++k) xw[k] = 0.0;
#pragma unroll 4
  for (int c = n - 1; c >= 0; --c) {
    const double* Lc = lt + static_cast<std::int64_t>(c) * (2 * P + 1);
    double s = active ? dst[static_cast<std::int64_t>(c) * dstr] : 0.0;
#pragma unroll
    for (int k = 1; k <= P; ++k) s = fma(-Lc[P + k], xw[k - 1], s);
    const double x = s * Lc[0];
    if (active) dst[static_cast<std::int64_t>(c) * dstr] = x;
#pragma unroll
    for (int k = P - 1; k >= 1; --k) xw[k] = xw[k - 1];
    xw[0] = x;
  }
}

constexpr int kLastCols = 32;     // columns staged per chunk (last-axis pass)
constexpr int kLastThreads = 128;  // lines per CTA

template <int P>
__global__ void __launch_bounds__(kLastThreads) k_fit_last(FitArgs a) {
  extern __shared__ double smem[];
  constexpr int CW = kLastCols, SP = CW + 1;
  double* s_q = smem;                          // LT x SP
  double* s_v = s_q + kLastThreads * SP;       // CW x (P+1)
  int* s_g0 = reinterpret_cast<int*>(s_v + CW * (P + 1));
  __shared__ unsigned long long s_red[32];
  const int d = a.D - 1;
  const int b = blockIdx.y;
  const BlockDev blk = a.blocks[b];
  const AxisProb pr = a.probs[blk.ax[d]];
  const int m = pr.m, n = pr.n;
  std::int64_t L = 1;
  for (int k = 0; k < d; ++k) L *= a.probs[blk.ax[k]].n;
  const std::int64_t l0 = static_cast<std::int64_t>(blockIdx.x) * kLastThreads;
  if (l0 >= L) return;
  const int nl = static_cast<int>((L - l0) < kLastThreads ? (L - l0) : kLastThreads);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kLastThreads / 32;
  const bool active = tid < nl;
  const std::int64_t lpitch = a.D == 1 ? m : a.pitch_last;
  const double* src = (a.D == 1 ? a.field + blk.fbase : (a.D == 2 ? a.t1 + blk.t1off : a.t2 + blk.t2off)) + l0 * lpitch;
  double* Pb = a.P + blk.poff + l0 * n;
  double* Yb = a.Y + blk.poff + l0 + tid;  // transposed scratch: Y[c*L + l]
#ifdef MFB_DEBUG
  {
    const double* sb = a.D == 1 ? a.field : (a.D == 2 ? a.t1 : a.t2);
    const std::int64_t sn = a.D == 1 ? a.n_field : (a.D == 2 ? a.n_t1 : a.n_t2);
    MFB_ASSERT(src - sb >= 0 && (src - sb) + static_cast<std::int64_t>(nl - 1) * lpitch + m <= sn, "last src");
    MFB_ASSERT(blk.poff + l0 * n + static_cast<std::int64_t>(nl) * n <= a.n_P, "last P");
    MFB_ASSERT(blk.poff + L * n <= a.n_P, "last Y");
  }
#endif
  const int* g0g = a.g0 + pr.row_off;
  const double* vg = a.vals + pr.row_off * (P + 1);
  const double* lt = a.ltab + pr.col_off * (2 * P + 1);

  double acc[P + 1], yw[P];
#pragma unroll
  for (int k = 0; k <= P; ++k) acc[k] = 0.0;
#pragma unroll
  for (int k = 0; k < P; ++k) yw[k] = 0.0;
  int cbase = g0g[0] < 0 ? g0g[0] : 0;
  for (int j0 = 0; j0 < m; j0 += CW) {
    const int jn = (m - j0) < CW ? (m - j0) : CW;
    __syncthreads();
    for (int li = warp; li < nl; li += nwarps)
      s_q[li * SP + lane] = lane < jn ? src[static_cast<std::int64_t>(li) * lpitch + j0 + lane] : 0.0;
    for (int e = tid; e < jn; e += kLastThreads) s_g0[e] = g0g[j0 + e];
    for (int e = tid; e < jn * (P + 1); e += kLastThreads) s_v[e] = vg[static_cast<std::int64_t>(j0) * (P + 1) + e];
    __syncthreads();
    for (int jj = 0; jj < jn; ++jj) {
      const int g = s_g0[jj];
      while (cbase < g) MFB_FLUSH_FWD(if (active) Yb[static_cast<std::int64_t>(c_) * L] = y_)
      const double q = s_q[tid * SP + jj];
      const double* vr = s_v + jj * (P + 1);
#pragma unroll
      for (int k = 0; k <= P; ++k) acc[k] = fma(vr[k], q, acc[k]);
    }
  }
  while (cbase < n) MFB_FLUSH_FWD(if (active) Yb[static_cast<std::int64_t>(c_) * L] = y_)

  // Is this line's lead index shared along any leading dim?
  bool lead_shared = false;
  {
    std::int64_t r = l0 + tid;
    for (int k = d - 1; k >= 0; --k) {
      const AxisProb pk = a.probs[blk.ax[k]];
      const std::int64_t ik = r % pk.n;
      r /= pk.n;
      if (active && a.shared_flag[a.sflag_off[k] + pk.col_lo + ik]) lead_shared = true;
    }
  }
  const unsigned char* sf_last = a.shared_flag + a.sflag_off[d] + pr.col_lo;

  double xw[P];
#pragma unroll
  for (int k = 0; k < P; ++k) xw[k] = 0.0;
  unsigned long long lmax = 0ull;
  for (int chi = n - 1; chi >= 0; chi -= CW) {
    const int clo = chi - CW + 1 > 0 ? chi - CW + 1 : 0;
    const int cn = chi - clo + 1;
#pragma unroll 4
    for (int c = chi; c >= clo; --c) {
      const double* Lc = lt + static_cast<std::int64_t>(c) * (2 * P + 1);
      double s = active ? Yb[static_cast<std::int64_t>(c) * L] : 0.0;
#pragma unroll
      for (int k = 1; k <= P; ++k) s = fma(-Lc[P + k], xw[k - 1], s);
      const double x = s * Lc[0];
#pragma unroll
      for (int k = P - 1; k >= 1; --k) xw[k] = xw[k - 1];
      xw[0] = x;
      s_q[tid * SP + (c - clo)] = x;
      if (active && !lead_shared && !sf_last[c]) lmax = umax(lmax, dbits(fabs(x)));
    }
    __syncthreads();
    for (int li = warp; li < nl; li += nwarps)
      if (lane < cn) Pb[static_cast<std::int64_t>(li) * n + clo + lane] = s_q[li * SP + lane];
    __syncthreads();
  }
  lmax = block_umax(lmax, s_red);
  if (tid == 0 && lmax) atomicMax(a.linf_int + b, lmax);
}

// ------------------------------------------------------------------- K4
// Decompose a flat shared-dof index into per-dim global indices.  Shared
// dofs are enumerated as D disjoint "pieces": piece k = C_0 x .. x C_{k-1} x
// S_k x A_{k+1} x .. (C = non-shared indices, S = shared, A = all).
__device__ __forceinline__ bool piece_index(const EpochArgs& a, std::int64_t g, std::int64_t* idx) {
  int pc = 0;
  while (pc < a.D && g >= a.piece[pc]) {
    g -= a.piece[pc];
    ++pc;
  }
  if (pc >= a.D) return false;
  for (int k = a.D - 1; k >= 0; --k) {
    const std::int64_t ext = k < pc ? a.nC[k] : (k == pc ? a.nS[k] : a.N[k]);
    const std::int64_t r = g % ext;
    g /= ext;
    idx[k] = k < pc ? a.clist[a.c_off[k] + r] : (k == pc ? a.slist[a.s_off[k] + r] : r);
#ifdef MFB_DEBUG
    if (idx[k] < 0 || idx[k] >= a.N[k]) {
      atomicCAS(&g_mfb_debug_line, 0, __LINE__);
      return false;
    }
#endif
  }
  return true;
}

constexpr int kEpochThreads = 256;
constexpr int kEpochSmemBlocks = 1024;  // per-CTA smem reduction slots

// True when two block ids are neighbours in the reference's sense (all
// coordinate distances <= 1, layout.cpp:328-340; holders share the dof, so
// their shared box is non-empty).  Writes the 3^D neighbour code.
__device__ __forceinline__ bool neighbour_code(const EpochArgs& a, int ia, int ib, int* code) {
  int c = 0, mul = 1;
  for (int k = a.D - 1; k >= 0; --k) {
    const int ca = ia % a.B[k], cb = ib % a.B[k];
    ia /= a.B[k];
    ib /= a.B[k];
    const int df = cb - ca;
    if (df < -1 || df > 1) return false;
    c += (df + 1) * mul;
    mul *= 3;
  }
  *code = c;
  return true;
}

// MAXH = 8 when every control has at most 2 holders per axis (all holders are
// then mutual neighbours); MAXH = 27 otherwise (only measurement modes run:
// the reference throws before averaging, solver.cpp:134-141).
template <int MAXH>
__global__ void __launch_bounds__(kEpochThreads) k_epoch(EpochArgs a) {
  __shared__ unsigned long long s_change[kEpochSmemBlocks];
  __shared__ unsigned long long s_linf[kEpochSmemBlocks];
  const bool use_smem = a.nblocks <= kEpochSmemBlocks && a.mode != 3;
  if (use_smem) {
    for (int i = threadIdx.x; i < a.nblocks; i += blockDim.x) {
      s_change[i] = 0ull;
      s_linf[i] = 0ull;
    }
    __syncthreads();
  }
  unsigned long long jss = 0ull, jms = 0ull;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t g = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g < a.total; g += stride) {
    std::int64_t idx[3] = {0, 0, 0};
    if (!piece_index(a, g, idx)) continue;
    int f[3] = {0, 0, 0}, e[3] = {1, 1, 1};
    int ns = 1;
    for (int k = 0; k < a.D; ++k) {
      const int2 r = a.hr[a.hr_off[k] + idx[k]];
      f[k] = r.x;
      e[k] = r.y - r.x + 1;
      ns *= e[k];
      MFB_ASSERT(r.x >= 0 && r.y < a.B[k] && r.y >= r.x, "epoch holder range");
    }
    MFB_ASSERT(ns >= 1 && ns <= MAXH, "epoch ns");
    // holders in ascending block id (layout.cpp:177-195): lexicographic coords
    std::int64_t off[MAXH];
    int ids[MAXH];
    double v[MAXH];
    for (int h = 0; h < ns; ++h) {
      int rr = h, c[3] = {0, 0, 0};
      for (int k = a.D - 1; k >= 0; --k) {
        c[k] = f[k] + rr % e[k];
        rr /= e[k];
      }
      int id = 0;
      std::int64_t o = 0;
      for (int k = 0; k < a.D; ++k) {
        id = id * a.B[k] + c[k];
        const AxisProb& pk = a.probs[a.axbase[k] + c[k]];
        MFB_ASSERT(idx[k] - pk.col_lo >= 0 && idx[k] - pk.col_lo < pk.n, "epoch local index");
        o = o * pk.n + (idx[k] - pk.col_lo);
      }
      MFB_ASSERT(id >= 0 && id < a.nblocks, "epoch id");
      ids[h] = id;
      off[h] = a.poff[id] + o;
      MFB_ASSERT(off[h] >= 0 && off[h] < a.n_P, "epoch off");
      v[h] = a.P[off[h]];
    }
    if (a.mode == 3) {  // final per-pair jumps (solver.cpp:416 -> :166-193)
      for (int h1 = 0; h1 < ns; ++h1)
        for (int h2 = h1 + 1; h2 < ns; ++h2) {
          int code;
          if (!neighbour_code(a, ids[h1], ids[h2], &code)) continue;
          const int slot = a.pair_slot[ids[h1] * 27 + code];
          if (slot >= 0) atomicMax(a.pair_jumps + 2 * slot + (ns > 2 ? 1 : 0), dbits(fabs(v[h1] - v[h2])));
        }
      continue;
    }
    const bool update = MAXH == 8 && ((a.mode == 2) || (a.mode == 1 && ns == 2));
    if (update) {
      // solver.cpp:147-159: ordered sum in ascending holder id, divide once
      double sum = 0.0;
      for (int h = 0; h < ns; ++h) sum = __dadd_rn(sum, v[h]);
      const double avg = __ddiv_rn(sum, static_cast<double>(ns));
      const unsigned long long la = dbits(fabs(avg));
      for (int h = 0; h < ns; ++h) {
        const unsigned long long ch = dbits(fabs(avg - v[h]));
        a.P[off[h]] = avg;
        if (use_smem) {
          atomicMax(s_change + ids[h], ch);
          atomicMax(s_linf + ids[h], la);
        } else {
          atomicMax(a.change + ids[h], ch);
          atomicMax(a.linf_sh + ids[h], la);
        }
      }
      // all copies now bit-identical: post-update jumps are exactly zero
    } else {
      double jd = 0.0;
      if (MAXH == 8) {  // all holders are mutual neighbours: max |Pa-Pb| = max - min
        double mn = v[0], mx = v[0];
        for (int h = 1; h < ns; ++h) {
          mn = fmin(mn, v[h]);
          mx = fmax(mx, v[h]);
        }
        jd = mx - mn;
      } else {
        for (int h1 = 0; h1 < ns; ++h1)
          for (int h2 = h1 + 1; h2 < ns; ++h2) {
            int code;
            if (neighbour_code(a, ids[h1], ids[h2], &code)) jd = fmax(jd, fabs(v[h1] - v[h2]));
          }
      }
      for (int h = 0; h < ns; ++h) {
        const unsigned long long lv = dbits(fabs(v[h]));
        if (use_smem)
          atomicMax(s_linf + ids[h], lv);
        else
          atomicMax(a.linf_sh + ids[h], lv);
      }
      if (ns == 2)
        jss = umax(jss, dbits(jd));
      else
        jms = umax(jms, dbits(jd));
    }
  }
  if (a.mode == 3) return;
  jss = warp_umax(jss);
  jms = warp_umax(jms);
  if ((threadIdx.x & 31) == 0) {
    if (jss) atomicMax(&a.acc->jump_ss, jss);
    if (jms) atomicMax(&a.acc->jump_ms, jms);
  }
  if (use_smem) {
    __syncthreads();
    for (int i = threadIdx.x; i < a.nblocks; i += blockDim.x) {
      if (s_change[i]) atomicMax(a.change + i, s_change[i]);
      if (s_linf[i]) atomicMax(a.linf_sh + i, s_linf[i]);
    }
  }
}

// Common case: every control has <= 2 holders per axis (n_s <= 8).  Holder
// loops are fully unrolled (registers, no local memory) and the per-(dim,
// coordinate) window tables and block offsets live in shared memory.
constexpr int kMaxCoords = 128;

// 32-bit piece decomposition (every extent and piece count < 2^31).
__device__ __forceinline__ bool piece_index32(const EpochArgs& a, unsigned g, int* idx) {
  int pc = 0;
  while (pc < a.D && g >= static_cast<unsigned>(a.piece[pc])) {
    g -= static_cast<unsigned>(a.piece[pc]);
    ++pc;
  }
  if (pc >= a.D) return false;
  for (int k = a.D - 1; k >= 0; --k) {
    const unsigned ext = static_cast<unsigned>(k < pc ? a.nC[k] : (k == pc ? a.nS[k] : a.N[k]));
    const unsigned q = g / ext, r = g - q * ext;
    g = q;
    idx[k] = k < pc ? a.clist[a.c_off[k] + r] : (k == pc ? a.slist[a.s_off[k] + r] : static_cast<int>(r));
  }
  return true;
}

// Max-reduce `val` into slot[key] for the whole warp: one shared atomic per
// warp when all participating lanes share the key (the common case), else
// one per lane.  key < 0 marks a non-participating lane.
__device__ __forceinline__ void warp_atomic_max(unsigned long long* slot, int key, unsigned long long val) {
  const unsigned part = __ballot_sync(kFull, key >= 0);
  if (!part) return;
  const int leader = __ffs(part) - 1;
  const int keyL = __shfl_sync(kFull, key, leader);
  if (__all_sync(kFull, key < 0 || key == keyL)) {
    val = warp_umax(key < 0 ? 0ull : val);
    if ((threadIdx.x & 31) == leader && val) atomicMax(slot + keyL, val);
  } else if (key >= 0 && val) {
    atomicMax(slot + key, val);
  }
}

__global__ void __launch_bounds__(kEpochThreads) k_epoch8(EpochArgs a) {
  __shared__ unsigned long long s_change[kEpochSmemBlocks];
  __shared__ unsigned long long s_linf[kEpochSmemBlocks];
  __shared__ long long s_poff[kEpochSmemBlocks];
  __shared__ int s_lo[3][kMaxCoords], s_n[3][kMaxCoords];
  const int tid = threadIdx.x;
  for (int i = tid; i < a.nblocks; i += blockDim.x) {
    s_change[i] = 0ull;
    s_linf[i] = 0ull;
    s_poff[i] = a.poff[i];
  }
  for (int k = 0; k < a.D; ++k)
    for (int c = tid; c < a.B[k]; c += blockDim.x) {
      const AxisProb pk = a.probs[a.axbase[k] + c];
      s_lo[k][c] = static_cast<int>(pk.col_lo);
      s_n[k][c] = pk.n;
    }
  __syncthreads();
  const bool measure = a.mode == 0, pairs = a.mode == 3;
  unsigned long long jss = 0ull, jms = 0ull;
  const unsigned total = static_cast<unsigned>(a.total);
  const unsigned stride = gridDim.x * blockDim.x;
  // warp-uniform trip count so the warp collectives below see all lanes
  for (unsigned g0 = blockIdx.x * blockDim.x + (tid & ~31u); g0 < total; g0 += stride) {
    const unsigned g = g0 + (tid & 31);
    int idx[3] = {0, 0, 0};
    const bool valid = g < total && piece_index32(a, g, idx);
    int f[3] = {0, 0, 0}, e[3] = {1, 1, 1};
    int ns = valid ? 1 : 0;
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (valid && k < a.D) {
        const int2 r = a.hr[a.hr_off[k] + idx[k]];
        f[k] = r.x;
        e[k] = r.y - r.x + 1;
        ns *= e[k];
      }
    double v[8];
    int ids[8];
    long long off[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      ids[h] = -1;
      off[h] = 0;
      v[h] = 0.0;
      if (h < ns) {
        int c[3] = {0, 0, 0}, rr = h;
#pragma unroll
        for (int k = 2; k >= 0; --k)
          if (k < a.D) {
            c[k] = f[k] + (e[k] == 2 ? (rr & 1) : 0);
            rr = e[k] == 2 ? (rr >> 1) : rr;
          }
        int id = 0;
        long long o = 0;
#pragma unroll
        for (int k = 0; k < 3; ++k)
          if (k < a.D) {
            id = id * a.B[k] + c[k];
            o = o * s_n[k][c[k]] + (idx[k] - s_lo[k][c[k]]);
          }
        ids[h] = id;
        off[h] = s_poff[id] + o;
        v[h] = a.P[off[h]];
      }
    }
    if (pairs) {  // final per-pair jumps (solver.cpp:416 -> :166-193)
#pragma unroll
      for (int h1 = 0; h1 < 8; ++h1)
#pragma unroll
        for (int h2 = h1 + 1; h2 < 8; ++h2)
          if (h2 < ns) {
            int code;
            if (!neighbour_code(a, ids[h1], ids[h2], &code)) continue;
            const int slot = a.pair_slot[ids[h1] * 27 + code];
            if (slot >= 0) atomicMax(a.pair_jumps + 2 * slot + (ns > 2 ? 1 : 0), dbits(fabs(v[h1] - v[h2])));
          }
      continue;
    }
    const bool update = !measure && ns >= 2 && (a.mode == 2 || ns == 2);
    unsigned long long ch[8], lv[8];
    if (update) {
      // solver.cpp:147-159: ordered sum in ascending holder id, divide once
      double sum = 0.0;
#pragma unroll
      for (int h = 0; h < 8; ++h)
        if (h < ns) sum = __dadd_rn(sum, v[h]);
      const double avg = __ddiv_rn(sum, static_cast<double>(ns));
      const unsigned long long la = dbits(fabs(avg));
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        ch[h] = h < ns ? dbits(fabs(avg - v[h])) : 0ull;
        lv[h] = h < ns ? la : 0ull;
        if (h < ns) a.P[off[h]] = avg;
      }
    } else {
      double mn = v[0], mx = v[0];
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        if (h < ns) {
          mn = fmin(mn, v[h]);
          mx = fmax(mx, v[h]);
        }
        ch[h] = 0ull;
        lv[h] = h < ns ? dbits(fabs(v[h])) : 0ull;
      }
      if (ns == 2)
        jss = umax(jss, dbits(mx - mn));
      else if (ns > 2)
        jms = umax(jms, dbits(mx - mn));
    }
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      if (!__any_sync(kFull, h < ns)) break;
      if (!measure) warp_atomic_max(s_change, ids[h], ch[h]);
      warp_atomic_max(s_linf, ids[h], lv[h]);
    }
  }
  if (pairs) return;
  jss = warp_umax(jss);
  jms = warp_umax(jms);
  if ((tid & 31) == 0) {
    if (jss) atomicMax(&a.acc->jump_ss, jss);
    if (jms) atomicMax(&a.acc->jump_ms, jms);
  }
  __syncthreads();
  for (int i = tid; i < a.nblocks; i += blockDim.x) {
    if (s_change[i]) atomicMax(a.change + i, s_change[i]);
    if (s_linf[i]) atomicMax(a.linf_sh + i, s_linf[i]);
  }
}

// ------------------------------------------------------- K4 (region form)
// enforce_constraints (solver.cpp:112-164) + record_epoch jumps (:166-193)
// over one tile of a region.  Every control of the region has the same NS
// holders, so holder ids, offsets and the per-holder reductions are uniform
// across the CTA: one atomic per holder per CTA instead of per control.
constexpr int kRegionThreads = 256;
constexpr int kRegionWarps = kRegionThreads / 32;

__device__ __forceinline__ double warp_dmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

// CTA max of K non-negative doubles with one barrier; thread j < K receives
// value j's CTA max (as a bit pattern, ordered like the value).
template <int K>
__device__ __forceinline__ unsigned long long cta_dmax_multi(double (&v)[K], double (*s_w)[kRegionWarps]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const double r = warp_dmax(v[j]);
    if (lane == 0) s_w[j][w] = r;
  }
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < K)
    for (int i = 0; i < kRegionWarps; ++i) r = fmax(r, s_w[threadIdx.x][i]);
  return dbits(r);
}

// u64 max over the warp in two 32-bit REDUX steps (high words, then the low
// words of the lanes holding the maximal high word).
__device__ __forceinline__ unsigned long long warp_umax64(unsigned long long v) {
  const unsigned hi = static_cast<unsigned>(v >> 32);
  const unsigned mhi = __reduce_max_sync(kFull, hi);
  const unsigned mlo = __reduce_max_sync(kFull, hi == mhi ? static_cast<unsigned>(v) : 0u);
  return (static_cast<unsigned long long>(mhi) << 32) | mlo;
}

// CTA max of K u64 bit patterns (non-negative doubles) with one barrier;
// thread j < K receives value j's CTA max.
template <int K>
__device__ __forceinline__ unsigned long long cta_umax_multi(unsigned long long (&v)[K], double (*s_w)[kRegionWarps]) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned long long(*s_u)[kRegionWarps] = reinterpret_cast<unsigned long long(*)[kRegionWarps]>(s_w);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const unsigned long long r = warp_umax64(v[j]);
    if (lane == 0) s_u[j][w] = r;
  }
  __syncthreads();
  unsigned long long r = 0ull;
  if (threadIdx.x < K)
#pragma unroll
    for (int i = 0; i < kRegionWarps; ++i) r = umax(r, s_u[threadIdx.x][i]);
  return r;
}

struct RegionRegs {
  long long base;
  int s0, s1, s2;
};

// q = n / d, r = n % d for 0 <= n < 2^24, 1 <= d: fp32 reciprocal estimate
// (off by at most one) plus one correction step, instead of the ~20-instruction
// integer division by a run-time divisor.
__device__ __forceinline__ void fast_divmod(int n, int d, float rcp, int& q, int& r) {
  q = __float2int_rz(__int2float_rz(n) * rcp);
  r = n - q * d;
  if (r < 0) {
    --q;
    r += d;
  } else if (r >= d) {
    ++q;
    r -= d;
  }
}

// fast_divmod without branches (the correction as selects).
__device__ __forceinline__ void divmod_nb(int n, int d, float rcp, int& q, int& r) {
  q = __float2int_rz(__int2float_rz(n) * rcp);
  r = n - q * d;
  const int lo = r < 0 ? 1 : 0, hi = r >= d ? 1 : 0;
  q += hi - lo;
  r += (lo - hi) * d;
}

// region_tile for a tile whose holders are all local (rmask == 0): 32-bit
// element offsets (the engine keeps the held lattices below 2^31 doubles),
// the last box dim contiguous in every copy (stride 1), branch-free index
// arithmetic, and for FLAT boxes (ext[0] == 1: every 1-D/2-D region) a single
// division.  Elements past the tile are loaded at a clamped index and not
// used.  Same arithmetic and reduction as region_tile.
template <int NS, bool FLAT, bool SNAP>
__device__ __forceinline__ void region_tile_local(const EpochRegionArgs& a, const RegionDev& R, const TileDev& t,
                                                  int mode, int se, double (*s_w)[kRegionWarps]) {
  constexpr int PT = NS == 2 ? 4 : (NS == 4 ? 2 : 1);
  // mode 4 = epoch 0 fused with iteration 1: as mode 1, plus the pre-average
  // SS jump of the n_s == 2 controls (epoch 0's measurement)
  const bool update = mode == 2 || ((mode == 1 || mode == 4) && NS == 2);
  const bool pre = mode == 4 && NS == 2;
  int base[NS], s0[NS], s1[NS];
#pragma unroll
  for (int h = 0; h < NS; ++h) {
    base[h] = static_cast<int>(R.base[h]);
    s0[h] = R.str[h][0];
    s1[h] = R.str[h][1];
  }
  const int e1 = R.ext[1], e2 = R.ext[2];
  const float rc1 = 1.0f / static_cast<float>(e1), rc2 = 1.0f / static_cast<float>(e2);
  double* __restrict__ P = a.P;
  // log_errors snapshots (residual_tma.cu): epoch se's value of every copy,
  // and in mode 4 also epoch 0's (the pre-average value)
  double* __restrict__ snap = (SNAP && se >= 0) ? a.snap + static_cast<long long>(se) * a.snap_stride : nullptr;
  double* __restrict__ snap0 = (SNAP && se >= 0 && mode == 4) ? a.snap : nullptr;
  unsigned long long red[NS + 2];  // [NS + 1]: mode 4's pre-average jump
#pragma unroll
  for (int j = 0; j <= NS + 1; ++j) red[j] = 0ull;
  const int end = t.start + t.count;
  for (int i0 = t.start + threadIdx.x; i0 < end; i0 += kRegionThreads * PT) {
    int off[PT][NS];
    double v[PT][NS];
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int i = min(i0 + u * kRegionThreads, end - 1);
      int q, r2, r0 = 0, r1;
      divmod_nb(i, e2, rc2, q, r2);
      if (FLAT)
        r1 = q;
      else
        divmod_nb(q, e1, rc1, r0, r1);
#pragma unroll
      for (int h = 0; h < NS; ++h) {
        off[u][h] = base[h] + r0 * s0[h] + r1 * s1[h] + r2;
        v[u][h] = P[off[u][h]];
      }
    }
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      if (i0 + u * kRegionThreads < end) {
        if (update) {
          if (pre) {
            double mn = v[u][0], mx = v[u][0];
#pragma unroll
            for (int h = 1; h < NS; ++h) {
              mn = fmin(mn, v[u][h]);
              mx = fmax(mx, v[u][h]);
            }
            red[NS + 1] = umax(red[NS + 1], dbits(mx - mn));
          }
          double sum = 0.0;  // solver.cpp:147-159: ascending holder id, divide once
#pragma unroll
          for (int h = 0; h < NS; ++h) sum = __dadd_rn(sum, v[u][h]);
          const double avg = sum * (1.0 / NS);  // NS is a power of two: bitwise equal to sum / NS
#pragma unroll
          for (int h = 0; h < NS; ++h) {
            red[h] = umax(red[h], dbits(fabs(avg - v[u][h])));
            P[off[u][h]] = avg;
            if (SNAP && snap) snap[off[u][h]] = avg;
            if (SNAP && snap0) snap0[off[u][h]] = v[u][h];
          }
          red[NS] = umax(red[NS], dbits(fabs(avg)));
        } else {
          double mn = v[u][0], mx = v[u][0];
#pragma unroll
          for (int h = 0; h < NS; ++h) {
            mn = fmin(mn, v[u][h]);
            mx = fmax(mx, v[u][h]);
            red[h] = umax(red[h], dbits(fabs(v[u][h])));
            if (SNAP && snap) snap[off[u][h]] = v[u][h];
            if (SNAP && snap0) snap0[off[u][h]] = v[u][h];
          }
          red[NS] = umax(red[NS], dbits(mx - mn));
        }
      }
    }
  }
  const unsigned long long b = cta_umax_multi<NS + 2>(red, s_w);
  const int j = threadIdx.x;
  if (b && j < NS) {
    atomicMax((update ? a.change : a.linf_sh) + R.ids[j], b);
  } else if (b && j == NS) {
    if (update) {
#pragma unroll
      for (int h = 0; h < NS; ++h) atomicMax(a.linf_sh + R.ids[h], b);
    } else {
      atomicMax(NS == 2 ? &a.st->jump_ss : &a.st->jump_ms, b);
    }
  } else if (b && j == NS + 1) {
    atomicMax(&a.st->jump0_ss, b);
  }
  __syncthreads();  // s_w and the tile descriptor are reused by the next tile
}

// R is the CTA's shared-memory copy of the region descriptor.  PT controls
// per thread per pass (PT loads per holder in flight); the n_s = 8 form keeps
// offsets in shared memory to stay within the register budget.
template <int NS>
__device__ __forceinline__ void region_tile(const EpochRegionArgs& a, const RegionDev& R, const TileDev& t, int mode,
                                            double (*s_w)[kRegionWarps]) {
  constexpr int PT = NS == 2 ? 4 : (NS == 4 ? 2 : 1);  // controls per thread per pass: 8 loads in flight
  const bool update = mode == 2 || (mode == 1 && NS == 2);  // (mode 4 runs on local tiles only)
  RegionRegs hr[NS <= 4 ? NS : 1];
#pragma unroll
  for (int h = 0; h < (NS <= 4 ? NS : 1); ++h) hr[h] = RegionRegs{R.base[h], R.str[h][0], R.str[h][1], R.str[h][2]};
  auto offset = [&](int h, int r0, int r1, int r2) -> long long {
    if (NS <= 4) return hr[h].base + static_cast<long long>(r0) * hr[h].s0 + r1 * hr[h].s1 + r2 * hr[h].s2;
    return R.base[h] + static_cast<long long>(r0) * R.str[h][0] + r1 * R.str[h][1] + r2 * R.str[h][2];
  };
  const int e1 = R.ext[1], e2 = R.ext[2];
  const int rmask = R.rmask;  // remote holders: read from the receive buffer, never written
  const float rc1 = 1.0f / static_cast<float>(e1), rc2 = 1.0f / static_cast<float>(e2);
  // update: red[h] = change of holder h, red[NS] = max |avg| (every copy);
  // measure: red[h] = max |copy of holder h|, red[NS] = jump
  unsigned long long red[NS + 1];  // bit patterns of non-negative doubles (ordered like the values)
#pragma unroll
  for (int j = 0; j <= NS; ++j) red[j] = 0ull;
  const int end = t.start + t.count;
  for (int i0 = t.start + threadIdx.x; i0 < end; i0 += kRegionThreads * PT) {
    long long off[PT][NS];
    double v[PT][NS];
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      const int i = i0 + u * kRegionThreads;
      int q, r2, r0, r1;
      fast_divmod(i, e2, rc2, q, r2);
      fast_divmod(q, e1, rc1, r0, r1);
#pragma unroll
      for (int h = 0; h < NS; ++h) {
        off[u][h] = offset(h, r0, r1, r2);
        v[u][h] = i < end ? ((rmask >> h) & 1 ? a.recv[off[u][h]] : a.P[off[u][h]]) : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < PT; ++u) {
      if (i0 + u * kRegionThreads >= end) break;
      if (update) {
        double sum = 0.0;  // solver.cpp:147-159: ascending holder id, divide once
#pragma unroll
        for (int h = 0; h < NS; ++h) sum = __dadd_rn(sum, v[u][h]);
        const double avg = sum * (1.0 / NS);  // NS is a power of two: bitwise equal to sum / NS
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          red[h] = umax(red[h], dbits(fabs(avg - v[u][h])));
          if (!((rmask >> h) & 1)) a.P[off[u][h]] = avg;
        }
        red[NS] = umax(red[NS], dbits(fabs(avg)));  // every holder's copy is now avg
      } else {
        double mn = v[u][0], mx = v[u][0];
#pragma unroll
        for (int h = 0; h < NS; ++h) {
          mn = fmin(mn, v[u][h]);
          mx = fmax(mx, v[u][h]);
          red[h] = umax(red[h], dbits(fabs(v[u][h])));
        }
        red[NS] = umax(red[NS], dbits(mx - mn));  // all holders are mutual neighbours
      }
    }
  }
  const unsigned long long b = cta_umax_multi<NS + 1>(red, s_w);
  const int j = threadIdx.x;
  if (b && j < NS) {
    if (!((rmask >> j) & 1)) atomicMax((update ? a.change : a.linf_sh) + R.ids[j], b);
  } else if (b && j == NS) {
    if (update) {
#pragma unroll
      for (int h = 0; h < NS; ++h)
        if (!((rmask >> h) & 1)) atomicMax(a.linf_sh + R.ids[h], b);
    } else {
      atomicMax(NS == 2 ? &a.st->jump_ss : &a.st->jump_ms, b);
    }
  }
  __syncthreads();  // s_w and the tile descriptor are reused by the next tile
}

template <int NS, bool SNAP>
__device__ __forceinline__ void region_tile_any(const EpochRegionArgs& a, const TileDev& t, int mode, int se,
                                                double (*s_w)[kRegionWarps]) {
  if (t.r.rmask != 0)
    region_tile<NS>(a, t.r, t, mode, s_w);  // (sharded solves keep no snapshots)
  else if (t.r.ext[0] == 1)
    region_tile_local<NS, true, SNAP>(a, t.r, t, mode, se, s_w);
  else
    region_tile_local<NS, false, SNAP>(a, t.r, t, mode, se, s_w);
}

// dp = max_b change_b / max(1, ||P_b||_inf) (solver.cpp:398-405) into
// epoch_out[3*slot], jumps, accumulator reset; loop bookkeeping in loop mode.
__device__ void epoch_finalize(const EpochRegionArgs& a, int mode, int slot, unsigned long long* s_red) {
  unsigned long long dp = 0ull;
  for (int b = threadIdx.x; b < a.nblocks; b += blockDim.x) {
    const unsigned long long li = umax(a.linf_int[b], __ldcg(a.linf_sh + b));
    const double lin = __longlong_as_double(static_cast<long long>(li));
    const double chv = __longlong_as_double(static_cast<long long>(__ldcg(a.change + b)));
    dp = umax(dp, dbits(chv / (lin > 1.0 ? lin : 1.0)));
    a.change[b] = 0ull;
    a.linf_sh[b] = 0ull;
  }
  for (int q = threadIdx.x; q < a.zero_pairs; q += blockDim.x) a.pair_jumps[q] = 0ull;
  dp = block_umax(dp, s_red);
  if (threadIdx.x == 0) {
    const double dpv = mode == 0 ? 0.0 : __longlong_as_double(static_cast<long long>(dp));  // record_epoch(0, 0.0)
    const unsigned long long js = atomicExch(&a.st->jump_ss, 0ull), jm = atomicExch(&a.st->jump_ms, 0ull);
    if (mode == 4) {  // epoch 0: jumps of the fit (the n_s > 2 ones are untouched by iteration 1)
      const unsigned long long j0 = atomicExch(&a.st->jump0_ss, 0ull);
      double* o0 = a.epoch_out;
      o0[0] = 0.0;
      o0[1] = __longlong_as_double(static_cast<long long>(j0));
      o0[2] = __longlong_as_double(static_cast<long long>(jm));
    }
    double* out = a.epoch_out + 3 * slot;
    out[0] = dpv;
    out[1] = __longlong_as_double(static_cast<long long>(js));
    out[2] = __longlong_as_double(static_cast<long long>(jm));
    a.st->done = 0;
    if (a.mode < 0 || a.mode == 4) {  // loop bookkeeping (solver.cpp:406-412)
      const bool conv = dpv < a.tol;
      a.st->last_iter = slot;
      a.st->converged = conv ? 1 : 0;
      a.st->iter = slot;
      cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(a.cond),
                              (!conv && slot < a.max_iter) ? 1u : 0u);
    }
  }
}

// MAXNS = 4 for 1-D/2-D decompositions (tighter register budget, 3 CTAs/SM),
// 8 for 3-D.
// SNAP: the log_errors form that also writes the epoch snapshots of the
// shared copies (residual_tma.cu); the plain form is the solve's hot epoch.
#ifndef MFB_EPOCH8_CTAS
#define MFB_EPOCH8_CTAS 3  // resident CTAs per SM of the n_s = 8 (3-D) form (3: C4 epochs 347 -> 327 us, C3 82 -> 80 us)
#endif
template <int MAXNS, bool SNAP>
__global__ void __launch_bounds__(kRegionThreads, MAXNS == 8 ? MFB_EPOCH8_CTAS : 3) k_epoch_regions(EpochRegionArgs a) {
  __shared__ double s_w[2 * kRegionMaxHolders + 1][kRegionWarps];
  __shared__ unsigned long long s_red[32];
  __shared__ int s_last;
  __shared__ TileDev s_T;
  pdl_enter();
  constexpr int kWords = static_cast<int>(sizeof(TileDev) / 4);
  static_assert(kWords <= kRegionThreads, "one descriptor word per thread");
  const int iter = a.mode < 0 ? a.st->iter + 1 : (a.mode == 4 ? 1 : 0);
  const int mode = a.mode < 0 ? (iter >= 2 ? 2 : 1) : a.mode;  // solver.cpp:397
  // an unrolled loop iteration ahead of the WHILE node: nothing to do once the
  // previous epoch converged or the iteration budget is spent (its finalize
  // then already cleared the WHILE condition)
  if (a.predicated && (a.st->converged || iter > a.max_iter)) return;
  // log_errors snapshot slot of this epoch (explicit-mode launches of the
  // host-driven loop name their epoch in a.slot)
  const int se = (a.snap && mode != 3) ? ((a.mode < 0 || a.mode == 4) ? iter : a.slot) : -1;
  // persistent CTAs: the next tile's descriptor is fetched while this one runs
  const int tid = threadIdx.x;
  int w = 0;
  if (tid < kWords && static_cast<int>(blockIdx.x) < a.ntiles)
    w = __ldg(reinterpret_cast<const int*>(a.tiles + blockIdx.x) + tid);
  for (int tb = blockIdx.x; tb < a.ntiles; tb += gridDim.x) {
    if (tid < kWords) reinterpret_cast<int*>(&s_T)[tid] = w;
    __syncthreads();
    const int tn = tb + gridDim.x;
    if (tid < kWords && tn < a.ntiles) w = __ldg(reinterpret_cast<const int*>(a.tiles + tn) + tid);
    const TileDev& t = s_T;
    switch (t.r.ns) {
      case 2: region_tile_any<2, SNAP>(a, t, mode, se, s_w); break;
      case 4: region_tile_any<4, SNAP>(a, t, mode, se, s_w); break;
      default: region_tile_any<MAXNS, SNAP>(a, t, mode, se, s_w); break;
    }
  }
  if (!a.finalize) return;
  // last CTA: dp = max_b change_b / max(1, ||P_b||_inf) (solver.cpp:398-405)
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(&a.st->done, 1) == static_cast<int>(gridDim.x) - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  epoch_finalize(a, mode, iter, s_red);
}

// One-CTA epoch bookkeeping after separately launched region kernels (the
// sharded path, where dp is then max-reduced across ranks).
__global__ void __launch_bounds__(kRegionThreads) k_epoch_finalize(EpochRegionArgs a) {
  __shared__ unsigned long long s_red[32];
  if (a.predicated && a.st->converged) return;  // a speculated epoch after convergence
  epoch_finalize(a, a.mode, a.slot, s_red);
}

// Sharded solve: the loop bookkeeping of epoch `slot` (solver.cpp:406-412) on
// the device, after dp has been max-reduced over the ranks, so that the host
// can enqueue several iterations (predicated on st->converged) per sync.
__global__ void k_shard_advance(EpochState* st, const double* epoch_out, int slot, double tol) {
  if (st->converged) return;
  st->iter = slot;
  st->last_iter = slot;
  if (slot >= 1 && epoch_out[3 * slot] < tol) st->converged = 1;
}

// Final per-pair jumps (solver.cpp:416 -> :166-193): L-inf of |P_a - P_b| per
// holder pair of each region, split SS/MS by the region's n_s.  Only needed
// when the last epoch did not average every shared control.
template <int NS>
__device__ __forceinline__ void region_pairs(const EpochRegionArgs& a, const RegionDev& R, const TileDev& t,
                                             double (*s_w)[kRegionWarps]) {
  constexpr int NP = NS * (NS - 1) / 2;
  double pj[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) pj[q] = 0.0;
  const int e1 = R.ext[1], e2 = R.ext[2];
  for (int i = t.start + threadIdx.x; i < t.start + t.count; i += kRegionThreads) {
    const int r2 = i % e2, q = i / e2;
    const int r1 = q % e1, r0 = q / e1;
    double v[NS];
#pragma unroll
    for (int h = 0; h < NS; ++h) {
      const long long o = R.base[h] + static_cast<long long>(r0) * R.str[h][0] + r1 * R.str[h][1] + r2 * R.str[h][2];
      v[h] = (R.rmask >> h) & 1 ? a.recv[o] : a.P[o];  // remote holder: its copy from the exchange
    }
    int q2 = 0;
#pragma unroll
    for (int h1 = 0; h1 < NS; ++h1)
#pragma unroll
      for (int h2 = h1 + 1; h2 < NS; ++h2, ++q2) pj[q2] = fmax(pj[q2], fabs(v[h1] - v[h2]));
  }
  // NP <= 28 > 2*kRegionMaxHolders+1 slots: reduce in chunks of 16
#pragma unroll
  for (int c0 = 0; c0 < NP; c0 += 16) {
    double part[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) part[j] = c0 + j < NP ? pj[c0 + j] : 0.0;
    const unsigned long long b = cta_dmax_multi<16>(part, s_w);
    const int q = c0 + static_cast<int>(threadIdx.x);
    if (threadIdx.x < 16 && q < NP && R.pslot[q] >= 0 && b)
      atomicMax(a.pair_jumps + 2 * R.pslot[q] + (NS > 2 ? 1 : 0), b);
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kRegionThreads) k_pair_jumps_regions(EpochRegionArgs a) {
  pdl_enter();
  __shared__ double s_w[2 * kRegionMaxHolders + 1][kRegionWarps];
  if (a.st->last_iter >= 2) return;  // after a mode-2 epoch all copies agree bitwise
  for (int tb = blockIdx.x; tb < a.ntiles; tb += gridDim.x) {
    const TileDev& t = a.tiles[tb];
    switch (t.r.ns) {
      case 2: region_pairs<2>(a, t.r, t, s_w); break;
      case 4: region_pairs<4>(a, t.r, t, s_w); break;
      default: region_pairs<8>(a, t.r, t, s_w); break;
    }
  }
}

// ------------------------------------------------------------------- K9
// residual_error (lsq.cpp:66-85) per local block: decode the block's held
// lattice P_b with its own (window-clipped) collocation rows at every point of
// its input box.  One thread per trailing point (j1[, j2]) sweeps axis 0 with a
// window of P+1 trailing-contracted control planes (D = 1: thread per row).
// Out-of-window basis values are zero in the row tables; their column indices
// are clamped so every lattice read stays inside P_b.
constexpr int kResThreads = 128;

template <int P>
__global__ void __launch_bounds__(kResThreads) k_block_residual(BlockResArgs a) {
  __shared__ double s_red[2][kResThreads / 32];
  if (a.expect_iter >= 0 && a.st->iter != a.expect_iter) return;  // its epoch did not run
  const int b = blockIdx.y;
  const BlockDev& blk = a.blocks[b];
  const int D = a.D;
  const AxisProb p0 = a.probs[blk.ax[0]];
  const int m0 = p0.m, n0 = p0.n;
  const int* g00 = a.g0 + p0.row_off;
  const double* v00 = a.vals + p0.row_off * (P + 1);
  const double* Pb = a.P + blk.poff;
  double l2 = 0.0, li = 0.0;
  auto clampi = [](int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); };
  if (D == 1) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < m0; j += gridDim.x * blockDim.x) {
      const int g = __ldg(g00 + j);
      double s = 0.0;
#pragma unroll
      for (int k = 0; k <= P; ++k) s = fma(__ldg(v00 + j * (P + 1) + k), Pb[clampi(g + k, n0)], s);
      const double e = a.field[blk.fbase + j * a.fs[0]] - s;
      l2 = fma(e, e, l2);
      li = fmax(li, fabs(e));
    }
  } else {
    const AxisProb p1 = a.probs[blk.ax[1]];
    const AxisProb p2 = D == 3 ? a.probs[blk.ax[2]] : p1;
    const int m1 = p1.m, n1 = p1.n, m2 = D == 3 ? p2.m : 1, n2 = D == 3 ? p2.n : 1;
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < m1 * m2) {
      const int j1 = D == 3 ? t / m2 : t, j2 = D == 3 ? t - (t / m2) * m2 : 0;
      double w1[P + 1], w2[P + 1];
      const int g1 = __ldg(a.g0 + p1.row_off + j1);
      const int g2 = D == 3 ? __ldg(a.g0 + p2.row_off + j2) : 0;
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        w1[k] = __ldg(a.vals + (p1.row_off + j1) * (P + 1) + k);
        w2[k] = D == 3 ? __ldg(a.vals + (p2.row_off + j2) * (P + 1) + k) : 0.0;
      }
      const std::int64_t plane_sz = static_cast<std::int64_t>(n1) * n2;
      auto plane = [&](int ai) -> double {  // trailing contraction of held plane ai
        const double* L0 = Pb + static_cast<std::int64_t>(clampi(ai, n0)) * plane_sz;
        double s = 0.0;
#pragma unroll
        for (int k1 = 0; k1 <= P; ++k1) {
          const std::int64_t r1 = static_cast<std::int64_t>(clampi(g1 + k1, n1)) * n2;
          if (D == 2) {
            s = fma(w1[k1], L0[r1], s);
          } else {
            double r = 0.0;
#pragma unroll
            for (int k2 = 0; k2 <= P; ++k2) r = fma(w2[k2], L0[r1 + clampi(g2 + k2, n2)], r);
            s = fma(w1[k1], r, s);
          }
        }
        return s;
      };
      int abase = __ldg(g00);
      double Tw[P + 1];
#pragma unroll
      for (int k = 0; k <= P; ++k) Tw[k] = plane(abase + k);
      const double* q = a.field + blk.fbase + j1 * a.fs[1] + (D == 3 ? j2 * a.fs[2] : 0);
      for (int j = 0; j < m0; ++j) {
        const int g = __ldg(g00 + j);
        while (abase < g) {
#pragma unroll
          for (int k = 0; k < P; ++k) Tw[k] = Tw[k + 1];
          ++abase;
          Tw[P] = plane(abase + P);
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k <= P; ++k) s = fma(__ldg(v00 + j * (P + 1) + k), Tw[k], s);
        const double e = q[static_cast<std::int64_t>(j) * a.fs[0]] - s;
        l2 = fma(e, e, l2);
        li = fmax(li, fabs(e));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l2 += __shfl_xor_sync(kFull, l2, o);
    li = fmax(li, __shfl_xor_sync(kFull, li, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_red[0][w] = l2;
    s_red[1][w] = li;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sl = 0.0, sm = 0.0;
    for (int i = 0; i < kResThreads / 32; ++i) {
      sl += s_red[0][i];
      sm = fmax(sm, s_red[1][i]);
    }
    a.partial[2 * (static_cast<std::int64_t>(b) * a.ntile + blockIdx.x)] = sl;
    a.partial[2 * (static_cast<std::int64_t>(b) * a.ntile + blockIdx.x) + 1] = sm;
  }
}

// D = 2, 3 form of K9 with the block's axis-0 row table staged in shared
// memory (broadcast reads: no global load on the per-row chain), the next
// control plane's lattice values fetched one advance ahead (the decode's
// scheme, k_decode_tma) and the field rows RB at a time ahead of use.  Same
// arithmetic, in the same order, as k_block_residual.
template <int P, int D>
__global__ void __launch_bounds__(kResThreads) k_block_residual_staged(BlockResArgs a) {
  extern __shared__ __align__(16) double s_rows[];  // m0 x (P+1) basis values, then m0 first columns
  __shared__ double s_red[2][kResThreads / 32];
  if (a.expect_iter >= 0 && a.st->iter != a.expect_iter) return;  // its epoch did not run
  const int b = blockIdx.y;
  const BlockDev& blk = a.blocks[b];
  const AxisProb p0 = a.probs[blk.ax[0]], p1 = a.probs[blk.ax[1]];
  const AxisProb p2 = D == 3 ? a.probs[blk.ax[2]] : p1;
  const int m0 = p0.m, n0 = p0.n, m1 = p1.m, n1 = p1.n;
  const int m2 = D == 3 ? p2.m : 1, n2 = D == 3 ? p2.n : 1;
  double* sv = s_rows;
  int* sg = reinterpret_cast<int*>(s_rows + m0 * (P + 1));
  {
    const double* v00 = a.vals + p0.row_off * (P + 1);
    const int* g00 = a.g0 + p0.row_off;
    for (int e = threadIdx.x; e < m0 * (P + 1); e += kResThreads) sv[e] = __ldg(v00 + e);
    for (int e = threadIdx.x; e < m0; e += kResThreads) sg[e] = __ldg(g00 + e);
  }
  __syncthreads();
  const double* Pb = a.P + blk.poff;
  double l2 = 0.0, li = 0.0;
  auto clampi = [](int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); };
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < m1 * m2) {
    const int j1 = D == 3 ? t / m2 : t, j2 = D == 3 ? t - (t / m2) * m2 : 0;
    double w1[P + 1], w2[P + 1];
    int r1[P + 1], c2[P + 1];  // clamped lattice row / column offsets of this point's window
    const int g1 = __ldg(a.g0 + p1.row_off + j1);
    const int g2 = D == 3 ? __ldg(a.g0 + p2.row_off + j2) : 0;
#pragma unroll
    for (int k = 0; k <= P; ++k) {
      w1[k] = __ldg(a.vals + (p1.row_off + j1) * (P + 1) + k);
      w2[k] = D == 3 ? __ldg(a.vals + (p2.row_off + j2) * (P + 1) + k) : 0.0;
      r1[k] = clampi(g1 + k, n1) * n2;
      c2[k] = D == 3 ? clampi(g2 + k, n2) : 0;
    }
    const std::int64_t plane_sz = static_cast<std::int64_t>(n1) * n2;
    constexpr int NV = D == 2 ? (P + 1) : (P + 1) * (P + 1);
    double nxt[NV];  // raw lattice values of the plane after the window
    auto fetch = [&](int ai) {
      const double* L0 = Pb + static_cast<std::int64_t>(clampi(ai, n0)) * plane_sz;
#pragma unroll
      for (int k1 = 0; k1 <= P; ++k1) {
        if (D == 2) {
          nxt[k1] = L0[r1[k1]];
        } else {
#pragma unroll
          for (int k2 = 0; k2 <= P; ++k2) nxt[(k1 * (P + 1) + k2) % NV] = L0[r1[k1] + c2[k2]];
        }
      }
    };
    auto reduce = [&]() -> double {  // plane() of k_block_residual on the fetched values
      double s = 0.0;
#pragma unroll
      for (int k1 = 0; k1 <= P; ++k1) {
        if (D == 2) {
          s = fma(w1[k1], nxt[k1], s);
        } else {
          double r = 0.0;
#pragma unroll
          for (int k2 = 0; k2 <= P; ++k2) r = fma(w2[k2], nxt[(k1 * (P + 1) + k2) % NV], r);
          s = fma(w1[k1], r, s);
        }
      }
      return s;
    };
    int abase = sg[0];
    double Tw[P + 1];
#pragma unroll
    for (int k = 0; k <= P; ++k) {
      fetch(abase + k);
      Tw[k] = reduce();
    }
    // D = 2: the next plane's P+1 values ride along in registers; D = 3 would
    // hold (P+1)^2 of them across the row loop, so it fetches at the advance
    constexpr bool AHEAD = D == 2;
    if (AHEAD) fetch(abase + P + 1);
    const double* q = a.field + blk.fbase + j1 * a.fs[1] + (D == 3 ? j2 * a.fs[2] : 0);
    const std::int64_t fs0 = a.fs[0];
    constexpr int RB = 4;
    double qn[RB];
#pragma unroll
    for (int u = 0; u < RB; ++u) qn[u] = u < m0 ? __ldcs(q + u * fs0) : 0.0;
    for (int j0 = 0; j0 < m0; j0 += RB) {
      double qc[RB];
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        qc[u] = qn[u];
        const int jn = j0 + RB + u;
        qn[u] = jn < m0 ? __ldcs(q + jn * fs0) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < RB; ++u) {
        const int j = j0 + u;
        if (j < m0) {
          const int g = sg[j];
          while (abase < g) {
#pragma unroll
            for (int k = 0; k < P; ++k) Tw[k] = Tw[k + 1];
            ++abase;
            if (!AHEAD) fetch(abase + P);
            Tw[P] = reduce();  // plane abase + P
            if (AHEAD) fetch(abase + P + 1);
          }
          const double* vr = sv + j * (P + 1);
          double s = 0.0;
#pragma unroll
          for (int k = 0; k <= P; ++k) s = fma(vr[k], Tw[k], s);
          const double e = qc[u] - s;
          l2 = fma(e, e, l2);
          li = fmax(li, fabs(e));
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l2 += __shfl_xor_sync(kFull, l2, o);
    li = fmax(li, __shfl_xor_sync(kFull, li, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_red[0][w] = l2;
    s_red[1][w] = li;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sl = 0.0, sm = 0.0;
    for (int i = 0; i < kResThreads / 32; ++i) {
      sl += s_red[0][i];
      sm = fmax(sm, s_red[1][i]);
    }
    a.partial[2 * (static_cast<std::int64_t>(b) * a.ntile + blockIdx.x)] = sl;
    a.partial[2 * (static_cast<std::int64_t>(b) * a.ntile + blockIdx.x) + 1] = sm;
  }
}

// Fixed-order reduction of the per-tile partials: errs[slot][b] = {sqrt(sum), max}.
__global__ void k_block_residual_reduce(BlockResArgs a) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblocks) return;
  if (a.expect_iter >= 0 && a.st->iter != a.expect_iter) return;
  const int slot = a.st ? a.st->iter : a.slot;
  double sl = 0.0, sm = 0.0;
  for (int t = 0; t < a.ntile; ++t) {
    sl += a.partial[2 * (static_cast<std::int64_t>(b) * a.ntile + t)];
    sm = fmax(sm, a.partial[2 * (static_cast<std::int64_t>(b) * a.ntile + t) + 1]);
  }
  const std::int64_t o = 2 * (static_cast<std::int64_t>(slot) * a.nglobal + a.boff + b);
  a.errs[o] = sqrt(sl);
  a.errs[o + 1] = sm;
}

template <int P>
struct BlockResLaunch {
  static int run(const BlockResArgs& a, cudaStream_t s) {
    dim3 grid(a.ntile, a.nblocks);
    const size_t smem = static_cast<size_t>(a.max_m0) * ((P + 1) * 8 + 4) + 16;
    static const bool plain = std::getenv("MFADD_RES_PLAIN") != nullptr;  // A/B: the unstaged kernel
    // D = 3 stays on the unstaged kernel (the staged form holds about 30% more
    // registers there; not measured faster)
    if (a.D == 2 && !plain && smem <= 160 * 1024) {
      cudaFuncSetAttribute(k_block_residual_staged<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      k_block_residual_staged<P, 2><<<grid, kResThreads, smem, s>>>(a);
    } else {
      k_block_residual<P><<<grid, kResThreads, 0, s>>>(a);
    }
    k_block_residual_reduce<<<(a.nblocks + 127) / 128, 128, 0, s>>>(a);
    return 2;
  }
};

// ------------------------------------------------------------------- K5
__global__ void __launch_bounds__(1024) k_dp(DpArgs a) {
  __shared__ unsigned long long red[32];
  unsigned long long dp = 0ull;
  for (int b = threadIdx.x; b < a.nblocks; b += blockDim.x) {
    const unsigned long long li = umax(a.linf_int[b], a.linf_sh[b]);
    const double lin = __longlong_as_double(static_cast<long long>(li));
    const double ch = __longlong_as_double(static_cast<long long>(a.change[b]));
    const double r = ch / (lin > 1.0 ? lin : 1.0);  // solver.cpp:404-405
    dp = umax(dp, dbits(r));
    a.change[b] = 0ull;
    a.linf_sh[b] = 0ull;
  }
  dp = block_umax(dp, red);
  if (threadIdx.x == 0) {
    const double dpv = __longlong_as_double(static_cast<long long>(dp));
    const double js = __longlong_as_double(static_cast<long long>(a.acc->jump_ss));
    const double jm = __longlong_as_double(static_cast<long long>(a.acc->jump_ms));
    a.epoch_out[0] = dpv;
    a.epoch_out[1] = js;
    a.epoch_out[2] = jm;
    if (a.host_mirror) {
      a.host_mirror[0] = dpv;
      a.host_mirror[1] = js;
      a.host_mirror[2] = jm;
    }
    a.acc->jump_ss = 0ull;
    a.acc->jump_ms = 0ull;
  }
}

// ------------------------------------------------------------------- K6
// One CTA per lattice row (all dims but the last): the lead-dim owner
// coordinates and local indices are CTA-uniform; the last dim's owner table and
// per-owner window origins sit in shared memory.
constexpr int kAsmMaxLast = 4096;  // last-dim extent handled by the smem owner table
constexpr int kAsmMaxB = 256;

constexpr int kAsmRows = 4;  // lattice rows per CTA (owner table loaded once)

__global__ void __launch_bounds__(256) k_assemble(AssembleArgs a) {
  pdl_enter();
  __shared__ short s_own[kAsmMaxLast];
  __shared__ long long s_base[kAsmRows][kAsmMaxB];  // P offset of the row in block (lead, c) minus col_lo
  const int D = a.D, dl = D - 1;
  const int Nl = static_cast<int>(a.N[dl]), Bl = a.B[dl];
  const bool own_smem = Nl <= kAsmMaxLast;
  if (own_smem)
    for (int i = threadIdx.x; i < Nl; i += blockDim.x) s_own[i] = static_cast<short>(__ldg(a.own_coord + a.oc_off[dl] + i));
  const std::int64_t r0 = static_cast<std::int64_t>(blockIdx.x) * kAsmRows;
  const int nr = static_cast<int>(a.nrows - r0 < kAsmRows ? a.nrows - r0 : kAsmRows);
  // s_base per (row, last-dim block coordinate): the plan's row-base table
  for (int e = threadIdx.x; e < nr * Bl; e += blockDim.x) {
    const int r = e / Bl, c = e - r * Bl;
    s_base[r][c] = __ldg(a.rowbase + (a.row0 + r0 + r) * Bl + c);
  }
  __syncthreads();
  const int i0 = static_cast<int>(a.col0), i1 = static_cast<int>(a.col0 + a.ncols);
  double* out = a.lattice + (a.row0 + r0) * Nl;
  // all rows' loads of one column sweep in flight before the stores
  for (int i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const int c = own_smem ? s_own[i] : a.own_coord[a.oc_off[dl] + i];
    double v[kAsmRows];
#pragma unroll
    for (int r = 0; r < kAsmRows; ++r) v[r] = (r < nr && s_base[r][c] != kAsmOtherRank) ? a.P[s_base[r][c] + i] : 0.0;
#pragma unroll
    for (int r = 0; r < kAsmRows; ++r)
      if (r < nr) out[static_cast<std::int64_t>(r) * Nl + i] = v[r];
  }
}

// ------------------------------------------------------------------- K7
constexpr int kDecodeThreads = 256;

template <int P>
__global__ void __launch_bounds__(kDecodeThreads) k_decode(DecodeArgs a) {
  extern __shared__ double sm[];
  __shared__ double s_red[64];
  std::int64_t t = blockIdx.x;
  std::int64_t tc[3];
  tc[2] = t % a.ntiles[2];
  t /= a.ntiles[2];
  tc[1] = t % a.ntiles[1];
  tc[0] = t / a.ntiles[1];
  std::int64_t o[3];
  int e[3], base[3], w[3];
  for (int k = 0; k < 3; ++k) {
    o[k] = tc[k] * a.T[k];
    const std::int64_t rem = a.M[k] - o[k];
    e[k] = static_cast<int>(rem < a.T[k] ? rem : a.T[k]);
    base[k] = a.g0[k][o[k]];
    w[k] = a.g0[k][o[k] + e[k] - 1] + a.pk[k] + 1 - base[k];
  }
  const int T1 = a.T[1], T2 = a.T[2];
  double* pbox = sm;                               // w0*w1*w2
  double* s1 = pbox + a.W[0] * a.W[1] * a.W[2];    // w0*w1*T2
  double* s2 = s1 + a.W[0] * a.W[1] * T2;          // w0*T1*T2
  const int tid = threadIdx.x;
  // stage 0: control box (global lattice, L2 resident)
  for (int i = tid; i < w[0] * w[1] * w[2]; i += kDecodeThreads) {
    const int c2 = i % w[2], c01 = i / w[2], c1 = c01 % w[1], c0 = c01 / w[1];
    const std::int64_t i0 = base[0] + c0, i1 = base[1] + c1, i2 = base[2] + c2;
    // windowed lattices (decode.hpp col_offset): clipped basis entries are zero
    const bool in = i0 >= 0 && i0 < a.N[0] && i1 >= 0 && i1 < a.N[1] && i2 >= 0 && i2 < a.N[2];
    pbox[i] = in ? a.lattice[(i0 * a.N[1] + i1) * a.N[2] + i2] : 0.0;
  }
  __syncthreads();
  const int sv0 = a.pk[0] + 1, sv1 = a.pk[1] + 1, sv2 = a.pk[2] + 1;
  // stage 1: contract the contiguous axis
  for (int i = tid; i < w[0] * w[1] * e[2]; i += kDecodeThreads) {
    const int x = i % e[2], c01 = i / e[2];
    const std::int64_t gx = o[2] + x;
    const int g = a.g0[2][gx] - base[2];
    const double* vr = a.vals[2] + gx * sv2;
    const double* pr = pbox + c01 * w[2] + g;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k <= P; ++k)
      if (k <= a.pk[2]) s = fma(vr[k], pr[k], s);
    s1[c01 * T2 + x] = s;
  }
  __syncthreads();
  // stage 2: middle axis
  for (int i = tid; i < w[0] * e[1] * e[2]; i += kDecodeThreads) {
    const int x = i % e[2], r = i / e[2], y = r % e[1], c0 = r / e[1];
    const std::int64_t gy = o[1] + y;
    const int g = a.g0[1][gy] - base[1];
    const double* vr = a.vals[1] + gy * sv1;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k <= P; ++k)
      if (k <= a.pk[1]) s = fma(vr[k], s1[(c0 * w[1] + g + k) * T2 + x], s);
    s2[(c0 * T1 + y) * T2 + x] = s;
  }
  __syncthreads();
  // stage 3: leading axis + error + reductions
  double l2 = 0.0, li = 0.0;
  for (int i = tid; i < e[0] * e[1] * e[2]; i += kDecodeThreads) {
    const int x = i % e[2], r = i / e[2], y = r % e[1], z = r / e[1];
    const std::int64_t gz = o[0] + z;
    const int g = a.g0[0][gz] - base[0];
    const double* vr = a.vals[0] + gz * sv0;
    double s = 0.0;
#pragma unroll
    for (int k = 0; k <= P; ++k)
      if (k <= a.pk[0]) s = fma(vr[k], s2[((g + k) * T1 + y) * T2 + x], s);
    const std::int64_t gi = ((o[0] + z) * a.M[1] + o[1] + y) * a.M[2] + o[2] + x;
    if (a.field) {
      const double err = a.field[gi] - s;
      if (a.out) a.out[gi] = err;
      l2 = fma(err, err, l2);
      li = fmax(li, fabs(err));
    } else if (a.out) {
      a.out[gi] = s;
    }
  }
  if (!a.partial) return;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    l2 += __shfl_xor_sync(kFull, l2, off);
    li = fmax(li, __shfl_xor_sync(kFull, li, off));
  }
  const int wid = tid >> 5;
  if ((tid & 31) == 0) {
    s_red[wid] = l2;
    s_red[32 + wid] = li;
  }
  __syncthreads();
  if (tid == 0) {
    double sl = 0.0, sm2 = 0.0;
    for (int ww = 0; ww < kDecodeThreads / 32; ++ww) {
      sl += s_red[ww];
      sm2 = fmax(sm2, s_red[32 + ww]);
    }
    a.partial[2 * blockIdx.x] = sl;
    a.partial[2 * blockIdx.x + 1] = sm2;
  }
}

// residual_error of one local problem (lsq.cpp:66-85): the decode of
// apply_along_axis over d = 0..D-1 (apply_line, collocation.cpp:37-45: acc +=
// v * x from 0.0, no FMA in the reference build) at one point, q - decoded.
// Out-of-window basis entries are exact zeros and add exact zeros, so the
// clipped row of the reference and the aligned row here sum identically.
constexpr int kResPtThreads = 256;
template <int P>
__global__ void __launch_bounds__(kResPtThreads) k_residual_points(ResidualArgs a) {
  __shared__ double s_red[2][kResPtThreads / 32];
  auto clampi = [](int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); };
  double l2 = 0.0, li = 0.0;
  const std::int64_t stride = static_cast<std::int64_t>(gridDim.x) * blockDim.x;
  for (std::int64_t i = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < a.total; i += stride) {
    int j[3] = {0, 0, 0};
    {
      std::int64_t r = i;
      for (int k = a.D - 1; k >= 0; --k) {
        j[k] = static_cast<int>(r % a.m[k]);
        r /= a.m[k];
      }
    }
    int g[3] = {0, 0, 0};
    double v[3][P + 1];
    for (int k = 0; k < 3; ++k) {
      if (k < a.D) {
        g[k] = a.g0[k][j[k]];
#pragma unroll
        for (int t = 0; t <= P; ++t) v[k][t] = a.vals[k][static_cast<std::int64_t>(j[k]) * (P + 1) + t];
      } else {
#pragma unroll
        for (int t = 0; t <= P; ++t) v[k][t] = t == 0 ? 1.0 : 0.0;
      }
    }
    const int n1 = a.D >= 2 ? a.n[1] : 1, n2 = a.D >= 3 ? a.n[2] : 1;
    const int K1 = a.D >= 2 ? P : 0, K2 = a.D >= 3 ? P : 0;
    double acc2 = 0.0;  // outermost: the last axis applied
    for (int k2 = 0; k2 <= K2; ++k2) {
      const int c2 = a.D >= 3 ? clampi(g[2] + k2, n2) : 0;
      double acc1 = 0.0;
      for (int k1 = 0; k1 <= K1; ++k1) {
        const int c1 = a.D >= 2 ? clampi(g[1] + k1, n1) : 0;
        double acc0 = 0.0;
#pragma unroll
        for (int k0 = 0; k0 <= P; ++k0) {
          const int c0 = clampi(g[0] + k0, a.n[0]);
          const double x = a.controls[(static_cast<std::int64_t>(c0) * n1 + c1) * n2 + c2];
          acc0 = __dadd_rn(acc0, __dmul_rn(v[0][k0], x));
        }
        acc1 = a.D >= 2 ? __dadd_rn(acc1, __dmul_rn(v[1][k1], acc0)) : acc0;
      }
      acc2 = a.D >= 3 ? __dadd_rn(acc2, __dmul_rn(v[2][k2], acc1)) : acc1;
    }
    const double e = __dsub_rn(a.q[i], acc2);
    if (a.pointwise) a.pointwise[i] = e;
    l2 = fma(e, e, l2);
    li = fmax(li, fabs(e));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    l2 += __shfl_xor_sync(kFull, l2, o);
    li = fmax(li, __shfl_xor_sync(kFull, li, o));
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_red[0][w] = l2;
    s_red[1][w] = li;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sl = 0.0, sm = 0.0;
    for (int t = 0; t < kResPtThreads / 32; ++t) {
      sl += s_red[0][t];
      sm = fmax(sm, s_red[1][t]);
    }
    a.partial[2 * blockIdx.x] = sl;
    a.partial[2 * blockIdx.x + 1] = sm;
  }
}

__global__ void __launch_bounds__(1024) k_reduce_partials(const double* p, std::int64_t n, double* out) {
  __shared__ double s_l2[1024], s_li[1024];
  double l2 = 0.0, li = 0.0;
  for (std::int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    l2 += p[2 * i];
    li = fmax(li, p[2 * i + 1]);
  }
  s_l2[threadIdx.x] = l2;
  s_li[threadIdx.x] = li;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      s_l2[threadIdx.x] += s_l2[threadIdx.x + s];
      s_li[threadIdx.x] = fmax(s_li[threadIdx.x], s_li[threadIdx.x + s]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s_l2[0];
    out[1] = s_li[0];
  }
}

// Degree dispatch: instantiate the templated kernels for p = 1..kMaxDegree.
template <template <int> class F, class... Args>
int dispatch_degree(int p, Args&&... args) {
  switch (p) {
    case 1: return F<1>::run(args...);
    case 2: return F<2>::run(args...);
    case 3: return F<3>::run(args...);
    case 4: return F<4>::run(args...);
    case 5: return F<5>::run(args...);
    case 6: return F<6>::run(args...);
    case 7: return F<7>::run(args...);
    case 8: return F<8>::run(args...);
    case 9: return F<9>::run(args...);
    default: return -1;
  }
}

template <int P>
struct ResidualPointsLaunch {
  static int run(const ResidualArgs& a, int ctas, cudaStream_t s) {
    k_residual_points<P><<<ctas, kResPtThreads, 0, s>>>(a);
    return 1;
  }
};

template <int P>
struct RowsLaunch {
  static int run(const RowsArgs& a, cudaStream_t s) {
    if (a.nprobs == 0 || a.max_m == 0) return 0;
    dim3 grid((a.max_m + 255) / 256, a.nprobs);
    launch_pdl(k_basis_rows<P>, grid, dim3(256), 0, s, a);
    return 1;
  }
};

template <int P>
struct CholLaunch {
  static int run(const CholArgs& a, cudaStream_t s) {
    if (a.nfactor == 0) return 0;
    CholArgs b = a;
    size_t smem = static_cast<size_t>(a.max_n) * (P + 1) * sizeof(double);
    const size_t twb = a.tw ? 2 * smem : 0;  // pristine band + reversed factor
    // staged rows: vals, then g0 as ints (rounded up to whole doubles)
    const size_t staged = smem + static_cast<size_t>(a.max_m) * (P + 1) * sizeof(double) +
                          static_cast<size_t>((a.max_m + 1) / 2) * sizeof(double);
    b.stage_rows = !a.light && staged + twb <= 200 * 1024;
    if (b.stage_rows) smem = staged;
    smem += twb;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_gram_chol<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (!a.light) {
      k_gram_chol<P><<<a.nfactor, 256, smem, s>>>(b);
      return 1;
    }
    // light (beside the axis-0 sweep): the parallel Gram phase, then the
    // serial Cholesky as one warp per problem with only the band in shared
    // memory, so its CTAs co-reside with the sweep's instead of holding a
    // full CTA's resources for the length of the dependent chain
    b.light = 1;
    b.stage_rows = 0;  // rows through L1: no shared-memory footprint beyond the band
    const size_t band = static_cast<size_t>(a.max_n) * (P + 1) * sizeof(double);
    k_gram_chol<P><<<a.nfactor, 256, band + twb, s>>>(b);
    b.light = 2;
    b.stage_rows = 0;
    k_gram_chol<P><<<a.nfactor, a.tw ? 64 : 32, band + twb, s>>>(b);
    return 2;
    return 1;
  }
};

template <int P>
struct FitStridedLaunch {
  static int run(const FitArgs& a, int d, cudaStream_t s) {
    dim3 grid((a.max_lines_strided[d] + kStridedThreads - 1) / kStridedThreads, a.nblocks);
    k_fit_strided<P><<<grid, kStridedThreads, 0, s>>>(a, d);
    return 1;
  }
};

// 1-D fit (lsq.cpp:39-64 with D = 1): one CTA per block.  Thread per output
// column c accumulates R^T q over the contiguous run of rows whose basis
// covers c (g0 in [c-P, c]), in row order; one thread then runs the banded
// forward / back substitution (n steps each) and the L-inf of the non-shared
// controls.
template <int P>
__global__ void __launch_bounds__(256) k_fit_1d(FitArgs a) {
  extern __shared__ double s_z[];  // n, then the factor table n x (2P+1)
  const int b = blockIdx.x;
  const BlockDev& blk = a.blocks[b];
  const AxisProb pr = a.probs[blk.ax[0]];
  const int m = pr.m, n = pr.n;
  const int* g0 = a.g0 + pr.row_off;
  const double* v = a.vals + pr.row_off * (P + 1);
  const double* q = a.field + blk.fbase;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    int lo = 0, hi = m;  // first row with g0 >= c - P
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(g0 + mid) < c - P)
        lo = mid + 1;
      else
        hi = mid;
    }
    double z = 0.0;
    for (int j = lo; j < m; ++j) {
      const int g = __ldg(g0 + j);
      if (g > c) break;
      z = fma(__ldg(v + static_cast<std::int64_t>(j) * (P + 1) + (c - g)), q[static_cast<std::int64_t>(j) * a.fs[0]], z);
    }
    s_z[c] = z;
  }
  double* s_lt = s_z + n;  // factor staged in smem: the serial solve never waits on L2
  for (int i = threadIdx.x; i < n * (2 * P + 1); i += blockDim.x) s_lt[i] = a.ltab[pr.col_off * (2 * P + 1) + i];
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double* lt = s_lt;
  double w[P];
#pragma unroll
  for (int k = 0; k < P; ++k) w[k] = 0.0;
  for (int c = 0; c < n; ++c) {  // forward: y_c = (z_c - sum_k L(c,c-k) y_{c-k}) / L(c,c)
    const double* Lc = lt + static_cast<std::int64_t>(c) * (2 * P + 1);
    double sacc = s_z[c];
#pragma unroll
    for (int k = P; k >= 1; --k) sacc = fma(-Lc[k], w[k - 1], sacc);
    const double y = sacc * Lc[0];
#pragma unroll
    for (int k = P - 1; k >= 1; --k) w[k] = w[k - 1];
    w[0] = y;
    s_z[c] = y;
  }
#pragma unroll
  for (int k = 0; k < P; ++k) w[k] = 0.0;
  double* Pb = a.P + blk.poff;
  const unsigned char* sf = a.shared_flag + a.sflag_off[0] + pr.col_lo;
  unsigned long long lmax = 0ull;
  for (int c = n - 1; c >= 0; --c) {  // back: x_c = (y_c - sum_k L(c+k,c) x_{c+k}) / L(c,c)
    const double* Lc = lt + static_cast<std::int64_t>(c) * (2 * P + 1);
    double sacc = s_z[c];
#pragma unroll
    for (int k = P; k >= 1; --k) sacc = fma(-Lc[P + k], w[k - 1], sacc);
    const double x = sacc * Lc[0];
#pragma unroll
    for (int k = P - 1; k >= 1; --k) w[k] = w[k - 1];
    w[0] = x;
    Pb[c] = x;
    if (!sf[c]) lmax = umax(lmax, dbits(fabs(x)));
  }
  if (lmax) atomicMax(a.linf_int + b, lmax);
}

template <int P>
struct Fit1DLaunch {
  static int run(const FitArgs& a, int max_n, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(max_n) * (2 * P + 2) * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_fit_1d<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_fit_1d<P><<<a.nblocks, 256, smem, s>>>(a);
    return 1;
  }
};

template <int P>
struct FitLastLaunch {
  static int run(const FitArgs& a, cudaStream_t s) {
    const size_t smem = (static_cast<size_t>(kLastThreads) * (kLastCols + 1) + kLastCols * (P + 1)) * sizeof(double) +
                        kLastCols * sizeof(int);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_fit_last<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dim3 grid((a.max_lines_last + kLastThreads - 1) / kLastThreads, a.nblocks);
    k_fit_last<P><<<grid, kLastThreads, smem, s>>>(a);
    return 1;
  }
};

template <int P>
struct DecodeLaunch {
  static int run(const DecodeArgs& a, cudaStream_t s) {
    const std::int64_t tiles = a.ntiles[0] * a.ntiles[1] * a.ntiles[2];
    const size_t smem = (static_cast<size_t>(a.W[0]) * a.W[1] * a.W[2] + static_cast<size_t>(a.W[0]) * a.W[1] * a.T[2] +
                         static_cast<size_t>(a.W[0]) * a.T[1] * a.T[2]) * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_decode<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_decode<P><<<static_cast<unsigned>(tiles), kDecodeThreads, smem, s>>>(a);
    return 1;
  }
};

}  // namespace

int debug_fail_line() {
#ifdef MFB_DEBUG
  int line = 0;
  cudaMemcpyFromSymbol(&line, g_mfb_debug_line, sizeof(int));
  return line;
#else
  return 0;
#endif
}

int launch_residual_points(int degree, const ResidualArgs& a, int ctas, cudaStream_t s) {
  return dispatch_degree<ResidualPointsLaunch>(degree, a, ctas, s);
}
int launch_basis_rows(int degree, const RowsArgs& a, cudaStream_t s) {
  return dispatch_degree<RowsLaunch>(degree, a, s);
}
int launch_block_residual(int degree, const BlockResArgs& a, cudaStream_t s) {
  if (a.nblocks <= 0) return 0;
  return dispatch_degree<BlockResLaunch>(degree, a, s);
}
int launch_gram_chol(int degree, const CholArgs& a, cudaStream_t s) {
  return dispatch_degree<CholLaunch>(degree, a, s);
}
int launch_fit_strided(int degree, const FitArgs& a, int axis, cudaStream_t s) {
  return dispatch_degree<FitStridedLaunch>(degree, a, axis, s);
}
int launch_fit_last(int degree, const FitArgs& a, cudaStream_t s) {
  return dispatch_degree<FitLastLaunch>(degree, a, s);
}
int launch_fit_1d(int degree, const FitArgs& a, int max_n, cudaStream_t s) {
  return dispatch_degree<Fit1DLaunch>(degree, a, max_n, s);
}
int launch_decode(int degree, const DecodeArgs& a, cudaStream_t s) {
  return dispatch_degree<DecodeLaunch>(degree, a, s);
}

int launch_epoch(const EpochArgs& a, cudaStream_t s) {
  if (a.total == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  std::int64_t want = (a.total + kEpochThreads - 1) / kEpochThreads;
  const std::int64_t cap = static_cast<std::int64_t>(sms) * 4;
  const unsigned grid = static_cast<unsigned>(want < cap ? want : cap);
  bool small = a.nblocks <= kEpochSmemBlocks;
  for (int k = 0; k < a.D; ++k) small = small && a.B[k] <= kMaxCoords;
  if (a.max_holders <= 8 && small)
    k_epoch8<<<grid, kEpochThreads, 0, s>>>(a);
  else if (a.max_holders <= 8)
    k_epoch<8><<<grid, kEpochThreads, 0, s>>>(a);
  else
    k_epoch<27><<<grid, kEpochThreads, 0, s>>>(a);
  return 1;
}

__global__ void __launch_bounds__(256) k_pack(const PackTile* tiles, const double* P, double* send) {
  const PackTile t = tiles[blockIdx.x];
  const float rc1 = 1.0f / static_cast<float>(t.ext1), rc2 = 1.0f / static_cast<float>(t.ext2);
  for (int i = t.start + threadIdx.x; i < t.start + t.count; i += blockDim.x) {
    int q, r2, r0, r1;
    fast_divmod(i, t.ext2, rc2, q, r2);
    fast_divmod(q, t.ext1, rc1, r0, r1);
    send[t.dst + i] = P[t.base + static_cast<long long>(r0) * t.str[0] + r1 * t.str[1] + r2 * t.str[2]];
  }
}

int launch_pack(const PackTile* tiles, int ntiles, const double* P, double* send, cudaStream_t s) {
  if (ntiles <= 0) return 0;
  k_pack<<<ntiles, 256, 0, s>>>(tiles, P, send);
  return 1;
}

int launch_epoch_finalize(const EpochRegionArgs& a, cudaStream_t s) {
  k_epoch_finalize<<<1, kRegionThreads, 0, s>>>(a);
  return 1;
}
int launch_shard_advance(EpochState* st, const double* epoch_out, int slot, double tol, cudaStream_t s) {
  k_shard_advance<<<1, 1, 0, s>>>(st, epoch_out, slot, tol);
  return 1;
}

int launch_epoch_regions(const EpochRegionArgs& a, cudaStream_t s) {
  if (a.ntiles <= 0) return 0;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  if (a.mode == 3)  // persistent over the tiles: one wave (usually it exits at once)
    launch_pdl(k_pair_jumps_regions, dim3(a.ntiles < 2 * sms ? a.ntiles : 2 * sms), dim3(kRegionThreads), 0, s, a);
  else {
    const int per_sm = a.max_ns > 4 ? MFB_EPOCH8_CTAS : 3;  // __launch_bounds__ residency
    const int grid = a.ntiles < sms * per_sm ? a.ntiles : sms * per_sm;
    if (a.max_ns > 4)
      a.snap ? launch_pdl(k_epoch_regions<8, true>, dim3(grid), dim3(kRegionThreads), 0, s, a)
             : launch_pdl(k_epoch_regions<8, false>, dim3(grid), dim3(kRegionThreads), 0, s, a);
    else
      a.snap ? launch_pdl(k_epoch_regions<4, true>, dim3(grid), dim3(kRegionThreads), 0, s, a)
             : launch_pdl(k_epoch_regions<4, false>, dim3(grid), dim3(kRegionThreads), 0, s, a);
  }
  return 1;
}

int launch_dp(const DpArgs& a, cudaStream_t s) {
  k_dp<<<1, 1024, 0, s>>>(a);
  return 1;
}

int launch_assemble(const AssembleArgs& a, cudaStream_t s) {
  if (a.B[a.D - 1] > kAsmMaxB) return -1;  // host validates blocks_per_dim first
  if (a.nrows <= 0) return 0;
  launch_pdl(k_assemble, dim3(static_cast<unsigned>((a.nrows + kAsmRows - 1) / kAsmRows)), dim3(256), 0, s, a);
  return 1;
}

int launch_reduce_partials(const double* partial, std::int64_t n, double* out2, cudaStream_t s) {
  k_reduce_partials<<<1, 1024, 0, s>>>(partial, n, out2);
  return 1;
}

}  // namespace mfb
