// solve_tma.cu — the solve stage of the fit on shared-memory tiles
// (lsq.cpp:59-60 on each axis, after the pure contractions of stream_tma.cu):
//
//   k_rl_tables     right-looking step tables of every factored axis problem
//   k_solve2d       D = 2: one CTA per block, G1^-1 then G0^-1 on Z = R0^T Q_b R1
//   k_solve2d_tw    the same with twisted (two-sided) passes (MFADD_TWIST)
//   k_solve3d       D = 3: slabs of axis-0 indices, G2^-1 and G1^-1 (and G0^-1)
//   k_axis0_slab    D = 3: G0^-1 on slabs of axis-1 indices of the held lattice
//
// (a translation unit of its own: these kernels are instantiated for every
// degree and line count and were two thirds of stream_tma.cu's compile time)
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "tma.cuh"

namespace mfb {

namespace {

constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ unsigned long long dbits_s(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

// ------------------------------------------- fused 2-D solve (CTA per block)
// D = 2 with the axis-0 sweep as a pure contraction (defer_back == 2): after
// k_last_contract_tma the block's whole right-hand side Z = R0^T Q_b R1 is
// n0 x n1 values, which fit in one CTA's shared memory.  One CTA per block
// pulls Z in with 1-D bulk copies (one per contraction segment, plus the
// segment carries), runs the banded G1 solve along every row (thread per
// row, lsq.cpp:59-60 on axis 1), then the banded G0 solve along every column
// (thread per column, lsq.cpp:59-60 on axis 0), and writes P_b once plus the
// per-block L-inf over non-shared controls (solver.cpp:97-101).  Replaces
// k_last_solve + k_axis0_solve_part: no y scratch round trip through HBM,
// one launch, no per-element index arithmetic on the load path.
//
// Shared-memory tile: X[c][i] in Z's own column-major layout (pitch zl lines,
// even so every column is 16-B aligned for the bulk copies, = 2 mod 4 so the
// column-parallel phase has at most 2-way bank conflicts).
constexpr int kSolve2dThreads = 256;

// Right-looking banded substitution passes on one line of a shared-memory
// tile.  A pass walks steps t = 0..n-1 over x0[t*ds] (ds < 0 walks a line
// backwards) with a step table of W doubles per step:
//   forward  (L y = z,   column c = t):      [L(c+k,c)/L(c+k,c+k) k=1..P, 1/L(c+P,c+P)]
//   backward (L^T x = y, column c = n-1-t):  [L(c,c-k)/L(c-k,c-k) k=1..P, 1/L(c-P,c-P)]
// Rows -P..-1 carry only the last entry (the scale of the first P values);
// rows past the line are zero.  The P pending sums of the next steps sit in
// static register slots (slot = step mod P; U is a multiple of P).  A
// finished value updates the pending sums at once, the next step's first,
// so the dependent chain per step is one FMA; the value P steps ahead enters
// scaled by its 1/L(c,c).  The arithmetic is the reference's solve
// (lsq.cpp:59-60) up to rounding order (1e-10 contract).  Full batches run
// without bounds tests; the last < 2U+P steps run guarded.
#ifndef MFB_RL_U
#define MFB_RL_U 8  // unrolled steps per batch of the right-looking passes (rounded up to a multiple of P)
#endif
template <int P>
struct RL {
  static constexpr int W = (P + 2) & ~1;  // table row (16-B multiple)
  static constexpr int U = P * ((MFB_RL_U + P - 1) / P);
};

__host__ __device__ inline int rl_rows(int n, int P) {  // table rows incl. the P leading ones
  const int U = P * ((MFB_RL_U + P - 1) / P);
  return P + n + 2 * U + P;
}

struct RLFinal {  // last pass of a tile: results also go to HBM (+ L-inf)
  double* dst;            // global base of this line's outputs
  std::int64_t dstride;   // global stride per step (signed)
  int t_lo, t_hi;         // steps [t_lo, t_hi) hold non-shared entries (shared ones sit at both ends of a line)
  bool line_shared;
  unsigned long long lmax;
};

// MFB_RL_GTAB=1 (measurement knob): the plain passes read the step tables from
// global memory through L1 instead of staging them in shared memory.  Measured
// slower on C5 (fit_last 193 us against 121 us; 181 / 177 us with the rows
// loaded 2 / 3 steps ahead): a broadcast 16-byte load costs four shared-memory
// wavefronts, but the L1 path's latency costs more.
#ifndef MFB_RL_GTAB
#define MFB_RL_GTAB 0
#endif
template <int P>
__device__ __forceinline__ void rl_load_step(const double* row, double (&cf)[RL<P>::W]) {
#pragma unroll
  for (int h = 0; h < RL<P>::W / 2; ++h) {
#if MFB_RL_GTAB
    const double2 v = __ldg(reinterpret_cast<const double2*>(row) + h);
#else
    const double2 v = reinterpret_cast<const double2*>(row)[h];
#endif
    cf[2 * h] = v.x;
    cf[2 * h + 1] = v.y;
  }
}

// cf holds the table rows of steps t0 .. t0+PF-1 on entry and of steps
// t0+U .. t0+U+PF-1 on exit: each step's coefficients are loaded PF steps
// ahead (MFB_RL_PF), off the dependent chain and past the shared-memory
// latency with one warp per scheduler.
#ifndef MFB_RL_PF
#define MFB_RL_PF 1
#endif
// SIDE (twisted forward passes): steps [side_e, n) hold the pending sums of
// the middle rows, which go to side[(t - side_e) * side_stride] instead of the
// line (the other half of the line still reads those rows).
struct RLSide {
  double* side;
  int stride, e;
};
template <int P, bool TAIL, bool FINAL, bool SIDE = false>
__device__ __forceinline__ void rl_batch(double* __restrict__ x0, const int ds, const int n, const int t0,
                                         const double* __restrict__ tab, double (&acc)[P], double (&zin)[RL<P>::U],
                                         double (&cf)[MFB_RL_PF][RL<P>::W], RLFinal& fin, const RLSide sd = RLSide{}) {
  constexpr int U = RL<P>::U, W = RL<P>::W, PF = MFB_RL_PF;
  double znx[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int te = t0 + U + P + u;
    znx[u] = (!TAIL || te < n) ? x0[te * ds] : 0.0;
  }
  const double* tb = tab + t0 * W;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    double cfn[W];
    rl_load_step<P>(tb + (u + PF) * W, cfn);  // the row PF steps ahead (tables are padded past the line)
    const double y = acc[u % P];
#pragma unroll
    for (int k = 1; k < P; ++k) acc[(u + k) % P] = fma(-cf[0][k - 1], y, acc[(u + k) % P]);
    acc[u % P] = fma(-cf[0][P - 1], y, zin[u] * cf[0][P]);
    const int t = t0 + u;
    if (!TAIL || t < n) {
      if (SIDE && TAIL && t >= sd.e)  // (a full batch ends U + P steps before n: below sd.e)
        sd.side[(t - sd.e) * sd.stride] = y;
      else
        x0[t * ds] = y;
      if (FINAL) {
        fin.dst[t * fin.dstride] = y;
        if (!fin.line_shared && t >= fin.t_lo && t < fin.t_hi) {  // no shared-memory flag on the chain
          const unsigned long long bits = dbits_s(fabs(y));
          fin.lmax = fin.lmax > bits ? fin.lmax : bits;
        }
      }
    }
#pragma unroll
    for (int q = 0; q + 1 < PF; ++q)
#pragma unroll
      for (int k = 0; k < W; ++k) cf[q][k] = cf[q + 1][k];
#pragma unroll
    for (int k = 0; k < W; ++k) cf[PF - 1][k] = cfn[k];
  }
#pragma unroll
  for (int u = 0; u < U; ++u) zin[u] = znx[u];
}

// init (twisted backward passes): the first P values come from registers
// instead of the line.
template <int P, bool FINAL, bool SIDE = false, bool INIT = false>
__device__ __forceinline__ void rl_pass(double* __restrict__ x0, const int ds, const int n,
                                        const double* __restrict__ tab, RLFinal& fin, const RLSide sd = RLSide{},
                                        const double* init = nullptr) {
  constexpr int U = RL<P>::U, W = RL<P>::W, PF = MFB_RL_PF;
  double acc[P], zin[U];
#pragma unroll
  for (int k = 0; k < P; ++k)
    acc[k] = (INIT ? init[k] : (k < n ? x0[k * ds] : 0.0)) * (MFB_RL_GTAB ? __ldg(tab + (k - P) * W + P) : tab[(k - P) * W + P]);
#pragma unroll
  for (int u = 0; u < U; ++u) zin[u] = P + u < n ? x0[(P + u) * ds] : 0.0;
  double cf[PF][W];
#pragma unroll
  for (int q = 0; q < PF; ++q) rl_load_step<P>(tab + q * W, cf[q]);
  int t0 = 0;
  for (; t0 + 2 * U + P <= n; t0 += U) rl_batch<P, false, FINAL, SIDE>(x0, ds, n, t0, tab, acc, zin, cf, fin, sd);
  for (; t0 < n; t0 += U) rl_batch<P, true, FINAL, SIDE>(x0, ds, n, t0, tab, acc, zin, cf, fin, sd);
}

// ---- twisted (two-sided) solve of one banded SPD system G x = z
// Rows [0, a) are eliminated from the top with the standard factor L, rows
// [a+P, n) from the bottom with the factor L' of the index-reversed matrix,
// and the P rows between them last, through the explicit inverse of their
// dense Schur complement S.  Two threads share a line: each runs a forward
// pass over its outer part (leaving its contribution to the middle rows'
// right-hand side in a side buffer), both form x_M = S^-1 r, and each runs the
// backward pass of its part outwards from the middle.  The arithmetic per row
// is that of lsq.cpp:59-60 with another elimination order (1e-10 contract);
// the dependent chain is n/2 + P steps per pass instead of n.
// Table set of one problem: [TF | TB | BF | BB | S^-1 (P*P, padded even)],
// step tables in the layout of rl_pass over a + P (top) / nb + P (bottom)
// steps, the last P forward steps (first P backward steps) being the middle
// rows.
__host__ __device__ inline int tw_top(int n, int P) { return (n - P) / 2; }
__host__ __device__ inline int tw_bot(int n, int P) { return n - P - (n - P) / 2; }
__host__ __device__ inline int tw_table_doubles(int n, int P) {
  const int W = (P + 2) & ~1;
  return 2 * (rl_rows(tw_top(n, P) + P, P) + rl_rows(tw_bot(n, P) + P, P)) * W + ((P * P + 1) & ~1);
}

// Forward / backward step tables of one half.  rec(i, 0) = 1/Lh(i,i) and
// rec(i, k) = Lh(i, i-k) in the half's own index space (bottom: reversed),
// e = rows eliminated by the half, top = the half whose forward pass carries
// the middle rows' own right-hand side.
template <int P, class Rec>
__device__ __forceinline__ void build_tw_half(Rec rec, int e, bool top, double* f, double* b, int tid, int nthr) {
  constexpr int W = RL<P>::W;
  const int rows = rl_rows(e + P, P);
  for (int i = tid; i < rows * W; i += nthr) {
    const int t = i / W - P, k = i - (t + P) * W;
    double fv = 0.0, bv = 0.0;
    if (k < P) {
      const int j = k + 1;
      if (t >= 0 && t < e) fv = rec(t + j, j) * (t + j < e ? rec(t + j, 0) : 1.0);
      if (t >= 0 && t < e + P) {
        const int rho = e + P - 1 - t, tgt = rho - j;
        if (tgt >= 0 && tgt < e) bv = rec(rho, j) * rec(tgt, 0);
      }
    } else if (k == P) {
      const int te = t + P;  // the step whose value enters here
      fv = te < e ? rec(te, 0) : (te < e + P ? (top ? 1.0 : 0.0) : 0.0);
      const int r = e - 1 - t;
      bv = t < 0 ? 1.0 : (r >= 0 ? rec(r, 0) : 0.0);
    }
    f[i] = fv;
    b[i] = bv;
  }
}

// lt: standard factor table (2P+1 per column), rv: reversed factor ([n][P+1]),
// gb: Gram band ([n][P+1]); out: the problem's table set.
template <int P>
__device__ void build_tw_tables(const double* lt, const double* rv, const double* gb, int n, double* out, int tid,
                                int nthr) {
  constexpr int LW = 2 * P + 1, W = RL<P>::W;
  const int a = tw_top(n, P), nb = tw_bot(n, P);
  double* tf = out;
  double* tb = tf + rl_rows(a + P, P) * W;
  double* bf = tb + rl_rows(a + P, P) * W;
  double* bb = bf + rl_rows(nb + P, P) * W;
  double* sinv = bb + rl_rows(nb + P, P) * W;
  auto rt = [lt](int i, int k) { return __ldg(lt + i * LW + k); };
  auto rb = [rv](int i, int k) { return __ldg(rv + i * (P + 1) + k); };
  build_tw_half<P>(rt, a, true, tf + 0, tb + 0, tid, nthr);
  build_tw_half<P>(rb, nb, false, bf + 0, bb + 0, tid, nthr);
  if (tid == nthr - 1) {
    // S = S_top + S_bot - G_MM with S_top = L_MM L_MM^T (what is left of the
    // middle block after the top eliminations), S_bot likewise from below.
    // Everything in registers (compile-time indices).
    double Lt[P][P], Lb[P][P];  // Lh(base+i, base+j), j <= i
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        Lt[i][j] = j > i ? 0.0 : (i == j ? 1.0 / rt(a + i, 0) : rt(a + i, i - j));
        Lb[i][j] = j > i ? 0.0 : (i == j ? 1.0 / rb(nb + i, 0) : rb(nb + i, i - j));
      }
    double S[P][P], I[P][P];
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        if (j > i) continue;  // actual rows (a+i, a+j)
        double st = 0.0, sb = 0.0;
#pragma unroll
        for (int m = 0; m < P; ++m)
          if (m <= j) st = fma(Lt[i][m], Lt[j][m], st);
        // reversed middle indices: row a+i <-> nb + (P-1-i), so (i, j) is the
        // reversed block's entry (P-1-j, P-1-i) with P-1-j >= P-1-i
#pragma unroll
        for (int m = 0; m < P; ++m)
          if (m <= P - 1 - i) sb = fma(Lb[P - 1 - j][m], Lb[P - 1 - i][m], sb);
        const double g = __ldg(gb + (a + i) * (P + 1) + (i - j));
        S[i][j] = st + sb - g;
        S[j][i] = S[i][j];
      }
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) I[i][j] = i == j ? 1.0 : 0.0;
#pragma unroll
    for (int c = 0; c < P; ++c) {  // Gauss-Jordan (S is SPD: no pivoting)
      const double pv = 1.0 / S[c][c];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        S[c][j] *= pv;
        I[c][j] *= pv;
      }
#pragma unroll
      for (int r = 0; r < P; ++r) {
        if (r == c) continue;
        const double fct = S[r][c];
#pragma unroll
        for (int j = 0; j < P; ++j) {
          S[r][j] = fma(-fct, S[c][j], S[r][j]);
          I[r][j] = fma(-fct, I[c][j], I[r][j]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) sinv[i * P + j] = I[i][j];
    if ((P * P) & 1) sinv[P * P] = 0.0;
  }
}

// ---- NL lines per thread
// The step-table row of a pass is the same for every line, and a broadcast
// 16-byte shared-memory load still costs four wavefronts: with one line per
// thread 12 of a step's 16 wavefronts are table reads, and the passes run
// against the shared-memory pipe (k_solve3d: 66% of its peak).  A thread that
// carries NL lines through the same steps reads each row once for all of
// them and has NL independent chains in flight.  Line j of a thread sits at
// element offset lo[j] from x0 (callers interleave the lines over the
// threads, so a warp's accesses to line j stay contiguous); lines past the
// end alias the thread's line 0 (same values, same stores).
template <int P, int NL>
struct RLN {
  static constexpr int UB = NL >= 4 ? 4 : 8;
  static constexpr int U = P * ((UB + P - 1) / P);  // <= RL<P>::U: the tables' padding covers it
};
template <int NL>
struct RLFinalN {         // last pass of a tile: results also go to HBM (+ L-inf)
  double* dst[NL];        // global base of each line's outputs
  std::int64_t dstride;   // global stride per step (signed)
  int t_lo, t_hi;         // steps [t_lo, t_hi) hold non-shared entries
  bool line_shared[NL];
  unsigned long long lmax;
};

template <int P, int NL, bool TAIL, bool FINAL>
__device__ __forceinline__ void rln_batch(double* __restrict__ x0, const int (&lo)[NL], const int ds, const int n,
                                          const int t0, const double* __restrict__ tab, double (&acc)[NL][P],
                                          double (&zin)[NL][RLN<P, NL>::U], double (&cf)[RL<P>::W], RLFinalN<NL>& fin) {
  constexpr int U = RLN<P, NL>::U, W = RL<P>::W;
  double znx[NL][U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int te = t0 + U + P + u;
#pragma unroll
    for (int j = 0; j < NL; ++j) znx[j][u] = (!TAIL || te < n) ? x0[te * ds + lo[j]] : 0.0;
  }
  const double* tb = tab + t0 * W;
#pragma unroll
  for (int u = 0; u < U; ++u) {
    double cfn[W];
    rl_load_step<P>(tb + (u + 1) * W, cfn);  // the next step's row (tables are padded past the line)
    const int t = t0 + u;
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const double y = acc[j][u % P];
#pragma unroll
      for (int k = 1; k < P; ++k) acc[j][(u + k) % P] = fma(-cf[k - 1], y, acc[j][(u + k) % P]);
      acc[j][u % P] = fma(-cf[P - 1], y, zin[j][u] * cf[P]);
      if (!TAIL || t < n) {
        x0[t * ds + lo[j]] = y;
        if (FINAL) {
          fin.dst[j][t * fin.dstride] = y;
          if (!fin.line_shared[j] && t >= fin.t_lo && t < fin.t_hi) {
            const unsigned long long bits = dbits_s(fabs(y));
            fin.lmax = fin.lmax > bits ? fin.lmax : bits;
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < W; ++k) cf[k] = cfn[k];
  }
#pragma unroll
  for (int j = 0; j < NL; ++j)
#pragma unroll
    for (int u = 0; u < U; ++u) zin[j][u] = znx[j][u];
}

template <int P, int NL, bool FINAL>
__device__ __forceinline__ void rln_pass(double* __restrict__ x0, const int (&lo)[NL], const int ds, const int n,
                                         const double* __restrict__ tab, RLFinalN<NL>& fin) {
  constexpr int U = RLN<P, NL>::U, W = RL<P>::W;
  double acc[NL][P], zin[NL][U];
#pragma unroll
  for (int j = 0; j < NL; ++j) {
#pragma unroll
    for (int k = 0; k < P; ++k) acc[j][k] = (k < n ? x0[k * ds + lo[j]] : 0.0) * tab[(k - P) * W + P];
#pragma unroll
    for (int u = 0; u < U; ++u) zin[j][u] = P + u < n ? x0[(P + u) * ds + lo[j]] : 0.0;
  }
  double cf[W];
  rl_load_step<P>(tab, cf);
  int t0 = 0;
  for (; t0 + 2 * U + P <= n; t0 += U) rln_batch<P, NL, false, FINAL>(x0, lo, ds, n, t0, tab, acc, zin, cf, fin);
  for (; t0 < n; t0 += U) rln_batch<P, NL, true, FINAL>(x0, lo, ds, n, t0, tab, acc, zin, cf, fin);
}

__host__ __device__ inline size_t solve2d_smem_bytes(int n0, int n1, int zl, int P, int kseg, bool tw = false) {
  const int W = (P + 2) & ~1;
  // step tables (only when staged in shared memory) / the twisted passes' two side buffers
  const size_t tabs = tw ? 2 * static_cast<size_t>(P) * (kSolve2dThreads / 2)
                         : (MFB_RL_GTAB ? 0 : 2 * static_cast<size_t>(rl_rows(n0, P) + rl_rows(n1, P)) * W);
  return 128 + (static_cast<size_t>(n1) * zl + static_cast<size_t>(kseg > 1 ? kseg - 1 : 0) * (P + 1) * zl + tabs) * 8 +
         static_cast<size_t>(n0 + n1 + 16);
}

// Forward / backward step tables of one axis problem (layout above) from the
// Cholesky table (2P+1 per column: [1/L(c,c), L(c,c-k), L(c+k,c)]).  f and b
// point at row -P of their rl_rows(n) rows.
template <int P>
__device__ __forceinline__ void build_rl_tables(const double* lt, int n, double* f, double* b, int tid, int nthr) {
  constexpr int LW = 2 * P + 1, W = RL<P>::W;
  const int rows = rl_rows(n, P);
  for (int e = tid; e < rows * W; e += nthr) {
    const int t = e / W - P, k = e - (t + P) * W;
    double fv = 0.0, bv = 0.0;
    if (k < P) {
      if (t >= 0 && t < n) {
        const int c = t, cb = n - 1 - t, j = k + 1;
        fv = c + j < n ? __ldg(lt + c * LW + P + j) * __ldg(lt + (c + j) * LW) : 0.0;
        bv = cb - j >= 0 ? __ldg(lt + cb * LW + j) * __ldg(lt + (cb - j) * LW) : 0.0;
      }
    } else if (k == P) {
      const int te = t + P;  // the step whose value enters here
      if (te >= 0 && te < n) {
        fv = __ldg(lt + te * LW);
        bv = __ldg(lt + (n - 1 - te) * LW);
      }
    }
    f[e] = fv;
    b[e] = bv;
  }
}

// The right-looking step tables of every factored axis problem, once per
// solve after the factorizations (the solve kernels bulk-copy them instead of
// deriving them from the Cholesky table in every CTA).
template <int P>
__global__ void __launch_bounds__(256) k_rl_tables(const CholArgs a, double* rlt, std::int64_t stride, int tw) {
  constexpr int W = RL<P>::W;
  const int pid = a.prob_ids[blockIdx.x];
  const AxisProb pr = a.probs[pid];
  double* f = rlt + static_cast<std::int64_t>(pid) * stride;
  if (tw) {
    const double* twp = a.tw + static_cast<std::int64_t>(pid) * a.tw_stride;
    build_tw_tables<P>(a.ltab + pr.col_off * (2 * P + 1), twp, twp + pr.n * (P + 1), pr.n, f, threadIdx.x, blockDim.x);
    return;
  }
  build_rl_tables<P>(a.ltab + pr.col_off * (2 * P + 1), pr.n, f, f + rl_rows(pr.n, P) * W, threadIdx.x, blockDim.x);
}

// A problem's tables into shared memory: bulk copies (rlt) on `bar`, or
// built from the Cholesky table by the CTA.  Returns the bytes the copies add.
template <int P>
__device__ __forceinline__ unsigned stage_rl_tables(const FitArgs& a, const AxisProb& pr, int pid, double* f, double* b,
                                                    std::uint64_t* bar, int tid, int nthr) {
  constexpr int W = RL<P>::W;
  const unsigned bytes = static_cast<unsigned>(rl_rows(pr.n, P) * W) * 8;
  if (a.rlt) {
    if (tid == 0) {
      const double* src = a.rlt + static_cast<std::int64_t>(pid) * a.rlt_stride;
      bulk_load_1d(f, src, bytes, bar);
      bulk_load_1d(b, src + rl_rows(pr.n, P) * W, bytes, bar);
    }
    return 2 * bytes;
  }
  build_rl_tables<P>(a.ltab + pr.col_off * (2 * P + 1), pr.n, f, b, tid, nthr);
  return 0;
}

#ifndef MFB_S2_NL
#define MFB_S2_NL 1  // lines per thread of k_solve2d's passes
#endif
template <int P>
__global__ void __launch_bounds__(kSolve2dThreads) k_solve2d(const FitArgs a) {
  pdl_enter();
  extern __shared__ __align__(128) double s2d[];
  __shared__ unsigned long long s_red[32];
  constexpr int PADC = P + 1, W = RL<P>::W;
  const int bid = blockIdx.x;
  const BlockDev& blk = a.blocks[bid];
  const AxisProb p0 = a.probs[blk.ax[0]], p1 = a.probs[blk.ax[1]];
  const int n0 = p0.n, n1 = p1.n, zl = blk.zl;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int* seg = a.segtab + blk.ax[1] * kSegStride;
  const int K = seg[0];
  const int* g0g = a.g0 + p1.row_off;
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(s2d);
  double* X = s2d + 16;                                   // [n1][zl]
  double* C = X + static_cast<std::int64_t>(n1) * zl;     // [(K-1)(P+1)][zl] carries
#if MFB_RL_GTAB
  // the step tables stay in global memory (k_rl_tables), read through L1
  const double* f0 = a.rlt + static_cast<std::int64_t>(blk.ax[0]) * a.rlt_stride;
  const double* b0 = f0 + rl_rows(n0, P) * W;
  const double* f1 = a.rlt + static_cast<std::int64_t>(blk.ax[1]) * a.rlt_stride;
  const double* b1 = f1 + rl_rows(n1, P) * W;
  unsigned char* sf0 = reinterpret_cast<unsigned char*>(C + static_cast<std::int64_t>(K - 1) * PADC * zl);
#else
  double* f0 = C + static_cast<std::int64_t>(K - 1) * PADC * zl;
  double* b0 = f0 + rl_rows(n0, P) * W;
  double* f1 = b0 + rl_rows(n0, P) * W;
  double* b1 = f1 + rl_rows(n1, P) * W;
  unsigned char* sf0 = reinterpret_cast<unsigned char*>(b1 + rl_rows(n1, P) * W);  // n0: axis-0 index shared
#endif
  unsigned char* sf1 = sf0 + n0;                                                   // n1: axis-1 index shared
  const double* zb = a.Y + blk.zoff + static_cast<std::int64_t>(PADC) * zl;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    unsigned bytes = static_cast<unsigned>(n1) * zl * 8 + static_cast<unsigned>(K - 1) * PADC * zl * 8;
#if !MFB_RL_GTAB
    if (a.rlt) bytes += 2 * static_cast<unsigned>((rl_rows(n0, P) + rl_rows(n1, P)) * W) * 8;
#endif
    mbar_arrive_expect_tx(bar, bytes);
    int cs = 0;
    for (int sg = 0; sg < K; ++sg) {  // segment sg owns columns [cs_sg, cs_sg+1) in parity sg & 1
      const int ce = sg + 1 < K ? __ldg(g0g + seg[2 + sg]) : n1;
      const double* src = zb + (sg & 1) * a.zhalf + static_cast<std::int64_t>(cs) * zl;
      if (ce > cs) bulk_load_1d(X + static_cast<std::int64_t>(cs) * zl, src, static_cast<unsigned>(ce - cs) * zl * 8, bar);
      if (sg + 1 < K)  // its partial sums of the next segment's first P+1 columns
        bulk_load_1d(C + static_cast<std::int64_t>(sg) * PADC * zl, zb + (sg & 1) * a.zhalf + static_cast<std::int64_t>(ce) * zl,
                     static_cast<unsigned>(PADC) * zl * 8, bar);
      cs = ce;
    }
  }
#if !MFB_RL_GTAB
  stage_rl_tables<P>(a, p0, blk.ax[0], f0, b0, bar, tid, nthr);
  stage_rl_tables<P>(a, p1, blk.ax[1], f1, b1, bar, tid, nthr);
#endif
  for (int c = tid; c < n1; c += nthr) sf1[c] = a.shared_flag[a.sflag_off[1] + p1.col_lo + c];
  __shared__ int s_ns[2];  // non-shared axis-0 indices: [s_ns[0], s_ns[1])
  if (tid == 0) {
    s_ns[0] = n0;
    s_ns[1] = 0;
  }
  __syncthreads();
  for (int i = tid; i < n0; i += nthr) {
    const unsigned char f = a.shared_flag[a.sflag_off[0] + p0.col_lo + i];
    sf0[i] = f;
    if (!f) {
      atomicMin(&s_ns[0], i);
      atomicMax(&s_ns[1], i + 1);
    }
  }
  __syncthreads();  // barrier init visible before any wait
  mbar_wait(bar, 0);
  // carries: X[cs_s + k] += C[s-1][k] for boundaries s = 1..K-1
  for (int e = tid; e < (K - 1) * PADC * n0; e += nthr) {
    const int r = e / n0, i = e - r * n0;  // r = (s-1)*(P+1) + k
    const int sb = r / PADC + 1, k = r - (sb - 1) * PADC;
    const int c = __ldg(g0g + seg[1 + sb]) + k;
    X[static_cast<std::int64_t>(c) * zl + i] += C[static_cast<std::int64_t>(r) * zl + i];
  }
  __syncthreads();
  double* Pb = a.P + blk.poff;
#if MFB_S2_NL > 1
  // NL lines per thread (rln_pass): a thread's lines are T apart
  constexpr int NL = MFB_S2_NL;
  RLFinalN<NL> fin{};
  int lo[NL];
  {  // G1^-1 along the rows (line i: X[.][i], stride zl)
    const int T = (n0 + NL - 1) / NL;
    for (int i = tid; i < T; i += nthr) {
#pragma unroll
      for (int j = 0; j < NL; ++j) lo[j] = i + j * T < n0 ? j * T : 0;
      rln_pass<P, NL, false>(X + i, lo, zl, n1, f1 + P * W, fin);
      rln_pass<P, NL, false>(X + i + (n1 - 1) * zl, lo, -zl, n1, b1 + P * W, fin);
    }
  }
  __syncthreads();
  {  // G0^-1 along the columns (line c: X[c][.], stride 1), P_b and the L-inf from the backward pass
    const int T = (n1 + NL - 1) / NL;
    for (int c = tid; c < T; c += nthr) {
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int cj = c + j * T < n1 ? c + j * T : c;
        lo[j] = (cj - c) * zl;
        fin.dst[j] = Pb + static_cast<std::int64_t>(n0 - 1) * n1 + cj;
        fin.line_shared[j] = sf1[cj] != 0;
      }
      double* xc = X + static_cast<std::int64_t>(c) * zl;
      rln_pass<P, NL, false>(xc, lo, 1, n0, f0 + P * W, fin);
      fin.dstride = -n1;
      fin.t_lo = n0 - s_ns[1];  // step t is axis-0 index n0 - 1 - t
      fin.t_hi = n0 - s_ns[0];
      rln_pass<P, NL, true>(xc + (n0 - 1), lo, -1, n0, b0 + P * W, fin);
    }
  }
#else
  RLFinal fin{};
  // G1^-1 along the rows (thread per row; stride zl)
  for (int i = tid; i < n0; i += nthr) {
    rl_pass<P, false>(X + i, zl, n1, f1 + P * W, fin);
    rl_pass<P, false>(X + i + (n1 - 1) * zl, -zl, n1, b1 + P * W, fin);
  }
  __syncthreads();
  // G0^-1 along the columns (thread per column); the backward pass writes
  // P_b[i][c] (coalesced over the warp's columns) and the L-inf over
  // non-shared controls.
  for (int c = tid; c < n1; c += nthr) {
    double* xc = X + static_cast<std::int64_t>(c) * zl;
    rl_pass<P, false>(xc, 1, n0, f0 + P * W, fin);
    fin.dst = Pb + static_cast<std::int64_t>(n0 - 1) * n1 + c;
    fin.dstride = -n1;
    fin.t_lo = n0 - s_ns[1];  // step t is axis-0 index n0 - 1 - t
    fin.t_hi = n0 - s_ns[0];
    fin.line_shared = sf1[c] != 0;
    rl_pass<P, true>(xc + (n0 - 1), -1, n0, b0 + P * W, fin);
  }
#endif
  unsigned long long lmax = fin.lmax;
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_xor_sync(kFullMask, lmax, o);
    lmax = lmax > t2 ? lmax : t2;
  }
  if (lane == 0) s_red[warp] = lmax;
  __syncthreads();
  if (tid == 0) {
    unsigned long long mx = 0ull;
    for (int w2 = 0; w2 < nw; ++w2) mx = mx > s_red[w2] ? mx : s_red[w2];
    if (mx) atomicMax(a.linf_int + bid, mx);
  }
}

// ---- k_solve2d_tw: the fused 2-D solve with twisted passes (MFADD_TWIST=1)
// Measured on C5 (round 2): 104 us as four inlined pass instantiations (a
// quarter of the issue slots waited for instructions), 119 us in this compact
// form (53 instructions per step against the plain kernel's 32, and the same
// 0.27 instructions per cycle per scheduler with twice the warps: a third of
// the warp time is spent at the per-pass barriers), against 70 us for
// k_solve2d.  Parity-green (the whole GPU suite passes with it), kept as a
// measurement knob, off by default.
// Same tile, carries and outputs as k_solve2d; a thread pair per line (top /
// bottom half).  All four passes of a thread (forward and backward, along the
// rows then along the columns) run the SAME compiled loop, tw_pass, whose
// per-pass differences are run-time values: the kernel body executes once per
// block, so its instruction footprint, not its branch count, is what matters
// (the four-instantiation form spent a quarter of its issue slots waiting for
// instructions).  Addresses are 32-bit shared-memory byte offsets.
__device__ __forceinline__ double lds_f64(std::uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void sts_f64(std::uint32_t addr, double v) {
  asm volatile("st.shared.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
template <int P>
struct TwPass {
  std::uint32_t x0;   // byte address of step 0's line element
  int dsb;            // byte stride per step (signed)
  int S;              // steps
  int e;              // steps [e, S) are stored to the side column (forward pass; S: none)
  const double* tab;  // the step table's row 0 (global memory, read through L1)
  std::uint32_t side; // byte address of the side column
  int sstb;           // its byte stride
  int use_init;       // backward pass: the first P values are init[]
  double init[P];
  double* gdst;       // final pass: global destination of step 0 (null: none)
  std::int64_t gstride;
  int t_lo, t_hi;     // steps that count towards the L-inf (empty: none)
};

template <int P>
__device__ __noinline__ unsigned long long tw_pass(const TwPass<P> q, unsigned long long lmax) {
  constexpr int U = RL<P>::U, W = RL<P>::W;
  const int S = q.S;
  double acc[P], zin[U], cf[W];
#pragma unroll
  for (int k = 0; k < P; ++k) {
    const double v = q.use_init ? q.init[k] : (k < S ? lds_f64(q.x0 + k * q.dsb) : 0.0);
    acc[k] = v * __ldg(q.tab + (k - P) * W + P);
  }
#pragma unroll
  for (int u = 0; u < U; ++u) zin[u] = P + u < S ? lds_f64(q.x0 + (P + u) * q.dsb) : 0.0;
#pragma unroll
  for (int h = 0; h < W / 2; ++h) {
    const double2 v = __ldg(reinterpret_cast<const double2*>(q.tab) + h);
    cf[2 * h] = v.x;
    cf[2 * h + 1] = v.y;
  }
  std::uint32_t xa = q.x0;           // line element of step t0
  const double* ta = q.tab + W;  // table row of step t0 + 1
  double* gp = q.gdst;
#pragma unroll 1
  for (int t0 = 0; t0 < S; t0 += U) {
    double znx[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int te = t0 + U + P + u;
      znx[u] = te < S ? lds_f64(xa + (U + P + u) * q.dsb) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      double cfn[W];
#pragma unroll
      for (int h = 0; h < W / 2; ++h) {  // the next step's row (tables are padded past the line)
        const double2 v = __ldg(reinterpret_cast<const double2*>(ta + u * W) + h);
        cfn[2 * h] = v.x;
        cfn[2 * h + 1] = v.y;
      }
      const double y = acc[u % P];
#pragma unroll
      for (int k = 1; k < P; ++k) acc[(u + k) % P] = fma(-cf[k - 1], y, acc[(u + k) % P]);
      acc[u % P] = fma(-cf[P - 1], y, zin[u] * cf[P]);
      const int t = t0 + u;
      if (t < S) {
        sts_f64(t < q.e ? xa + u * q.dsb : q.side + (t - q.e) * q.sstb, y);
        if (gp) {
          gp[u * q.gstride] = y;
          if (t >= q.t_lo && t < q.t_hi) {
            const unsigned long long bits = dbits_s(fabs(y));
            lmax = lmax > bits ? lmax : bits;
          }
        }
      }
#pragma unroll
      for (int k = 0; k < W; ++k) cf[k] = cfn[k];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) zin[u] = znx[u];
    xa += U * q.dsb;
    ta += U * W;
    if (gp) gp += U * q.gstride;
  }
  return lmax;
}

template <int P>
__global__ void __launch_bounds__(kSolve2dThreads) k_solve2d_tw(const FitArgs a) {
  pdl_enter();
  extern __shared__ __align__(128) double s2d[];
  __shared__ unsigned long long s_red[32];
  __shared__ int s_ns[2];  // non-shared axis-0 indices: [s_ns[0], s_ns[1])
  constexpr int PADC = P + 1, W = RL<P>::W, HALF = kSolve2dThreads / 2;
  const int bid = blockIdx.x;
  const BlockDev& blk = a.blocks[bid];
  const AxisProb p0 = a.probs[blk.ax[0]], p1 = a.probs[blk.ax[1]];
  const int n0 = p0.n, n1 = p1.n, zl = blk.zl;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int* seg = a.segtab + blk.ax[1] * kSegStride;
  const int K = seg[0];
  const int* g0g = a.g0 + p1.row_off;
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(s2d);
  double* X = s2d + 16;                                   // [n1][zl]
  double* C = X + static_cast<std::int64_t>(n1) * zl;     // [(K-1)(P+1)][zl] carries
  // the problems' table sets stay in global memory (k_rl_tables), read through L1
  const double* tab0 = a.rlt + static_cast<std::int64_t>(blk.ax[0]) * a.rlt_stride;
  const double* tab1 = a.rlt + static_cast<std::int64_t>(blk.ax[1]) * a.rlt_stride;
  double* mtop = C + static_cast<std::int64_t>(K - 1) * PADC * zl;  // side buffers [P][HALF]
  double* mbot = mtop + P * HALF;
  unsigned char* sf1 = reinterpret_cast<unsigned char*>(mbot + P * HALF);  // n1: axis-1 index shared
  const double* zb = a.Y + blk.zoff + static_cast<std::int64_t>(PADC) * zl;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, static_cast<unsigned>(n1) * zl * 8 + static_cast<unsigned>(K - 1) * PADC * zl * 8);
    int cs = 0;
    for (int sg = 0; sg < K; ++sg) {  // segment sg owns columns [cs_sg, cs_sg+1) in parity sg & 1
      const int ce = sg + 1 < K ? __ldg(g0g + seg[2 + sg]) : n1;
      const double* src = zb + (sg & 1) * a.zhalf + static_cast<std::int64_t>(cs) * zl;
      if (ce > cs) bulk_load_1d(X + static_cast<std::int64_t>(cs) * zl, src, static_cast<unsigned>(ce - cs) * zl * 8, bar);
      if (sg + 1 < K)  // its partial sums of the next segment's first P+1 columns
        bulk_load_1d(C + static_cast<std::int64_t>(sg) * PADC * zl, zb + (sg & 1) * a.zhalf + static_cast<std::int64_t>(ce) * zl,
                     static_cast<unsigned>(PADC) * zl * 8, bar);
      cs = ce;
    }
    s_ns[0] = n0;
    s_ns[1] = 0;
  }
  for (int c = tid; c < n1; c += nthr) sf1[c] = a.shared_flag[a.sflag_off[1] + p1.col_lo + c];
  __syncthreads();
  for (int i = tid; i < n0; i += nthr)
    if (!a.shared_flag[a.sflag_off[0] + p0.col_lo + i]) {
      atomicMin(&s_ns[0], i);
      atomicMax(&s_ns[1], i + 1);
    }
  __syncthreads();  // barrier init visible before any wait
  mbar_wait(bar, 0);
  // carries: X[cs_s + k] += C[s-1][k] for boundaries s = 1..K-1
  for (int e = tid; e < (K - 1) * PADC * n0; e += nthr) {
    const int r = e / n0, i = e - r * n0;  // r = (s-1)*(P+1) + k
    const int sb = r / PADC + 1, k = r - (sb - 1) * PADC;
    const int c = __ldg(g0g + seg[1 + sb]) + k;
    X[static_cast<std::int64_t>(c) * zl + i] += C[static_cast<std::int64_t>(r) * zl + i];
  }
  __syncthreads();
  const int role = tid >= HALF ? 1 : 0, pr = tid - role * HALF;
  const std::uint32_t xs = smem_u32(X), mts = smem_u32(mtop + pr), mbs = smem_u32(mbot + pr);
  double* Pb = a.P + blk.poff;
  unsigned long long lmax = 0ull;
  // phase 0: G1^-1 along the rows (line i: X[.][i], stride zl);
  // phase 1: G0^-1 along the columns (line c: X[c][.], stride 1), whose
  // backward passes write P_b[i][c] and the L-inf over non-shared controls
#pragma unroll 1
  for (int ph = 0; ph < 2; ++ph) {
    const int n = ph ? n0 : n1, nl = ph ? n1 : n0;   // line length, line count
    const int stb = (ph ? 1 : zl) * 8;               // byte stride along a line
    const double* tb = ph ? tab0 : tab1;
    const int ta = tw_top(n, P), nb = tw_bot(n, P);
    const int rt = rl_rows(ta + P, P) * W, rb = rl_rows(nb + P, P) * W;
    const double* fwd = tb + (role ? 2 * rt : 0) + P * W;
    const double* bwd = tb + (role ? 2 * rt + rb : rt) + P * W;
    const double* sinv = tb + 2 * rt + 2 * rb;
    const int e = role ? nb : ta, S = e + P;
#pragma unroll 1
    for (int l0 = 0; l0 < nl; l0 += HALF) {
      const int l = l0 + pr;
      const bool act = l < nl;
      const std::uint32_t line = xs + static_cast<std::uint32_t>(act ? l : 0) * (ph ? zl * 8 : 8);
      TwPass<P> q;
      q.S = S;
      q.tab = fwd;
      q.side = role ? mbs : mts;
      q.sstb = HALF * 8;
      q.gdst = nullptr;
      q.gstride = 0;
      q.t_lo = q.t_hi = 0;
      // forward: top walks rows 0, 1, ..; bottom rows n-1, n-2, ..
      q.x0 = role ? line + static_cast<std::uint32_t>(n - 1) * stb : line;
      q.dsb = role ? -stb : stb;
      q.e = e;
      q.use_init = 0;
#pragma unroll
      for (int k = 0; k < P; ++k) q.init[k] = 0.0;
      if (act) lmax = tw_pass<P>(q, lmax);
      __syncthreads();
      if (act) {
        double r[P];
#pragma unroll
        for (int j = 0; j < P; ++j) r[j] = mtop[j * HALF + pr] + mbot[(P - 1 - j) * HALF + pr];  // row ta+j
        // x_M = S^-1 r; backward: top walks rows ta+P-1 down to 0, bottom
        // rows ta up to n-1; the first P steps are the middle rows in the
        // pass's own order
#pragma unroll
        for (int i = 0; i < P; ++i) {
          double sacc = 0.0;
#pragma unroll
          for (int j = 0; j < P; ++j) sacc = fma(__ldg(sinv + i * P + j), r[j], sacc);
          q.init[role ? i : P - 1 - i] = sacc;
        }
        q.use_init = 1;
        q.tab = bwd;
        q.e = S;
        q.x0 = line + static_cast<std::uint32_t>(role ? ta : ta + P - 1) * stb;
        q.dsb = role ? stb : -stb;
        if (ph) {
          q.gdst = Pb + static_cast<std::int64_t>(role ? ta : ta + P - 1) * n1 + l;
          q.gstride = role ? n1 : -n1;
          if (!sf1[l]) {  // step t <-> row ta + t (bottom) / ta + P - 1 - t (top)
            q.t_lo = role ? s_ns[0] - ta : ta + P - s_ns[1];
            q.t_hi = role ? s_ns[1] - ta : ta + P - s_ns[0];
          }
        }
        lmax = tw_pass<P>(q, lmax);
      }
      __syncthreads();
    }
  }
  const int lane = tid & 31, warp = tid >> 5, nw = nthr >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_xor_sync(kFullMask, lmax, o);
    lmax = lmax > t2 ? lmax : t2;
  }
  if (lane == 0) s_red[warp] = lmax;
  __syncthreads();
  if (tid == 0) {
    unsigned long long mx = 0ull;
    for (int w2 = 0; w2 < nw; ++w2) mx = mx > s_red[w2] ? mx : s_red[w2];
    if (mx) atomicMax(a.linf_int + bid, mx);
  }
}

// ------------------------------------------- fused 3-D solve (CTA per slab)
// D = 3 with all three passes as pure contractions (FitArgs::fuse3d): after
// k_last_contract_tma the block's right-hand side Z = Q_b x0 R0 x1 R1 x2 R2 is
// n0 n1 n2 values in the layout Z[c][l], l = i0 n1 + i1 (column pitch zl).  A
// CTA takes the slab i0 in [i0a, i0b) of one block (FitArgs::s3_slab indices;
// C4: 36^3 controls per block, slabs of 6 = 61 KB), pulls its n2 column runs
// in with 1-D bulk copies into X[c][ls] (pitch s3_zs), and applies G2^-1 along
// c (a thread per line ls) and G1^-1 along i1 (a thread per (i0, c)) with the
// right-looking passes of k_solve2d (lsq.cpp:59-60 on each axis; the axis
// operators commute).  With several slabs per block the axis-1 backward pass
// writes P_b and the axis-0 solve follows on the held lattices
// (k_axis0_backsub / k_axis0_solve_part, which also take the L-inf).  When the
// whole block is one slab, G0^-1 along i0 (a thread per (i1, c)) runs here
// too, its backward pass writing P_b and the per-block L-inf over non-shared
// controls (solver.cpp:97-101).  Replaces the middle pass's in-place solve on
// T2 and k_last_solve (strided walks over HBM-resident intermediates).
constexpr int kSolve3dMaxThreads = 640;
// Lines per thread of k_solve3d's passes (FitArgs::s3_nl): 4 where the grid
// fills the GPU many times over (C4: 3072 slabs; 271 vs 320 us for the
// last-axis group), 1 where CTAs are scarce (C3: 512 slabs; 62 vs 81 us).

// Shared memory: the slab tile, the segment carries, two step-table slots
// (each a forward + backward table of the largest extent: axis 2's and axis
// 1's tables arrive with the tile, axis 0's replaces axis 2's during the
// axis-1 phase) and the shared-index flags.
__host__ __device__ inline size_t solve3d_smem_bytes(int n0, int n1, int n2, int zs, int P, int kseg) {
  const int W = (P + 2) & ~1;
  const int nm = n0 > n1 ? (n0 > n2 ? n0 : n2) : (n1 > n2 ? n1 : n2);
  return 128 + (static_cast<size_t>(n2) * zs + static_cast<size_t>(kseg > 1 ? kseg - 1 : 0) * (P + 1) * zs +
                4 * static_cast<size_t>(rl_rows(nm, P)) * W) *
                   8 +
         static_cast<size_t>(n0 + n1 + n2 + 16);
}

template <int P, int NL>
__global__ void __launch_bounds__((kSolve3dMaxThreads / NL + 31) / 32 * 32) k_solve3d(const FitArgs a) {
  pdl_enter();
  extern __shared__ __align__(128) double s2d[];
  __shared__ unsigned long long s_red[32];
  __shared__ int s_ns[2];  // non-shared axis-0 indices: [s_ns[0], s_ns[1])
  constexpr int PADC = P + 1, W = RL<P>::W;
  const int bid = blockIdx.x;
  const BlockDev& blk = a.blocks[bid];
  const AxisProb p0 = a.probs[blk.ax[0]], p1 = a.probs[blk.ax[1]], p2 = a.probs[blk.ax[2]];
  const int n0 = p0.n, n1 = p1.n, n2 = p2.n, zl = blk.zl, zs = a.s3_zs;
  const int i0a = static_cast<int>(blockIdx.y) * a.s3_slab;
  if (i0a >= n0) return;
  const int i0b = i0a + a.s3_slab < n0 ? i0a + a.s3_slab : n0;
  const int S0 = i0b - i0a, L = S0 * n1, l_off = i0a * n1;
  const bool whole = a.s3_nslab == 1;  // the block is one slab: axis 0 is solved here too
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int* seg = a.segtab + blk.ax[2] * kSegStride;
  const int K = seg[0];
  const int* g0g = a.g0 + p2.row_off;
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(s2d);
  double* X = s2d + 16;                                   // [n2][zs]
  double* C = X + static_cast<std::int64_t>(n2) * zs;     // [(K-1)(P+1)][zs] carries
  const int slot = 2 * rl_rows(a.max_n0 > a.max_n1 ? (a.max_n0 > a.max_n2 ? a.max_n0 : a.max_n2)
                                                     : (a.max_n1 > a.max_n2 ? a.max_n1 : a.max_n2), P) * W;
  double* f2 = C + static_cast<std::int64_t>(K - 1) * PADC * zs;  // slot 0: axis 2, later axis 0
  double* b2 = f2 + rl_rows(n2, P) * W;
  double* f0 = f2;
  double* b0 = f0 + rl_rows(n0, P) * W;
  double* f1 = f2 + slot;                                         // slot 1: axis 1
  double* b1 = f1 + rl_rows(n1, P) * W;
  unsigned char* sf0 = reinterpret_cast<unsigned char*>(f1 + slot);  // n0: axis-0 index shared
  unsigned char* sf1 = sf0 + n0;
  unsigned char* sf2 = sf1 + n1;
  const double* zb = a.Y + blk.zoff + static_cast<std::int64_t>(PADC) * zl + l_off;
  // bytes of one column run, rounded up to a 16-B multiple (an odd line count
  // copies one more value: inside Z's column pitch and the tile's)
  const unsigned run = static_cast<unsigned>((L + 1) & ~1) * 8;
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
    unsigned bytes = static_cast<unsigned>(n2 + (K - 1) * PADC) * run;
    bytes += 2 * static_cast<unsigned>((rl_rows(n1, P) + rl_rows(n2, P)) * W) * 8;
    mbar_arrive_expect_tx(bar, bytes);
    s_ns[0] = n0;
    s_ns[1] = 0;
  }
  __syncthreads();  // barrier init visible before the copies are issued by other threads
  {
    // column c's run comes from the parity buffer of the segment that owns it;
    // carry column (s, k) = segment s-1's partial sums of column cs_s + k
    for (int c = tid; c < n2 + (K - 1) * PADC; c += nthr) {
      if (c < n2) {
        int own = 0;
        for (int s2 = 1; s2 < K; ++s2)
          if (c >= __ldg(g0g + seg[1 + s2])) own = s2;
        bulk_load_1d(X + static_cast<std::int64_t>(c) * zs, zb + (own & 1) * a.zhalf + static_cast<std::int64_t>(c) * zl, run, bar);
      } else {
        const int r = c - n2, sb = r / PADC + 1, k = r - (sb - 1) * PADC;
        const int col = __ldg(g0g + seg[1 + sb]) + k;
        bulk_load_1d(C + static_cast<std::int64_t>(r) * zs, zb + ((sb - 1) & 1) * a.zhalf + static_cast<std::int64_t>(col) * zl, run, bar);
      }
    }
  }
  stage_rl_tables<P>(a, p1, blk.ax[1], f1, b1, bar, tid, nthr);
  stage_rl_tables<P>(a, p2, blk.ax[2], f2, b2, bar, tid, nthr);
  for (int c = tid; c < n1; c += nthr) sf1[c] = a.shared_flag[a.sflag_off[1] + p1.col_lo + c];
  for (int c = tid; c < n2; c += nthr) sf2[c] = a.shared_flag[a.sflag_off[2] + p2.col_lo + c];
  for (int i = tid; i < n0; i += nthr) {
    const unsigned char f = a.shared_flag[a.sflag_off[0] + p0.col_lo + i];
    sf0[i] = f;
    if (!f) {
      atomicMin(&s_ns[0], i);
      atomicMax(&s_ns[1], i + 1);
    }
  }
  __syncthreads();
  mbar_wait(bar, 0);
  // carries: X[cs_s + k] += C[s-1][k] for boundaries s = 1..K-1
  for (int e = tid; e < (K - 1) * PADC * L; e += nthr) {
    const int r = e / L, i = e - r * L;  // r = (s-1)*(P+1) + k
    const int sb = r / PADC + 1, k = r - (sb - 1) * PADC;
    const int c = __ldg(g0g + seg[1 + sb]) + k;
    X[static_cast<std::int64_t>(c) * zs + i] += C[static_cast<std::int64_t>(r) * zs + i];
  }
  __syncthreads();
  RLFinalN<NL> fin{};
  int lo[NL];
  // G2^-1 along c (line ls: X[.][ls], stride zs); a thread's lines are T apart
  {
    const int T = (L + NL - 1) / NL;
    for (int l = tid; l < T; l += nthr) {
#pragma unroll
      for (int j = 0; j < NL; ++j) lo[j] = l + j * T < L ? j * T : 0;
      rln_pass<P, NL, false>(X + l, lo, zs, n2, f2 + P * W, fin);
      rln_pass<P, NL, false>(X + l + (n2 - 1) * zs, lo, -zs, n2, b2 + P * W, fin);
    }
  }
  __syncthreads();
  if (whole) {  // axis 0's tables over axis 2's, behind the axis-1 phase
    if (tid == 0) {
      fence_proxy_async();
      mbar_arrive_expect_tx(bar + 1, 2 * static_cast<unsigned>(rl_rows(n0, P) * W) * 8);
    }
    stage_rl_tables<P>(a, p0, blk.ax[0], f0, b0, bar + 1, tid, nthr);
  }
  // G1^-1 along i1 (line (i0, c), c fastest: X[c][i0 n1 + .], stride 1).
  // Several slabs: the backward pass writes P_b[i0][i1][c] (coalesced over
  // the warp's c).
  double* Pb = a.P + blk.poff;
  {
    const int NQ = S0 * n2, T = (NQ + NL - 1) / NL;
    for (int q0 = tid; q0 < T; q0 += nthr) {
      double* x = nullptr;
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int q = q0 + j * T < NQ ? q0 + j * T : q0;
        const int i0r = q / n2, c = q - i0r * n2;
        double* xj = X + static_cast<std::int64_t>(c) * zs + i0r * n1;
        if (j == 0) x = xj;
        lo[j] = static_cast<int>(xj - x);
        fin.dst[j] = Pb + (static_cast<std::int64_t>(i0a + i0r) * n1 + (n1 - 1)) * n2 + c;
        fin.line_shared[j] = true;  // (the L-inf is taken by the axis-0 solve)
      }
      rln_pass<P, NL, false>(x, lo, 1, n1, f1 + P * W, fin);
      if (whole) {
        rln_pass<P, NL, false>(x + (n1 - 1), lo, -1, n1, b1 + P * W, fin);
      } else {
        fin.dstride = -n2;
        fin.t_lo = fin.t_hi = 0;
        rln_pass<P, NL, true>(x + (n1 - 1), lo, -1, n1, b1 + P * W, fin);
      }
    }
  }
  if (!whole) return;
  __syncthreads();
  mbar_wait(bar + 1, 0);
  // G0^-1 along i0 (thread per (i1, c), c fastest; stride n1); the backward
  // pass writes P_b[i0][i1][c] and the L-inf over non-shared controls
  {
    const int NQ = n1 * n2, T = (NQ + NL - 1) / NL;
    for (int q0 = tid; q0 < T; q0 += nthr) {
      double* x = nullptr;
#pragma unroll
      for (int j = 0; j < NL; ++j) {
        const int q = q0 + j * T < NQ ? q0 + j * T : q0;
        const int i1 = q / n2, c = q - i1 * n2;
        double* xj = X + static_cast<std::int64_t>(c) * zs + i1;
        if (j == 0) x = xj;
        lo[j] = static_cast<int>(xj - x);
        fin.dst[j] = Pb + (static_cast<std::int64_t>(n0 - 1) * n1 + i1) * n2 + c;
        fin.line_shared[j] = (sf1[i1] | sf2[c]) != 0;
      }
      rln_pass<P, NL, false>(x, lo, n1, n0, f0 + P * W, fin);
      fin.dstride = -static_cast<std::int64_t>(n1) * n2;
      fin.t_lo = n0 - s_ns[1];  // step t is axis-0 index n0 - 1 - t
      fin.t_hi = n0 - s_ns[0];
      rln_pass<P, NL, true>(x + (n0 - 1) * n1, lo, -n1, n0, b0 + P * W, fin);
    }
  }
  unsigned long long lmax = fin.lmax;
  const int lane = tid & 31, warp = tid >> 5, nw = (nthr + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_xor_sync(kFullMask, lmax, o);
    lmax = lmax > t2 ? lmax : t2;
  }
  if (lane == 0) s_red[warp] = lmax;
  __syncthreads();
  if (tid == 0) {
    unsigned long long mx = 0ull;
    for (int w2 = 0; w2 < nw; ++w2) mx = mx > s_red[w2] ? mx : s_red[w2];
    if (mx) atomicMax(a.linf_int + bid, mx);
  }
}

// ------------------------------- axis-0 solve on shared-memory slabs (D = 3)
// After k_solve3d's slabs, P_b holds G2^-1 G1^-1 Z; this kernel applies G0^-1
// along i0 (lsq.cpp:59-60 on axis 0).  A CTA takes the slab i1 in [i1a, i1b) of
// one block: for every i0 the values P_b[i0][i1a..i1b)[.] are one contiguous
// run, copied (coalesced loads) into X[i0][r], r = (i1 - i1a) n2 + c.  The
// passes walk i0 with the tile's row pitch (a warp's lines are consecutive r:
// conflict-free); the backward pass writes P_b back in place (coalesced) and
// takes the per-block L-inf over non-shared controls (solver.cpp:97-101).
// Replaces k_axis0_backsub / k_axis0_solve_part, whose threads walk the
// HBM-resident lattice with a stride of n1 n2 values.
__host__ __device__ inline size_t axis0_slab_smem_bytes(int n0, int lines, int P) {
  const int W = (P + 2) & ~1;
  return 128 + (static_cast<size_t>(n0) * ((lines + 1) & ~1) + 2 * static_cast<size_t>(rl_rows(n0, P)) * W) * 8 + 64;
}

template <int P, int NL>
__global__ void __launch_bounds__((kSolve3dMaxThreads / NL + 31) / 32 * 32) k_axis0_slab(const FitArgs a) {
  pdl_enter();
  extern __shared__ __align__(128) double s2d[];
  __shared__ unsigned long long s_red[32];
  __shared__ int s_ns[2];  // non-shared axis-0 indices: [s_ns[0], s_ns[1])
  constexpr int W = RL<P>::W;
  const int bid = blockIdx.x;
  const BlockDev& blk = a.blocks[bid];
  const AxisProb p0 = a.probs[blk.ax[0]], p1 = a.probs[blk.ax[1]], p2 = a.probs[blk.ax[2]];
  const int n0 = p0.n, n1 = p1.n, n2 = p2.n;
  const int i1a = static_cast<int>(blockIdx.y) * a.a0_slab;
  if (i1a >= n1) return;
  const int i1b = i1a + a.a0_slab < n1 ? i1a + a.a0_slab : n1;
  const int L = (i1b - i1a) * n2, zr = a.a0_zr;
  const int tid = threadIdx.x, nthr = blockDim.x;
  std::uint64_t* bar = reinterpret_cast<std::uint64_t*>(s2d);
  double* X = s2d + 16;  // [n0][zr]
  double* f0 = X + static_cast<std::int64_t>(n0) * zr;
  double* b0 = f0 + rl_rows(n0, P) * W;
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
    mbar_arrive_expect_tx(bar, 2 * static_cast<unsigned>(rl_rows(n0, P) * W) * 8);
    s_ns[0] = n0;
    s_ns[1] = 0;
  }
  stage_rl_tables<P>(a, p0, blk.ax[0], f0, b0, bar, tid, nthr);
  double* Pb = a.P + blk.poff + static_cast<std::int64_t>(i1a) * n2;
  const std::int64_t grow = static_cast<std::int64_t>(n1) * n2;  // P_b values per i0
  {  // tile load: 8-byte asynchronous copies, all of a thread's in flight at once
     // (P_b rows are only 8-B aligned in general, and the CTA has few threads:
     // plain loads spent 45% of the kernel waiting on their round trips)
    const std::uint32_t xs = smem_u32(X);
    for (int i0 = 0; i0 < n0; ++i0)
      for (int r = tid; r < L; r += nthr)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(xs + static_cast<std::uint32_t>(i0 * zr + r) * 8u),
                     "l"(Pb + i0 * grow + r)
                     : "memory");
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  for (int i = tid; i < n0; i += nthr)
    if (!a.shared_flag[a.sflag_off[0] + p0.col_lo + i]) {
      atomicMin(&s_ns[0], i);
      atomicMax(&s_ns[1], i + 1);
    }
  __syncthreads();
  mbar_wait(bar, 0);
  RLFinalN<NL> fin{};
  int lo[NL];
  const int T = (L + NL - 1) / NL;
  for (int r0 = tid; r0 < T; r0 += nthr) {
#pragma unroll
    for (int j = 0; j < NL; ++j) {
      const int r = r0 + j * T < L ? r0 + j * T : r0;
      const int i1 = i1a + r / n2, c = r - (r / n2) * n2;
      lo[j] = r - r0;
      fin.dst[j] = Pb + static_cast<std::int64_t>(n0 - 1) * grow + r;
      fin.line_shared[j] = (a.shared_flag[a.sflag_off[1] + p1.col_lo + i1] | a.shared_flag[a.sflag_off[2] + p2.col_lo + c]) != 0;
    }
    rln_pass<P, NL, false>(X + r0, lo, zr, n0, f0 + P * W, fin);
    fin.dstride = -grow;
    fin.t_lo = n0 - s_ns[1];  // step t is axis-0 index n0 - 1 - t
    fin.t_hi = n0 - s_ns[0];
    rln_pass<P, NL, true>(X + r0 + static_cast<std::int64_t>(n0 - 1) * zr, lo, -zr, n0, b0 + P * W, fin);
  }
  unsigned long long lmax = fin.lmax;
  const int lane = tid & 31, warp = tid >> 5, nw = (nthr + 31) >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_xor_sync(kFullMask, lmax, o);
    lmax = lmax > t2 ? lmax : t2;
  }
  if (lane == 0) s_red[warp] = lmax;
  __syncthreads();
  if (tid == 0) {
    unsigned long long mx = 0ull;
    for (int w2 = 0; w2 < nw; ++w2) mx = mx > s_red[w2] ? mx : s_red[w2];
    if (mx) atomicMax(a.linf_int + bid, mx);
  }
}

template <template <int> class F, class... Args>
int dispatch_p(int p, Args&&... args) {
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

// The solve stage after the last-axis contraction (FitArgs::fuse3d / fuse2d);
// returns the launches made.
template <int P>
struct SolveStageLaunch {
  static int run(const FitArgs& a, int kseg, cudaStream_t s) {
    if (a.fuse3d) {
      const size_t sm3 = solve3d_smem_bytes(a.max_n0, a.max_n1, a.max_n2, a.s3_zs, P, kseg);
      const int nl = a.s3_nl >= 4 ? 4 : 1;
      const int thr3 = std::max(64, ((a.solve3d_threads + nl - 1) / nl + 31) / 32 * 32);
      if (nl == 4) {
        cudaFuncSetAttribute(k_solve3d<P, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm3));
        launch_pdl(k_solve3d<P, 4>, dim3(a.nblocks, a.s3_nslab), dim3(thr3), sm3, s, a);
      } else {
        cudaFuncSetAttribute(k_solve3d<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm3));
        launch_pdl(k_solve3d<P, 1>, dim3(a.nblocks, a.s3_nslab), dim3(thr3), sm3, s, a);
      }
      if (a.s3_nslab > 1 && a.a0_slab > 0) {  // the axis-0 solve on i1 slabs
        const int lines = a.a0_slab * a.max_n2;
        const size_t sma = axis0_slab_smem_bytes(a.max_n0, lines, P);
        const int thra = std::max(64, ((std::min(lines, kSolve3dMaxThreads) + nl - 1) / nl + 31) / 32 * 32);
        const dim3 ga(a.nblocks, (a.max_n1 + a.a0_slab - 1) / a.a0_slab);
        if (nl == 4) {
          cudaFuncSetAttribute(k_axis0_slab<P, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sma));
          launch_pdl(k_axis0_slab<P, 4>, ga, dim3(thra), sma, s, a);
        } else {
          cudaFuncSetAttribute(k_axis0_slab<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sma));
          launch_pdl(k_axis0_slab<P, 1>, ga, dim3(thra), sma, s, a);
        }
        return 2;
      }
      return 1;
    }
    const size_t sm2 = solve2d_smem_bytes(a.max_n0, a.max_n1, a.max_zl, P, kseg, a.tw2d != 0);
    if (a.tw2d) {
      cudaFuncSetAttribute(k_solve2d_tw<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm2));
      launch_pdl(k_solve2d_tw<P>, dim3(a.nblocks), dim3(kSolve2dThreads), sm2, s, a);
      return 1;
    }
    cudaFuncSetAttribute(k_solve2d<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm2));
    launch_pdl(k_solve2d<P>, dim3(a.nblocks), dim3(kSolve2dThreads), sm2, s, a);
    return 1;
  }
};

}  // namespace

int launch_solve_stage(int degree, const FitArgs& a, int kseg, cudaStream_t s) {
  return dispatch_p<SolveStageLaunch>(degree, a, kseg, s);
}

namespace {
template <int P>
struct RlTablesLaunch {
  static int run(const CholArgs& a, double* rlt, std::int64_t stride, cudaStream_t s, bool tw) {
    if (a.nfactor == 0) return 0;
    k_rl_tables<P><<<a.nfactor, 256, 0, s>>>(a, rlt, stride, tw ? 1 : 0);
    return 1;
  }
};
template <int P>
struct RlDoubles {
  static std::int64_t run(int n, bool tw) {
    const std::int64_t plain = 2 * static_cast<std::int64_t>(rl_rows(n, P)) * RL<P>::W;
    return tw && tw_ok(n, P) ? std::max<std::int64_t>(plain, tw_table_doubles(n, P)) : plain;
  }
};
}  // namespace

int launch_rl_tables(int degree, const CholArgs& a, double* rlt, std::int64_t stride, cudaStream_t s, bool tw) {
  return dispatch_p<RlTablesLaunch>(degree, a, rlt, stride, s, tw);
}
std::int64_t rl_table_doubles(int degree, int n, bool tw) {
  switch (degree) {
    case 1: return RlDoubles<1>::run(n, tw);
    case 2: return RlDoubles<2>::run(n, tw);
    case 3: return RlDoubles<3>::run(n, tw);
    case 4: return RlDoubles<4>::run(n, tw);
    case 5: return RlDoubles<5>::run(n, tw);
    case 6: return RlDoubles<6>::run(n, tw);
    case 7: return RlDoubles<7>::run(n, tw);
    case 8: return RlDoubles<8>::run(n, tw);
    case 9: return RlDoubles<9>::run(n, tw);
    default: return 0;
  }
}

size_t axis0_slab_smem(int degree, int n0, int lines) {
  const size_t b = axis0_slab_smem_bytes(n0, lines, degree);
  return b <= 227 * 1024 - 512 ? b : 0;
}

size_t solve3d_smem(int degree, int n0, int n1, int n2, int zs, int kseg) {
  const size_t b = solve3d_smem_bytes(n0, n1, n2, zs, degree, kseg);
  return b <= 227 * 1024 - 512 ? b : 0;
}

size_t solve2d_smem(int degree, int n0, int n1, int zl, int kseg, bool tw) {
  const size_t b = solve2d_smem_bytes(n0, n1, zl, degree, kseg, tw);
  return b <= 227 * 1024 - 512 ? b : 0;
}


}  // namespace mfb
