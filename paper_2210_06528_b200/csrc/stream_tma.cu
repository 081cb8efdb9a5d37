// TMA-pipelined streaming passes of the B200 MFA encode path (sm_100a).
//
//  k_fit_axis0_tma   axis-0 fit pass (lsq.cpp:57-61 on axis 0): the HBM-bound
//                    read of every block's input box Q_loc.
//  k_decode_tma      decode of the global lattice over the whole input grid
//                    + error field + L2^2/Linf partials (solver.cpp:298-328).
//  k_last_contract_tma / k_last_solve, k_axis0_backsub / k_axis0_solve_part
//                    the last-axis contraction and the per-line solve walkers.
//  (the solve stage on shared-memory tiles -- k_solve2d, k_solve3d,
//   k_axis0_slab -- lives in solve_tma.cu)
//
// The two sweeps go over axis 0 axis 0 with one thread per trailing grid point.  Input rows are
// staged through an S-stage shared-memory ring filled by the Tensor Memory
// Accelerator (one elected thread issues a tensor-map tile load of R rows
// plus 1-D bulk copies of the matching basis rows; an mbarrier with expect_tx
// completes each stage).  The per-thread arithmetic is the register-window
// R^T contraction / decode of kernels.cu; see DESIGN.md §4.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "tma.cuh"

#ifdef MFB_DEBUG
__device__ int g_tma_debug_line = 0;
#define MFB_ASSERT(c, tag)                       \
  do {                                           \
    if (!(c)) {                                  \
      atomicCAS(&g_tma_debug_line, 0, __LINE__); \
      return;                                    \
    }                                            \
  } while (0)
// record-only variant for checks between barriers (no early return)
#define MFB_CHECK(c) \
  do {               \
    if (!(c)) atomicCAS(&g_tma_debug_line, 0, __LINE__); \
  } while (0)
#else
#define MFB_ASSERT(c, tag) \
  do {                     \
  } while (0)
#endif

namespace mfb {

namespace {

constexpr unsigned kFullMask = 0xffffffffu;

template <int V>
struct Int {
  static constexpr int value = V;
};

__device__ __forceinline__ unsigned long long dbits_s(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

struct StageLayout {
  int q_bytes;     // R * nthr * 8 (the full TMA box)
  int v_off;       // offset of basis values in the stage
  int g_off;       // offset of g0 ints
  int stage_bytes;
};

__host__ __device__ inline StageLayout stage_layout(int R, int nthr, int P) {
  StageLayout L;
  L.q_bytes = R * nthr * 8;
  L.v_off = (L.q_bytes + 127) / 128 * 128;
  L.g_off = L.v_off + R * (P + 1) * 8;
  L.stage_bytes = ((L.g_off + R * 4) + 127) / 128 * 128;
  return L;
}

// ---------------------------------------------------------------- fit axis 0
constexpr int kFitR = 8;  // rows per TMA stage (fit axis 0)

// MID: the middle axis of D = 3 (lsq.cpp:57-61 on axis 1).  Each (block, c0)
// slice of T1 = [n0][m1][pitch] is a 2-D box of m1 rows x m2 columns read
// through the same kind of tensor map; the sweep runs over j1 and writes
// T2[c0][c1][j2] (row pitch = the common last-axis pitch).
// BACK = false (axis 0 when FitArgs::defer_back): forward substitution only;
// the L^-T half of the axis-0 solve then runs on the held lattice at the end
// (k_axis0_backsub): the axis operators commute, so the result is the same up
// to rounding while T1 is written once instead of written, re-read, rewritten.
// FWD = false (axis 0 when FitArgs::defer_back == 2): contraction only, the
// whole G0^-1 solve runs on the held lattices at the end (no factor needed
// during the sweep, so the Gram/Cholesky setup overlaps it).
template <int P, int S, int NC, bool MID, bool BACK = true, bool FWD = true>
__global__ void __launch_bounds__(256) k_fit_axis0_tma(const FitArgs a, const __grid_constant__ CUtensorMap map,
                                                       const TmaGeom geo) {
  pdl_enter();
  constexpr int R = kFitR;
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  const int b = blockIdx.y;
  const BlockDev& blk = a.blocks[b];
  const AxisProb pr = a.probs[blk.ax[MID ? 1 : 0]];
  const int m = pr.m, n = pr.n;
  const int D = MID ? 2 : a.D;  // MID sweeps a 2-D slice
  const int c0s = MID ? static_cast<int>(blockIdx.z) : 0;
  if (MID && c0s >= a.probs[blk.ax[0]].n) return;
  const int m1 = MID ? a.probs[blk.ax[2]].m : a.probs[blk.ax[1]].m;  // columns of the swept box
  const int m2 = D == 3 ? a.probs[blk.ax[2]].m : 1;
  // Box: W inner columns (even, 16-B multiple) x [B1] x R rows.  TMA tile
  // loads need a 16-B aligned innermost start coordinate, so the box starts
  // at the even column at or below the block's first column and the column
  // map is shifted by that parity (geo.B2 = W, one spare column).  Each
  // thread owns NC adjacent box columns (NC = 2: one LDS.128 per row, the
  // broadcast basis values and loop bookkeeping shared by two columns).
  const int B1 = geo.B1, W = geo.B2;
  const int nbox = B1 * W;  // doubles per box row
  const int tile = blockIdx.x;
  const int tid = threadIdx.x;
  const AxisProb p1 = a.probs[blk.ax[MID ? 2 : 1]];
  // first box row: the block's first input row (field), or the slice's first
  // T1 row (T1 rows are [block][c0][j1], all of width pitch)
  const int in0 = MID ? static_cast<int>(blk.t1off / a.pitch_last) + c0s * m : static_cast<int>(pr.in_lo);
  int c_inner, c_mid, bcol;  // bcol: first box column of this thread (row-major over [B1][W])
  int j1[NC], j2[NC];
  bool act[NC];
  if (D == 2) {
    const int cols = W - 2;  // columns owned per tile
    if (tile * cols >= m1) return;
    const int first = (MID ? 0 : static_cast<int>(p1.in_lo)) + tile * cols;
    c_inner = first & ~1;
    c_mid = 0;
    bcol = NC * tid;
#pragma unroll
    for (int e = 0; e < NC; ++e) {
      j1[e] = tile * cols + bcol + e - (first - c_inner);
      j2[e] = 0;
      act[e] = bcol + e < W && j1[e] >= tile * cols && j1[e] < tile * cols + cols && j1[e] < m1;
    }
  } else {
    if (tile * B1 >= m1) return;
    const int in2 = static_cast<int>(a.probs[blk.ax[2]].in_lo);
    c_inner = in2 & ~1;
    c_mid = static_cast<int>(p1.in_lo) + tile * B1;
    const int tpr = W / NC;  // threads per box row
    const int row = tid / tpr;
    bcol = row * W + NC * (tid - row * tpr);
#pragma unroll
    for (int e = 0; e < NC; ++e) {
      j1[e] = tile * B1 + row;
      j2[e] = NC * (tid - row * tpr) + e - (in2 - c_inner);
      act[e] = row < B1 && j1[e] < m1 && j2[e] >= 0 && j2[e] < m2;
    }
  }
  // output: T1[i0][m1][pitch] (D = 3), T1[i0][pitch] (D = 2), or for MID
  // T2[c0][c1][pitch]; dstr = the stride between consecutive output rows
  const std::int64_t pitch = a.pitch_last;
  double* dst[NC];
#pragma unroll
  for (int e = 0; e < NC; ++e) {
    const std::int64_t col = act[e] ? (D == 3 ? static_cast<std::int64_t>(j1[e]) * pitch + j2[e] : j1[e]) : 0;
    dst[e] = MID ? a.t2 + blk.t2off + static_cast<std::int64_t>(c0s) * n * pitch + col : a.t1 + blk.t1off + col;
  }
  const int* g0g = a.g0 + pr.row_off;
  const double* vg = a.vals + pr.row_off * (P + 1);
  const double* lt = a.ltab + pr.col_off * (2 * P + 1);

  const StageLayout SL = stage_layout(R, nbox, P);
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sm_raw + S * SL.stage_bytes);
  const int nchunks = (m + R - 1) / R;
  const unsigned tx_bytes = static_cast<unsigned>(SL.q_bytes + R * (P + 1) * 8 + R * 4);
  auto issue = [&](int c) {
    const int st = c % S;
    unsigned char* base = sm_raw + st * SL.stage_bytes;
    mbar_arrive_expect_tx(&bars[st], tx_bytes);
    if (D == 2)
      tma_load_2d(base, &map, c_inner, in0 + c * R, &bars[st]);
    else
      tma_load_3d(base, &map, c_inner, c_mid, in0 + c * R, &bars[st]);
    bulk_load_1d(base + SL.v_off, vg + static_cast<std::int64_t>(c) * R * (P + 1), R * (P + 1) * 8, &bars[st]);
    bulk_load_1d(base + SL.g_off, g0g + static_cast<std::int64_t>(c) * R, R * 4, &bars[st]);
  };
  if (tid == 0) {
    prefetch_tmap(&map);
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  // Cholesky coefficients of this block's axis-0 problem, staged in smem
  // with P+1 zero columns on both sides (fetches need no clamping; L1 is
  // mostly carved out for the TMA ring).
  double* s_lt = reinterpret_cast<double*>(sm_raw + S * SL.stage_bytes + 128);
  constexpr int LW = 2 * P + 1;
  if (FWD)
    for (int i = tid; i < (n + 2 * (P + 1)) * LW; i += blockDim.x) {
      const int cc = i / LW - (P + 1);
      s_lt[i] = (cc >= 0 && cc < n) ? __ldg(lt + static_cast<std::int64_t>(cc) * LW + (i - (i / LW) * LW)) : 0.0;
    }
  const double* slt = s_lt + (P + 1) * LW;  // slt[cc * LW + k], cc in [-(P+1), n+P]
  __syncthreads();
  if (tid == 0)
    for (int c = 0; c < S && c < nchunks; ++c) issue(c);

  // acc[e][u]: R^T q of column e's output column in slot u; yv[e][u]: its
  // forward-substitution value (y_{c-k} in slot (u - k) mod (P+1): no moves)
  double acc[NC][P + 1], yv[NC][P + 1];
#pragma unroll
  for (int e = 0; e < NC; ++e)
#pragma unroll
    for (int k = 0; k <= P; ++k) acc[e][k] = yv[e][k] = 0.0;
  int cbase = __ldg(g0g) < 0 ? __ldg(g0g) : 0;
  const std::int64_t dstr = D == 2 ? pitch : static_cast<std::int64_t>(m1) * pitch;  // output row stride
  // Column-ordered accumulation with static register slots (as in
  // k_last_contract_tma): output columns are visited in groups of P+1, slot
  // u = the unrolled loop index; before column c is completed, the run of
  // rows whose span starts at c is accumulated into slots (u + k) mod (P+1).
  double Lnx[P + 1];  // forward coefficients of column cbase, fetched one column ahead
  auto fetch_fwd = [&](int cc) {
    if (!FWD) return;
    const double* Lc = slt + (cc < -(P + 1) ? -(P + 1) : cc) * LW;
#pragma unroll
    for (int k = 0; k <= P; ++k) Lnx[k] = Lc[k];
  };
  fetch_fwd(cbase);
  std::int64_t yoff = static_cast<std::int64_t>(cbase) * dstr;  // T1 offset of output column cbase
  // row cursor over the TMA stages
  int c = 0, jl = 0, jn = 0, gnext = 0x7fffffff;
  const double* sq = nullptr;
  const double* sv = nullptr;
  const int* sg = nullptr;
  auto open_chunk = [&]() {
    const int st = c % S;
    const unsigned char* base = sm_raw + st * SL.stage_bytes;
    sq = reinterpret_cast<const double*>(base) + bcol;
    sv = reinterpret_cast<const double*>(base + SL.v_off);
    sg = reinterpret_cast<const int*>(base + SL.g_off);
    jn = (m - c * R) < R ? (m - c * R) : R;
    jl = 0;
    mbar_wait(&bars[st], (c / S) & 1);
    gnext = sg[0];
  };
  // the staged-row stride in a register (the compiler otherwise re-derives
  // it from the kernel parameters on every row)
  int nbox_r = nbox;
  asm volatile("" : "+r"(nbox_r));
  auto advance = [&]() {
    if (++jl < jn) {
      gnext = sg[jl];
      sq += nbox_r;  // this thread's column in the next staged row
      return;
    }
    __syncthreads();  // every column is done with chunk c: refill its stage
    if (tid == 0 && c + S < nchunks) {
      fence_proxy_async();
      issue(c + S);
    }
    if (++c < nchunks)
      open_chunk();
    else
      gnext = 0x7fffffff;
  };
  if (nchunks > 0) open_chunk();
  while (cbase < n) {
#pragma unroll
    for (int u = 0; u <= P; ++u) {
      while (gnext == cbase) {  // CTA-uniform
        if (NC == 1 && jl + 1 < jn && sg[jl + 1] == cbase) {  // two rows of the same column run (CTA-uniform)
          const double q0 = sq[0], q1 = sq[nbox_r];
          const double* vr = sv + jl * (P + 1);
#pragma unroll
          for (int k = 0; k <= P; ++k) {
            const double v0 = vr[k], v1 = vr[P + 1 + k];
            acc[0][(u + k) % (P + 1)] = fma(v1, q1, fma(v0, q0, acc[0][(u + k) % (P + 1)]));
          }
          ++jl;
          sq += nbox_r;
          advance();
          continue;
        }
        double q[NC];
        if (NC == 4) {
          const double2 qa = *reinterpret_cast<const double2*>(sq), qb = *reinterpret_cast<const double2*>(sq + 2);
          q[0] = qa.x;
          q[1 % NC] = qa.y;
          q[2 % NC] = qb.x;
          q[NC - 1] = qb.y;
        } else if (NC == 2) {
          const double2 q2 = *reinterpret_cast<const double2*>(sq);
          q[0] = q2.x;
          q[NC - 1] = q2.y;
        } else {
          q[0] = *sq;
        }
        const double* vr = sv + jl * (P + 1);
#pragma unroll
        for (int k = 0; k <= P; ++k) {
          const double v = vr[k];
#pragma unroll
          for (int e = 0; e < NC; ++e) acc[e][(u + k) % (P + 1)] = fma(v, q[e], acc[e][(u + k) % (P + 1)]);
        }
        advance();
      }
      if (cbase >= 0) {  // forward substitution of column cbase (< n), or just R^T q
#pragma unroll
        for (int e = 0; e < NC; ++e) {
          if (FWD) {
            double sacc = acc[e][u];
#pragma unroll
            for (int k = P; k >= 1; --k) sacc = fma(-Lnx[k], yv[e][(u + P + 1 - k) % (P + 1)], sacc);
            const double y = sacc * Lnx[0];
            if (act[e]) dst[e][yoff] = y;
            yv[e][u] = y;
          } else if (act[e]) {
            dst[e][yoff] = acc[e][u];
          }
        }
      }
      yoff += dstr;
#pragma unroll
      for (int e = 0; e < NC; ++e) acc[e][u] = 0.0;
      fetch_fwd(++cbase);
      if (cbase >= n) break;
    }
  }
  if (!BACK) return;
  // Back substitution in place, y values prefetched PF columns ahead.  PF is a
  // multiple of P: x_{c+k} sits in the static slot (u - k) mod P of xw.
  bool any = false;
#pragma unroll
  for (int e = 0; e < NC; ++e) any = any || act[e];
  if (!any) return;
  constexpr int PF = P * ((16 / NC + P - 1) / P);
  double yr[NC][PF];
#pragma unroll
  for (int u = 0; u < PF; ++u)
#pragma unroll
    for (int e = 0; e < NC; ++e)
      yr[e][u] = (act[e] && n - 1 - u >= 0) ? dst[e][static_cast<std::int64_t>(n - 1 - u) * dstr] : 0.0;
  double xw[NC][P];
#pragma unroll
  for (int e = 0; e < NC; ++e)
#pragma unroll
    for (int k = 0; k < P; ++k) xw[e][k] = 0.0;
  double Lb[P + 1];  // backward coefficients of the current column, fetched ahead
  auto fetch_bwd = [&](int cc) {
    const double* Lc = slt + cc * LW;  // cc >= -1
    Lb[0] = Lc[0];
#pragma unroll
    for (int k = 1; k <= P; ++k) Lb[k] = Lc[P + k];
  };
  fetch_bwd(n - 1);
  for (int c0 = n - 1; c0 >= 0; c0 -= PF) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int cc = c0 - u;
      if (cc >= 0) {
        const int cn = cc - PF;
        const double Lb0 = Lb[0];
        double Lk[P + 1];
#pragma unroll
        for (int k = 1; k <= P; ++k) Lk[k] = Lb[k];
        fetch_bwd(cc - 1);
#pragma unroll
        for (int e = 0; e < NC; ++e) {
          double sacc = yr[e][u];
          yr[e][u] = (act[e] && cn >= 0) ? dst[e][static_cast<std::int64_t>(cn) * dstr] : 0.0;
#pragma unroll
          for (int k = P; k >= 1; --k) sacc = fma(-Lk[k], xw[e][(u - k + PF) % P], sacc);
          const double x = sacc * Lb0;
          if (act[e]) dst[e][static_cast<std::int64_t>(cc) * dstr] = x;
          xw[e][u % P] = x;
        }
      }
    }
  }
}

// ---------------------------------------------------------------- fit last axis
// The last-axis pass (lsq.cpp:57-61 on axis D-1) in two kernels:
//
//  k_last_contract_tma  Z = R^T y per line (collocation.cpp:46-54), each line
//                       split into up to kMaxSeg row segments so that
//                       lines x segments threads stream the input (4x the
//                       parallelism of one thread per line).  Segment s owns
//                       the columns below the next segment's first column
//                       cs_{s+1} = g0(js_{s+1}); its partial sums for columns
//                       cs_{s+1} .. cs_{s+1}+P go to a carry buffer.
//  k_last_solve         per line: add the carries, forward and back
//                       substitution with the banded Cholesky factor
//                       (lsq.cpp:59-60), write P, per-block max |P| over
//                       non-shared controls.
//
// Input boxes: 16 columns x LT lines, SWIZZLE_128B (16-B chunk k of line t at
// chunk k ^ (t & 7): the per-thread LDS.128 of two columns is conflict-free),
// plus the chunk's basis rows by 1-D bulk copies, in an S-stage TMA ring.
constexpr int kLastCW = 16;
#ifndef MFB_LAST_S
#define MFB_LAST_S 2
#endif
constexpr int kLastS = MFB_LAST_S;  // TMA ring stages of the last-axis contraction

__host__ __device__ inline int last_stage_bytes(int LT, int P) {
  return ((LT * 128 + kLastCW * (P + 1) * 8 + kLastCW * 4) + 1023) / 1024 * 1024;
}

template <int P>
__global__ void __launch_bounds__(256) k_last_contract_tma(const FitArgs a, const __grid_constant__ CUtensorMap map,
                                                           const int LT) {
  pdl_enter();
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  constexpr int S = kLastS, CW = kLastCW, PADC = P + 1;
  const int D = a.D, d = D - 1;
  const int b = blockIdx.y, sgi = blockIdx.z;
  const BlockDev& blk = a.blocks[b];  // by reference: ax[] is indexed at run time
  const int pid = blk.ax[d];
  const int* seg = a.segtab + pid * kSegStride;
  const int K = seg[0];
  if (sgi >= K) return;
  const AxisProb pr = a.probs[pid];
  std::int64_t L = 1;
  for (int k = 0; k < d; ++k) L *= a.probs[blk.ax[k]].n;
  const std::int64_t l0 = static_cast<std::int64_t>(blockIdx.x) * LT;
  if (l0 >= L) return;
  const int tid = threadIdx.x;
  const bool active = l0 + tid < L;
  const int js = seg[1 + sgi], je = seg[2 + sgi];
  const int* g0g = a.g0 + pr.row_off;
  const double* vg = a.vals + pr.row_off * (P + 1);
  const int row0 = static_cast<int>((D == 2 ? blk.t1off : blk.t2off) / a.pitch_last + l0);

  const int SB = last_stage_bytes(LT, P);
  const int v_off = LT * 128, g_off = v_off + CW * (P + 1) * 8;
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sm_raw + S * SB);
  const int c_first = js / CW, nchunks = (je + CW - 1) / CW - c_first;
  const unsigned tx_bytes = static_cast<unsigned>(LT * 128 + CW * (P + 1) * 8 + CW * 4);
  auto issue = [&](int c) {  // c: chunk index within the segment
    const int st = c % S;
    unsigned char* base = sm_raw + st * SB;
    const int col = (c_first + c) * CW;
    mbar_arrive_expect_tx(&bars[st], tx_bytes);
    tma_load_2d(base, &map, col, row0, &bars[st]);
    bulk_load_1d(base + v_off, vg + static_cast<std::int64_t>(col) * (P + 1), CW * (P + 1) * 8, &bars[st]);
    bulk_load_1d(base + g_off, g0g + col, CW * 4, &bars[st]);
  };
  if (tid == 0) {
    prefetch_tmap(&map);
    for (int st = 0; st < S; ++st) mbar_init(&bars[st], 1);
    fence_mbar_init();
    for (int c = 0; c < S && c < nchunks; ++c) issue(c);
  }
  __syncthreads();

  // Column-ordered accumulation with static register slots: columns are
  // visited in groups of P+1 (slot u = column mod P+1, the unrolled loop
  // index), and before column c is flushed the run of rows whose span starts
  // at c (g0 == c) is accumulated into slots (u + k) mod (P+1).  All register
  // indices are compile-time constants.  Columns go to this segment's parity
  // buffer at padded index c + P + 1 (a store through an incrementing pointer).
  double acc[P + 1];
#pragma unroll
  for (int k = 0; k <= P; ++k) acc[k] = 0.0;
  int cbase = __ldg(g0g + js);
  if (sgi == 0 && cbase > 0) cbase = 0;
  const int zl = blk.zl;
  double* zp = a.Y + (sgi & 1) * a.zhalf + blk.zoff + static_cast<std::int64_t>(cbase + PADC) * zl + l0 + tid;
  const int cend = sgi + 1 < K ? __ldg(g0g + je) + P + 1 : pr.n;
  const int swz = tid & 7;
  // row cursor over the TMA stages: chunk c, local row jl in [.., jhi)
  int c = 0, jl = 0, jhi = 0, gnext = 0x7fffffff;
  const unsigned char* lineb = nullptr;
  const int* sg = nullptr;
  const double* sv = nullptr;
  auto open_chunk = [&]() {
    const int st = c % S;
    const unsigned char* base = sm_raw + st * SB;
    sg = reinterpret_cast<const int*>(base + g_off);
    sv = reinterpret_cast<const double*>(base + v_off);
    lineb = base + tid * 128;
    const int jb = (c_first + c) * CW;
    jl = (js > jb ? js : jb) - jb;
    jhi = (je < jb + CW ? je : jb + CW) - jb;
    mbar_wait(&bars[st], (c / S) & 1);
    gnext = sg[jl];
  };
  auto advance = [&]() {
    if (++jl < jhi) {
      gnext = sg[jl];
      return;
    }
    __syncthreads();  // every line is done with chunk c: refill its stage
    if (tid == 0 && c + S < nchunks) {
      fence_proxy_async();
      issue(c + S);
    }
    if (++c < nchunks)
      open_chunk();
    else
      gnext = 0x7fffffff;
  };
  if (nchunks > 0) open_chunk();
  while (cbase < cend) {
#pragma unroll
    for (int u = 0; u <= P; ++u) {
      while (gnext == cbase) {  // CTA-uniform
        const double q = *reinterpret_cast<const double*>(lineb + ((((jl >> 1) ^ swz) << 4) | ((jl & 1) << 3)));
        const double* vr = sv + jl * (P + 1);
#pragma unroll
        for (int k = 0; k <= P; ++k) acc[(u + k) % (P + 1)] = fma(vr[k], q, acc[(u + k) % (P + 1)]);
        advance();
      }
      if (active) *zp = acc[u];
      zp += zl;
      acc[u] = 0.0;
      if (++cbase >= cend) break;
    }
  }
}

template <int P>
__global__ void __launch_bounds__(128) k_last_solve(const FitArgs a) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  __shared__ unsigned long long s_red[32];
  constexpr int LW = 2 * P + 1, XP = 33, PADC = P + 1;
  constexpr int U = P * ((8 + P - 1) / P);  // batch of columns, a multiple of P (static window slots)
  constexpr int F = (P + 2) & ~1;  // coefficients per column, padded to 16 B
  const int D = a.D, d = D - 1;
  const int b = blockIdx.y;
  const BlockDev& blk = a.blocks[b];
  const int pid = blk.ax[d];
  const AxisProb pr = a.probs[pid];
  const int n = pr.n;
  std::int64_t L = 1;
  for (int k = 0; k < d; ++k) L *= a.probs[blk.ax[k]].n;
  const std::int64_t l0 = static_cast<std::int64_t>(blockIdx.x) * blockDim.x;
  if (l0 >= L) return;
  const int nl = static_cast<int>((L - l0) < blockDim.x ? (L - l0) : blockDim.x);
  const int tid = threadIdx.x;
  const bool active = tid < nl;
  // smem: x staging | fwd coefficients | bwd coefficients | column codes | line flags
  double* s_x = reinterpret_cast<double*>(sm_raw);
  double* s_f = s_x + blockDim.x * XP;          // (n + 1) x F: [1/L(c,c), L(c,c-1) .. L(c,c-P)]
  double* s_b = s_f + (n + 1) * F;              // (n + 1) x F: [1/L(c,c), L(c+1,c) .. L(c+P,c)]
  unsigned char* s_code = reinterpret_cast<unsigned char*>(s_b + (n + 1) * F);  // n: owner parity | 2*(carry)
  unsigned char* s_sf = s_code + n;             // n: column shared along the last dim
  unsigned char* s_lead = s_sf + n;             // blockDim: line's lead index shared
  const double* lt = a.ltab + pr.col_off * LW;
  for (int i = tid; i < n * F; i += blockDim.x) {
    const int c = i / F, k = i - c * F;
    const double* Lc = lt + static_cast<std::int64_t>(c) * LW;
    s_f[i] = k == 0 ? Lc[0] : (k <= P ? Lc[k] : 0.0);
    s_b[i] = k == 0 ? Lc[0] : (k <= P ? Lc[P + k] : 0.0);
  }
  const int* seg = a.segtab + pid * kSegStride;
  const int K = seg[0];
  const int* g0g = a.g0 + pr.row_off;
  for (int c = tid; c < n; c += blockDim.x) {
    int own = 0, carry = 0;
    for (int s2 = 1; s2 < K; ++s2) {
      const int cs = __ldg(g0g + seg[1 + s2]);
      if (c >= cs) own = s2;
      if (c >= cs && c <= cs + P) carry = 1;
    }
    s_code[c] = static_cast<unsigned char>((own & 1) | (carry << 1));
    s_sf[c] = a.shared_flag[a.sflag_off[d] + pr.col_lo + c];
  }
  {
    bool lead_shared = false;
    std::int64_t r = l0 + tid;
    for (int k = d - 1; k >= 0; --k) {
      const AxisProb pk = a.probs[blk.ax[k]];
      const std::int64_t ik = r % pk.n;
      r /= pk.n;
      if (active && a.shared_flag[a.sflag_off[k] + pk.col_lo + ik]) lead_shared = true;
    }
    s_lead[tid] = lead_shared ? 1 : 0;
  }
  __syncthreads();
  // the two parity buffers of this line, padded column 0
  const std::int64_t zbase = blk.zoff + static_cast<std::int64_t>(PADC) * blk.zl + l0 + tid;
  const double* z0 = a.Y + zbase;
  const double* z1 = a.Y + a.zhalf + zbase;
  double* yb = a.Y + a.zhalf * 2 + blk.poff + l0 + tid;  // y scratch Y2[c*L + l]
  auto zload = [&](int c) -> double {
    if (!active || c >= n) return 0.0;
    const unsigned code = s_code[c];
    const std::int64_t o = static_cast<std::int64_t>(c) * blk.zl;
    double z = (code & 1) ? z1[o] : z0[o];
    if (code & 2) z += (code & 1) ? z0[o] : z1[o];  // carry of the previous segment
    return z;
  };
  // forward substitution, U columns of Z in flight.  U is a multiple of P, so
  // y_{c-k} lives in the static slot (c - k) mod P of yw (no window moves).
  double yw[P];
#pragma unroll
  for (int k = 0; k < P; ++k) yw[k] = 0.0;
  double zn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) zn[u] = zload(u);
  double* yp = yb;
  for (int c0 = 0; c0 < n; c0 += U) {
    double z[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      z[u] = zn[u];
      zn[u] = zload(c0 + U + u);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = c0 + u;
      if (c < n) {
        const double2* Lc = reinterpret_cast<const double2*>(s_f + c * F);
        double cf[F];
#pragma unroll
        for (int h = 0; h < F / 2; ++h) {
          const double2 t = Lc[h];
          cf[2 * h] = t.x;
          cf[2 * h + 1] = t.y;
        }
        double sacc = z[u];
#pragma unroll
        for (int k = P; k >= 1; --k) sacc = fma(-cf[k], yw[(u - k + U) % P], sacc);
        const double y = sacc * cf[0];
        if (active) *yp = y;
        yp += L;
        yw[u % P] = y;
      }
    }
  }
  // back substitution; x staged through smem for coalesced P rows
  double* Pb = a.P + blk.poff + l0 * n;
  // back substitution from the last column down, U columns per batch (x_{c+k}
  // in static slot (n - 1 - c - k) mod P counted from the top); x staged
  // through smem in 32-column chunks for coalesced P rows.
  double xw[P];
#pragma unroll
  for (int k = 0; k < P; ++k) xw[k] = 0.0;
  unsigned long long lmax = 0ull;
  const double* ybp = yb + static_cast<std::int64_t>(n - 1) * L;  // y of column n-1-t at ybp - t*L
  double yn[U];
#pragma unroll
  for (int u = 0; u < U; ++u) yn[u] = (active && u < n) ? *(ybp - static_cast<std::int64_t>(u) * L) : 0.0;
  constexpr int XC = 32 / U * U;  // columns per staging chunk (multiple of U)
  for (int t0 = 0; t0 < n; t0 += XC) {  // t = n - 1 - c counts columns from the top
    for (int t1 = t0; t1 < t0 + XC && t1 < n; t1 += U) {
      double y[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        y[u] = yn[u];
        const int tn = t1 + U + u;
        yn[u] = (active && tn < n) ? *(ybp - static_cast<std::int64_t>(tn) * L) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int t = t1 + u, c = n - 1 - t;
        if (t < n) {
          const double2* Lc = reinterpret_cast<const double2*>(s_b + c * F);
          double cf[F];
#pragma unroll
          for (int h = 0; h < F / 2; ++h) {
            const double2 v2 = Lc[h];
            cf[2 * h] = v2.x;
            cf[2 * h + 1] = v2.y;
          }
          double sacc = y[u];
#pragma unroll
          for (int k = P; k >= 1; --k) sacc = fma(-cf[k], xw[(u - k + U) % P], sacc);
          const double x = sacc * cf[0];
          xw[u % P] = x;
          s_x[tid * XP + (t - t0)] = x;
        }
      }
    }
    const int cn = (n - t0) < XC ? (n - t0) : XC;  // columns c = n-1-t0 down to n-t0-cn
    const int clo = n - t0 - cn;
    __syncthreads();
    // coalesced P rows; L-inf over non-shared controls (dp denominator)
    for (int e = tid; e < nl * 32; e += blockDim.x) {
      const int li = e >> 5, cl = e & 31;
      if (cl < cn) {  // column clo + cl was staged at t - t0 = cn - 1 - cl
        const double x = s_x[li * XP + (cn - 1 - cl)];
        Pb[static_cast<std::int64_t>(li) * n + clo + cl] = x;
        if (!a.defer_back && !s_lead[li] && !s_sf[clo + cl]) lmax = lmax > dbits_s(fabs(x)) ? lmax : dbits_s(fabs(x));
      }
    }
    __syncthreads();
  }
  // block-wide max of lmax -> linf_int[b]
  const int lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_xor_sync(kFullMask, lmax, o);
    lmax = lmax > t2 ? lmax : t2;
  }
  if (lane == 0) s_red[warp] = lmax;
  __syncthreads();
  if (tid == 0) {
    unsigned long long mx = 0ull;
    for (int w = 0; w < nwarps; ++w) mx = mx > s_red[w] ? mx : s_red[w];
    if (mx) atomicMax(a.linf_int + b, mx);
  }
}


// ------------------------------------------------------- deferred axis-0 L^-T
// x = L0^-T y along axis 0 of every held lattice P_b = [n0][rest] (rest =
// n1 [x n2]): thread per trailing index, in place, y values prefetched PF
// rows ahead, static window slots; then the per-block L-inf over non-shared
// controls (the dp denominator, solver.cpp:402-405).
constexpr int kBacksubThreads = 64;

template <int P>
__global__ void __launch_bounds__(kBacksubThreads) k_axis0_backsub(const FitArgs a) {
  extern __shared__ __align__(16) double s_lt0[];  // (n0 + 1) x (P+1) backward, then (n0 + 1) x (P+1) forward
  __shared__ unsigned long long s_red[32];
  constexpr int PF = P * ((32 + P - 1) / P);  // rows of y in flight per thread (latency-bound chain)
  const int b = blockIdx.y;
  const BlockDev& blk = a.blocks[b];
  const AxisProb p0 = a.probs[blk.ax[0]];
  const int n0 = p0.n, D = a.D;
  std::int64_t rest = 1;
  for (int k = 1; k < D; ++k) rest *= a.probs[blk.ax[k]].n;
  const std::int64_t t = static_cast<std::int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (static_cast<std::int64_t>(blockIdx.x) * blockDim.x >= rest) return;
  const bool active = t < rest;
  const double* lt = a.ltab + p0.col_off * (2 * P + 1);
  const bool fwd = a.defer_back == 2;  // full G0^-1 (forward then back), else L0^-T only
  double* s_f0 = s_lt0 + (n0 + 1) * (P + 1);  // [1/L(c,c), L(c,c-1) .. L(c,c-P)]
  for (int i = threadIdx.x; i < (n0 + 1) * (P + 1); i += blockDim.x) {
    const int c = i / (P + 1), k = i - c * (P + 1);
    s_lt0[i] = c < n0 ? lt[static_cast<std::int64_t>(c) * (2 * P + 1) + (k == 0 ? 0 : P + k)] : 0.0;
    if (fwd) s_f0[i] = c < n0 ? lt[static_cast<std::int64_t>(c) * (2 * P + 1) + k] : 0.0;
  }
  __syncthreads();
  // is this trailing index shared along dims >= 1?
  bool trail_shared = false;
  {
    std::int64_t r = active ? t : 0;
    for (int k = D - 1; k >= 1; --k) {
      const AxisProb pk = a.probs[blk.ax[k]];
      const std::int64_t ik = r % pk.n;
      r /= pk.n;
      if (a.shared_flag[a.sflag_off[k] + pk.col_lo + ik]) trail_shared = true;
    }
  }
  const unsigned char* sf0 = a.shared_flag + a.sflag_off[0] + p0.col_lo;
  double* col = a.P + blk.poff + (active ? t : 0);
  if (fwd) {  // y = L0^-1 w in place, w values prefetched PF rows ahead
    double wr[PF], yw[P];
#pragma unroll
    for (int u = 0; u < PF; ++u) wr[u] = (active && u < n0) ? col[static_cast<std::int64_t>(u) * rest] : 0.0;
#pragma unroll
    for (int k = 0; k < P; ++k) yw[k] = 0.0;
    for (int c0 = 0; c0 < n0; c0 += PF) {
#pragma unroll
      for (int u = 0; u < PF; ++u) {
        const int c = c0 + u;
        if (c < n0) {
          const double* Lc = s_f0 + c * (P + 1);
          double sacc = wr[u];
          const int cn = c + PF;
          wr[u] = (active && cn < n0) ? col[static_cast<std::int64_t>(cn) * rest] : 0.0;
#pragma unroll
          for (int k = P; k >= 1; --k) sacc = fma(-Lc[k], yw[(u - k + PF) % P], sacc);
          const double y = sacc * Lc[0];
          yw[u % P] = y;
          if (active) col[static_cast<std::int64_t>(c) * rest] = y;
        }
      }
    }
  }
  double yr[PF];
#pragma unroll
  for (int u = 0; u < PF; ++u) yr[u] = (active && n0 - 1 - u >= 0) ? col[static_cast<std::int64_t>(n0 - 1 - u) * rest] : 0.0;
  double xw[P];
#pragma unroll
  for (int k = 0; k < P; ++k) xw[k] = 0.0;
  unsigned long long lmax = 0ull;
  for (int c0 = n0 - 1; c0 >= 0; c0 -= PF) {
#pragma unroll
    for (int u = 0; u < PF; ++u) {
      const int c = c0 - u;
      if (c >= 0) {
        const double* Lc = s_lt0 + c * (P + 1);
        double sacc = yr[u];
        const int cn = c - PF;
        yr[u] = (active && cn >= 0) ? col[static_cast<std::int64_t>(cn) * rest] : 0.0;
#pragma unroll
        for (int k = P; k >= 1; --k) sacc = fma(-Lc[k], xw[(u - k + PF) % P], sacc);
        const double x = sacc * Lc[0];
        xw[u % P] = x;
        if (active) {
          col[static_cast<std::int64_t>(c) * rest] = x;
          if (!trail_shared && !sf0[c]) lmax = lmax > dbits_s(fabs(x)) ? lmax : dbits_s(fabs(x));
        }
      }
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_xor_sync(kFullMask, lmax, o);
    lmax = lmax > t2 ? lmax : t2;
  }
  if (lane == 0) s_red[warp] = lmax;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long mx = 0ull;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) mx = mx > s_red[w] ? mx : s_red[w];
    if (mx) atomicMax(a.linf_int + b, mx);
  }
}

// Partitioned form of the same solve (FitArgs::defer_back == 2: forward then
// back substitution with the axis-0 factor) for more parallelism per column:
// each column is cut into K segments, one thread each.  A segment is first
// solved with zero carry-in (y0); the true solution is y0 + F_k c_k where c_k
// holds the P values just before the segment and F_k (len x P) is the
// segment's response to unit carries, a property of the factor alone (built
// per CTA in smem).  Carries are propagated segment to segment with the last
// P rows of F_k (P x P), then every segment is corrected.  The back
// substitution runs the same scheme from the bottom.  P is L2-resident here,
// so the extra passes over it are cheap next to the latency they hide.
constexpr int kPartSeg = 4;
constexpr int kPartCols = 32;

template <int P>
__global__ void __launch_bounds__(kPartSeg * kPartCols) k_axis0_solve_part(const FitArgs a) {
  extern __shared__ __align__(16) double s_part[];
  __shared__ unsigned long long s_red[32];
  constexpr int K = kPartSeg, NCOL = kPartCols, LW = 2 * P + 1;
  const int b = blockIdx.y;
  const BlockDev& blk = a.blocks[b];
  const AxisProb p0 = a.probs[blk.ax[0]];
  const int n0 = p0.n, D = a.D;
  std::int64_t rest = 1;
  for (int k = 1; k < D; ++k) rest *= a.probs[blk.ax[k]].n;
  const std::int64_t col0 = static_cast<std::int64_t>(blockIdx.x) * NCOL;
  if (col0 >= rest) return;
  const int tid = threadIdx.x, cl = tid % NCOL, sg = tid / NCOL;
  const std::int64_t t = col0 + cl;
  const bool active = t < rest;
  // smem: factor (n0 x LW) | F responses (n0 x P) | B responses (n0 x P) | carries K x NCOL x P (x2)
  double* s_l = s_part;
  double* s_F = s_l + n0 * LW;
  double* s_B = s_F + n0 * P;
  double* s_tail = s_B + n0 * P;         // [K][NCOL][P]: last P values of each segment's zero-carry solve
  double* s_car = s_tail + K * NCOL * P;  // [K][NCOL][P]: carry into each segment
  double* s_x = s_car + K * NCOL * P;     // [n0][NCOL]: the CTA's column tile of P_b
  const double* lt = a.ltab + p0.col_off * LW;
  // global -> smem with 8 independent loads in flight per thread (the copies
  // are otherwise serialised on each load's latency)
  auto stage = [&](double* dst, auto src_of, int count) {
    constexpr int B = 8;
    for (int i0 = tid; i0 < count; i0 += B * static_cast<int>(blockDim.x)) {
      double v[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int i = i0 + u * static_cast<int>(blockDim.x);
        v[u] = i < count ? src_of(i) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int i = i0 + u * static_cast<int>(blockDim.x);
        if (i < count) dst[i] = v[u];
      }
    }
  };
  stage(s_l, [&](int i) { return __ldg(lt + i); }, n0 * LW);
  __syncthreads();
  auto seg_lo = [&](int k) { return static_cast<int>(static_cast<std::int64_t>(k) * n0 / K); };
  // response matrices: thread (k, j) for k = 1..K-1, j < P
  if (tid < (K - 1) * P) {
    const int k = 1 + tid / P, j = tid % P, lo = seg_lo(k), hi = seg_lo(k + 1);
    double w[P];  // w[m-1] = value at row c-m (carry unit vector e_j: row lo-1-j)
#pragma unroll
    for (int m = 0; m < P; ++m) w[m] = m == j ? 1.0 : 0.0;
    for (int c = lo; c < hi; ++c) {  // forward: y_c = -(sum_m L(c,c-m) y_{c-m}) / L(c,c)
      const double* Lc = s_l + c * LW;
      double sacc = 0.0;
#pragma unroll
      for (int m = P; m >= 1; --m) sacc = fma(-Lc[m], w[m - 1], sacc);
      const double y = sacc * Lc[0];
#pragma unroll
      for (int m = P - 1; m >= 1; --m) w[m] = w[m - 1];
      w[0] = y;
      s_F[c * P + j] = y;
    }
  } else if (tid >= 64 && tid < 64 + (K - 1) * P) {
    const int q = tid - 64, k = q / P, j = q % P, lo = seg_lo(k), hi = seg_lo(k + 1);  // k = 0..K-2
    double w[P];  // w[m-1] = value at row c+m (carry unit vector e_j: row hi+j)
#pragma unroll
    for (int m = 0; m < P; ++m) w[m] = m == j ? 1.0 : 0.0;
    for (int c = hi - 1; c >= lo; --c) {  // back: x_c = -(sum_m L(c+m,c) x_{c+m}) / L(c,c)
      const double* Lc = s_l + c * LW;
      double sacc = 0.0;
#pragma unroll
      for (int m = P; m >= 1; --m) sacc = fma(-Lc[P + m], w[m - 1], sacc);
      const double x = sacc * Lc[0];
#pragma unroll
      for (int m = P - 1; m >= 1; --m) w[m] = w[m - 1];
      w[0] = x;
      s_B[c * P + j] = x;
    }
  }
  // the column tile -> smem (independent coalesced loads), solved there, written back once
  double* Pt = a.P + blk.poff + col0;
  const int ncl = static_cast<int>(rest - col0 < NCOL ? rest - col0 : NCOL);
  stage(s_x, [&](int i) {
    const int c = i / NCOL, j = i - c * NCOL;
    return j < ncl ? Pt[static_cast<std::int64_t>(c) * rest + j] : 0.0;
  }, n0 * NCOL);
  __syncthreads();
  double* xs = s_x + cl;  // this thread's column: xs[c * NCOL]
  const int lo = seg_lo(sg), hi = seg_lo(sg + 1);
  // (1) forward, zero carry-in
  {
    double w[P];
#pragma unroll
    for (int m = 0; m < P; ++m) w[m] = 0.0;
    for (int c = lo; c < hi; ++c) {
      const double* Lc = s_l + c * LW;
      double sacc = xs[c * NCOL];
#pragma unroll
      for (int m = P; m >= 1; --m) sacc = fma(-Lc[m], w[m - 1], sacc);
      const double y = sacc * Lc[0];
#pragma unroll
      for (int m = P - 1; m >= 1; --m) w[m] = w[m - 1];
      w[0] = y;
      xs[c * NCOL] = y;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) s_tail[(sg * NCOL + cl) * P + m] = w[m];  // w[m] = y at row hi-1-m
  }
  __syncthreads();
  // (2) carries: c_0 = 0, c_{k+1}[m] = y0_k(hi-1-m) + sum_j F_k(hi-1-m, j) c_k[j]
  if (sg == 0) {
    double c[P];
#pragma unroll
    for (int m = 0; m < P; ++m) c[m] = 0.0;
    for (int k = 0; k + 1 < K; ++k) {
      const int hk = seg_lo(k + 1);
      double nc[P];
#pragma unroll
      for (int m = 0; m < P; ++m) {
        double v = s_tail[(k * NCOL + cl) * P + m];
        if (k > 0)
#pragma unroll
          for (int j = 0; j < P; ++j) v = fma(s_F[(hk - 1 - m) * P + j], c[j], v);
        nc[m] = v;
      }
#pragma unroll
      for (int m = 0; m < P; ++m) {
        c[m] = nc[m];
        s_car[((k + 1) * NCOL + cl) * P + m] = nc[m];
      }
    }
  }
  __syncthreads();
  // (3) correct segments k >= 1 (y = y0 + F c), then (4) back, zero carry-in
  {
    double cf[P];
#pragma unroll
    for (int j = 0; j < P; ++j) cf[j] = sg > 0 ? s_car[(sg * NCOL + cl) * P + j] : 0.0;
    double w[P];
#pragma unroll
    for (int m = 0; m < P; ++m) w[m] = 0.0;
    // a segment's back pass needs its own corrected y: fuse (3) into (4) bottom-up
    for (int c = hi - 1; c >= lo; --c) {
      double y = xs[c * NCOL];
      if (sg > 0)
#pragma unroll
        for (int j = 0; j < P; ++j) y = fma(s_F[c * P + j], cf[j], y);
      const double* Lc = s_l + c * LW;
      double sacc = y;
#pragma unroll
      for (int m = P; m >= 1; --m) sacc = fma(-Lc[P + m], w[m - 1], sacc);
      const double x = sacc * Lc[0];
#pragma unroll
      for (int m = P - 1; m >= 1; --m) w[m] = w[m - 1];
      w[0] = x;
      xs[c * NCOL] = x;
    }
#pragma unroll
    for (int m = 0; m < P; ++m) s_tail[(sg * NCOL + cl) * P + m] = w[m];  // w[m] = x0 at row lo+m
  }
  __syncthreads();
  // (5) back carries from the bottom: d_{K-1} = 0, d_{k-1}[m] = x0_k(lo_k+m) + sum_j B_k(lo_k+m, j) d_k[j]
  if (sg == 0) {
    double d[P];
#pragma unroll
    for (int m = 0; m < P; ++m) d[m] = 0.0;
    for (int k = K - 1; k >= 1; --k) {
      const int lk = seg_lo(k);
      double nd[P];
#pragma unroll
      for (int m = 0; m < P; ++m) {
        double v = s_tail[(k * NCOL + cl) * P + m];
        if (k < K - 1)
#pragma unroll
          for (int j = 0; j < P; ++j) v = fma(s_B[(lk + m) * P + j], d[j], v);
        nd[m] = v;
      }
#pragma unroll
      for (int m = 0; m < P; ++m) {
        d[m] = nd[m];
        s_car[((k - 1) * NCOL + cl) * P + m] = nd[m];
      }
    }
  }
  __syncthreads();
  // (6) correct segments k < K-1 (x = x0 + B d) and the L-inf of non-shared controls
  bool trail_shared = false;
  {
    std::int64_t r = active ? t : 0;
    for (int k = D - 1; k >= 1; --k) {
      const AxisProb pk = a.probs[blk.ax[k]];
      const std::int64_t ik = r % pk.n;
      r /= pk.n;
      if (a.shared_flag[a.sflag_off[k] + pk.col_lo + ik]) trail_shared = true;
    }
  }
  const unsigned char* sf0 = a.shared_flag + a.sflag_off[0] + p0.col_lo;
  unsigned long long lmax = 0ull;
  {
    double df[P];
#pragma unroll
    for (int j = 0; j < P; ++j) df[j] = sg < K - 1 ? s_car[(sg * NCOL + cl) * P + j] : 0.0;
    for (int c = lo; c < hi; ++c) {
      double x = xs[c * NCOL];
      if (sg < K - 1) {
#pragma unroll
        for (int j = 0; j < P; ++j) x = fma(s_B[c * P + j], df[j], x);
        xs[c * NCOL] = x;
      }
      if (active && !trail_shared && !sf0[c]) lmax = lmax > dbits_s(fabs(x)) ? lmax : dbits_s(fabs(x));
    }
  }
  __syncthreads();
  for (int i = tid; i < n0 * NCOL; i += blockDim.x) {
    const int c = i / NCOL, j = i - c * NCOL;
    if (j < ncl) Pt[static_cast<std::int64_t>(c) * rest + j] = s_x[i];
  }
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t2 = __shfl_xor_sync(kFullMask, lmax, o);
    lmax = lmax > t2 ? lmax : t2;
  }
  if (lane == 0) s_red[warp] = lmax;
  __syncthreads();
  if (tid == 0) {
    unsigned long long mx = 0ull;
    for (int w2 = 0; w2 < static_cast<int>(blockDim.x >> 5); ++w2) mx = mx > s_red[w2] ? mx : s_red[w2];
    if (mx) atomicMax(a.linf_int + b, mx);
  }
}

template <int P>
struct BacksubLaunch {
  static int run(const FitArgs& a, int max_n0, std::int64_t max_rest, cudaStream_t s) {
    static const bool no_part = std::getenv("MFADD_NO_PART") != nullptr;
    if (a.defer_back == 2 && !no_part && a.min_n0 >= kPartSeg * 2 * (P + 1)) {
      const size_t smem = (static_cast<size_t>(max_n0) * (2 * P + 1) + 2 * static_cast<size_t>(max_n0) * P +
                           2 * static_cast<size_t>(kPartSeg) * kPartCols * P + static_cast<size_t>(max_n0) * kPartCols) *
                          sizeof(double);
      cudaFuncSetAttribute(k_axis0_solve_part<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      dim3 grid(static_cast<unsigned>((max_rest + kPartCols - 1) / kPartCols), a.nblocks);
      k_axis0_solve_part<P><<<grid, kPartSeg * kPartCols, smem, s>>>(a);
      return 1;
    }
    const size_t smem = 2 * static_cast<size_t>(max_n0 + 1) * (P + 1) * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_axis0_backsub<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dim3 grid(static_cast<unsigned>((max_rest + kBacksubThreads - 1) / kBacksubThreads), a.nblocks);
    k_axis0_backsub<P><<<grid, kBacksubThreads, smem, s>>>(a);
    return 1;
  }
};

// ---------------------------------------------------------------- decode
// WIN (D = 3): the host has checked that every CTA's axis-2 window fits, so
// only the shared-window form is compiled (no (P+1)^2 per-thread plane
// registers: higher occupancy).
template <int P, int D, int S, int MB = 1, bool ERR = true, bool WIN = false>
__global__ void __launch_bounds__(256, MB) k_decode_tma(const DecodeSweepArgs a, const __grid_constant__ CUtensorMap map,
                                                    const TmaGeom geo) {
  pdl_enter();
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  __shared__ double s_red[64];
  constexpr int R = kFitR;  // same row stages as the fit pass
  const int B1 = geo.B1, B2 = geo.B2;
  const int nthr = B1 * B2;
  const int tid = threadIdx.x;
  // trailing tile
  const int tx = blockIdx.x % a.ntile2, ty = blockIdx.x / a.ntile2;
  int j1, j2;
  if (D == 2) {
    j1 = tx * B2 + tid;
    j2 = 0;
  } else {
    j1 = ty * B1 + tid / B2;
    j2 = tx * B2 + tid % B2;
  }
  const bool active = D == 2 ? j1 < a.M1 : (j1 < a.M1 && j2 < a.M2);
  const int y0 = a.ybeg + blockIdx.y * a.H;
  const int y1 = (y0 + a.H) < a.yend ? (y0 + a.H) : a.yend;
  const std::int64_t Tr = static_cast<std::int64_t>(a.M1) * a.M2;
  const std::int64_t t = static_cast<std::int64_t>(j1) * a.M2 + j2;
  // trailing basis of this thread (fixed for the whole sweep)
  double w1[P + 1], w2[P + 1];
  int g1 = 0, g2 = 0;
  const int j1c = active ? j1 : 0, j2c = active ? j2 : 0;
  if (D == 2) {
    g1 = __ldg(a.g0_1 + j1c);
#pragma unroll
    for (int k = 0; k <= P; ++k) w1[k] = __ldg(a.v_1 + static_cast<std::int64_t>(j1c) * (P + 1) + k);
  } else {
    g1 = __ldg(a.g0_1 + j1c);
    g2 = __ldg(a.g0_2 + j2c);
#pragma unroll
    for (int k = 0; k <= P; ++k) {
      w1[k] = __ldg(a.v_1 + static_cast<std::int64_t>(j1c) * (P + 1) + k);
      w2[k] = __ldg(a.v_2 + static_cast<std::int64_t>(j2c) * (P + 1) + k);
    }
  }
  const std::int64_t N12 = static_cast<std::int64_t>(a.N1) * a.N2;
  auto plane = [&](int ai) -> double {  // trailing contraction of control plane ai
    const double* L0 = a.lattice + static_cast<std::int64_t>(ai) * N12;
    double s = 0.0;
    if (D == 2) {
#pragma unroll
      for (int k = 0; k <= P; ++k) s = fma(w1[k], __ldg(L0 + g1 + k), s);
    } else {
#pragma unroll
      for (int k1 = 0; k1 <= P; ++k1) {
        const double* Lr = L0 + static_cast<std::int64_t>(g1 + k1) * a.N2 + g2;
        double r = 0.0;
#pragma unroll
        for (int k2 = 0; k2 <= P; ++k2) r = fma(w2[k2], __ldg(Lr + k2), r);
        s = fma(w1[k1], r, s);
      }
    }
    return s;
  };

  const StageLayout SL = stage_layout(R, nthr, P);
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sm_raw + S * SL.stage_bytes);
  // chunks start at a 4-row boundary (16-B aligned bulk copies of the int row
  // table); rows before y0 in the first chunk are skipped
  const int ya = y0 & ~3;
  const int nchunks = y1 > y0 ? (y1 - ya + R - 1) / R : 0;
  const unsigned tx_bytes = static_cast<unsigned>(SL.q_bytes + R * (P + 1) * 8 + R * 4);
  const int c_inner = D == 2 ? tx * B2 : tx * B2;
  const int c_mid = D == 2 ? 0 : ty * B1;
  auto issue = [&](int c) {
    const int st = c % S;
    unsigned char* base = sm_raw + st * SL.stage_bytes;
    mbar_arrive_expect_tx(&bars[st], tx_bytes);
    if (D == 2)
      tma_load_2d(base, &map, c_inner, ya + c * R, &bars[st]);
    else
      tma_load_3d(base, &map, c_inner, c_mid, ya + c * R, &bars[st]);
    bulk_load_1d(base + SL.v_off, a.v_0 + static_cast<std::int64_t>(ya + c * R) * (P + 1), R * (P + 1) * 8,
                 &bars[st]);
    bulk_load_1d(base + SL.g_off, a.g0_0 + ya + c * R, R * 4, &bars[st]);
  };
  if (tid == 0) {
    prefetch_tmap(&map);
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int c = 0; c < S && c < nchunks; ++c) issue(c);

  // Control-plane window in static register slots: plane a lives in slot
  // a mod (P+1).  Walking the planes in order (unrolled step u = slot of
  // plane abase), the run of rows whose window starts at abase is decoded
  // from slots (u + k) mod (P+1); advancing the window replaces slot u by
  // plane abase + P + 1, whose lattice values were fetched one step ahead.
  int abase = __ldg(a.g0_0 + y0);
  double Tw[P + 1];
#pragma unroll
  for (int k = 0; k <= P; ++k) Tw[k] = (active && !WIN) ? plane(abase + k) : 0.0;
  constexpr int NV = D == 2 ? (P + 1) : (WIN ? 1 : (P + 1) * (P + 1));
  double nxt[NV];
  auto fetch_plane = [&](int ai) {
    const int a2 = ai < a.N0 ? ai : a.N0 - 1;
    const double* L0 = a.lattice + static_cast<std::int64_t>(a2) * N12;
    if (D == 2) {
#pragma unroll
      for (int k = 0; k <= P; ++k) nxt[k] = __ldg(L0 + g1 + k);
    } else {
#pragma unroll
      for (int k1 = 0; k1 <= P; ++k1)
#pragma unroll
        for (int k2 = 0; k2 <= P; ++k2)
          nxt[(k1 * (P + 1) + k2) % NV] = __ldg(L0 + static_cast<std::int64_t>(g1 + k1) * a.N2 + g2 + k2);
    }
  };
  auto reduce_plane = [&]() -> double {
    double s = 0.0;
    if (D == 2) {
#pragma unroll
      for (int k = 0; k <= P; ++k) s = fma(w1[k], nxt[k], s);
    } else {
#pragma unroll
      for (int k1 = 0; k1 <= P; ++k1) {
        double r = 0.0;
#pragma unroll
        for (int k2 = 0; k2 <= P; ++k2) r = fma(w2[k2], nxt[(k1 * (P + 1) + k2) % NV], r);
        s = fma(w1[k1], r, s);
      }
    }
    return s;
  };
  // D = 3 with one row j1 per CTA (B1 == 1, C3/C4): every thread shares g1
  // and w1, so each control plane's axis-1 contraction is done once per CTA
  // for the tile's window of axis-2 columns (thread q of the window loads
  // P+1 values, coalesced), staged in shared memory (double-buffered by
  // plane), and each thread finishes with P+1 products: P+1 loads per plane
  // per thread instead of (P+1)^2.
  int g2base = 0, rw = 0;
  double* sR = reinterpret_cast<double*>(sm_raw + S * SL.stage_bytes + S * 8);
  if (D == 3 && B1 == 1) {
    const int jf = tx * B2, jl = (tx * B2 + B2 - 1) < a.M2 - 1 ? (tx * B2 + B2 - 1) : a.M2 - 1;
    g2base = __ldg(a.g0_2 + jf);
    rw = __ldg(a.g0_2 + jl) - g2base + P + 1;
  }
  const bool win = WIN || (D == 3 && B1 == 1 && rw <= geo.lt_cap && rw <= nthr);  // CTA-uniform
  double lv[P + 1];  // this thread's window column of the plane after next (raw lattice values)
  int rbuf = 0;
  auto fetch_window = [&](int ai) {
    const int a2 = ai < a.N0 ? ai : a.N0 - 1;
    if (tid < rw) {
      const double* L0 = a.lattice + static_cast<std::int64_t>(a2) * N12 + g2base + tid;
#pragma unroll
      for (int k1 = 0; k1 <= P; ++k1) lv[k1] = __ldg(L0 + static_cast<std::int64_t>(g1 + k1) * a.N2);
    }
  };
  // WIN: the CTA's axis-1-contracted window of every control plane its row
  // range touches, U[a - a_lo][t], staged once up front (independent loads,
  // no per-advance loads or barriers in the sweep)
  const int a_lo = WIN ? __ldg(a.g0_0 + y0) : 0;
  const int y1c = y1 > y0 ? y1 - 1 : y0;
  const int a_hi = WIN ? min(__ldg(a.g0_0 + y1c) + P, a.N0 - 1) : 0;
  const int na = a_hi - a_lo + 1;
  const int wo = g2 > g2base ? g2 - g2base : 0;  // (inactive threads: clamped, unused)
  bool wfits = true;
  if (WIN) {
    const bool fits = rw <= geo.lt_cap && na <= a.na_cap;  // host-sized exactly
    wfits = fits;
    if (fits && rw > 0) {
      const int tr = nthr / rw > 0 ? nthr / rw : 1;
      const int t = tid % rw, r0 = tid / rw;
      if (r0 < tr) {
        const double* Lc = a.lattice + g2base + t;
#pragma unroll 4
        for (int ai = r0; ai < na; ai += tr) {
          const double* L0 = Lc + static_cast<std::int64_t>(a_lo + ai) * N12;
          double r = 0.0;
#pragma unroll
          for (int k1 = 0; k1 <= P; ++k1) r = fma(w1[k1], __ldg(L0 + static_cast<std::int64_t>(g1 + k1) * a.N2), r);
          sR[ai * geo.lt_cap + t] = r;
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k <= P; ++k) {
      const double* Rg = sR + min(abase + k - a_lo, na - 1) * geo.lt_cap + wo;
      double sres = 0.0;
#pragma unroll
      for (int k2 = 0; k2 <= P; ++k2) sres = fma(w2[k2], Rg[k2], sres);
      Tw[k] = (active && fits) ? sres : 0.0;
    }
  }
  if (!WIN) {
    if (win)
      fetch_window(abase + P + 1);
    else if (active)
      fetch_plane(abase + P + 1);
  }
  double l2 = wfits ? 0.0 : __longlong_as_double(0x7ff8000000000000LL);  // NaN: never a silent wrong answer
  unsigned long long li = 0ull;  // L-inf as the bit pattern of |e| (ordered like the value)
  // error of the current row (ERR: the error field is stored); inactive
  // threads point at their clamped column and never store
  double* errp = ERR ? a.err + static_cast<std::int64_t>(y0) * Tr + (active ? t : 0) : nullptr;
  // row cursor over the TMA stages
  int c = 0, jl = 0, jn = 0, gnext = 0x7fffffff;
  const double* sq = nullptr;
  const double* sv = nullptr;
  const int* sg = nullptr;
  auto open_chunk = [&]() {
    const int st = c % S;
    const unsigned char* base = sm_raw + st * SL.stage_bytes;
    sq = reinterpret_cast<const double*>(base) + tid;
    sv = reinterpret_cast<const double*>(base + SL.v_off);
    sg = reinterpret_cast<const int*>(base + SL.g_off);
    const int yc = ya + c * R;
    jn = (y1 - yc) < R ? (y1 - yc) : R;
    jl = y0 > yc ? y0 - yc : 0;
    mbar_wait(&bars[st], (c / S) & 1);
    gnext = sg[jl];
  };
  auto advance = [&]() {
    if (++jl < jn) {
      gnext = sg[jl];
      return;
    }
    __syncthreads();  // every thread is done with chunk c: refill its stage
    if (tid == 0 && c + S < nchunks) {
      fence_proxy_async();
      issue(c + S);
    }
    if (++c < nchunks)
      open_chunk();
    else
      gnext = 0x7fffffff;
  };
  if (nchunks > 0) open_chunk();
  while (gnext != 0x7fffffff) {
#pragma unroll
    for (int u = 0; u <= P; ++u) {
      while (gnext == abase) {  // CTA-uniform
        const double* vr = sv + jl * (P + 1);
        double sd = 0.0;
#pragma unroll
        for (int k = 0; k <= P; ++k) sd = fma(vr[k], Tw[(u + k) % (P + 1)], sd);
        // no branches in the per-row body: inactive threads (box padding)
        // compute on their staged column, store nothing and count zero
        const double e = active ? sq[jl * nthr] - sd : 0.0;
        if (ERR) {
          if (active) *errp = e;
          errp += Tr;
        }
        l2 = fma(e, e, l2);
        const unsigned long long eb = dbits_s(e) & 0x7fffffffffffffffull;
        li = li > eb ? li : eb;
        advance();
      }
      if (gnext == 0x7fffffff) break;
      if (WIN) {  // plane abase + P + 1 replaces plane abase, from the staged windows
        const double* Rg = sR + min(abase + P + 1 - a_lo, na - 1) * geo.lt_cap + wo;
        double sres = 0.0;
#pragma unroll
        for (int k2 = 0; k2 <= P; ++k2) sres = fma(w2[k2], Rg[k2], sres);
        Tw[u] = active ? sres : 0.0;
        ++abase;
      } else if (win) {  // plane abase + P + 1 replaces plane abase, through the shared window
        double* R = sR + rbuf * geo.lt_cap;
        if (tid < rw) {
          double r = 0.0;
#pragma unroll
          for (int k1 = 0; k1 <= P; ++k1) r = fma(w1[k1], lv[k1], r);
          R[tid] = r;
        }
        __syncthreads();
        const double* Rg = R + (g2 > g2base ? g2 - g2base : 0);  // (inactive threads: clamped, unused)
        double sres = 0.0;
#pragma unroll
        for (int k2 = 0; k2 <= P; ++k2) sres = fma(w2[k2], Rg[k2], sres);
        Tw[u] = active ? sres : 0.0;
        rbuf ^= 1;
        ++abase;
        fetch_window(abase + P + 1);
      } else {
        Tw[u] = active ? reduce_plane() : 0.0;  // plane abase + P + 1 replaces plane abase
        ++abase;
        if (active) fetch_plane(abase + P + 1);
      }
    }
  }
  // CTA reduction -> partial[blockIdx]
  double lid = __longlong_as_double(static_cast<long long>(li));
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    l2 += __shfl_xor_sync(kFullMask, l2, off);
    lid = fmax(lid, __shfl_xor_sync(kFullMask, lid, off));
  }
  const int wid = tid >> 5;
  if ((tid & 31) == 0) {
    s_red[wid] = l2;
    s_red[32 + wid] = lid;
  }
  __syncthreads();
  if (tid == 0) {
    double sl = 0.0, sm2 = 0.0;
    for (int w = 0; w < (nthr + 31) / 32; ++w) {
      sl += s_red[w];
      sm2 = fmax(sm2, s_red[32 + w]);
    }
    const std::int64_t cta = static_cast<std::int64_t>(blockIdx.y) * gridDim.x + blockIdx.x;
    a.partial[2 * cta] = sl;
    a.partial[2 * cta + 1] = sm2;
  }
  // last CTA: fixed-order reduction of all partials into red2 (L2^2, L-inf)
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(a.ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const std::int64_t nparts = static_cast<std::int64_t>(gridDim.x) * gridDim.y;
  double pl = 0.0, pm = 0.0;
  for (std::int64_t i = tid; i < nparts; i += nthr) {
    pl += __ldcg(a.partial + 2 * i);
    pm = fmax(pm, __ldcg(a.partial + 2 * i + 1));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    pl += __shfl_xor_sync(kFullMask, pl, off);
    pm = fmax(pm, __shfl_xor_sync(kFullMask, pm, off));
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    s_red[wid] = pl;
    s_red[32 + wid] = pm;
  }
  __syncthreads();
  if (tid == 0) {
    double sl = 0.0, sm2 = 0.0;
    for (int w = 0; w < (nthr + 31) / 32; ++w) {
      sl += s_red[w];
      sm2 = fmax(sm2, s_red[32 + w]);
    }
    a.red2[0] = sl;
    a.red2[1] = sm2;
    *a.ticket = 0u;
  }
}

template <int P>
struct Axis0Launch {
  template <int S, int NC, bool MID = false>
  static void go(const FitArgs& a, const CUtensorMap& map, const TmaGeom& g, int ntiles, cudaStream_t s,
                 int zdim = 1) {
    const StageLayout SL = stage_layout(kFitR, g.B1 * g.B2, P);
    const size_t smem = static_cast<size_t>(S) * SL.stage_bytes + 128 + static_cast<size_t>(g.lt_cap) * 8;
    dim3 grid(ntiles, a.nblocks, zdim);
    if ((!MID && a.defer_back == 2) || (MID && a.fuse3d)) {  // contraction only: no factor table in smem
      const size_t smem_c = static_cast<size_t>(S) * SL.stage_bytes + 128;
      cudaFuncSetAttribute(k_fit_axis0_tma<P, S, NC, MID, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem_c));
      launch_pdl(k_fit_axis0_tma<P, S, NC, MID, false, false>, grid, dim3(g.B1 * g.B2 / NC), smem_c, s, a, map, g);
    } else if (!MID && a.defer_back) {
      cudaFuncSetAttribute(k_fit_axis0_tma<P, S, NC, MID, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      launch_pdl(k_fit_axis0_tma<P, S, NC, MID, false>, grid, dim3(g.B1 * g.B2 / NC), smem, s, a, map, g);
    } else {
      cudaFuncSetAttribute(k_fit_axis0_tma<P, S, NC, MID>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      launch_pdl(k_fit_axis0_tma<P, S, NC, MID>, grid, dim3(g.B1 * g.B2 / NC), smem, s, a, map, g);
    }
  }
  static int run(const FitArgs& a, const CUtensorMap& map, const TmaGeom& g, int ntiles, cudaStream_t s) {
    // NC = 2 (two columns per thread, one LDS.128 per row): slower on C5 (331 vs
    // 233 us: fewer resident warps), faster for D = 3 (C4 902 -> 798 us, C3 59.6 -> 55.5 us)
    static const int nc_env = std::getenv("MFADD_FIT_NC") ? std::atoi(std::getenv("MFADD_FIT_NC")) : 0;
    const int nc = nc_env > 0 ? nc_env : (a.D == 3 ? 2 : 1);
    if (nc == 1)
      g.S == 3 ? go<3, 1>(a, map, g, ntiles, s) : go<4, 1>(a, map, g, ntiles, s);
    else if (nc == 4 && g.B2 % 4 == 0 && a.D == 3)
      g.S == 3 ? go<3, 4>(a, map, g, ntiles, s) : go<4, 4>(a, map, g, ntiles, s);
    else
      g.S == 3 ? go<3, 2>(a, map, g, ntiles, s) : go<4, 2>(a, map, g, ntiles, s);
    return 1;
  }
};

template <int P>
struct DecodeSweepLaunch {
  template <int D, int S>
  static void go(const DecodeSweepArgs& a, const CUtensorMap& map, const TmaGeom& g, cudaStream_t s) {
    const StageLayout SL = stage_layout(kFitR, g.B1 * g.B2, P);
    const size_t smem = static_cast<size_t>(S) * SL.stage_bytes + S * 8 +
                        (D == 3 && a.win ? static_cast<size_t>(a.na_cap) : 2) * static_cast<size_t>(g.lt_cap) * 8;
    dim3 grid(a.ntile1 * a.ntile2, a.nrange);
    static const int mb = std::getenv("MFADD_DEC_MINB") ? std::atoi(std::getenv("MFADD_DEC_MINB")) : 1;
    if (mb >= 4) {
      cudaFuncSetAttribute(k_decode_tma<P, D, S, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      launch_pdl(k_decode_tma<P, D, S, 4>, grid, dim3(g.B1 * g.B2), smem, s, a, map, g);
      return;
    }
    if (D == 3 && a.win && a.err) {
      cudaFuncSetAttribute(k_decode_tma<P, D, S, 1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      launch_pdl(k_decode_tma<P, D, S, 1, true, true>, grid, dim3(g.B1 * g.B2), smem, s, a, map, g);
      return;
    }
    if (!a.err) {  // no error field: L2 / L-inf only
      cudaFuncSetAttribute(k_decode_tma<P, D, S, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(smem));
      launch_pdl(k_decode_tma<P, D, S, 1, false>, grid, dim3(g.B1 * g.B2), smem, s, a, map, g);
      return;
    }
    cudaFuncSetAttribute(k_decode_tma<P, D, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    launch_pdl(k_decode_tma<P, D, S>, grid, dim3(g.B1 * g.B2), smem, s, a, map, g);
  }
  static int run(const DecodeSweepArgs& a, const CUtensorMap& map, const TmaGeom& g, cudaStream_t s) {
    if (a.D == 2)
      g.S == 3 ? go<2, 3>(a, map, g, s) : go<2, 4>(a, map, g, s);
    else
      g.S == 3 ? go<3, 3>(a, map, g, s) : go<3, 4>(a, map, g, s);
    return 1;
  }
};

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

template <int P>
struct LastLaunch {
  static int run(const FitArgs& a, const CUtensorMap& map, int LT, int lt_cap, int kseg, cudaStream_t s) {
    const size_t smem = static_cast<size_t>(kLastS) * last_stage_bytes(LT, P) + 128;
    cudaFuncSetAttribute(k_last_contract_tma<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    dim3 grid((a.max_lines_last + LT - 1) / LT, a.nblocks, kseg);
    launch_pdl(k_last_contract_tma<P>, grid, dim3(LT), smem, s, a, map, LT);
    // the contraction needs no factor: the Gram/Cholesky side stream joins here
    if (a.join_event) cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(a.join_event), 0);
    if (a.fuse3d || a.fuse2d) return 1 + launch_solve_stage(P, a, kseg, s);  // solve_tma.cu
    constexpr int T2 = 64, F = (P + 2) & ~1;
    const int nmax = lt_cap / (2 * P + 1);  // max last-axis n (+ padding) from the L-table capacity
    const size_t smem2 = static_cast<size_t>(T2) * 33 * 8 + 2 * static_cast<size_t>(nmax + 1) * F * 8 +
                         2 * static_cast<size_t>(nmax) + T2;
    cudaFuncSetAttribute(k_last_solve<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem2));
    dim3 grid2((a.max_lines_last + T2 - 1) / T2, a.nblocks);
    k_last_solve<P><<<grid2, T2, smem2, s>>>(a);
    return 2;
  }
};

}  // namespace

int debug_fail_line_tma() {
  int line = 0;
#ifdef MFB_DEBUG
  cudaMemcpyFromSymbol(&line, g_tma_debug_line, sizeof(int));
#endif
  return line;
}

int launch_axis0_backsub(int degree, const FitArgs& a, int max_n0, std::int64_t max_rest, cudaStream_t s) {
  return dispatch_p<BacksubLaunch>(degree, a, max_n0, max_rest, s);
}

int launch_fit_last_tma(int degree, const FitArgs& a, const CUtensorMap& map, int LT, int lt_cap, int kseg,
                        cudaStream_t s) {
  return dispatch_p<LastLaunch>(degree, a, map, LT, lt_cap, kseg, s);
}

int launch_fit_axis0_tma(int degree, const FitArgs& a, const CUtensorMap& map, const TmaGeom& g, int ntiles,
                         cudaStream_t s) {
  return dispatch_p<Axis0Launch>(degree, a, map, g, ntiles, s);
}

namespace {
template <int P>
struct MidLaunch {
  static int run(const FitArgs& a, const CUtensorMap& map, const TmaGeom& g, int ntiles, int max_n0, cudaStream_t s) {
    static const int nc = std::getenv("MFADD_MID_NC") ? std::atoi(std::getenv("MFADD_MID_NC")) : 1;
    if (nc == 2)
      Axis0Launch<P>::template go<4, 2, true>(a, map, g, ntiles, s, max_n0);
    else
      Axis0Launch<P>::template go<4, 1, true>(a, map, g, ntiles, s, max_n0);
    return 1;
  }
};
}  // namespace

int launch_fit_mid_tma(int degree, const FitArgs& a, const CUtensorMap& map, const TmaGeom& g, int ntiles, int max_n0,
                       cudaStream_t s) {
  return dispatch_p<MidLaunch>(degree, a, map, g, ntiles, max_n0, s);
}

int launch_decode_tma(int degree, const DecodeSweepArgs& a, const CUtensorMap& map, const TmaGeom& g,
                      cudaStream_t s) {
  return dispatch_p<DecodeSweepLaunch>(degree, a, map, g, s);
}

}  // namespace mfb
