// residual_tma.cu — per-epoch block residuals of log_errors (record_epoch,
// solver.cpp:357-364 -> residual_error, lsq.cpp:66-85) in ONE pass over the
// blocks' input boxes after the epoch loop.
//
// The residuals never feed back into the iteration, so the solve keeps a
// snapshot of every epoch's shared controls (the region epoch kernel writes
// each shared copy's post-epoch value into snap[e] at its held-lattice
// offset; non-shared controls never change after the fit and are read from
// P).  This kernel then streams each block's input box once (TMA ring of R
// rows, as the decode sweep) and decodes it against EG epochs' lattices at a
// time, accumulating {sum e^2, max |e|} per epoch: Q_loc is read once instead
// of once per epoch.
//
// Thread per trailing point (D = 2: a column j1 of a column tile; D = 3: a
// column j2 of one row j1 per CTA), axis 0 swept with a window of P+1
// trailing-contracted control planes per epoch in static register slots.
// Before the sweep the CTA stages, for every control plane its rows touch,
// the lattice window of its points over the innermost axis (D = 3: already
// contracted along axis 1 with the CTA's common row j1) in shared memory,
// EG epochs at a time: one burst of independent loads, then the sweep
// streams Q through the TMA ring with no global-memory latency on its
// chain.  Per-CTA partials are reduced per (epoch, block) in a fixed order
// by k_res_reduce.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.cuh"
#include "tma.cuh"

namespace mfb {
namespace {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr int kResR = 8;  // rows per TMA stage
#ifndef MFB_RES_S
#define MFB_RES_S 3
#endif
constexpr int kResS = MFB_RES_S;  // TMA ring stages

struct ResStage {
  int q_bytes, v_off, g_off, stage_bytes;
};

__host__ __device__ inline ResStage res_stage(int nbox, int P) {
  ResStage L;
  L.q_bytes = kResR * nbox * 8;
  L.v_off = (L.q_bytes + 127) / 128 * 128;
  L.g_off = L.v_off + kResR * (P + 1) * 8;
  L.stage_bytes = ((L.g_off + kResR * 4) + 127) / 128 * 128;
  return L;
}

__host__ __device__ inline size_t res_tma_smem(int P, int W, int EG, int na_cap, int lt_cap, int S) {
  return static_cast<size_t>(S) * res_stage(W, P).stage_bytes + S * 8 + 8 +
         static_cast<size_t>(EG) * na_cap * lt_cap * 8;
}

// NG epoch groups: the CTA runs NG threads per point, each decoding EG / NG
// of the pass's epochs from the same staged rows (Q is still read once per
// pass; twice the warps per SM at half the registers per thread).
#ifndef MFB_RES_MAXREG
#define MFB_RES_MAXREG 128  // registers per thread of the one-thread-per-point form
#endif
template <int P, int D, int EG, int S, int NG>
__global__ void __maxnreg__(NG == 2 ? 84 : MFB_RES_MAXREG) k_residual_tma(const ResTmaArgs a, const __grid_constant__ CUtensorMap map) {
  extern __shared__ __align__(1024) unsigned char sm_raw[];
  __shared__ double s_red[2 * EG][16];
  const int b = blockIdx.y;
  const BlockDev blk = a.blocks[b];
  const AxisProb p0 = a.probs[blk.ax[0]], p1 = a.probs[blk.ax[1]];
  const AxisProb p2 = D == 3 ? a.probs[blk.ax[2]] : p1;
  const int m0 = p0.m, n0 = p0.n, m1 = p1.m, n1 = p1.n;
  const int m2 = D == 3 ? p2.m : 1, n2 = D == 3 ? p2.n : 1;
  const int W = a.W, tid = threadIdx.x, nthr = blockDim.x;
  constexpr int EGT = EG / NG;                   // epochs per thread
  const int Wt = nthr / NG;                      // threads per epoch group
  const int grp = tid / Wt, ct = tid - grp * Wt;  // epoch group, column thread
  const int ne = a.st ? a.st->iter + 1 : 1;  // epochs recorded (0 .. iter)
  // ---- this thread's point and the CTA's box origin
  const int tcol = blockIdx.x % a.ntc, rr = blockIdx.x / a.ntc;  // column tile, row range
  int j1, j2 = 0, c_inner, c_mid = 0;
  bool act, live;
  if (D == 2) {
    const int cols = W - 2;
    const int first = static_cast<int>(p1.in_lo) + tcol * cols;
    c_inner = first & ~1;  // 16-B aligned box start; the column map is shifted by its parity
    j1 = tcol * cols + ct - (first - c_inner);
    live = tcol * cols < m1;
    act = live && ct < W && j1 >= tcol * cols && j1 < tcol * cols + cols && j1 < m1;
  } else {
    j1 = tcol;
    live = j1 < m1;
    const int in2 = static_cast<int>(p2.in_lo);
    c_inner = in2 & ~1;
    c_mid = static_cast<int>(p1.in_lo) + (live ? j1 : 0);
    j2 = ct - (in2 - c_inner);
    act = live && ct < W && j2 >= 0 && j2 < m2;
  }
  // row range of this CTA (chunk-aligned)
  const int nch_all = (m0 + kResR - 1) / kResR;
  const int cpr = (nch_all + a.nrr - 1) / a.nrr;  // chunks per row range
  const int ch0 = rr * cpr, ch1 = min(nch_all, ch0 + cpr);
  live = live && ch0 < ch1;
  act = act && live;
  const int nchunks = live ? ch1 - ch0 : 0;
  // ---- trailing basis of this thread (clamped so every lattice read stays in P_b)
  auto clampi = [](int i, int n) { return i < 0 ? 0 : (i >= n ? n - 1 : i); };
  const int j1c = (j1 >= 0 && j1 < m1) ? j1 : 0, j2c = (j2 >= 0 && j2 < m2) ? j2 : 0;
  double w1[P + 1], w2[P + 1];
  int g1 = __ldg(a.g0 + p1.row_off + j1c), g2 = D == 3 ? __ldg(a.g0 + p2.row_off + j2c) : 0;
#pragma unroll
  for (int k = 0; k <= P; ++k) {
    w1[k] = __ldg(a.vals + (p1.row_off + j1c) * (P + 1) + k);
    w2[k] = D == 3 ? __ldg(a.vals + (p2.row_off + j2c) * (P + 1) + k) : 0.0;
  }
  const unsigned char* sf0 = a.sflag + a.sflag_off[0] + p0.col_lo;
  const unsigned char* sf1 = a.sflag + a.sflag_off[1] + p1.col_lo;
  const unsigned char* sf2 = a.sflag + a.sflag_off[D == 3 ? 2 : 1] + p2.col_lo;
  const double* Pb = a.P + blk.poff;
  const double* Sb = a.snap + blk.poff;
  const std::int64_t plane_sz = static_cast<std::int64_t>(n1) * n2;
  // Shared window over the innermost lattice axis of the CTA's points: the
  // lattice columns gbase .. gbase + rw - 1 (D = 2: axis 1, D = 3: axis 2).
  // Window thread tid stages column gbase + tid of each control plane (D = 3:
  // already contracted along axis 1 with the CTA's common row j1), every
  // thread then finishes its point with P+1 products from shared memory.
  int gbase = 0, rw = 0;
  {
    const AxisProb& pi = D == 2 ? p1 : p2;
    const int mi = D == 2 ? m1 : m2;
    int jf, jl;
    if (D == 2) {
      jf = tcol * (W - 2);
      jl = min(mi - 1, jf + W - 3);
    } else {
      jf = 0;
      jl = mi - 1;
    }
    if (jf < mi) {
      gbase = __ldg(a.g0 + pi.row_off + jf);
      rw = __ldg(a.g0 + pi.row_off + jl) - gbase + P + 1;
    }
  }
  const int ni = D == 2 ? n1 : n2;
  unsigned f1w = 0u;  // D = 3: shared flags of the CTA's P+1 lattice rows along axis 1
  if (D == 3) {
#pragma unroll
    for (int k = 0; k <= P; ++k)
      if (sf1[clampi(g1 + k, n1)]) f1w |= 1u << k;
  }
  const int gi = D == 2 ? g1 : g2;  // this point's first window column
  const int wo = act ? gi - gbase : 0;

  // ---- TMA ring
  const ResStage SL = res_stage(W, P);
  std::uint64_t* bars = reinterpret_cast<std::uint64_t*>(sm_raw + S * SL.stage_bytes);
  double* sR = reinterpret_cast<double*>(sm_raw + S * SL.stage_bytes + S * 8 + 8);  // [EG][na_cap][lt_cap]
  const unsigned tx_bytes = static_cast<unsigned>(SL.q_bytes + kResR * (P + 1) * 8 + kResR * 4);
  const int* g0g = a.g0 + p0.row_off;
  const double* vg = a.vals + p0.row_off * (P + 1);
  const int in0 = static_cast<int>(p0.in_lo);
  // global chunk g = pass * nchunks + c (parity bookkeeping continues across passes)
  auto issue = [&](int g) {
    const int st = g % S, c = ch0 + g % nchunks;
    unsigned char* base = sm_raw + st * SL.stage_bytes;
    mbar_arrive_expect_tx(&bars[st], tx_bytes);
    if (D == 2)
      tma_load_2d(base, &map, c_inner, in0 + c * kResR, &bars[st]);
    else
      tma_load_3d(base, &map, c_inner, c_mid, in0 + c * kResR, &bars[st]);
    bulk_load_1d(base + SL.v_off, vg + static_cast<std::int64_t>(c) * kResR * (P + 1), kResR * (P + 1) * 8, &bars[st]);
    bulk_load_1d(base + SL.g_off, g0g + static_cast<std::int64_t>(c) * kResR, kResR * 4, &bars[st]);
  };
  const int npass = (ne + EG - 1) / EG;
  const int gtotal = npass * nchunks;
  if (tid == 0) {
    prefetch_tmap(&map);
    for (int s = 0; s < S; ++s) mbar_init(&bars[s], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0)
    for (int g = 0; g < S && g < gtotal; ++g) issue(g);

  int g = 0;  // global chunk cursor
  for (int pass = 0; pass < npass; ++pass) {
    const int e0 = pass * EG;
    double l2[EGT];
    unsigned long long li[EGT];  // max |e| as bit patterns (ordered like the values)
#pragma unroll
    for (int q = 0; q < EGT; ++q) {
      l2[q] = 0.0;
      li[q] = 0ull;
    }
    if (nchunks > 0) {
      const int ybeg = ch0 * kResR;
      const int yend = min(m0, ch1 * kResR);
      // planes this row range touches (clamped like every lattice read)
      const int a_lo = clampi(__ldg(g0g + ybeg), n0), a_hi = clampi(__ldg(g0g + yend - 1) + P, n0);
      const int na = a_hi - a_lo + 1;
      // Phase 1: the CTA's window of every touched plane for this pass's
      // epochs, U[q][a - a_lo][t] (D = 3: contracted along axis 1 with the
      // CTA's common row j1), all loads independent (no per-advance latency
      // in the sweep).  Shared controls come from the epoch snapshot, the
      // others from P (they never change after the fit).
      const bool fits = rw <= a.lt_cap && na <= a.na_cap;  // (the host sizes the caps exactly)
      if (!fits)
#pragma unroll
        for (int q = 0; q < EGT; ++q) l2[q] = __longlong_as_double(0x7ff8000000000000LL);  // NaN: never silent
      if (fits) {
        // thread -> (window column t, plane phase r0): one division per thread
        const int tr = nthr / rw > 0 ? nthr / rw : 1;
        const int t = tid % rw, r0 = tid / rw;
        if (r0 < tr) {
          const int cwt = clampi(gbase + t, ni);
          const bool shc = (D == 2 ? sf1[cwt] : sf2[cwt]) != 0;
#pragma unroll 1
          for (int q = 0; q < EG; ++q) {
            const int e = e0 + q < ne ? e0 + q : ne - 1;
            const double* Ls0 = Sb + static_cast<std::int64_t>(e) * a.snap_stride;
#pragma unroll 4
            for (int ai = r0; ai < na; ai += tr) {
              const int a2 = a_lo + ai;
              const bool shw = shc || sf0[a2] != 0;
              const std::int64_t pb = static_cast<std::int64_t>(a2) * plane_sz;
              double r = 0.0;
              if (D == 2) {
                r = __ldg((shw ? Ls0 : Pb) + pb + cwt);
              } else {
#pragma unroll
                for (int k = 0; k <= P; ++k) {
                  const std::int64_t o = pb + static_cast<std::int64_t>(clampi(g1 + k, n1)) * n2 + cwt;
                  r = fma(w1[k], __ldg((shw || ((f1w >> k) & 1u) ? Ls0 : Pb) + o), r);
                }
              }
              sR[(q * a.na_cap + ai) * a.lt_cap + t] = r;
            }
          }
        }
      }
      __syncthreads();
      // trailing contraction of plane ai for every epoch -> Tw slot
      double Tw[EGT][P + 1];
      const double* wk = D == 2 ? w1 : w2;
      auto reduce_into = [&](int slot, int ai) {
        const double* Ub = sR + (static_cast<std::int64_t>(grp) * EGT * a.na_cap + clampi(ai, n0) - a_lo) * a.lt_cap + wo;
#pragma unroll
        for (int q = 0; q < EGT; ++q) {
          double sacc = 0.0;
#pragma unroll
          for (int k = 0; k <= P; ++k) sacc = fma(wk[k], Ub[q * a.na_cap * a.lt_cap + k], sacc);
          Tw[q][slot] = sacc;
        }
      };
      int abase = __ldg(g0g + ybeg);
#pragma unroll
      for (int k = 0; k <= P; ++k) reduce_into(k, abase + k);
      // row cursor over the TMA stages
      int c = 0, jl = 0, jn = 0, gnext = 0x7fffffff;
      const double* sq = nullptr;
      const double* sv = nullptr;
      const int* sg = nullptr;
      auto open_chunk = [&]() {
        const int st = g % S;
        const unsigned char* base = sm_raw + st * SL.stage_bytes;
        sq = reinterpret_cast<const double*>(base) + (ct < W ? ct : 0);
        sv = reinterpret_cast<const double*>(base + SL.v_off);
        sg = reinterpret_cast<const int*>(base + SL.g_off);
        const int yc = (ch0 + c) * kResR;
        jn = (m0 - yc) < kResR ? (m0 - yc) : kResR;
        jl = 0;
        mbar_wait(&bars[st], (g / S) & 1);
        gnext = sg[0];
      };
      auto advance = [&]() {
        if (++jl < jn) {
          gnext = sg[jl];
          return;
        }
        __syncthreads();  // every thread is done with this stage: refill it
        if (tid == 0 && g + S < gtotal) {
          fence_proxy_async();
          issue(g + S);
        }
        ++g;
        if (++c < nchunks)
          open_chunk();
        else
          gnext = 0x7fffffff;
      };
      open_chunk();
      while (gnext != 0x7fffffff) {
#pragma unroll
        for (int u = 0; u <= P; ++u) {
          while (gnext == abase) {  // CTA-uniform
            // e = q - sum_k v_k T_k as one FMA chain from q; L-inf as integer
            // max of |e|'s bit pattern (off the FP64 pipe); inactive (padding)
            // threads compute on finite staged values and are zeroed at the
            // end.  Two rows of the same window per step when the chunk has
            // them (twice the independent chains per thread).
            const bool two = jl + 1 < jn && sg[jl + 1] == abase;  // CTA-uniform
            const double* vr = sv + jl * (P + 1);
            if (two) {
              double v0[P + 1], v1[P + 1];
#pragma unroll
              for (int k = 0; k <= P; ++k) {
                v0[k] = vr[k];
                v1[k] = vr[P + 1 + k];
              }
              const double q0 = sq[jl * W], q1 = sq[(jl + 1) * W];
#pragma unroll
              for (int q = 0; q < EGT; ++q) {
                double e = q0, f = q1;
#pragma unroll
                for (int k = 0; k <= P; ++k) {
                  e = fma(-v0[k], Tw[q][(u + k) % (P + 1)], e);
                  f = fma(-v1[k], Tw[q][(u + k) % (P + 1)], f);
                }
                l2[q] = fma(e, e, l2[q]);
                l2[q] = fma(f, f, l2[q]);
                const unsigned long long eb = static_cast<unsigned long long>(__double_as_longlong(e)) & 0x7fffffffffffffffull;
                const unsigned long long fb = static_cast<unsigned long long>(__double_as_longlong(f)) & 0x7fffffffffffffffull;
                const unsigned long long mb = eb > fb ? eb : fb;
                li[q] = li[q] > mb ? li[q] : mb;
              }
              ++jl;  // (jl + 1 < jn: still inside the chunk)
            } else {
              double v[P + 1];
#pragma unroll
              for (int k = 0; k <= P; ++k) v[k] = vr[k];
              const double qv = sq[jl * W];
#pragma unroll
              for (int q = 0; q < EGT; ++q) {
                double e = qv;
#pragma unroll
                for (int k = 0; k <= P; ++k) e = fma(-v[k], Tw[q][(u + k) % (P + 1)], e);
                l2[q] = fma(e, e, l2[q]);
                const unsigned long long eb = static_cast<unsigned long long>(__double_as_longlong(e)) & 0x7fffffffffffffffull;
                li[q] = li[q] > eb ? li[q] : eb;
              }
            }
            advance();
          }
          if (gnext == 0x7fffffff) break;
          reduce_into(u, abase + P + 1);  // plane abase + P + 1 replaces plane abase
          ++abase;
        }
      }
    }
    // ---- CTA partials of this pass's epochs (group grp holds epochs grp*EGT ..)
    double lif[EGT];
#pragma unroll
    for (int q = 0; q < EGT; ++q) {
      if (!act) {
        l2[q] = 0.0;
        li[q] = 0ull;
      }
      lif[q] = __longlong_as_double(static_cast<long long>(li[q]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        l2[q] += __shfl_xor_sync(kFullMask, l2[q], o);
        lif[q] = fmax(lif[q], __shfl_xor_sync(kFullMask, lif[q], o));
      }
    }
    const int wg = ct >> 5;  // warp within the group
    if ((tid & 31) == 0)
#pragma unroll
      for (int q = 0; q < EGT; ++q) {
        s_red[2 * (grp * EGT + q)][wg] = l2[q];
        s_red[2 * (grp * EGT + q) + 1][wg] = lif[q];
      }
    __syncthreads();
    if (tid < EG && e0 + tid < ne) {
      double sl = 0.0, sm = 0.0;
      for (int w = 0; w < (Wt + 31) / 32; ++w) {
        sl += s_red[2 * tid][w];
        sm = fmax(sm, s_red[2 * tid + 1][w]);
      }
      const std::int64_t o =
          (static_cast<std::int64_t>(e0 + tid) * gridDim.y + b) * gridDim.x + blockIdx.x;
      a.partial[2 * o] = sl;
      a.partial[2 * o + 1] = sm;
    }
    __syncthreads();
  }
}

// errs[e][boff + b] = {sqrt(sum of the block's partials), max} for e < ne, in
// a fixed order (bitwise reproducible).
__global__ void k_res_reduce(const ResTmaArgs a, int nblocks, int ctas) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblocks) return;
  const int ne = a.st ? a.st->iter + 1 : 1;
  for (int e = 0; e < ne; ++e) {
    double sl = 0.0, sm = 0.0;
    const std::int64_t o = (static_cast<std::int64_t>(e) * nblocks + b) * ctas;
    for (int t = 0; t < ctas; ++t) {
      sl += a.partial[2 * (o + t)];
      sm = fmax(sm, a.partial[2 * (o + t) + 1]);
    }
    const std::int64_t w = 2 * (static_cast<std::int64_t>(e) * a.nglobal + a.boff + b);
    a.errs[w] = sqrt(sl);
    a.errs[w + 1] = sm;
  }
}

template <int P>
struct ResTmaLaunch {
  template <int D, int EG, int NG>
  static void go(const ResTmaArgs& a, const CUtensorMap& map, int threads, cudaStream_t s) {
    constexpr int S = kResS;
    const size_t smem = res_tma_smem(P, a.W, EG, a.na_cap, a.lt_cap, S);
    cudaFuncSetAttribute(k_residual_tma<P, D, EG, S, NG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
    dim3 grid(a.ntc * a.nrr, a.nblocks);
    k_residual_tma<P, D, EG, S, NG><<<grid, threads * NG, smem, s>>>(a, map);
    k_res_reduce<<<(a.nblocks + 127) / 128, 128, 0, s>>>(a, a.nblocks, a.ntc * a.nrr);
  }
  static int run(const ResTmaArgs& a, const CUtensorMap& map, int threads, cudaStream_t s) {
    const int eg = a.eg;
    const bool two = a.ng == 2 && threads * 2 <= 512;
    if (a.D == 2) {
      if (eg >= 4)
        two ? go<2, 4, 2>(a, map, threads, s) : go<2, 4, 1>(a, map, threads, s);
      else
        eg >= 2 ? go<2, 2, 1>(a, map, threads, s) : go<2, 1, 1>(a, map, threads, s);
    } else {
      if (eg >= 4)
        two ? go<3, 4, 2>(a, map, threads, s) : go<3, 4, 1>(a, map, threads, s);
      else
        eg >= 2 ? go<3, 2, 1>(a, map, threads, s) : go<3, 1, 1>(a, map, threads, s);
    }
    return 2;
  }
};

template <template <int> class F, class... Args>
int dispatch_res(int p, Args&&... args) {
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

}  // namespace

size_t residual_tma_smem(int degree, int W, int eg, int na_cap, int lt_cap) {
  return res_tma_smem(degree, W, eg, na_cap, lt_cap, kResS);
}

int launch_residual_tma(int degree, const ResTmaArgs& a, const CUtensorMap& map, int threads, cudaStream_t s) {
  return dispatch_res<ResTmaLaunch>(degree, a, map, threads, s);
}

}  // namespace mfb
