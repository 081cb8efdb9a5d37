// Device-side data layout shared by the engine (engine.cu) and the kernels
// (kernels.cu) of the B200 MFA encode path.  See DESIGN.md §3 for the HBM
// layout rationale.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mfb {

constexpr int kMaxDegree = 9;  // templated kernels are instantiated for p = 1..kMaxDegree

// One per-dimension collocation problem: a (dim, block-coordinate) pair of the
// decomposition (all blocks with that coordinate share the rows, solver.cpp:
// 59-66,83-88), one dimension of a stand-alone LocalProblem, or the global
// decode rows of one dimension (window = all controls).
struct AxisProb {
  int dim;
  int m;              // rows (input samples along the dim)
  int n;              // columns (controls in the window)
  int pad_;
  std::int64_t col_lo;  // global index of local column 0 (BlockDim::dof_lo)
  std::int64_t in_lo;   // global input index of row 0
  std::int64_t M;       // global input count: u_j = (in_lo+j)/(M-1); M<0 -> explicit params
  std::int64_t param_off;  // offset into the explicit parameter array
  std::int64_t row_off;    // first row in the rows tables
  std::int64_t col_off;    // first column in the Cholesky tables
  std::int64_t knot_off;   // first knot of this dim's knot vector
  int nknots;
  int pad2_;
};

// One block of the decomposition as the fit kernels see it.
struct BlockDev {
  int ax[3];           // AxisProb id per dim
  int zl;              // last-axis contraction buffer: column pitch in lines (even, = 2 mod 4)
  std::int64_t fbase;  // field offset of the input box origin (input_lo per dim)
  std::int64_t poff;   // offset of the held lattice P_b
  std::int64_t t1off;  // axis-0 intermediate   [n0][m1][m2]
  std::int64_t t2off;  // axis-1 intermediate   [n0][n1][m2]
  std::int64_t zoff;   // last-axis contraction buffer: [n + 2(P+1)][lines] per parity half
};

// Last-axis row segments (k_last_contract_tma): per axis problem
// {K, js[0..K]} padded to kSegStride ints.
constexpr int kMaxSeg = 8;
constexpr int kSegStride = kMaxSeg + 2;

// Status word written by kernels when the reference would throw.
struct DevStatus {
  int code;       // 0 ok, 1 invalid_argument (no active basis), 2 out_of_range, 3 singular
  int axis_prob;  // AxisProb id of the first failure
  int row;        // failing row / column
  int pad_;
};

// Per-epoch reduction slots (u64 bit patterns of non-negative doubles so that
// atomicMax orders them like the values).
struct EpochAcc {
  unsigned long long jump_ss, jump_ms;
};

// A region of shared controls: a box of global control indices over which the
// holder set is constant (the product of one constant-holder interval per
// dim).  Holders are listed in ascending block id (layout.cpp:177-195);
// holder h's copy of control lo + r sits at P[base[h] + sum_k r[k]*str[h][k]].
constexpr int kRegionMaxHolders = 8;
struct RegionDev {
  int ns;      // holders (2, 4 or 8)
  int rmask;   // bit h: holder h lives on another rank (value read from the receive buffer, not written)
  int ext[3];  // box extents (1 for unused dims)
  int ids[kRegionMaxHolders];
  long long base[kRegionMaxHolders];
  int str[kRegionMaxHolders][3];
  int pslot[kRegionMaxHolders * (kRegionMaxHolders - 1) / 2];  // final-jump slot per holder pair, -1 if none
};

// A CTA's slice [start, start + count) of one region's row-major box, with
// the region's descriptor inlined (one dependent load per tile).
struct TileDev {
  RegionDev r;
  int start, count;
};

// Sharded solve: copy [start, start+count) of one holder's copy of a region
// box (P offset base + r.str) into the send buffer at dst + i.
struct PackTile {
  long long base, dst;
  int str[3];
  int ext1, ext2;
  int start, count;
};

// Device-side epoch loop state (the loop runs without host round trips).
struct EpochState {
  int iter;          // last loop iteration that ran (0 before the loop)
  int done;          // CTA tickets of the running epoch (last-CTA pattern)
  int last_iter;     // last iteration that ran
  int converged;     // dp < tol at last_iter
  unsigned long long jump_ss, jump_ms;
  unsigned long long jump0_ss;  // fused epoch 0 + iteration 1 (mode 4): the SS jump before the averaging
};

}  // namespace mfb
