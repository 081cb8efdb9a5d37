// Host-side decomposition metadata for the B200 MFA encode path.
//
// Restates the reference's partition() (proj/core/src/layout.cpp:217-342),
// plan_dim (:81-121), SharedDofMap (:125-203) and shared_dof_box (:205-215).
// Every integer here is bit-exact with the reference; knots are generated with
// the same floating-point expressions (knots.cpp:58-79, layout.cpp:94-101).
// This is plan-time host work (the reference also runs partition() outside
// solve()); everything inside solve() runs on the GPU.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mfb {

// BlockDim field order (layout.hpp:47-57)
enum BlockDimField : int {
  SPAN_LO, SPAN_HI, DELTA_LO, DELTA_HI, OVL_LO, OVL_HI, LSPAN_LO, LSPAN_HI,
  DOF_LO, DOF_HI, OWN_LO, OWN_HI, IN_LO, IN_HI, OWNIN_LO, OWNIN_HI, BD_N
};

struct SingularFit : std::runtime_error {
  int dim;
  std::int64_t span;
  SingularFit(int d, std::int64_t s, const std::string& w) : std::runtime_error(w), dim(d), span(s) {}
};

struct Decomp {
  int rank = 0, degree = 0;
  bool clamp = false;
  std::int64_t overlap = 0;
  std::array<std::int64_t, 3> grid{1, 1, 1};
  std::array<int, 3> blocks{1, 1, 1};
  std::array<std::int64_t, 3> n_ctrl{1, 1, 1};
  std::array<std::int64_t, 3> spans{0, 0, 0};          // T: nonempty span count
  std::vector<std::array<double, 2>> bounds;
  std::array<std::vector<double>, 3> knots;
  std::array<std::vector<int>, 3> span_knot;
  int nblocks = 0;
  std::vector<std::array<int, 3>> coords;               // per block
  std::vector<std::int64_t> bd;                         // nblocks*rank*BD_N
  std::array<std::vector<std::array<int, 2>>, 3> holder;  // per dim per ctrl index
  std::vector<std::vector<int>> neighbors;
  bool any_shared = false;

  std::int64_t& at(int b, int k, int f) { return bd[(static_cast<std::size_t>(b) * rank + k) * BD_N + f]; }
  std::int64_t at(int b, int k, int f) const { return bd[(static_cast<std::size_t>(b) * rank + k) * BD_N + f]; }
  int block_id(const int* c) const {
    int id = 0;
    for (int k = 0; k < rank; ++k) id = id * blocks[k] + c[k];
    return id;
  }
  // Per-dim block coordinate -> BlockDim of any block with that coordinate
  // (ranges along dim k depend only on the coordinate along k).
  std::int64_t dim_field(int k, int c, int f) const;
  bool shared_box(int a, int b, std::array<std::array<std::int64_t, 2>, 3>& box) const;
  std::int64_t total_inputs() const;
  std::int64_t total_ctrl() const;
};

// layout.cpp:217-342.  Throws std::invalid_argument like the reference.
Decomp partition(int rank, const std::int64_t* grid, const double* bounds, const int* blocks, int degree,
                 const std::int64_t* nctrl_per_block, std::int64_t overlap, bool clamp_interfaces);

// knots.cpp:48-81 (uniform clamped/floating knot vector)
std::vector<double> make_knot_vector(int degree, int basis_count, double a, double b, bool clamp_left,
                                     bool clamp_right);

// runtime.cpp:160-171
std::vector<std::int64_t> exchange_volume(const Decomp& d);

// ------------------------------------------------------------ shared regions
// A box of shared controls with one holder set: the product of one
// constant-holder-range interval per dim (SharedDofMap::holder_span,
// layout.cpp:125-203) with n_s >= 2.  Holders in ascending block id
// (layout.cpp:177-195; last dim least significant).  Requires at most two
// holders per dim (n_s <= 8); enumeration order is deterministic.
struct Region {
  std::array<std::int64_t, 3> lo{0, 0, 0}, ext{1, 1, 1};
  int ns = 0;
  std::array<int, 8> ids{};
  std::array<std::array<int, 3>, 8> coords{};
  std::int64_t size() const { return ext[0] * ext[1] * ext[2]; }
};
std::vector<Region> enumerate_regions(const Decomp& d);

// ------------------------------------------------------------ sharding
// Rank r of n owns the contiguous block ids [blo, bhi) (ids are lexicographic
// with axis 0 slowest, layout.cpp:320-323).  With n <= B0 the ranges are whole
// block rows [row_lo, row_hi) along axis 0 (r*B0/n .. (r+1)*B0/n): a shared
// control then has holders on at most two adjacent ranks, and a rank decodes
// the input rows its block rows own.  With n > B0 (D >= 2, n <= nblocks) the
// ranges are [r*nblocks/n, (r+1)*nblocks/n) and may cut a block row
// (`partial`): holders then sit on any of the neighbouring ranks, the owned
// lattice entries are a subset of the rows [own_lo, own_hi), and the input
// rows are split evenly over the ranks for the decode (the reference deals any
// block count to any number of workers, runtime.cpp:115-121).
struct ShardRange {
  int row_lo = 0, row_hi = 0, blo = 0, bhi = 0;
  bool partial = false;                 // block-id ranges finer than block rows
  std::int64_t in_lo = 0, in_hi = 0;    // own input rows along axis 0 (decode)
  std::int64_t own_lo = 0, own_hi = 0;  // control rows along axis 0 the local blocks own entries of (assembly)
  std::int64_t box_lo = 0, box_hi = 0;  // input rows the rank reads: its blocks' fits and its decode rows
};
ShardRange shard_range(const Decomp& d, int rank, int nranks);
int shard_of_block(const Decomp& d, int nranks, int block);

// Per-epoch exchange with one peer rank: the buffer is the concatenation, over
// the regions holding controls on both ranks (ascending region index), of the
// sending rank's holders' copies (ascending holder slot), each region box in
// row-major order.  `send` lists (region, holder slot) of this rank's copies,
// `recv` those of the peer, in buffer order.
struct PeerLayout {
  int peer = -1;
  std::vector<std::pair<int, int>> send, recv;
  std::int64_t send_count = 0, recv_count = 0;
};
std::vector<PeerLayout> shard_peers(const Decomp& d, const std::vector<Region>& regions, int rank, int nranks);

}  // namespace mfb
