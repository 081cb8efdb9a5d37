// Host-side partition for the B200 MFA encode path; see layout.hpp.
#include "layout.hpp"

#include <algorithm>
#include <cstdlib>
#include <limits>

namespace mfb {

namespace {

// layout.cpp:63-65 — round-half-down of a*T/B (face Greville ties go low)
std::int64_t face_span(std::int64_t a, std::int64_t T, std::int64_t B) { return (2 * a * T + B - 1) / (2 * B); }

// layout.cpp:68-70 — first input j with j/(m-1) >= t/T, exact integers
std::int64_t input_floor(std::int64_t t, std::int64_t T, std::int64_t m) { return (t * (m - 1) + T - 1) / T; }

void validate_knots(const std::vector<double>& kn, int p) {  // knots.cpp:24-46 (clamped)
  for (std::size_t i = 1; i < kn.size(); ++i)
    if (kn[i] < kn[i - 1]) throw std::invalid_argument("KnotVector: knots must be non-decreasing");
  int run = 1;
  for (std::size_t i = 1; i < kn.size(); ++i) {
    run = (kn[i] == kn[i - 1]) ? run + 1 : 1;
    if (run > p + 1) throw std::invalid_argument("KnotVector: knot multiplicity exceeds p+1");
  }
}

}  // namespace

std::vector<double> make_knot_vector(int degree, int basis_count, double a, double b, bool clamp_left,
                                     bool clamp_right) {
  if (degree < 1) throw std::invalid_argument("make_knot_vector: degree must be >= 1");
  if (basis_count < degree + 1)
    throw std::invalid_argument("make_knot_vector: basis count must be at least p+1 (got " +
                                std::to_string(basis_count) + " for p=" + std::to_string(degree) + ")");
  if (!(a < b)) throw std::invalid_argument("make_knot_vector: range must satisfy a < b");
  const int p = degree, spans = basis_count - p;
  const double h = (b - a) / spans;
  std::vector<double> kn;
  kn.reserve(static_cast<std::size_t>(basis_count + p + 1));
  if (clamp_left) {
    for (int i = 0; i <= p; ++i) kn.push_back(a);
  } else {
    for (int i = p; i >= 1; --i) kn.push_back(a - i * h);
    kn.push_back(a);
  }
  for (int k = 1; k < spans; ++k) kn.push_back(a + k * h);
  if (clamp_right) {
    for (int i = 0; i <= p; ++i) kn.push_back(b);
  } else {
    kn.push_back(b);
    for (int i = 1; i <= p; ++i) kn.push_back(b + i * h);
  }
  return kn;
}

std::int64_t Decomp::dim_field(int k, int c, int f) const {
  // Block with coordinate c along k and 0 elsewhere.
  int cc[3] = {0, 0, 0};
  cc[k] = c;
  return at(block_id(cc), k, f);
}

bool Decomp::shared_box(int a, int b, std::array<std::array<std::int64_t, 2>, 3>& box) const {
  for (int k = 0; k < rank; ++k) {
    box[k][0] = std::max(at(a, k, DOF_LO), at(b, k, DOF_LO));
    box[k][1] = std::min(at(a, k, DOF_HI), at(b, k, DOF_HI));
    if (box[k][0] >= box[k][1]) return false;
  }
  return true;
}

std::int64_t Decomp::total_inputs() const {
  std::int64_t c = 1;
  for (int k = 0; k < rank; ++k) c *= grid[k];
  return c;
}

std::int64_t Decomp::total_ctrl() const {
  std::int64_t c = 1;
  for (int k = 0; k < rank; ++k) c *= n_ctrl[k];
  return c;
}

Decomp partition(int rank, const std::int64_t* grid, const double* bounds, const int* blocks, int degree,
                 const std::int64_t* nctrl_blk, std::int64_t overlap, bool clamp) {
  if (rank < 1 || rank > 3) throw std::invalid_argument("partition: 1, 2 or 3 dimensions supported");
  if (degree < 1) throw std::invalid_argument("partition: degree must be >= 1");
  if (overlap < 0) throw std::invalid_argument("partition: overlap must be >= 0");
  const int p = degree;
  const std::int64_t w = p / 2;  // delta_width, layout.cpp:11-14
  Decomp d;
  d.rank = rank;
  d.degree = p;
  d.clamp = clamp;
  d.overlap = clamp ? 0 : overlap;
  std::array<std::vector<std::int64_t>, 3> face;
  for (int k = 0; k < rank; ++k) {
    d.grid[k] = grid[k];
    d.blocks[k] = blocks[k];
    d.bounds.push_back({bounds ? bounds[2 * k] : 0.0, bounds ? bounds[2 * k + 1] : 1.0});
    if (blocks[k] < 1) throw std::invalid_argument("partition: blocks per dimension must be >= 1");
    if (nctrl_blk[k] < p + 1)
      throw std::invalid_argument("partition: nctrl per block must be at least p+1 in dimension " + std::to_string(k));
    if (!(d.bounds[k][0] < d.bounds[k][1]))
      throw std::invalid_argument("partition: bounds min must be < max in dimension " + std::to_string(k));
    const int B = blocks[k];
    const std::int64_t nb = nctrl_blk[k];
    // plan_dim, layout.cpp:81-121
    if (!clamp || B == 1) {
      d.n_ctrl[k] = static_cast<std::int64_t>(B) * nb;
      d.knots[k] = make_knot_vector(p, static_cast<int>(d.n_ctrl[k]), 0.0, 1.0, true, true);
    } else {
      d.n_ctrl[k] = static_cast<std::int64_t>(B) * (nb - 1) + 1;
      const std::int64_t seg = nb - p;
      if (seg < 1) throw std::invalid_argument("partition: clamp_interfaces requires nctrl per block > degree");
      const std::int64_t spans = static_cast<std::int64_t>(B) * seg;
      const double h = 1.0 / static_cast<double>(spans);
      auto& kn = d.knots[k];
      for (int i = 0; i <= p; ++i) kn.push_back(0.0);
      for (std::int64_t t = 1; t < spans; ++t) {
        const double v = static_cast<double>(t) * h;
        kn.push_back(v);
        if (t % seg == 0)
          for (int r = 1; r < p; ++r) kn.push_back(v);
      }
      for (int i = 0; i <= p; ++i) kn.push_back(1.0);
    }
    validate_knots(d.knots[k], p);
    const int n = static_cast<int>(d.knots[k].size()) - p - 1;
    for (int s = p; s < n; ++s)
      if (d.knots[k][static_cast<std::size_t>(s)] < d.knots[k][static_cast<std::size_t>(s) + 1])
        d.span_knot[k].push_back(s);
    const std::int64_t T = static_cast<std::int64_t>(d.span_knot[k].size());
    d.spans[k] = T;
    face[k].resize(static_cast<std::size_t>(B) + 1);
    for (int b = 0; b <= B; ++b)
      face[k][static_cast<std::size_t>(b)] =
          (!clamp || B == 1) ? face_span(b, T, B) : static_cast<std::int64_t>(b) * (nb - p);
    face[k][0] = 0;
    face[k][static_cast<std::size_t>(B)] = T;
    if (grid[k] < d.n_ctrl[k])
      throw std::invalid_argument("partition: input count must be >= control count in dimension " + std::to_string(k));
    if (!clamp && B > 1) {  // layout.cpp:257-267
      std::int64_t mn = std::numeric_limits<std::int64_t>::max();
      for (int b = 0; b < B; ++b)
        mn = std::min(mn, face[k][static_cast<std::size_t>(b) + 1] - face[k][static_cast<std::size_t>(b)]);
      if (w + d.overlap > mn)
        throw std::invalid_argument("partition: overlap too large in dimension " + std::to_string(k) +
                                    ": delta+overlap spans (" + std::to_string(w + d.overlap) +
                                    ") exceed the smallest block (" + std::to_string(mn) +
                                    " spans); exchanges would cross non-neighbor blocks");
    }
  }
  int nb = 1;
  for (int k = 0; k < rank; ++k) nb *= blocks[k];
  d.nblocks = nb;
  d.coords.assign(static_cast<std::size_t>(nb), {0, 0, 0});
  d.bd.assign(static_cast<std::size_t>(nb) * rank * BD_N, 0);
  const std::int64_t c_hi = p - w;
  std::array<int, 3> c{0, 0, 0};
  for (int id = 0; id < nb; ++id) {
    d.coords[static_cast<std::size_t>(id)] = c;
    for (int k = 0; k < rank; ++k) {
      const int b = c[k], B = blocks[k];
      const std::int64_t T = d.spans[k], m = grid[k];
      auto F = [&](int f) -> std::int64_t& { return d.at(id, k, f); };
      F(SPAN_LO) = face[k][static_cast<std::size_t>(b)];
      F(SPAN_HI) = face[k][static_cast<std::size_t>(b) + 1];
      if (!clamp) {
        F(DELTA_LO) = b > 0 ? w : 0;
        F(DELTA_HI) = b < B - 1 ? w : 0;
        F(OVL_LO) = b > 0 ? d.overlap : 0;
        F(OVL_HI) = b < B - 1 ? d.overlap : 0;
      }
      F(LSPAN_LO) = F(SPAN_LO) - F(DELTA_LO) - F(OVL_LO);
      F(LSPAN_HI) = F(SPAN_HI) + F(DELTA_HI) + F(OVL_HI);
      if (!clamp) {  // layout.cpp:298-305: residence by Greville point
        F(DOF_LO) = F(LSPAN_LO) == 0 ? 0 : F(LSPAN_LO) + c_hi;
        F(DOF_HI) = F(LSPAN_HI) == T ? d.n_ctrl[k] : F(LSPAN_HI) + c_hi;
        F(OWN_LO) = F(SPAN_LO) == 0 ? 0 : F(SPAN_LO) + c_hi;
        F(OWN_HI) = F(SPAN_HI) == T ? d.n_ctrl[k] : F(SPAN_HI) + c_hi;
      } else {  // layout.cpp:306-313
        F(DOF_LO) = d.span_knot[k][static_cast<std::size_t>(F(LSPAN_LO))] - p;
        F(DOF_HI) = d.span_knot[k][static_cast<std::size_t>(F(LSPAN_HI) - 1)] + 1;
        F(OWN_LO) = F(DOF_LO) + (b > 0 ? 1 : 0);
        F(OWN_HI) = F(DOF_HI);
      }
      F(IN_LO) = input_floor(F(LSPAN_LO), T, m);  // layout.cpp:315-318
      F(IN_HI) = F(LSPAN_HI) == T ? m : input_floor(F(LSPAN_HI), T, m);
      F(OWNIN_LO) = input_floor(F(SPAN_LO), T, m);
      F(OWNIN_HI) = F(SPAN_HI) == T ? m : input_floor(F(SPAN_HI), T, m);
    }
    for (int k = rank - 1; k >= 0; --k) {
      if (++c[k] < blocks[k]) break;
      c[k] = 0;
    }
  }
  // SharedDofMap holder ranges, layout.cpp:125-146
  for (int k = 0; k < rank; ++k) {
    d.holder[k].assign(static_cast<std::size_t>(d.n_ctrl[k]), {0, -1});
    for (int id = 0; id < nb; ++id) {
      const int cc = d.coords[static_cast<std::size_t>(id)][k];
      for (std::int64_t i = d.at(id, k, DOF_LO); i < d.at(id, k, DOF_HI); ++i) {
        auto& r = d.holder[k][static_cast<std::size_t>(i)];
        if (r[1] < r[0]) {
          r = {cc, cc};
        } else {
          r[0] = std::min(r[0], cc);
          r[1] = std::max(r[1], cc);
        }
      }
    }
    for (const auto& r : d.holder[k])
      if (r[1] > r[0]) d.any_shared = true;
  }
  // neighbors, layout.cpp:328-340
  d.neighbors.resize(static_cast<std::size_t>(nb));
  std::array<std::array<std::int64_t, 2>, 3> box;
  for (int id = 0; id < nb; ++id)
    for (int o = 0; o < nb; ++o) {
      if (o == id) continue;
      bool adj = true;
      for (int k = 0; k < rank; ++k)
        if (std::abs(d.coords[static_cast<std::size_t>(o)][k] - d.coords[static_cast<std::size_t>(id)][k]) > 1)
          adj = false;
      if (adj && d.shared_box(id, o, box)) d.neighbors[static_cast<std::size_t>(id)].push_back(o);
    }
  return d;
}

std::vector<std::int64_t> exchange_volume(const Decomp& d) {
  std::vector<std::int64_t> vol(static_cast<std::size_t>(d.nblocks), 0);
  std::array<std::array<std::int64_t, 2>, 3> box;
  for (int a = 0; a < d.nblocks; ++a)
    for (int j : d.neighbors[static_cast<std::size_t>(a)]) {
      if (!d.shared_box(a, j, box)) continue;
      std::int64_t c = 1;
      for (int k = 0; k < d.rank; ++k) c *= box[k][1] - box[k][0];
      vol[static_cast<std::size_t>(a)] += c;
    }
  return vol;
}

// ---------------------------------------------------------------- regions
std::vector<Region> enumerate_regions(const Decomp& d) {
  const int D = d.rank;
  struct Iv {
    std::int64_t lo, hi;
    int f, e;
  };
  std::vector<Iv> iv[3];
  for (int k = 0; k < D; ++k)
    for (std::int64_t i = 0; i < d.n_ctrl[k]; ++i) {
      const auto r = d.holder[k][static_cast<std::size_t>(i)];
      if (r[1] - r[0] > 1) throw std::logic_error("enumerate_regions: more than two holders along one axis");
      if (!iv[k].empty() && iv[k].back().f == r[0] && iv[k].back().e == r[1] - r[0] + 1 && iv[k].back().hi == i)
        ++iv[k].back().hi;
      else
        iv[k].push_back({i, i + 1, r[0], r[1] - r[0] + 1});
    }
  std::vector<Region> out;
  std::size_t cnt[3] = {1, 1, 1};
  for (int k = 0; k < D; ++k) cnt[k] = iv[k].size();
  for (std::size_t i0 = 0; i0 < cnt[0]; ++i0)
    for (std::size_t i1 = 0; i1 < cnt[1]; ++i1)
      for (std::size_t i2 = 0; i2 < cnt[2]; ++i2) {
        const std::size_t ii[3] = {i0, i1, i2};
        int ns = 1;
        for (int k = 0; k < D; ++k) ns *= iv[k][ii[k]].e;
        if (ns < 2) continue;
        Region R;
        R.ns = ns;
        for (int k = 0; k < D; ++k) {
          R.lo[static_cast<std::size_t>(k)] = iv[k][ii[k]].lo;
          R.ext[static_cast<std::size_t>(k)] = iv[k][ii[k]].hi - iv[k][ii[k]].lo;
        }
        for (int h = 0; h < ns; ++h) {
          int rr = h, c[3] = {0, 0, 0};
          for (int k = D - 1; k >= 0; --k) {
            const Iv& v = iv[k][ii[k]];
            c[k] = v.f + (v.e == 2 ? (rr & 1) : 0);
            rr = v.e == 2 ? (rr >> 1) : rr;
          }
          R.ids[static_cast<std::size_t>(h)] = d.block_id(c);
          for (int k = 0; k < 3; ++k) R.coords[static_cast<std::size_t>(h)][static_cast<std::size_t>(k)] = c[k];
        }
        out.push_back(R);
      }
  return out;
}

// ---------------------------------------------------------------- sharding
ShardRange shard_range(const Decomp& d, int rank, int nranks) {
  if (nranks < 1 || rank < 0 || rank >= nranks) throw std::invalid_argument("shard_range: bad rank");
  const int B0 = d.blocks[0];
  ShardRange s;
  if (nranks > B0) {  // contiguous block-id ranges finer than block rows
    if (d.rank < 2 || nranks > d.nblocks || nranks > d.grid[0])
      throw std::invalid_argument("shard_range: " + std::to_string(nranks) + " ranks for " + std::to_string(d.nblocks) +
                                  " blocks (" + std::to_string(B0) + " block rows along axis 0)");
    s.partial = true;
    s.blo = static_cast<int>(static_cast<std::int64_t>(rank) * d.nblocks / nranks);
    s.bhi = static_cast<int>(static_cast<std::int64_t>(rank + 1) * d.nblocks / nranks);
    s.row_lo = d.coords[static_cast<std::size_t>(s.blo)][0];
    s.row_hi = d.coords[static_cast<std::size_t>(s.bhi - 1)][0] + 1;
    s.in_lo = static_cast<std::int64_t>(rank) * d.grid[0] / nranks;
    s.in_hi = static_cast<std::int64_t>(rank + 1) * d.grid[0] / nranks;
  } else {
    s.row_lo = static_cast<int>(static_cast<std::int64_t>(rank) * B0 / nranks);
    s.row_hi = static_cast<int>(static_cast<std::int64_t>(rank + 1) * B0 / nranks);
    const int per_row = d.nblocks / B0;
    s.blo = s.row_lo * per_row;
    s.bhi = s.row_hi * per_row;
    s.in_lo = d.dim_field(0, s.row_lo, OWNIN_LO);
    s.in_hi = d.dim_field(0, s.row_hi - 1, OWNIN_HI);
  }
  s.own_lo = d.dim_field(0, s.row_lo, OWN_LO);
  s.own_hi = d.dim_field(0, s.row_hi - 1, OWN_HI);
  s.box_lo = std::min(d.dim_field(0, s.row_lo, IN_LO), s.in_lo);
  s.box_hi = std::max(d.dim_field(0, s.row_hi - 1, IN_HI), s.in_hi);
  return s;
}

int shard_of_block(const Decomp& d, int nranks, int block) {
  const int B0 = d.blocks[0];
  // inverse of lo(r) = r*N/n: the largest r with lo(r) <= x
  auto inv = [nranks](std::int64_t x, std::int64_t N) {
    int r = static_cast<int>((x * nranks + nranks - 1) / N);
    if (r >= nranks) r = nranks - 1;
    while (r > 0 && static_cast<std::int64_t>(r) * N / nranks > x) --r;
    while (r + 1 < nranks && static_cast<std::int64_t>(r + 1) * N / nranks <= x) ++r;
    return r;
  };
  if (nranks > B0) return inv(block, d.nblocks);
  return inv(d.coords[static_cast<std::size_t>(block)][0], B0);
}

std::vector<PeerLayout> shard_peers(const Decomp& d, const std::vector<Region>& regions, int rank, int nranks) {
  std::vector<PeerLayout> out;
  for (int q = 0; q < nranks; ++q) {
    if (q == rank) continue;
    PeerLayout pl;
    pl.peer = q;
    for (std::size_t ri = 0; ri < regions.size(); ++ri) {
      const Region& R = regions[ri];
      bool mine = false, theirs = false;
      for (int h = 0; h < R.ns; ++h) {
        const int s = shard_of_block(d, nranks, R.ids[static_cast<std::size_t>(h)]);
        mine = mine || s == rank;
        theirs = theirs || s == q;
      }
      if (!mine || !theirs) continue;
      for (int h = 0; h < R.ns; ++h) {
        const int s = shard_of_block(d, nranks, R.ids[static_cast<std::size_t>(h)]);
        if (s == rank) {
          pl.send.emplace_back(static_cast<int>(ri), h);
          pl.send_count += R.size();
        } else if (s == q) {
          pl.recv.emplace_back(static_cast<int>(ri), h);
          pl.recv_count += R.size();
        }
      }
    }
    if (!pl.send.empty() || !pl.recv.empty()) out.push_back(pl);
  }
  return out;
}

}  // namespace mfb
