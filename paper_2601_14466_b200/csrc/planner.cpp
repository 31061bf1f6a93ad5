// Host planner of the 1D block-cyclic redistribution.
//
// Column-level semantics are the reference's (pkg/src/bcmg/layout.py):
//   counts  layout.py:82-95     (tile t -> device t mod D, last tile partial)
//   dest_of layout.py:126-145   (position p -> offsets[(p/T) mod D] + ((p/T)/D)*T + p mod T)
//   cycles  layout.py:148-172   (fixed points dropped, each cycle headed by its
//                                smallest member, ascending heads)
//   inverse layout.py:175-183   (head kept, tail reversed)
// On top of that the B200 build plans at SEGMENT granularity: with
// S = gcd(T, N, offsets[1..D-1]) every run of S columns starting at a
// multiple of S stays contiguous and lands on a multiple of S, so the
// column permutation is S copies of one segment permutation.  At every
// BASELINE shape S = T (a tile is one contiguous N*T*esz byte block); for
// shapes like N=10, T=3, D=3 it degrades to S = 1, i.e. the reference's
// column-level plan.
#include <algorithm>
#include <numeric>
#include <stdexcept>

#include "ops.h"

namespace bcmg {

std::vector<int64_t> column_counts(int64_t n_cols, int64_t tile, int ndev) {
  if (ndev < 1) throw Error(CONFIG, "need at least one device");
  if (tile < 1 || tile > n_cols) throw Error(CONFIG, "tile width out of range");
  std::vector<int64_t> counts(ndev, 0);
  const int64_t nt = (n_cols + tile - 1) / tile;
  // full rounds of D tiles, then the remainder (closed form of the deal)
  for (int d = 0; d < ndev; ++d) {
    const int64_t tiles_d = nt / ndev + (d < nt % ndev ? 1 : 0);
    counts[d] = tiles_d * tile;
  }
  const int64_t last_dev = (nt - 1) % ndev;
  counts[last_dev] -= nt * tile - n_cols;  // partial final tile
  return counts;
}

static std::vector<int64_t> offsets_of(const std::vector<int64_t>& counts) {
  std::vector<int64_t> off(counts.size(), 0);
  for (size_t d = 1; d < counts.size(); ++d) off[d] = off[d - 1] + counts[d - 1];
  return off;
}

void build_dest(int64_t n_cols, int64_t tile, int ndev, int64_t* dest) {
  const auto off = offsets_of(column_counts(n_cols, tile, ndev));
  for (int64_t p = 0; p < n_cols; ++p) {
    const int64_t t = p / tile;
    dest[p] = off[t % ndev] + (t / ndev) * tile + p % tile;
  }
}

void decompose(int64_t n, const int64_t* dest, std::vector<int64_t>& members, std::vector<int64_t>& offsets) {
  std::vector<char> seen(n, 0);
  for (int64_t p = 0; p < n; ++p) {
    if (dest[p] < 0 || dest[p] >= n || seen[dest[p]]) throw Error(CONFIG, "dest_of is not a bijection");
    seen[dest[p]] = 1;
  }
  std::fill(seen.begin(), seen.end(), 0);
  members.clear();
  offsets.assign(1, 0);
  for (int64_t h = 0; h < n; ++h) {
    if (seen[h]) continue;
    seen[h] = 1;
    if (dest[h] == h) continue;
    members.push_back(h);
    for (int64_t q = dest[h]; q != h; q = dest[q]) {
      seen[q] = 1;
      members.push_back(q);
    }
    offsets.push_back((int64_t)members.size());
  }
}

void invert_cycles(std::vector<int64_t>& members, const std::vector<int64_t>& offsets) {
  for (size_t c = 0; c + 1 < offsets.size(); ++c)
    std::reverse(members.begin() + offsets[c] + 1, members.begin() + offsets[c + 1]);
}

SegPlan segment_plan(int64_t n_cols, int64_t tile, int ndev, bool inverse) {
  const auto counts = column_counts(n_cols, tile, ndev);
  const auto off = offsets_of(counts);
  int64_t s = std::gcd(tile, n_cols);
  for (int d = 1; d < ndev; ++d) s = std::gcd(s, off[d]);
  if (s < 1) s = 1;
  const int64_t nseg = n_cols / s;
  std::vector<int64_t> dest(nseg);
  for (int64_t i = 0; i < nseg; ++i) {
    const int64_t p = i * s, t = p / tile;
    dest[i] = (off[t % ndev] + (t / ndev) * tile + p % tile) / s;
  }
  SegPlan plan;
  plan.seg = s;
  decompose(nseg, dest.data(), plan.members, plan.offsets);
  if (inverse) invert_cycles(plan.members, plan.offsets);
  plan.seg_cols.assign(plan.offsets.size() - 1, s);
  return plan;
}

}  // namespace bcmg
