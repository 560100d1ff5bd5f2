// Host-side shard logic for the multi-GPU PAGANI loop (pure functions).
//
// Rank r owns the contiguous slice [B_r, B_{r+1}) of the GLOBAL region order,
// with every B_r a multiple of the 2048-region fold block (reduce.cpp:10), so
// a rank's local 2048-blocks are global blocks and every fp64 sum is the same
// bit pattern as on one GPU.  After bisection the children of the global kept
// region k sit at 2k, 2k+1 (geometry.cpp:124-125); rank r produced the
// contiguous range [2K_r, 2K_{r+1}) and the next batch is re-partitioned into
// balanced block ranges, moving the pieces that change owner (this exchange
// is also the rebalance).
#pragma once

#include <cstdint>
#include <vector>

namespace pgn {

constexpr int64_t kShardBlock = 2048;

// Balanced partition of m regions into nranks block-aligned ranges.
inline std::vector<int64_t> shard_bounds(int64_t m, int nranks) {
  const int64_t nb = (m + kShardBlock - 1) / kShardBlock;
  std::vector<int64_t> b(nranks + 1);
  for (int r = 0; r <= nranks; ++r) {
    const int64_t blk = (nb * r) / nranks;
    const int64_t v = blk * kShardBlock;
    b[r] = v < m ? v : m;
  }
  b[nranks] = m;
  return b;
}

// Largest number of blocks any rank owns under `bounds`.
inline int64_t max_blocks(const std::vector<int64_t>& bounds) {
  int64_t mb = 0;
  for (size_t r = 0; r + 1 < bounds.size(); ++r) {
    const int64_t nb = (bounds[r + 1] - bounds[r] + kShardBlock - 1) / kShardBlock;
    mb = nb > mb ? nb : mb;
  }
  return mb;
}

struct Piece {
  int peer;
  int64_t src_off;  // offset in the sender's child staging
  int64_t dst_off;  // offset in the receiver's next slice
  int64_t count;    // regions
};

// kept[r] = global kept index of rank r's first kept region (nranks+1 entries,
// kept[nranks] = total).  Children of rank r: global [2 kept[r], 2 kept[r+1]).
// next = shard_bounds(2 * kept[nranks], nranks).
inline void exchange_plan(int nranks, int rank, const std::vector<int64_t>& kept,
                          const std::vector<int64_t>& next, std::vector<Piece>& sends,
                          std::vector<Piece>& recvs) {
  sends.clear();
  recvs.clear();
  for (int s = 0; s < nranks; ++s)
    for (int d = 0; d < nranks; ++d) {
      if (s != rank && d != rank) continue;
      const int64_t c0 = 2 * kept[s], c1 = 2 * kept[s + 1];
      const int64_t lo = c0 > next[d] ? c0 : next[d];
      const int64_t hi = c1 < next[d + 1] ? c1 : next[d + 1];
      if (hi <= lo) continue;
      const Piece p{s == rank ? d : s, lo - c0, lo - next[d], hi - lo};
      if (s == rank) sends.push_back(p);
      if (d == rank) recvs.push_back(p);
    }
}

}  // namespace pgn
