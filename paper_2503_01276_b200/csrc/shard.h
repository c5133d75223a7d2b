// Multi-GPU sharding plan (host only): which rank solves which macropoint of each level, and which
// parent fine solutions move between ranks after each level.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "plan.h"

struct ShardPlan {
  int world = 1;
  // owner[level][pos]: rank owning position pos of S_level (lexicographic order)
  std::vector<std::vector<int>> owner;
  // xfer[level]: (macropoint, src rank, dst rank) of the parent solutions of S_level that a
  // child on another rank needs; sorted by (src, dst, macropoint).  Sent after level `level`.
  std::vector<std::vector<std::array<int64_t, 3>>> xfer;
  std::vector<int> owner_of;  // per lexicographic macropoint index
};

// Contiguous, cost-balanced ownership per level: S_level in lexicographic order (slowest axis
// first, i.e. slabs of the macrogrid) cut into `world` runs of near-equal total work, the work of a
// macropoint being the level-n node count of its (clipped) window.  Same macropoint -> same
// arithmetic on any rank, so results do not depend on world.
void shard_build(const HostPlan& pl, int world, ShardPlan& out);
