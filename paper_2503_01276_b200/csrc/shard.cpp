// Sharding plan of the multi-GPU layer: macropoints of one level are independent
// ("independent across different macropoints"); a child at level n reads only the
// fine solutions of its T_{n-1} parents (Eq. 11), so after each level the owners
// send exactly those parents to the ranks whose children use them.
#include "shard.h"

#include <algorithm>
#include <set>

void shard_build(const HostPlan& pl, int world, ShardPlan& out) {
  if (world < 1) world = 1;
  out.world = world;
  out.owner.assign(pl.L + 1, {});
  out.xfer.assign(pl.L + 1, {});
  out.owner_of.assign(pl.all.size(), 0);
  int64_t s = 1;
  for (int lev = 1; lev <= pl.L; lev++) {
    const std::vector<int64_t>& Sl = pl.S[lev];
    std::vector<double> w(Sl.size());
    double tot = 0.0;
    for (size_t i = 0; i < Sl.size(); i++) {
      const MacroHost& m = pl.all[Sl[i]];
      double nodes = 1.0;
      for (int d = 0; d < pl.D; d++) nodes *= (double)((m.hi[d] - m.lo[d]) / s + 1);
      w[i] = nodes;
      tot += nodes;
    }
    // position i goes to the rank whose share [r tot/world, (r+1) tot/world) holds the midpoint of
    // its work interval: contiguous runs, each rank within one macropoint of an equal share
    std::vector<int>& own = out.owner[lev];
    own.assign(Sl.size(), 0);
    double acc = 0.0;
    for (size_t i = 0; i < Sl.size(); i++) {
      const double mid = acc + 0.5 * w[i];
      int r = (tot > 0.0) ? (int)(mid * world / tot) : 0;
      r = std::min(std::max(r, 0), world - 1);
      own[i] = r;
      out.owner_of[Sl[i]] = r;
      acc += w[i];
    }
    s *= pl.eta;
  }
  // transfers: parent t of a child p needs to reach owner(p) if owner(t) differs; sent after
  // level(t)
  std::vector<std::set<std::array<int64_t, 3>>> xs(pl.L + 1);
  for (size_t lin = 0; lin < pl.all.size(); lin++) {
    const MacroHost& m = pl.all[lin];
    if (m.level < 2) continue;
    const int dst = out.owner_of[lin];
    for (int t = 0; t < m.npar; t++) {
      const int64_t par = m.par_lin[t];
      const int src = out.owner_of[par];
      if (src == dst) continue;
      xs[pl.all[par].level].insert({(int64_t)src, (int64_t)dst, par});
    }
  }
  for (int lev = 1; lev <= pl.L; lev++)
    for (const auto& e : xs[lev]) out.xfer[lev].push_back({e[2], e[0], e[1]});
}
