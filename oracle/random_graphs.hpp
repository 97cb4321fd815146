// random_graphs.hpp -- TEST INFRASTRUCTURE (oracle/): reference TaskGraphs
// built by random sequences of the reference's own mutators, shared by
// bridge_check (GPU, the C++ bridge) and engine_check (CPU, the width-1
// engine).  partition_task on random leaves, merge_cluster on random
// innermost clusters (the top one included: back to the bare root),
// repartition_cluster; a call the reference rejects leaves the graph as is.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <random>
#include <vector>

#include "hesp/graph.hpp"

namespace oracle {

struct GraphStats {
  int calls = 0, top_merges = 0;
  int dropped = 0;  // graphs a mutator left broken with a foreign exception (a reference defect)
};

inline std::vector<hesp::TaskGraph> random_graphs(int count, std::int64_t n, int elem, int s_base,
                                                  std::int64_t min_block, std::uint64_t seed, GraphStats* st) {
  std::mt19937_64 rng(seed);
  std::vector<hesp::TaskGraph> gs;
  for (int i = 0; i < count; ++i) {
    auto g = hesp::TaskGraph::root_cholesky(n, elem);
    const int s_choice[] = {2, 3, 4, 8, s_base, s_base};
    bool broken = false;
    auto try_call = [&](auto&& f) {
      if (broken) return;
      try {
        f();
        ++st->calls;
      } catch (const hesp::Error&) {
      } catch (const std::exception&) {
        // e.g. merge_cluster's prune erasing an intersection block a task
        // still references (graph.cpp:214-266): the graph is left half-mutated
        broken = true;
      }
    };
    try_call([&] { g.partition_task(0, 1.0 / s_choice[rng() % 6], min_block); });
    const int steps = static_cast<int>(rng() % 12);
    for (int k = 0; k < steps && !broken; ++k) {
      const int r = static_cast<int>(rng() % 100);
      const auto leaves = g.leaf_tasks();
      const auto inner = g.innermost_clusters();
      if (r < 55) {
        const int t = leaves[rng() % leaves.size()];
        const int s = 2 + static_cast<int>(rng() % 3);
        if (g.task(t).b / s >= min_block && g.task_depth(t) < 4)
          try_call([&] { g.partition_task(t, 1.0 / s, min_block); });
      } else if (r < 80 && !inner.empty()) {
        const int c = inner[rng() % inner.size()];
        if (g.cluster(c).parent_task == g.root_task()) ++st->top_merges;
        try_call([&] { g.merge_cluster(c); });
      } else if (!inner.empty()) {
        // a re-tiling of the root may take any choice; inner clusters stay
        // within the engine's slot sizing (<= 8 x 8 sub-tilings)
        const int c = inner[rng() % inner.size()];
        const bool top = g.cluster(c).parent_task == g.root_task();
        const int s = top ? s_choice[rng() % 6] : s_choice[rng() % 4];
        try_call([&] { g.repartition_cluster(c, 1.0 / s, min_block); });
      }
    }
    if (broken) {
      ++st->dropped;
      --i;  // draw another graph in its place
      continue;
    }
    gs.push_back(std::move(g));
  }
  return gs;
}

}  // namespace oracle
