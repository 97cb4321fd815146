// hesp_port.h — CPU restatement of the reference hot path.  TEST
// INFRASTRUCTURE ONLY (never linked into the product): a second, independent
// checker beside the compiled reference (oracle/_ref).  It restates the
// reference semantics directly -- link-based data DAG with BFS closures,
// explicit pairwise conflict edges, map-based per-space memory state, pin
// counters with release lists, an epoch heap -- rather than the engine's
// reformulations (DESIGN.md §3 E1, E3-E5).  Only E2 (edges matter through
// their transitive closure) is shared: the port keeps the
// full conflict relation instead of transitively reducing it.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "hesp_workload.h"

namespace port {

struct Space {
  int id;
  long long cap;
  bool main;
};
struct Proc {
  int id, type, space;
};
struct Link {
  int src, dst;
  double lat, bw;
};
struct Platform {
  std::vector<Space> spaces;  // sorted by id
  std::vector<std::string> types;
  std::vector<Proc> procs;    // dense ids
  std::vector<Link> links;
};

struct Model {
  bool analytic = true;
  struct A {
    int kind;
    std::string type;
    double peak, bhalf;
  };
  struct R {
    int kind;
    std::string type;
    long long b;
    double sec;
  };
  std::vector<A> entries;
  std::vector<R> rows;
};

struct Sched {
  int ordering = 1;   // 0 FCFS, 1 PL
  int selection = 3;  // 0 R-P, 1 F-P, 2 EIT-P, 3 EFT-P
  int caching = 1;    // 0 WT, 1 WB, 2 WA
  uint64_t seed = 0;
  long long min_block = 64;
};

struct Result {
  int status = 0;  // 0 ok, 1 + hesp::Err ordinal
  int leaves = 0;
  double makespan = 0;
  uint64_t ahash = 0, xhash = 0;
};

// root_cholesky(n, elem) + partition_task(0, 1/s_base) + ops, then simulate.
Result evaluate(const Platform& plat, const Model& model, const Sched& sched, long long n, int elem,
                int s_base, const hesp_cand_desc& desc);

}  // namespace port
