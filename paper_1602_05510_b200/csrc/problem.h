// problem.h — host-side construction of the engine's Problem tables.
#pragma once

#include <string>
#include <vector>

#include "engine_types.h"
#include "hesp_engine.h"

namespace hx {

// Host copy of a fully built problem: the POD tables plus the base graph
// arrays the device copies point at after upload.
struct HostProblem {
  Problem p{};
  // every top-level tiling's arrays, concatenated (TIL_BASE first)
  std::vector<TaskMeta> base_tasks;
  std::vector<BlockMeta> base_blocks;
  std::vector<BasePreds> base_preds;
  std::vector<int32_t> base_plist;
  struct TilingOff {
    int s, n_tasks, n_blocks;
    long long base_b;
    size_t tasks, blocks, preds, plist;  // offsets into the arrays above
  };
  std::vector<TilingOff> til;
};

// Points p's base arrays and tilings at copies of hp's arrays (host vectors
// or their device uploads).
void bind_tilings(Problem& p, const HostProblem& hp, const TaskMeta* tasks, const BlockMeta* blocks,
                  const BasePreds* preds, const int32_t* plist);

// Validates (Platform::validate, platform.cpp:91-138; PerfModel::analytic,
// platform.cpp:312-325) and precomputes everything; throws std::runtime_error.
HostProblem build_problem(const hesp_platform& plat, const hesp_perf_model& model,
                          const hesp_sched_config& sched, const hesp_workload& wl);

// Sets the message hesp_last_error() returns (engine_kernels.cu).
void set_last_error(const std::string& msg);

// PerfModel::task_time restated for one (kind, b, type); throws on miss.
double host_task_time(const hesp_perf_model& m, int kind, long long b, int type, bool* known);

}  // namespace hx
