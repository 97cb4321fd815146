// hesp_b200_bridge.hpp — reference-side binding of the B200 engine (header-only).
//
// What a maintainer of the reference adds to use the GPU engine from code
// that already holds hesp::Platform / hesp::SchedConfig values
// (platform.hpp:50-86, sim.hpp:26-32) and the tuples it passes to
// PerfModel::analytic / PerfModel::tabulated (platform.hpp:118-121).
// It maps those types field for field onto the C ABI (hesp_engine.h) and
// turns ABI errors back into hesp::Error, so callers keep the reference's
// error behaviour.  Candidates are partition-op sequences applied after
// root_cholesky(n, elem) + partition_task(0, 1/s_base) (graph.hpp:119,136).
//
//   hesp::b200::BatchSimulator gpu(platform, analytic_entries, cfg, n, elem, s_base, gen);
//   std::vector<hesp_outcome> out = gpu.evaluate(descs, &best);   // per-candidate status/makespan
//
// Link with paper_1602_05510_b200/libhesp_b200.so; include paths: this
// directory and the reference's proj/include.
#pragma once

#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "hesp/platform.hpp"
#include "hesp/sim.hpp"
#include "hesp_engine.h"

namespace hesp::b200 {

using AnalyticEntry = std::tuple<TaskKind, std::string, double, double>;   // platform.hpp:118-119
using TableRow = std::tuple<TaskKind, std::string, std::int64_t, double>;  // platform.hpp:120-121

class BatchSimulator {
 public:
  BatchSimulator(const Platform& platform, const std::vector<AnalyticEntry>& analytic,
                 const std::vector<TableRow>& table, const SchedConfig& cfg, std::int64_t n, int elem_size,
                 int s_base, const hesp_gen_config& gen, int device = 0) {
    std::vector<hesp_space> spaces;
    for (const auto& s : platform.spaces()) spaces.push_back({s.id, s.capacity_bytes, s.is_main ? 1 : 0});
    std::vector<const char*> names;
    for (const auto& t : platform.types()) names.push_back(t.name.c_str());
    std::vector<hesp_processor> procs;
    for (const auto& p : platform.processors()) procs.push_back({p.id, p.type, p.space});
    std::vector<hesp_link> links;
    for (const auto& l : platform.links()) links.push_back({l.src, l.dst, l.latency_s, l.bandwidth_bps});
    auto type_index = [&](const std::string& name) {
      for (std::size_t i = 0; i < platform.types().size(); ++i)
        if (platform.types()[i].name == name) return static_cast<int>(i);
      return -1;
    };
    std::vector<hesp_analytic_entry> ents;
    for (const auto& [k, ty, peak, bh] : analytic)
      if (type_index(ty) >= 0) ents.push_back({static_cast<int32_t>(k), type_index(ty), peak, bh});
    std::vector<hesp_table_row> rows;
    for (const auto& [k, ty, b, sec] : table)
      if (type_index(ty) >= 0) rows.push_back({static_cast<int32_t>(k), type_index(ty), b, sec});
    const hesp_platform hp{static_cast<int32_t>(spaces.size()), spaces.data(), static_cast<int32_t>(names.size()),
                           names.data(), static_cast<int32_t>(procs.size()), procs.data(),
                           static_cast<int32_t>(links.size()), links.data()};
    const hesp_perf_model hm{table.empty() ? HESP_MODEL_ANALYTIC : HESP_MODEL_TABULATED,
                             static_cast<int32_t>(ents.size()), ents.data(), static_cast<int32_t>(rows.size()),
                             rows.data()};
    const hesp_sched_config hs{static_cast<int32_t>(cfg.ordering), static_cast<int32_t>(cfg.selection),
                               static_cast<int32_t>(cfg.caching), 0, cfg.seed, cfg.min_block};
    const hesp_workload wl{n, elem_size, s_base, gen};
    engine_ = hesp_engine_create(device, &hp, &hm, &hs, &wl);
    if (!engine_) fail(Err::Validation, std::string("hesp_engine_create: ") + hesp_last_error());
  }
  ~BatchSimulator() { hesp_engine_destroy(engine_); }
  BatchSimulator(const BatchSimulator&) = delete;
  BatchSimulator& operator=(const BatchSimulator&) = delete;

  // Explicit candidates from host memory; outcome k belongs to descs[k].
  std::vector<hesp_outcome> evaluate(const std::vector<hesp_cand_desc>& descs, hesp_best* best = nullptr,
                                     std::uint64_t first_index = 0) {
    std::vector<hesp_outcome> out(descs.size());
    check(hesp_eval_descs(engine_, descs.data(), descs.size(), first_index, out.data(), best));
    return out;
  }

  // Candidates first..first+count-1 of the workload generator, generated on the device.
  hesp_best evaluate_generated(std::uint64_t first, std::uint64_t count, std::vector<hesp_outcome>* out = nullptr) {
    hesp_best best{};
    if (out) out->resize(count);
    check(hesp_eval_generated(engine_, first, count, out ? out->data() : nullptr, &best));
    return best;
  }

  // The reference's per-candidate exception, if any (errors.hpp:10-32).
  static void rethrow(const hesp_outcome& o) {
    if (o.status > 0 && o.status <= 21) fail(static_cast<Err>(o.status - 1), hesp_status_name(o.status));
    if (o.status != 0) fail(Err::Internal, hesp_status_name(o.status));
  }

 private:
  static void check(int rc) {
    if (rc != HESP_OK) fail(Err::Internal, std::string("hesp engine: ") + hesp_last_error());
  }
  hesp_engine* engine_ = nullptr;
};

}  // namespace hesp::b200
