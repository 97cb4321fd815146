// hesp_b200_bridge.hpp — reference-side binding of the B200 engine (header-only).
//
// What a maintainer of the reference adds to use the GPU engine from code
// that already holds hesp::Platform / hesp::SchedConfig values
// (platform.hpp:50-86, sim.hpp:26-32) and the tuples it passes to
// PerfModel::analytic / PerfModel::tabulated (platform.hpp:118-121).
// It maps those types field for field onto the C ABI (hesp_engine.h) and
// turns ABI errors back into hesp::Error, so callers keep the reference's
// error behaviour.  Candidates are partition/merge-op sequences applied after
// root_cholesky(n, elem) + partition_task(0, 1/s_base) (graph.hpp:119,136).
//
//   hesp::b200::BatchSimulator gpu(platform, analytic_entries, cfg, n, elem, s_base, gen);
//   std::vector<hesp_outcome> out = gpu.evaluate(descs, &best);   // per-candidate status/makespan
//   hesp::SimResult r = gpu.simulate(descs[best.index], elem);     // the winner's full SimResult
//
// Link with paper_1602_05510_b200/libhesp_b200.so; include paths: this
// directory and the reference's proj/include.
#pragma once

#include <algorithm>
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

  // The full hesp::SimResult of one candidate, simulated on the device
  // (hesp_eval_trace): the value simulate(graph, platform, model, cfg)
  // (sim.hpp:150-151) returns for the graph the descriptor describes, in the
  // reference's own types and container orders.  Throws the reference's
  // hesp::Error for a failing candidate.
  SimResult simulate(const hesp_cand_desc& desc, int elem_size) {
    std::vector<hesp_assignment> a(4096);
    std::vector<hesp_transfer> x(8192);
    std::vector<hesp_residency> r(16384);
    std::vector<hesp_event> e(32768);
    std::vector<hesp_load_step> st(8192);
    hesp_trace t{};
    int rc;
    for (;;) {
      t = hesp_trace{};
      t.cap_assign = (int32_t)a.size();
      t.cap_xfer = (int32_t)x.size();
      t.cap_res = (int32_t)r.size();
      t.cap_events = (int32_t)e.size();
      t.cap_steps = (int32_t)st.size();
      t.assignments = a.data();
      t.transfers = x.data();
      t.residency = r.data();
      t.events = e.data();
      t.steps = st.data();
      rc = hesp_eval_trace(engine_, &desc, &t);
      if (rc != HESP_E_LIMIT) break;
      a.resize(std::max<size_t>(a.size(), t.n_assign));
      x.resize(std::max<size_t>(x.size(), t.n_xfer));
      r.resize(std::max<size_t>(r.size(), t.n_res));
      e.resize(std::max<size_t>(e.size(), t.n_events));
      st.resize(std::max<size_t>(st.size(), t.n_steps));
    }
    if (rc < 0) check(rc);
    if (rc > 0) {
      hesp_outcome o{};
      o.status = rc;
      rethrow(o);
    }
    static const char* kinds[] = {"CHOL", "TRSM", "SYRK", "GEMM"};
    SimResult res;
    res.makespan = t.outcome.makespan;
    for (int i = 0; i < t.n_assign; ++i) {
      res.assignments[a[i].task] = {a[i].task, a[i].proc, a[i].start, a[i].end};
      res.idle_avg[a[i].task] = a[i].idle_avg;
    }
    for (int i = 0; i < t.n_xfer; ++i) {
      TransferRec rec;
      rec.block = x[i].block;
      if (x[i].has_fragment)
        rec.fragment = Region{x[i].frag_row, x[i].frag_col, x[i].frag_rows, x[i].frag_cols, elem_size};
      for (int h = 0; h < x[i].n_hops; ++h) rec.route.emplace_back(x[i].hop_src[h], x[i].hop_dst[h]);
      rec.start = x[i].start;
      rec.end = x[i].end;
      rec.bytes = x[i].bytes;
      rec.dst_space = x[i].dst_space;
      res.transfers.push_back(rec);
    }
    for (int i = 0; i < t.n_events; ++i) {
      EventRec ev;
      ev.kind = static_cast<EventRec::Kind>(e[i].kind);
      ev.time = e[i].time;
      if (e[i].kind <= HESP_EV_TASK_END) {
        ev.subject = "T" + std::to_string(e[i].id) + ":" + kinds[e[i].task_kind] + ":b" + std::to_string(e[i].b);
        ev.resource = std::to_string(e[i].res_a);
      } else {
        ev.subject = "B" + std::to_string(e[i].id);
        ev.resource = std::to_string(e[i].res_a) + "->" + std::to_string(e[i].res_b);
      }
      res.events.push_back(std::move(ev));
    }
    for (int i = 0; i < t.n_res; ++i)
      res.residency_log.push_back({r[i].time, r[i].space, r[i].delta_bytes, r[i].block});
    return res;
  }

  // The iterative solver (hesp_solve; solver.hpp:83-84 semantics).
  hesp_solver_result solve(const hesp_solver_config& cfg, std::vector<hesp_solver_iteration>& history,
                           const hesp_cand_desc* initial = nullptr) {
    history.resize(cfg.iterations > 0 ? cfg.iterations : 1);
    hesp_solver_result out{};
    out.cap_history = (int32_t)history.size();
    out.history = history.data();
    const int rc = hesp_solve(engine_, initial, &cfg, &out);
    if (rc < 0) check(rc);
    if (rc > 0) {
      hesp_outcome o{};
      o.status = rc;
      rethrow(o);
    }
    history.resize(out.n_history);
    return out;
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
