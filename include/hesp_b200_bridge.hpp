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
// or, with the reference's own graphs (root_cholesky(n, elem) followed by any
// partition_task / merge_cluster / repartition_cluster calls):
//
//   hesp::SimResult r = gpu.simulate(graph);         // == hesp::simulate(graph, platform, model, cfg)
//   std::vector<hesp_outcome> o = gpu.evaluate(graphs, &best);
//
// Link with paper_1602_05510_b200/libhesp_b200.so; include paths: this
// directory and the reference's proj/include.
#pragma once

#include <algorithm>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include <cmath>
#include <map>

#include "hesp/graph.hpp"
#include "hesp/platform.hpp"
#include "hesp/sim.hpp"
#include "hesp_engine.h"

namespace hesp::b200 {

using AnalyticEntry = std::tuple<TaskKind, std::string, double, double>;   // platform.hpp:118-119
using TableRow = std::tuple<TaskKind, std::string, std::int64_t, double>;  // platform.hpp:120-121

// ---- a reference TaskGraph as an engine descriptor (see BatchSimulator::simulate(const TaskGraph&)) ----
struct Plan {
  hesp_cand_desc desc{};
  std::vector<int> task_of;   // replay (reference) task id -> graph task id, -1 = none
  std::vector<int> block_of;  // replay block id -> graph block id (blocks_checked only)
  bool blocks_checked = false;
};

// n, elem: the engine's workload; s_base: its base tiling (snapped);
// n_base_tasks / n_base_blocks: the ids that tiling consumes (root included).
inline Plan plan_graph(const TaskGraph& g, std::int64_t n_, int elem_, std::int64_t s_base_, int n_base_tasks_,
                       int n_base_blocks_) {
  if (g.root_n() != n_ || g.elem_size() != elem_)
    fail(Err::Validation, "graph root differs from the engine's workload (n, elem_size)");
  const int root = g.root_task();
  const Task& rt = g.task(root);
  const Region whole{0, 0, n_, n_, elem_};
  const auto& blocks = g.data().blocks();
  bool rooted = rt.kind == TaskKind::CHOL && rt.writes.size() == 1 && rt.reads == rt.writes &&
                g.data().block(rt.writes[0]).region == whole;
  for (const auto& [id, t] : g.tasks())
    if (id != root && !t.cluster) rooted = false;
  if (!rooted) fail(Err::UnknownPartitioner, "graph with explicit edges has no partitioners");
  auto s_of = [](const TaskCluster& c) { return static_cast<int>(std::llround(1.0 / c.p)); };
  Plan pl;
  std::map<int, int> rid;  // graph task id -> replay id
  rid[root] = 0;
  std::vector<std::pair<int, int>> ops;  // (task or cluster, s or HESP_OP_MERGE)
  int next_t = 1, next_b = 1;
  bool shifted = false;
  std::vector<const TaskCluster*> order;  // clusters in replay order
  if (!rt.is_leaf()) {
    const TaskCluster& top = g.cluster(*rt.subcluster);
    if (s_of(top) != s_base_) {
      ops.push_back({0, HESP_OP_MERGE});
      ops.push_back({0, s_of(top)});
      shifted = true;
    }
    order.push_back(&top);
  } else {
    ops.push_back({0, HESP_OP_MERGE});
    shifted = true;
  }
  if (shifted) {
    next_t = n_base_tasks_;
    next_b = n_base_blocks_;
  }
  for (const auto& [cid, c] : g.clusters())
    if (c.parent_task != root) order.push_back(&c);
  for (const TaskCluster* c : order) {
    if (c->parent_task != root) ops.push_back({rid.at(c->parent_task), s_of(*c)});
    for (int m : c->members) rid[m] = next_t++;
  }
  if (ops.size() > HESP_MAX_OPS) fail(Err::Internal, "graph needs more partition ops than a descriptor holds");
  pl.desc.n_ops = static_cast<int32_t>(ops.size());
  for (std::size_t k = 0; k < ops.size(); ++k) pl.desc.ops[k] = hesp_op{ops[k].first, ops[k].second};
  pl.task_of.assign(next_t, -1);
  for (const auto& [gid, r] : rid) pl.task_of[r] = gid;
  // Blocks: without intersection descriptors and partial overlaps the replay
  // creates exactly the graph's blocks, in first-use order over the
  // clusters' members (reads, then the write); their graph ids must ascend.
  bool simple = true;
  for (const auto& [id, b] : blocks)
    if (b.is_intersection) simple = false;
  std::vector<int> created;
  if (simple) {
    std::vector<char> seen(blocks.empty() ? 1 : blocks.rbegin()->first + 1, 0);
    seen[rt.writes[0]] = 1;
    for (const TaskCluster* c : order)
      for (int m : c->members) {
        const Task& t = g.task(m);
        for (int b : t.reads)
          if (!seen[b]) seen[b] = 1, created.push_back(b);
        for (int b : t.writes)
          if (!seen[b]) seen[b] = 1, created.push_back(b);
      }
    if (created.size() + 1 != blocks.size()) simple = false;
    for (std::size_t k = 1; k < created.size() && simple; ++k)
      if (created[k] <= created[k - 1]) simple = false;
    for (std::size_t a = 0; a < created.size() && simple; ++a)
      for (std::size_t b = a + 1; b < created.size() && simple; ++b) {
        const Region& x = g.data().block(created[a]).region;
        const Region& y = g.data().block(created[b]).region;
        if (regions_overlap(x, y) && !region_contains(x, y) && !region_contains(y, x)) simple = false;
      }
  }
  if (simple) {
    const int off = shifted ? n_base_blocks_ - 1 : 0;
    pl.block_of.assign(off + created.size() + 1, -1);
    pl.block_of[0] = rt.writes[0];
    for (std::size_t k = 0; k < created.size(); ++k) pl.block_of[off + 1 + k] = created[k];
    pl.blocks_checked = true;
  }
  return pl;
}


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
    hesp_engine_info info{};
    check(hesp_engine_get_info(engine_, &info));
    n_ = n;
    elem_ = elem_size;
    s_base_ = hesp_snap_tiles(n, s_base, gen.min_block);
    n_base_tasks_ = info.n_base_tasks;
    n_base_blocks_ = info.n_base_blocks;
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

  // ---- the reference's own graphs (graph.hpp:114-185) ----
  //
  // A TaskGraph built by root_cholesky(n, elem) and any sequence of
  // partition_task / merge_cluster / repartition_cluster calls is replayed on
  // the device as the descriptor of its live clusters in cluster-id order
  // (the top one as a merge of the engine's base cluster plus a partition of
  // the root when its tiling differs from s_base).  The replay creates the
  // live tasks and blocks in the same relative order as the graph's own ids,
  // which is all simulate() depends on (ties break by id order); the result is
  // relabelled with the graph's ids.  The block order is verified: a graph
  // whose history cannot be reproduced that way (a merged cluster created a
  // block a later cluster still uses, in an order the replay cannot give)
  // throws Err::Internal rather than risk a different schedule.  Custom graphs
  // (TaskGraph::custom) have no partitioners: Err::UnknownPartitioner, as
  // partition_task throws on them (graph.cpp:460-461).

  // == hesp::simulate(g, platform, model, cfg) (sim.hpp:150-151), on the device.
  SimResult simulate(const TaskGraph& g) {
    const Plan pl = plan(g);
    SimResult r = simulate(pl.desc, elem_);
    relabel(g, pl, r);
    return r;
  }

  // Status and makespan of every graph (the makespan simulate() would give),
  // one device batch; outcome k belongs to graphs[k] (best.index = k).  A
  // graph whose history the replay cannot reproduce (see above) gets status
  // HESP_ST_UNREPRODUCIBLE instead of a possibly different makespan.
  std::vector<hesp_outcome> evaluate(const std::vector<TaskGraph>& graphs, hesp_best* best = nullptr) {
    std::vector<hesp_cand_desc> descs(graphs.size());
    std::vector<Plan> plans;
    plans.reserve(graphs.size());
    for (std::size_t k = 0; k < graphs.size(); ++k) {
      plans.push_back(plan(graphs[k]));
      descs[k] = plans.back().desc;
    }
    std::vector<hesp_outcome> out = evaluate(descs, best);
    bool recheck = false;
    for (std::size_t k = 0; k < graphs.size(); ++k) {
      if (plans[k].blocks_checked || out[k].status != 0) continue;
      // the block order could not be settled on the host: verify it through a trace of this one
      try {
        SimResult r = simulate(plans[k].desc, elem_);
        relabel(graphs[k], plans[k], r);
      } catch (const Error&) {
        out[k] = hesp_outcome{};
        out[k].status = HESP_ST_UNREPRODUCIBLE;
        recheck = true;
      }
    }
    if (recheck && best) {  // the winner (and the valid count) among the graphs that stand
      best->makespan = 0.0;
      best->index = -1;
      best->n_ok = 0;
      for (std::size_t k = 0; k < out.size(); ++k) {
        if (out[k].status != 0) continue;
        ++best->n_ok;
        if (best->index < 0 || out[k].makespan < best->makespan) {
          best->makespan = out[k].makespan;
          best->index = (std::int64_t)k;
        }
      }
    }
    return out;
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

  Plan plan(const TaskGraph& g) const { return plan_graph(g, n_, elem_, s_base_, n_base_tasks_, n_base_blocks_); }

 public:
  // The engine descriptor a graph is replayed as (its live clusters in id order).
  hesp_cand_desc describe(const TaskGraph& g) const { return plan(g).desc; }

 private:
  // Graph ids into a SimResult of the plan's descriptor (after a trace when
  // the block order could not be settled on the host).
  void relabel(const TaskGraph& g, Plan pl, SimResult& r) const {
    if (!pl.blocks_checked) {
      std::int32_t nb = 0;
      check(hesp_trace_blocks(engine_, nullptr, 0, &nb));
      std::vector<hesp_block_info> bi(nb);
      check(hesp_trace_blocks(engine_, bi.data(), nb, &nb));
      pl.block_of.assign(nb, -1);
      int last = -1;
      std::size_t live = 0;
      for (int b = 0; b < nb; ++b) {
        if (bi[b].rows == 0) continue;
        const auto id = g.data().find_by_region(Region{bi[b].row, bi[b].col, bi[b].rows, bi[b].cols, elem_});
        if (!id || *id <= last || g.data().block(*id).is_intersection != (bi[b].is_intersection != 0))
          fail(Err::Internal, "graph history not reproducible on the B200 engine (block order)");
        pl.block_of[b] = last = *id;
        ++live;
      }
      if (live != g.data().blocks().size())
        fail(Err::Internal, "graph history not reproducible on the B200 engine (block set)");
    }
    auto tk = [&](int id) {
      if (id < 0 || id >= (int)pl.task_of.size() || pl.task_of[id] < 0) fail(Err::Internal, "unmapped task id");
      return pl.task_of[id];
    };
    auto bk = [&](int id) {
      if (id < 0 || id >= (int)pl.block_of.size() || pl.block_of[id] < 0) fail(Err::Internal, "unmapped block id");
      return pl.block_of[id];
    };
    SimResult o;
    o.makespan = r.makespan;
    for (const auto& [id, a] : r.assignments) {
      Assignment b = a;
      b.task = tk(id);
      o.assignments[b.task] = b;
      o.idle_avg[b.task] = r.idle_avg.at(id);
    }
    for (auto x : r.transfers) {
      x.block = bk(x.block);
      o.transfers.push_back(x);
    }
    for (auto ev : r.events) {  // subjects "T<id>:<kind>:b<side>" / "B<id>"
      const std::size_t colon = ev.subject.find(':');
      if (ev.subject[0] == 'T')
        ev.subject = "T" + std::to_string(tk(std::stoi(ev.subject.substr(1, colon - 1)))) + ev.subject.substr(colon);
      else
        ev.subject = "B" + std::to_string(bk(std::stoi(ev.subject.substr(1))));
      o.events.push_back(std::move(ev));
    }
    // the reference orders events by (time, kind, resource, subject) (sim.cpp:812-818):
    // relabelled subjects may compare differently; block ids keep their order
    std::stable_sort(o.events.begin(), o.events.end(), [](const EventRec& a, const EventRec& b) {
      if (a.time != b.time) return a.time < b.time;
      if (a.kind != b.kind) return a.kind < b.kind;
      if (a.resource != b.resource) return a.resource < b.resource;
      return a.subject < b.subject;
    });
    for (auto x : r.residency_log) {
      x.block = bk(x.block);
      o.residency_log.push_back(x);
    }
    r = std::move(o);
  }

  hesp_engine* engine_ = nullptr;
  std::int64_t n_ = 0, s_base_ = 0;
  int elem_ = 0, n_base_tasks_ = 0, n_base_blocks_ = 0;
};

}  // namespace hesp::b200
