// ref_harness.cpp — drives the UNMODIFIED reference simulator (compiled from
// /root/reference/proj/src into oracle/_ref/libhesp_ref.so) over a batch of
// candidate partitionings.  TEST INFRASTRUCTURE ONLY: used to generate the
// golden fixtures, to pin the CPU restatement (oracle/port) and as the
// bench's CPU baseline / reference arm.  Never linked into the product.
//
// Per candidate:
//   TaskGraph::root_cholesky(n, elem)                       graph.cpp:397
//   partition_task(0, 1.0/s_base, min_block)                graph.cpp:456
//   partition_task(op.task, 1.0/op.s, min_block) per op     graph.cpp:456
//   simulate(graph, platform, model, cfg)                   sim.cpp:838
// and records status (0 ok, 1 + hesp::Err ordinal, 100 foreign exception),
// makespan bits, and order-independent hashes of every Assignment and
// TransferRec (include/hesp_workload.h), so a single 40-byte record pins the
// whole schedule bit-for-bit.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "hesp/graph.hpp"
#include "hesp/platform.hpp"
#include "hesp/sim.hpp"
#include "hesp_workload.h"

namespace {

struct Record {
  uint64_t index;
  int32_t status;
  int32_t n_leaves;
  double makespan;
  uint64_t assign_hash;
  uint64_t xfer_hash;
};
static_assert(sizeof(Record) == 40, "record layout");

struct Args {
  std::string platform, model, out, detail_out, descs;
  bool model_csv = false;
  int64_t n = 16384;
  int elem = 4;
  int s_base = 16;
  hesp_gen_config gen{};
  std::string ordering = "PL", selection = "EFT-P", caching = "WB";
  uint64_t sched_seed = 0;
  uint64_t first = 0, count = 100;
  int threads = 1;
  double time_limit = 0;  // seconds; 0 = none
  long detail = -1;
  bool quiet = false;
  long trace = -1;  // --trace: full SimResult dump (JSON) of one candidate
  std::string trace_out;
  int shift_task = -1;  // --shift-task T --shift-by X: move T's interval by -X before verify
  double shift_by = 0;
  // --solve N: the SPEC solver restated over the reference
  // TaskGraph/simulate, for hesp_solve parity
  int solve = -1;
  std::string solve_sel = "All", solve_samp = "Hard";
  int solve_kmax = 8;
  uint64_t solve_seed = 0;
  double overhead = 1.1;
};

std::string slurp(const std::string& path) {
  std::ifstream f(path);
  if (!f) {
    std::fprintf(stderr, "cannot open %s\n", path.c_str());
    std::exit(2);
  }
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

uint64_t bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}

struct Ctx {
  const Args* a;
  const hesp::Platform* plat;
  const hesp::PerfModel* model;
  hesp::SchedConfig cfg;
  int32_t n_base;
  int64_t base_b;
  int32_t s_base_snapped;
};

std::vector<hesp_cand_desc> g_descs;  // --descs: explicit candidates (index = position)

Record evaluate(const Ctx& c, uint64_t index, hesp::SimResult* keep, hesp::TaskGraph** keep_graph) {
  Record r{};
  r.index = index;
  hesp_cand_desc d;
  if (!g_descs.empty()) d = g_descs.at(index);
  else hesp_generate(&c.a->gen, c.s_base_snapped, c.n_base, c.base_b, index, &d);
  try {
    auto g = hesp::TaskGraph::root_cholesky(c.a->n, c.a->elem);
    g.partition_task(0, 1.0 / c.a->s_base, c.a->gen.min_block);
    for (int k = 0; k < d.n_ops; ++k) {
      if (d.ops[k].s == HESP_OP_MERGE) g.merge_cluster(d.ops[k].task);  // graph.cpp:521-534
      else g.partition_task(d.ops[k].task, 1.0 / d.ops[k].s, c.a->gen.min_block);
    }
    r.n_leaves = static_cast<int32_t>(g.leaf_tasks().size());
    auto res = hesp::simulate(g, *c.plat, *c.model, c.cfg);
    r.makespan = res.makespan;
    uint64_t ah = 0, xh = 0;
    for (const auto& [id, asg] : res.assignments)
      ah += hesp_assign_term(asg.task, asg.proc, bits(asg.start), bits(asg.end));
    for (const auto& x : res.transfers) {
      int64_t fr = 0, fc = 0, frs = 0, fcs = 0;
      if (x.fragment) {
        fr = x.fragment->row;
        fc = x.fragment->col;
        frs = x.fragment->rows;
        fcs = x.fragment->cols;
      }
      xh += hesp_xfer_term(x.block, x.route.front().first, x.dst_space, x.bytes, bits(x.start),
                           bits(x.end), fr, fc, frs, fcs);
    }
    r.assign_hash = ah;
    r.xfer_hash = xh;
    if (keep) *keep = std::move(res);
    if (keep_graph) *keep_graph = new hesp::TaskGraph(std::move(g));
  } catch (const hesp::Error& e) {
    r.status = 1 + static_cast<int32_t>(e.code());
    r.makespan = 0;
  } catch (const std::exception& e) {
    r.status = 100;
    r.makespan = 0;
  }
  return r;
}

bool parse_int_list(const char* s, hesp_gen_config* g) {
  g->n_s_choices = 0;
  const char* p = s;
  while (*p && g->n_s_choices < 4) {
    g->s_choices[g->n_s_choices++] = std::atoi(p);
    while (*p && *p != ',') ++p;
    if (*p == ',') ++p;
  }
  return g->n_s_choices > 0;
}

// Full SimResult of one candidate as JSON, doubles as 16-hex-digit bit
// patterns, in the reference's own container orders (sim.cpp:813-832), plus
// compute_load_trace, the summary metrics and verify_schedule's messages.
void dump_trace(FILE* f, const Record& r, hesp::SimResult& res, const hesp::TaskGraph* g, const hesp::Platform& plat,
                const Args& a) {
  auto hx = [](double x) {
    char b[24];
    std::snprintf(b, sizeof b, "\"%016llx\"", (unsigned long long)bits(x));
    return std::string(b);
  };
  auto q = [](const std::string& x) { return "\"" + x + "\""; };
  std::fprintf(f, "{\"index\": %llu, \"status\": %d, \"leaves\": %d, \"makespan\": %s",
               (unsigned long long)r.index, r.status, r.n_leaves, hx(r.makespan).c_str());
  if (r.status != 0 || !g) {
    std::fprintf(f, "}\n");
    return;
  }
  std::fprintf(f, ",\n\"assignments\": [");
  bool first = true;
  for (const auto& [id, x] : res.assignments) {
    std::fprintf(f, "%s[%d, %d, %s, %s, %s]", first ? "" : ", ", x.task, x.proc, hx(x.start).c_str(),
                 hx(x.end).c_str(), hx(res.idle_avg.at(id)).c_str());
    first = false;
  }
  std::fprintf(f, "],\n\"transfers\": [");
  first = true;
  for (const auto& x : res.transfers) {
    std::string fr = "null", route = "[";
    if (x.fragment)
      fr = "[" + std::to_string(x.fragment->row) + ", " + std::to_string(x.fragment->col) + ", " +
           std::to_string(x.fragment->rows) + ", " + std::to_string(x.fragment->cols) + "]";
    for (size_t h = 0; h < x.route.size(); ++h)
      route += (h ? ", [" : "[") + std::to_string(x.route[h].first) + ", " + std::to_string(x.route[h].second) + "]";
    route += "]";
    std::fprintf(f, "%s[%d, %d, %d, %lld, %s, %s, %s, %s]", first ? "" : ", ", x.block, x.route.front().first,
                 x.dst_space, (long long)x.bytes, hx(x.start).c_str(), hx(x.end).c_str(), fr.c_str(), route.c_str());
    first = false;
  }
  std::fprintf(f, "],\n\"events\": [");
  first = true;
  for (const auto& e : res.events) {
    std::fprintf(f, "%s[%d, %s, %s, %s]", first ? "" : ", ", static_cast<int>(e.kind), hx(e.time).c_str(),
                 q(e.subject).c_str(), q(e.resource).c_str());
    first = false;
  }
  std::fprintf(f, "],\n\"residency\": [");
  first = true;
  for (const auto& c : res.residency_log) {
    std::fprintf(f, "%s[%s, %d, %lld, %d]", first ? "" : ", ", hx(c.time).c_str(), c.space, (long long)c.delta_bytes,
                 c.block);
    first = false;
  }
  const auto lt = hesp::compute_load_trace(res, plat);
  std::fprintf(f, "],\n\"load\": [");
  first = true;
  for (const auto& [t, n] : lt.steps) {
    std::fprintf(f, "%s[%s, %d]", first ? "" : ", ", hx(t).c_str(), n);
    first = false;
  }
  std::fprintf(f, "],\n\"busy\": %s, \"avg_load\": %s, \"integral\": %s", hx(res.busy_time()).c_str(),
               hx(res.avg_load(plat.processor_count())).c_str(), hx(lt.integral()).c_str());
  if (a.shift_task >= 0) {
    auto it = res.assignments.find(a.shift_task);
    if (it != res.assignments.end()) {
      it->second.start -= a.shift_by;
      it->second.end -= a.shift_by;
    }
  }
  const auto v = hesp::verify_schedule(res, *g, plat);
  std::fprintf(f, ",\n\"violations\": [");
  for (size_t i = 0; i < v.size(); ++i) std::fprintf(f, "%s%s", i ? ", " : "", q(v[i]).c_str());
  std::fprintf(f, "]}\n");
}

// ---------------------------------------------------------------------------
// Solver oracle.  TEST INFRASTRUCTURE: the declared-only solver
// (solver.hpp:57-86) restated from SPEC.md:410-461 with the decisions of
// DESIGN.md §10, driving the UNMODIFIED reference TaskGraph (partition_task,
// merge_cluster, repartition_cluster) and simulate().
struct OCand {
  int action;  // 0 partition, 1 merge, 2 repartition
  int target, parent;
  int64_t k;
  double score;
  int64_t d;
};

int64_t o_snap(int64_t d, int64_t k, int64_t mb) {  // TaskGraph::snap_tiling
  return hesp::TaskGraph::snap_tiling(d, k, mb);
}

void run_solve(const Ctx& c, FILE* f) {
  const Args& a = *c.a;
  const hesp::Platform& plat = *c.plat;
  const hesp::PerfModel& model = *c.model;
  const int64_t mb = a.gen.min_block;
  const int sel = a.solve_sel == "CP" ? 1 : a.solve_sel == "Shallow" ? 2 : 0;
  const bool soft = a.solve_samp == "Soft";
  hesp::Rng rng(a.solve_seed);
  auto g = hesp::TaskGraph::root_cholesky(a.n, a.elem);
  g.partition_task(0, 1.0 / a.s_base, mb);
  auto choose_k = [&](double idle, int64_t d) -> int64_t {
    if (d < 2 * mb) return 0;
    const int64_t lim = std::min<int64_t>(a.solve_kmax, d / mb);
    int64_t k = (int64_t)std::ceil(std::sqrt(idle + 1.0)) + 1;
    k = std::max<int64_t>(2, std::min(k, lim));
    return o_snap(d, k, mb);
  };
  auto w_sub = [&](const hesp::Task& t, int64_t k, const std::string& type, double* w) {
    std::vector<hesp::Region> rr;
    for (int r : t.reads)
      if (std::find(t.writes.begin(), t.writes.end(), r) == t.writes.end()) rr.push_back(g.data().block(r).region);
    const auto specs = hesp::enumerate_partition(t.kind, rr, g.data().block(t.writes.front()).region, k);
    double sum = 0;
    for (const auto& sp : specs) {
      if (!model.knows(sp.kind, type)) return false;
      sum += model.task_time(sp.kind, sp.write.rows, type);
    }
    *w = sum;
    return true;
  };
  std::fprintf(f, "{\"history\": [");
  double best = 0;
  int best_it = -1;
  for (int it = 0; it < a.solve; ++it) {
    hesp::SimResult res;
    try {
      res = hesp::simulate(g, plat, model, c.cfg);
    } catch (const hesp::Error& e) {
      std::fprintf(f, "], \"status\": %d}\n", 1 + static_cast<int>(e.code()));
      return;
    }
    int depth = 0;
    double num = 0, den = 0;
    for (const auto& [id, t] : g.tasks()) {
      if (!t.is_leaf()) continue;
      depth = std::max(depth, g.task_depth(id));
      const double fl = hesp::task_flops(t.kind, t.b);
      num += fl * (double)t.b;
      den += fl;
    }
    const double avgb = den > 0 ? num / den : 0.0;
    const double load = 100.0 * res.avg_load(plat.processor_count());
    if (best_it < 0 || res.makespan < best) {
      best = res.makespan;
      best_it = it;
    }
    int action = -1, target = -1, ncand = 0, nvalid = 0;
    int64_t dd = 0;
    double pp = 0, sc = 0;
    if (it + 1 < a.solve) {
      std::vector<int> tasks;
      if (sel == 0) {
        for (const auto& [id, x] : res.assignments) tasks.push_back(id);
      } else if (sel == 2) {
        int dmin = 1 << 30;
        for (const auto& [id, x] : res.assignments) dmin = std::min(dmin, g.task_depth(id));
        for (const auto& [id, x] : res.assignments)
          if (g.task_depth(id) == dmin) tasks.push_back(id);
      } else {
        int cur = -1;
        for (const auto& [id, x] : res.assignments)
          if (cur < 0 || x.end > res.assignments.at(cur).end) cur = id;
        while (cur >= 0) {
          tasks.push_back(cur);
          int nxt = -1;
          for (int pr : g.preds(cur))
            if (nxt < 0 || res.assignments.at(pr).end > res.assignments.at(nxt).end) nxt = pr;
          cur = nxt;
        }
        std::sort(tasks.begin(), tasks.end());
      }
      std::vector<OCand> cands;
      for (int id : tasks) {
        const auto& x = res.assignments.at(id);
        const auto& t = g.task(id);
        const double idle = res.idle_avg.at(id);
        const int64_t k = choose_k(idle, t.b);
        if (k == 0) continue;
        double w;
        if (!w_sub(t, k, plat.type_name(x.proc), &w)) continue;
        const double est = a.overhead * w / std::min(idle + 1.0, (double)k);
        const double score = std::max(0.0, (x.end - x.start) - est);
        if (score > 0) cands.push_back({0, id, id, k, score, t.b});
      }
      for (int cid : g.innermost_clusters()) {
        if (cid == 0) continue;  // the base cluster stays
        const auto& cl = g.cluster(cid);
        double lo = 0, hi = 0, isum = 0;
        bool first = true;
        for (int m : cl.members) {
          const auto& x = res.assignments.at(m);
          if (first || x.start < lo) lo = x.start;
          if (first || x.end > hi) hi = x.end;
          first = false;
          isum += res.idle_avg.at(m);
        }
        const auto& par = g.task(cl.parent_task);
        double tmin = 0;
        std::string tbest;
        bool have = false;
        for (const auto& ty : plat.types()) {
          if (!model.knows(par.kind, ty.name)) continue;
          const double tt = model.task_time(par.kind, par.b, ty.name);
          if (!have || tt < tmin) {
            tmin = tt;
            tbest = ty.name;
            have = true;
          }
        }
        if (!have) continue;
        const double span = hi - lo;
        const double merge = std::max(0.0, span - tmin);
        if (merge > 0) cands.push_back({1, cid, cl.parent_task, 0, merge, par.b});
        const double ic = isum / (double)cl.members.size();
        const int64_t k = choose_k(ic, par.b);
        const int64_t kc = par.b / g.task(cl.members.front()).b;
        double w;
        if (k == 0 || k == kc || !w_sub(par, k, tbest, &w)) continue;
        const double est = a.overhead * w / std::min(ic + 1.0, (double)k);
        const double rep = merge + std::max(0.0, span - est);
        if (rep > 0) cands.push_back({2, cid, cl.parent_task, k, rep, par.b});
      }
      ncand = (int)cands.size();
      auto mutated = [&](const OCand& x) {
        hesp::TaskGraph h = g;
        if (x.action == 0) h.partition_task(x.target, 1.0 / (double)x.k, mb);
        else if (x.action == 1) h.merge_cluster(x.target);
        else h.repartition_cluster(x.target, 1.0 / (double)x.k, mb);
        return h;
      };
      std::vector<char> ok(cands.size(), 0);
      {
        std::atomic<size_t> next{0};
        auto worker = [&]() {
          for (;;) {
            const size_t i = next.fetch_add(1);
            if (i >= cands.size()) return;
            try {
              auto h = mutated(cands[i]);
              hesp::simulate(h, plat, model, c.cfg);
              ok[i] = 1;
            } catch (const std::exception&) {
            }
          }
        };
        std::vector<std::thread> pool;
        for (int t = 0; t < std::max(1, a.threads); ++t) pool.emplace_back(worker);
        for (auto& t : pool) t.join();
      }
      std::vector<OCand> valid;
      for (size_t i = 0; i < cands.size(); ++i)
        if (ok[i]) valid.push_back(cands[i]);
      nvalid = (int)valid.size();
      if (!valid.empty()) {
        size_t pick = 0;
        if (!soft) {  // argmax score, ties: lowest target id, then candidate order
          for (size_t i = 1; i < valid.size(); ++i)
            if (valid[i].score > valid[pick].score ||
                (valid[i].score == valid[pick].score && valid[i].target < valid[pick].target))
              pick = i;
        } else {
          double total = 0;
          for (const auto& x : valid) total += x.score;
          const double u = rng.uniform() * total;
          double acc = 0;
          pick = valid.size() - 1;
          for (size_t i = 0; i < valid.size(); ++i) {
            acc += valid[i].score;
            if (u < acc) {
              pick = i;
              break;
            }
          }
        }
        const OCand& x = valid[pick];
        action = x.action;
        target = x.target;
        dd = x.d;
        pp = x.action == 1 ? 1.0 : 1.0 / (double)x.k;
        sc = x.score;
        g = mutated(x);
      }
    }
    std::fprintf(f, "%s[%d, %d, %d, %d, %d, %d, %lld, \"%016llx\", \"%016llx\", \"%016llx\", \"%016llx\", \"%016llx\"]",
                 it ? ", " : "", it, action, target, ncand, nvalid, depth, (long long)dd, (unsigned long long)bits(pp),
                 (unsigned long long)bits(sc), (unsigned long long)bits(res.makespan), (unsigned long long)bits(avgb),
                 (unsigned long long)bits(load));
  }
  std::fprintf(f, "], \"status\": 0, \"best\": \"%016llx\", \"best_iteration\": %d}\n",
               (unsigned long long)bits(best), best_it);
}

}  // namespace

int main(int argc, char** argv) {
  Args a;
  a.gen.seed = 1;
  a.gen.k_max = 8;
  a.gen.max_depth = 3;
  a.gen.min_block = 64;
  a.gen.n_s_choices = 2;
  a.gen.s_choices[0] = 2;
  a.gen.s_choices[1] = 4;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto v = [&]() -> const char* {
      if (i + 1 >= argc) {
        std::fprintf(stderr, "missing value for %s\n", k.c_str());
        std::exit(2);
      }
      return argv[++i];
    };
    if (k == "--platform") a.platform = v();
    else if (k == "--model") a.model = v();
    else if (k == "--model-csv") { a.model = v(); a.model_csv = true; }
    else if (k == "--n") a.n = std::atoll(v());
    else if (k == "--elem") a.elem = std::atoi(v());
    else if (k == "--sbase") a.s_base = std::atoi(v());
    else if (k == "--seed") a.gen.seed = std::strtoull(v(), nullptr, 0);
    else if (k == "--kmax") a.gen.k_max = std::atoi(v());
    else if (k == "--maxdepth") a.gen.max_depth = std::atoi(v());
    else if (k == "--min-block") a.gen.min_block = std::atoll(v());
    else if (k == "--s-choices") parse_int_list(v(), &a.gen);
    else if (k == "--ordering") a.ordering = v();
    else if (k == "--selection") a.selection = v();
    else if (k == "--caching") a.caching = v();
    else if (k == "--sched-seed") a.sched_seed = std::strtoull(v(), nullptr, 0);
    else if (k == "--merge-pct") a.gen.merge_pct = std::atoi(v());
    else if (k == "--first") a.first = std::strtoull(v(), nullptr, 0);
    else if (k == "--count") a.count = std::strtoull(v(), nullptr, 0);
    else if (k == "--threads") a.threads = std::atoi(v());
    else if (k == "--time-limit") a.time_limit = std::atof(v());
    else if (k == "--out") a.out = v();
    else if (k == "--detail") a.detail = std::atol(v());
    else if (k == "--detail-out") a.detail_out = v();
    else if (k == "--quiet") a.quiet = true;
    else if (k == "--descs") a.descs = v();
    else if (k == "--trace") a.trace = std::atol(v());
    else if (k == "--solve") a.solve = std::atoi(v());
    else if (k == "--solve-selection") a.solve_sel = v();
    else if (k == "--solve-sampling") a.solve_samp = v();
    else if (k == "--solve-kmax") a.solve_kmax = std::atoi(v());
    else if (k == "--solve-seed") a.solve_seed = std::strtoull(v(), nullptr, 0);
    else if (k == "--overhead") a.overhead = std::atof(v());
    else if (k == "--trace-out") a.trace_out = v();
    else if (k == "--shift-task") a.shift_task = std::atoi(v());
    else if (k == "--shift-by") a.shift_by = std::atof(v());
    else {
      std::fprintf(stderr, "unknown argument %s\n", k.c_str());
      return 2;
    }
  }
  if (a.threads <= 0) a.threads = static_cast<int>(std::thread::hardware_concurrency());
  if (!a.descs.empty()) {
    std::ifstream f(a.descs, std::ios::binary);
    hesp_cand_desc d;
    while (f.read(reinterpret_cast<char*>(&d), sizeof d)) g_descs.push_back(d);
    a.first = 0;
    a.count = g_descs.size();
  }

  const auto plat = hesp::Platform::from_json(slurp(a.platform));
  const auto model = a.model_csv ? hesp::PerfModel::from_table_csv(slurp(a.model))
                                 : hesp::PerfModel::from_analytic_json(slurp(a.model));
  Ctx c{&a, &plat, &model, {}, 0, 0, 0};
  c.cfg.ordering = hesp::ordering_from(a.ordering);
  c.cfg.selection = hesp::selection_from(a.selection);
  c.cfg.caching = hesp::caching_from(a.caching);
  c.cfg.seed = a.sched_seed;
  c.cfg.min_block = a.gen.min_block;
  {
    // base tiling facts for the generator, taken from the reference itself
    auto g = hesp::TaskGraph::root_cholesky(a.n, a.elem);
    const int cl = g.partition_task(0, 1.0 / a.s_base, a.gen.min_block);
    c.n_base = static_cast<int32_t>(g.cluster(cl).members.size());
    c.base_b = g.task(g.cluster(cl).members.front()).b;
    c.s_base_snapped = static_cast<int32_t>(a.n / c.base_b);
  }

  if (a.solve >= 0) {
    FILE* f = a.trace_out.empty() ? stdout : std::fopen(a.trace_out.c_str(), "w");
    run_solve(c, f);
    if (f != stdout) std::fclose(f);
    return 0;
  }
  if (a.trace >= 0) {
    hesp::SimResult res;
    hesp::TaskGraph* g = nullptr;
    Record r = evaluate(c, static_cast<uint64_t>(a.trace), &res, &g);
    FILE* f = a.trace_out.empty() ? stdout : std::fopen(a.trace_out.c_str(), "w");
    dump_trace(f, r, res, g, plat, a);
    if (f != stdout) std::fclose(f);
    delete g;
    return 0;
  }
  if (a.detail >= 0) {
    hesp::SimResult res;
    hesp::TaskGraph* g = nullptr;
    Record r = evaluate(c, static_cast<uint64_t>(a.detail), &res, &g);
    FILE* f = a.detail_out.empty() ? stdout : std::fopen(a.detail_out.c_str(), "w");
    hesp_cand_desc d;
    if (!g_descs.empty()) d = g_descs.at(r.index);
    else hesp_generate(&a.gen, c.s_base_snapped, c.n_base, c.base_b, r.index, &d);
    std::fprintf(f, "index %llu status %d leaves %d makespan %.17g bits %016llx ah %016llx xh %016llx\n",
                 (unsigned long long)r.index, r.status, r.n_leaves, r.makespan,
                 (unsigned long long)bits(r.makespan), (unsigned long long)r.assign_hash,
                 (unsigned long long)r.xfer_hash);
    std::fprintf(f, "ops");
    for (int k = 0; k < d.n_ops; ++k)
      if (d.ops[k].s == HESP_OP_MERGE) std::fprintf(f, " m%d", d.ops[k].task);
      else std::fprintf(f, " %d/%d", d.ops[k].task, d.ops[k].s);
    std::fprintf(f, "\n");
    if (g) {
      for (const auto& [id, blk] : g->data().blocks())
        std::fprintf(f, "B %d %lld %lld %lld %lld %d\n", id, (long long)blk.region.row,
                     (long long)blk.region.col, (long long)blk.region.rows,
                     (long long)blk.region.cols, blk.is_intersection ? 1 : 0);
      for (int id : g->leaf_tasks()) {
        const auto& t = g->task(id);
        std::fprintf(f, "L %d %d %lld r", id, static_cast<int>(t.kind), (long long)t.b);
        for (int b : t.reads) std::fprintf(f, " %d", b);
        std::fprintf(f, " w");
        for (int b : t.writes) std::fprintf(f, " %d", b);
        std::fprintf(f, " p");
        for (int p : g->preds(id)) std::fprintf(f, " %d", p);
        std::fprintf(f, "\n");
      }
      delete g;
    }
    for (const auto& [id, asg] : res.assignments)
      std::fprintf(f, "A %d %d %.17g %.17g %016llx %016llx\n", asg.task, asg.proc, asg.start, asg.end,
                   (unsigned long long)bits(asg.start), (unsigned long long)bits(asg.end));
    for (const auto& x : res.transfers) {
      std::fprintf(f, "X %d %d->%d %lld %.17g %.17g", x.block, x.route.front().first, x.dst_space,
                   (long long)x.bytes, x.start, x.end);
      if (x.fragment)
        std::fprintf(f, " frag %lld %lld %lld %lld", (long long)x.fragment->row,
                     (long long)x.fragment->col, (long long)x.fragment->rows,
                     (long long)x.fragment->cols);
      std::fprintf(f, "\n");
    }
    if (f != stdout) std::fclose(f);
    return 0;
  }

  std::vector<Record> recs(a.count);
  std::vector<char> done(a.count, 0);
  std::atomic<uint64_t> next{0};
  std::atomic<bool> stop{false};
  const auto t0 = std::chrono::steady_clock::now();
  auto worker = [&]() {
    for (;;) {
      if (stop.load(std::memory_order_relaxed)) return;
      const uint64_t k = next.fetch_add(1);
      if (k >= a.count) return;
      recs[k] = evaluate(c, a.first + k, nullptr, nullptr);
      done[k] = 1;
      if (a.time_limit > 0) {
        const double el =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (el > a.time_limit) stop = true;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < a.threads; ++t) pool.emplace_back(worker);
  for (auto& t : pool) t.join();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();

  uint64_t n_done = 0, n_ok = 0;
  std::vector<Record> out;
  out.reserve(a.count);
  for (uint64_t k = 0; k < a.count; ++k)
    if (done[k]) {
      ++n_done;
      n_ok += recs[k].status == 0;
      out.push_back(recs[k]);
    }
  if (!a.out.empty()) {
    FILE* f = std::fopen(a.out.c_str(), "wb");
    const char magic[8] = {'H', 'E', 'S', 'P', 'G', 'L', 'D', '1'};
    std::fwrite(magic, 1, 8, f);
    const uint64_t n = out.size();
    std::fwrite(&n, 8, 1, f);
    std::fwrite(out.data(), sizeof(Record), out.size(), f);
    std::fclose(f);
  }
  if (!a.quiet) {
    std::printf(
        "{\"candidates\": %llu, \"ok\": %llu, \"failed\": %llu, \"wall_s\": %.6f, "
        "\"cand_per_s\": %.6f, \"threads\": %d, \"hw_threads\": %u}\n",
        (unsigned long long)n_done, (unsigned long long)n_ok, (unsigned long long)(n_done - n_ok), wall,
        n_done / wall, a.threads, std::thread::hardware_concurrency());
  }
  return 0;
}
