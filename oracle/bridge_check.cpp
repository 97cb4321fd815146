// bridge_check.cpp — the reference-side C++ binding (include/hesp_b200_bridge.hpp)
// used as a maintainer would: the GPU engine's SimResult, in the reference's
// own hesp:: types, against hesp::simulate of the UNMODIFIED reference on the
// same graph, field by field; and the reference's own verify_schedule applied
// to the GPU result.  TEST INFRASTRUCTURE (needs a GPU; built here, run on the
// GPU box: links oracle/_ref/libhesp_ref.so and the engine library).
#include <cstdio>
#include <cstring>
#include <random>
#include <fstream>
#include <sstream>
#include <string>

#include "hesp/graph.hpp"
#include "hesp/platform.hpp"
#include "hesp/sim.hpp"
#include "hesp_b200_bridge.hpp"
#include "json.hpp"
#include "random_graphs.hpp"  // nlohmann 3.11.3 (the reference's own parser dependency), for the fixture entries

namespace {
std::string slurp(const std::string& p) {
  std::ifstream f(p);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
bool same_events(const hesp::SimResult& a, const hesp::SimResult& b) {
  if (a.events.size() != b.events.size()) return false;
  for (size_t i = 0; i < a.events.size(); ++i) {
    const auto &x = a.events[i], &y = b.events[i];
    if (x.kind != y.kind || std::memcmp(&x.time, &y.time, 8) || x.subject != y.subject || x.resource != y.resource)
      return false;
  }
  return true;
}
bool same(const hesp::SimResult& a, const hesp::SimResult& b, std::string* why) {
  auto eqd = [](double x, double y) { return std::memcmp(&x, &y, 8) == 0; };
  if (!eqd(a.makespan, b.makespan)) return *why = "makespan", false;
  if (a.assignments.size() != b.assignments.size()) return *why = "assignment count", false;
  for (const auto& [id, x] : a.assignments) {
    auto it = b.assignments.find(id);
    if (it == b.assignments.end() || x.proc != it->second.proc || !eqd(x.start, it->second.start) ||
        !eqd(x.end, it->second.end))
      return *why = "assignment " + std::to_string(id), false;
    if (!eqd(a.idle_avg.at(id), b.idle_avg.at(id))) return *why = "idle_avg " + std::to_string(id), false;
  }
  if (a.transfers.size() != b.transfers.size()) return *why = "transfer count", false;
  for (size_t i = 0; i < a.transfers.size(); ++i) {
    const auto &x = a.transfers[i], &y = b.transfers[i];
    if (x.block != y.block || x.route != y.route || !eqd(x.start, y.start) || !eqd(x.end, y.end) ||
        x.bytes != y.bytes || x.dst_space != y.dst_space || x.fragment.has_value() != y.fragment.has_value() ||
        (x.fragment && !(*x.fragment == *y.fragment)))
      return *why = "transfer " + std::to_string(i), false;
  }
  if (!same_events(a, b)) return *why = "events", false;
  if (a.residency_log.size() != b.residency_log.size()) return *why = "residency count", false;
  for (size_t i = 0; i < a.residency_log.size(); ++i) {
    const auto &x = a.residency_log[i], &y = b.residency_log[i];
    if (!eqd(x.time, y.time) || x.space != y.space || x.delta_bytes != y.delta_bytes || x.block != y.block)
      return *why = "residency " + std::to_string(i), false;
  }
  return true;
}
}  // namespace

int main(int argc, char** argv) {
  std::string plat_p, model_p;
  bool csv = false;
  int64_t n = 16384;
  int elem = 4, s_base = 16, count = 8;
  uint64_t first = 0, sseed = 0;
  hesp_gen_config gen{1, 8, 3, 64, 2, {2, 4, 0, 0}, 0};
  std::string ordering = "PL", selection = "EFT-P", caching = "WB";
  int graphs = 0;  // --graphs N: N graphs built by random reference partition/merge/repartition calls
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto v = [&]() { return std::string(argv[++i]); };
    if (k == "--platform") plat_p = v();
    else if (k == "--model") model_p = v();
    else if (k == "--model-csv") { model_p = v(); csv = true; }
    else if (k == "--n") n = std::stoll(v());
    else if (k == "--elem") elem = std::stoi(v());
    else if (k == "--sbase") s_base = std::stoi(v());
    else if (k == "--seed") gen.seed = std::stoull(v());
    else if (k == "--kmax") gen.k_max = std::stoi(v());
    else if (k == "--maxdepth") gen.max_depth = std::stoi(v());
    else if (k == "--min-block") gen.min_block = std::stoll(v());
    else if (k == "--s-choices") {
      std::stringstream ss(v());
      std::string t;
      gen.n_s_choices = 0;
      while (std::getline(ss, t, ',')) gen.s_choices[gen.n_s_choices++] = std::stoi(t);
    } else if (k == "--ordering") ordering = v();
    else if (k == "--selection") selection = v();
    else if (k == "--caching") caching = v();
    else if (k == "--sched-seed") sseed = std::stoull(v());
    else if (k == "--merge-pct") gen.merge_pct = std::stoi(v());
    else if (k == "--first") first = std::stoull(v());
    else if (k == "--count") count = std::stoi(v());
    else if (k == "--threads") v();
    else if (k == "--graphs") graphs = std::stoi(v());
  }
  const auto plat = hesp::Platform::from_json(slurp(plat_p));
  const auto text = slurp(model_p);
  const auto model = csv ? hesp::PerfModel::from_table_csv(text) : hesp::PerfModel::from_analytic_json(text);
  hesp::SchedConfig cfg;
  cfg.ordering = hesp::ordering_from(ordering);
  cfg.selection = hesp::selection_from(selection);
  cfg.caching = hesp::caching_from(caching);
  cfg.seed = sseed;
  cfg.min_block = gen.min_block;
  // the model as the bridge takes it: the fixture's own entries
  std::vector<hesp::b200::AnalyticEntry> an;
  std::vector<hesp::b200::TableRow> tab;
  if (csv) {
    std::stringstream ss(text);
    std::string line;
    std::getline(ss, line);
    while (std::getline(ss, line)) {
      if (line.find_first_not_of(" \r\t") == std::string::npos) continue;
      std::stringstream ls(line);
      std::string kd, ty, b, sec;
      std::getline(ls, kd, ',');
      std::getline(ls, ty, ',');
      std::getline(ls, b, ',');
      std::getline(ls, sec, ',');
      auto trim = [](std::string x) {
        x.erase(0, x.find_first_not_of(" \t"));
        x.erase(x.find_last_not_of(" \t\r") + 1);
        return x;
      };
      tab.emplace_back(hesp::task_kind_from(trim(kd)), trim(ty), std::stoll(trim(b)), std::stod(trim(sec)));
    }
  } else {
    const auto j = nlohmann::json::parse(text);
    for (const auto& e : j)
      an.emplace_back(hesp::task_kind_from(e["kind"].get<std::string>()), e["proc_type"].get<std::string>(),
                      e["peak_flops"].get<double>(), e["b_half"].get<double>());
  }
  hesp::b200::BatchSimulator gpu(plat, an, tab, cfg, n, elem, s_base, gen);
  if (graphs > 0) {
    // The TaskGraph drop-in: graphs built by arbitrary sequences of the
    // reference's own mutators (partition_task / merge_cluster incl. the base
    // cluster / repartition_cluster; failing calls leave the graph as is),
    // simulated by hesp::simulate and by BatchSimulator::simulate(graph), and
    // batch-evaluated by BatchSimulator::evaluate(graphs).
    oracle::GraphStats gst_;
    std::vector<hesp::TaskGraph> gs =
        oracle::random_graphs(graphs, n, elem, s_base, gen.min_block, gen.seed * 7919 + first, &gst_);
    const int calls = gst_.calls, base_merges = gst_.top_merges;
    int ok = 0, failed = 0, bad = 0, unrepro = 0;
    std::vector<int> ref_status(gs.size(), 0);
    std::vector<double> ref_mk(gs.size(), 0.0);
    for (std::size_t i = 0; i < gs.size(); ++i) {
      hesp::SimResult ref, mine;
      int gst = 0;
      try {
        ref = hesp::simulate(gs[i], plat, model, cfg);
        ref_mk[i] = ref.makespan;
      } catch (const hesp::Error& e) {
        ref_status[i] = 1 + static_cast<int>(e.code());
      }
      try {
        mine = gpu.simulate(gs[i]);
      } catch (const hesp::Error& e) {
        gst = 1 + static_cast<int>(e.code());
      }
      if (gst == 1 + static_cast<int>(hesp::Err::Internal) && ref_status[i] != gst) {
        ++unrepro;  // the bridge refused: history not reproducible by the replay (explicit, never a wrong result)
        continue;
      }
      if (ref_status[i] || gst) {
        ++failed;
        if (ref_status[i] != gst) {
          ++bad;
          const hesp_cand_desc d = gpu.describe(gs[i]);
          std::printf("graph %zu: status ref %d gpu %d; ops", i, ref_status[i], gst);
          for (int k = 0; k < d.n_ops; ++k) std::printf(" (%d,%d)", d.ops[k].task, d.ops[k].s);
          std::printf("\n");
        }
        continue;
      }
      std::string why;
      if (!same(ref, mine, &why)) {
        ++bad;
        std::printf("graph %zu: %s differs\n", i, why.c_str());
        continue;
      }
      if (hesp::verify_schedule(mine, gs[i], plat) != hesp::verify_schedule(ref, gs[i], plat)) {
        ++bad;
        std::printf("graph %zu: verify_schedule differs\n", i);
        continue;
      }
      ++ok;
    }
    hesp_best best{};
    const auto out = gpu.evaluate(gs, &best);
    int unrepro_batch = 0;
    for (std::size_t i = 0; i < gs.size(); ++i) {
      if (out[i].status == HESP_ST_UNREPRODUCIBLE) {
        ++unrepro_batch;
        continue;
      }
      if (out[i].status != ref_status[i] || std::memcmp(&out[i].makespan, &ref_mk[i], 8)) {
        ++bad;
        std::printf("graph %zu: evaluate gives status %d makespan %.17g, reference %d %.17g\n", i, out[i].status,
                    out[i].makespan, ref_status[i], ref_mk[i]);
      }
    }
    if (unrepro_batch != unrepro) {
      ++bad;
      std::printf("simulate refused %d graphs, evaluate %d\n", unrepro, unrepro_batch);
    }
    std::printf("bridge_check graphs: %d graphs (%d mutator calls, %d merges of the top cluster, %d redrawn after a "
                "reference defect), %d identical SimResults, %d failing in both, %d refused as unreproducible, "
                "mismatches %d\n",
                graphs, calls, base_merges, gst_.dropped, ok, failed, unrepro, bad);
    return bad ? 1 : 0;
  }
  auto g0 = hesp::TaskGraph::root_cholesky(n, elem);
  const int cl = g0.partition_task(0, 1.0 / s_base, gen.min_block);
  const int n_base = (int)g0.cluster(cl).members.size();
  const int64_t base_b = g0.task(g0.cluster(cl).members.front()).b;
  int bad = 0, ok = 0, failed = 0;
  for (uint64_t c = first; c < first + (uint64_t)count; ++c) {
    hesp_cand_desc d;
    hesp_generate(&gen, (int32_t)(n / base_b), n_base, base_b, c, &d);
    hesp::SimResult ref;
    int ref_status = 0;
    hesp::TaskGraph g = g0;
    try {
      for (int k = 0; k < d.n_ops; ++k) {
        if (d.ops[k].s == HESP_OP_MERGE) g.merge_cluster(d.ops[k].task);
        else g.partition_task(d.ops[k].task, 1.0 / d.ops[k].s, gen.min_block);
      }
      ref = hesp::simulate(g, plat, model, cfg);
    } catch (const hesp::Error& e) {
      ref_status = 1 + static_cast<int>(e.code());
    }
    int gpu_status = 0;
    hesp::SimResult mine;
    try {
      mine = gpu.simulate(d, elem);
    } catch (const hesp::Error& e) {
      gpu_status = 1 + static_cast<int>(e.code());
    }
    if (ref_status || gpu_status) {
      ++failed;
      if (ref_status != gpu_status) {
        ++bad;
        std::printf("cand %llu: status ref %d gpu %d\n", (unsigned long long)c, ref_status, gpu_status);
      }
      continue;
    }
    std::string why;
    if (!same(ref, mine, &why)) {
      ++bad;
      std::printf("cand %llu: %s differs\n", (unsigned long long)c, why.c_str());
      continue;
    }
    // the reference's own verifier on the GPU result
    if (hesp::verify_schedule(mine, g, plat) != hesp::verify_schedule(ref, g, plat)) {
      ++bad;
      std::printf("cand %llu: verify_schedule differs\n", (unsigned long long)c);
      continue;
    }
    ++ok;
  }
  std::printf("bridge_check: %d candidates, %d identical SimResults, %d failing in both, mismatches %d\n", count, ok,
              failed, bad);
  return bad ? 1 : 0;
}
