// engine_check.cpp — TEST INFRASTRUCTURE: runs the engine's width-1 host
// instantiation (paper_1602_05510_b200/csrc/engine.h, Engine<HostWarp>) and
// the unmodified reference (oracle/_ref/libhesp_ref.so) on the same
// candidates and reports the first mismatches with per-task detail.  Used
// to develop the engine on a CPU; the GPU parity tests compare the CUDA
// instantiation against golden records produced by ref_harness.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "engine.h"
#include "hesp/graph.hpp"
#include "hesp/platform.hpp"
#include "hesp/sim.hpp"
#include "json.hpp"
#include "problem.h"
#include "hesp_b200_bridge.hpp"
#include "random_graphs.hpp"

using nlohmann::json;

static std::string slurp(const std::string& path) {
  std::ifstream f(path);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
static uint64_t bits(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}
static int kind_of(const std::string& k) {
  return k == "CHOL" ? 0 : k == "TRSM" ? 1 : k == "SYRK" ? 2 : 3;
}

int main(int argc, char** argv) {
  std::string platform, modelp;
  bool csv = false;
  long long n = 16384;
  int elem = 4, s_base = 16;
  hesp_gen_config gen{};
  gen.seed = 1;
  gen.k_max = 8;
  gen.max_depth = 3;
  gen.min_block = 64;
  gen.n_s_choices = 2;
  gen.s_choices[0] = 2;
  gen.s_choices[1] = 4;
  std::string ordering = "PL", selection = "EFT-P", caching = "WB";
  unsigned long long first = 0, count = 100, sseed = 0;
  int verbose = 0;
  std::string descs_path;  // --descs: explicit candidates (520-byte hesp_cand_desc records)
  int graphs = 0;          // --graphs N: random reference TaskGraphs through the bridge's replay plan
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto v = [&]() { return std::string(argv[++i]); };
    if (k == "--platform") platform = v();
    else if (k == "--model") modelp = v();
    else if (k == "--model-csv") { modelp = v(); csv = true; }
    else if (k == "--n") n = std::stoll(v());
    else if (k == "--elem") elem = std::stoi(v());
    else if (k == "--sbase") s_base = std::stoi(v());
    else if (k == "--seed") gen.seed = std::stoull(v(), nullptr, 0);
    else if (k == "--kmax") gen.k_max = std::stoi(v());
    else if (k == "--maxdepth") gen.max_depth = std::stoi(v());
    else if (k == "--min-block") gen.min_block = std::stoll(v());
    else if (k == "--s-choices") {
      std::string s = v();
      gen.n_s_choices = 0;
      std::stringstream ss(s);
      std::string tok;
      while (std::getline(ss, tok, ',')) gen.s_choices[gen.n_s_choices++] = std::stoi(tok);
    } else if (k == "--ordering") ordering = v();
    else if (k == "--selection") selection = v();
    else if (k == "--caching") caching = v();
    else if (k == "--sched-seed") sseed = std::stoull(v());
    else if (k == "--merge-pct") gen.merge_pct = std::stoi(v());
    else if (k == "--first") first = std::stoull(v());
    else if (k == "--count") count = std::stoull(v());
    else if (k == "--verbose") verbose = std::stoi(v());
    else if (k == "--descs") descs_path = v();
    else if (k == "--graphs") graphs = std::stoi(v());
    else {
      std::fprintf(stderr, "unknown arg %s\n", k.c_str());
      return 2;
    }
  }
  // ---- reference objects
  const auto rplat = hesp::Platform::from_json(slurp(platform));
  const auto rmodel = csv ? hesp::PerfModel::from_table_csv(slurp(modelp))
                          : hesp::PerfModel::from_analytic_json(slurp(modelp));
  hesp::SchedConfig rcfg;
  rcfg.ordering = hesp::ordering_from(ordering);
  rcfg.selection = hesp::selection_from(selection);
  rcfg.caching = hesp::caching_from(caching);
  rcfg.seed = sseed;
  rcfg.min_block = gen.min_block;
  // ---- engine inputs (C-ABI structs) from the same files
  json pj = json::parse(slurp(platform));
  std::vector<hesp_space> spaces;
  for (auto& s : pj["spaces"])
    spaces.push_back({s["id"].get<int>(), s["capacity_bytes"].get<long long>(), s.value("is_main", false) ? 1 : 0});
  std::vector<std::string> tnames;
  for (auto& t : pj["types"]) tnames.push_back(t["name"].get<std::string>());
  std::vector<const char*> tptr;
  for (auto& t : tnames) tptr.push_back(t.c_str());
  auto tindex = [&](const std::string& nm) {
    for (size_t i = 0; i < tnames.size(); ++i)
      if (tnames[i] == nm) return (int)i;
    return -1;
  };
  std::vector<hesp_processor> procs;
  for (auto& p : pj["processors"])
    procs.push_back({p["id"].get<int>(), tindex(p["type"].get<std::string>()), p["space"].get<int>()});
  std::vector<hesp_link> links;
  if (pj.contains("links"))
    for (auto& l : pj["links"])
      links.push_back({l["src"].get<int>(), l["dst"].get<int>(), l["latency_s"].get<double>(),
                       l["bandwidth_Bps"].get<double>()});
  hesp_platform hplat{(int)spaces.size(), spaces.data(), (int)tnames.size(), tptr.data(),
                      (int)procs.size(), procs.data(), (int)links.size(), links.data()};
  std::vector<hesp_analytic_entry> ents;
  std::vector<hesp_table_row> rows;
  hesp_perf_model hmodel{};
  if (!csv) {
    json mj = json::parse(slurp(modelp));
    for (auto& e : mj) {
      int ti = tindex(e["proc_type"].get<std::string>());
      if (ti < 0) continue;
      ents.push_back({kind_of(e["kind"].get<std::string>()), ti, e["peak_flops"].get<double>(),
                      e["b_half"].get<double>()});
    }
    hmodel.variant = HESP_MODEL_ANALYTIC;
    hmodel.n_entries = (int)ents.size();
    hmodel.entries = ents.data();
  } else {
    std::stringstream ss(slurp(modelp));
    std::string line;
    std::getline(ss, line);
    while (std::getline(ss, line)) {
      if (line.empty()) continue;
      std::stringstream ls(line);
      std::string kk, tt, bb, sec;
      std::getline(ls, kk, ',');
      std::getline(ls, tt, ',');
      std::getline(ls, bb, ',');
      std::getline(ls, sec, ',');
      int ti = tindex(tt);
      if (ti < 0) continue;
      rows.push_back({kind_of(kk), ti, std::stoll(bb), std::stod(sec)});
    }
    hmodel.variant = HESP_MODEL_TABULATED;
    hmodel.n_rows = (int)rows.size();
    hmodel.rows = rows.data();
  }
  auto sel_of = [](const std::string& s) {
    return s == "R-P" ? 0 : s == "F-P" ? 1 : s == "EIT-P" ? 2 : 3;
  };
  hesp_sched_config hs{ordering == "PL" ? 1 : 0, sel_of(selection),
                       caching == "WT" ? 0 : caching == "WB" ? 1 : 2, 0, sseed, gen.min_block};
  hesp_workload wl{n, elem, s_base, gen};
  hx::HostProblem hp = hx::build_problem(hplat, hmodel, hs, wl);
  hx::bind_tilings(hp.p, hp, hp.base_tasks.data(), hp.base_blocks.data(), hp.base_preds.data(),
                   hp.base_plist.data());
  const hx::SlotLayout L = hp.p.lay;
  std::vector<uint8_t> slot(L.total);
  hx::Small sm{};
  std::printf("base: tasks %d blocks %d slot %zu bytes, bvals %d\n", hp.p.n_base_tasks,
              hp.p.n_base_blocks, L.total, hp.p.nbv);

  std::vector<hesp_cand_desc> descs;
  std::vector<hesp::TaskGraph> gs;
  if (graphs > 0) {  // BatchSimulator::simulate(const TaskGraph&)'s replay, on the host engine
    oracle::GraphStats gst;
    gs = oracle::random_graphs(graphs, n, elem, s_base, gen.min_block, gen.seed * 7919 + first, &gst);
    const int s0 = (int)hesp_snap_tiles(n, s_base, gen.min_block);
    for (const auto& g : gs)
      descs.push_back(hesp::b200::plan_graph(g, n, elem, s0, hp.p.n_base_tasks, hp.p.n_base_blocks).desc);
    first = 0;
    count = descs.size();
  } else if (!descs_path.empty()) {
    const std::string raw = slurp(descs_path);
    descs.resize(raw.size() / sizeof(hesp_cand_desc));
    std::memcpy(descs.data(), raw.data(), descs.size() * sizeof(hesp_cand_desc));
    first = 0;
    count = descs.size();
  }
  double t_eng = 0, t_ref = 0;
  int bad = 0, ok_both = 0;
  std::map<int, int> hist;
  for (unsigned long long c = first; c < first + count; ++c) {
    hesp_cand_desc d;
    if (!descs.empty()) d = descs[c];
    else hesp_generate(&gen, (int)(n / hp.p.base_b), hp.p.n_base_leaves, hp.p.base_b, c, &d);
    auto t0 = std::chrono::steady_clock::now();
    hx::Engine<hx::HostWarp> eng(hx::HostWarp{}, hp.p, slot.data(), &sm);
    std::vector<double> tr_s, tr_e;
    std::vector<int> tr_p;
    const hx::Outcome o = eng.run(d);
    auto t1 = std::chrono::steady_clock::now();
    // reference
    int rstatus = 0, rleaves = 0;
    double rmk = 0;
    uint64_t rah = 0, rxh = 0;
    hesp::SimResult res;
    std::map<int, std::vector<int>> rpreds;
    try {
      auto g = hesp::TaskGraph::root_cholesky(n, elem);
      if (!gs.empty()) {
        g = gs[c];  // the caller's own graph (ids differ from the replay's: compare id-free fields)
      } else {
        g.partition_task(0, 1.0 / s_base, gen.min_block);
        for (int k = 0; k < d.n_ops; ++k) {
          if (d.ops[k].s == HESP_OP_MERGE) g.merge_cluster(d.ops[k].task);
          else g.partition_task(d.ops[k].task, 1.0 / d.ops[k].s, gen.min_block);
        }
      }
      rleaves = (int)g.leaf_tasks().size();
      res = hesp::simulate(g, rplat, rmodel, rcfg);
      rmk = res.makespan;
      for (auto& [id, a] : res.assignments) rah += hesp_assign_term(a.task, a.proc, bits(a.start), bits(a.end));
      for (auto& x : res.transfers) {
        long long fr = 0, fc = 0, frs = 0, fcs = 0;
        if (x.fragment) {
          fr = x.fragment->row;
          fc = x.fragment->col;
          frs = x.fragment->rows;
          fcs = x.fragment->cols;
        }
        rxh += hesp_xfer_term(x.block, x.route.front().first, x.dst_space, x.bytes, bits(x.start),
                              bits(x.end), fr, fc, frs, fcs);
      }
    } catch (const hesp::Error& e) {
      rstatus = 1 + (int)e.code();
      rmk = 0;
      rah = rxh = 0;
    } catch (const std::exception& e) {
      rstatus = 100;
    }
    auto t2 = std::chrono::steady_clock::now();
    t_eng += std::chrono::duration<double>(t1 - t0).count();
    t_ref += std::chrono::duration<double>(t2 - t1).count();
    hist[o.status]++;
    const bool same = o.status == rstatus && o.n_leaves == rleaves && bits(o.makespan) == bits(rmk) &&
                      (!gs.empty() || (o.assign_hash == rah && o.xfer_hash == rxh));
    if (same) {
      ok_both += rstatus == 0;
      continue;
    }
    ++bad;
    if (bad <= 5 || verbose) {
      if (!gs.empty()) {
        std::printf("graph %llu ops", c);
        for (int k = 0; k < d.n_ops; ++k) std::printf(" (%d,%d)", d.ops[k].task, d.ops[k].s);
        std::printf("; clusters");
        for (const auto& [id, cl] : gs[c].clusters()) std::printf(" %d:%d/%.4g", id, cl.parent_task, 1.0 / cl.p);
        std::printf("\n");
      }
      std::printf("MISMATCH cand %llu ops=%d: eng st=%d leaves=%d mk=%.17g ah=%016llx xh=%016llx | ref st=%d leaves=%d mk=%.17g ah=%016llx xh=%016llx\n",
                  c, d.n_ops, o.status, o.n_leaves, o.makespan, (unsigned long long)o.assign_hash,
                  (unsigned long long)o.xfer_hash, rstatus, rleaves, rmk, (unsigned long long)rah,
                  (unsigned long long)rxh);
    }
  }
  std::printf("checked %llu: mismatches %d, both-ok %d; engine(host, 1 lane) %.3f ms/cand, reference %.3f ms/cand\n",
              count, bad, ok_both, 1e3 * t_eng / count, 1e3 * t_ref / count);
  std::printf("status histogram:");
  for (auto& [k, v] : hist) std::printf(" %d:%d", k, v);
  std::printf("\n");
  return bad ? 1 : 0;
}
