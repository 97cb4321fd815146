// port_harness.cpp — drives the CPU restatement (oracle/port) over a batch of
// candidates with the same CLI and 40-byte record format as ref_harness.
// TEST INFRASTRUCTURE ONLY (golden pinning of the port; optional "port" CPU baseline).
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "json.hpp"
#include "port/hesp_port.h"

namespace {
struct Record {
  uint64_t index;
  int32_t status, n_leaves;
  double makespan;
  uint64_t assign_hash, xfer_hash;
};
std::string slurp(const std::string& p) {
  std::ifstream f(p);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}
int kind_of(const std::string& k) { return k == "CHOL" ? 0 : k == "TRSM" ? 1 : k == "SYRK" ? 2 : 3; }
}  // namespace

int main(int argc, char** argv) {
  std::string platform, model, out, descs_path, ordering = "PL", selection = "EFT-P", caching = "WB";
  bool csv = false;
  long long n = 16384, first = 0, count = 10;
  int elem = 4, s_base = 16, threads = 1;
  double time_limit = 0;
  hesp_gen_config gen{};
  gen.seed = 1;
  gen.k_max = 8;
  gen.max_depth = 3;
  gen.min_block = 64;
  gen.n_s_choices = 2;
  gen.s_choices[0] = 2;
  gen.s_choices[1] = 4;
  port::Sched sched;
  for (int i = 1; i < argc; ++i) {
    std::string k = argv[i];
    auto v = [&]() { return std::string(argv[++i]); };
    if (k == "--platform") platform = v();
    else if (k == "--model") model = v();
    else if (k == "--model-csv") { model = v(); csv = true; }
    else if (k == "--n") n = std::stoll(v());
    else if (k == "--elem") elem = std::stoi(v());
    else if (k == "--sbase") s_base = std::stoi(v());
    else if (k == "--seed") gen.seed = std::stoull(v(), nullptr, 0);
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
    else if (k == "--sched-seed") sched.seed = std::stoull(v());
    else if (k == "--merge-pct") {
      gen.merge_pct = std::stoi(v());
      if (gen.merge_pct) {
        std::fprintf(stderr, "port_harness: merge ops are not restated in oracle/port (partitions only)\n");
        return 2;
      }
    }
    else if (k == "--first") first = std::stoll(v());
    else if (k == "--count") count = std::stoll(v());
    else if (k == "--threads") threads = std::stoi(v());
    else if (k == "--time-limit") time_limit = std::stod(v());
    else if (k == "--out") out = v();
    else if (k == "--quiet") {}
    else if (k == "--descs") descs_path = v();
    else {
      std::fprintf(stderr, "unknown argument %s\n", k.c_str());
      return 2;
    }
  }
  if (threads <= 0) threads = static_cast<int>(std::thread::hardware_concurrency());
  sched.ordering = ordering == "PL" ? 1 : 0;
  sched.selection = selection == "R-P" ? 0 : selection == "F-P" ? 1 : selection == "EIT-P" ? 2 : 3;
  sched.caching = caching == "WT" ? 0 : caching == "WB" ? 1 : 2;
  sched.min_block = gen.min_block;
  port::Platform plat;
  auto pj = nlohmann::json::parse(slurp(platform));
  for (auto& s : pj["spaces"]) plat.spaces.push_back({s["id"].get<int>(), s["capacity_bytes"].get<long long>(), s.value("is_main", false)});
  std::sort(plat.spaces.begin(), plat.spaces.end(), [](auto& a, auto& b) { return a.id < b.id; });
  for (auto& t : pj["types"]) plat.types.push_back(t["name"].get<std::string>());
  for (auto& p : pj["processors"]) {
    const std::string tn = p["type"].get<std::string>();
    const int ti = static_cast<int>(std::find(plat.types.begin(), plat.types.end(), tn) - plat.types.begin());
    plat.procs.push_back({p["id"].get<int>(), ti, p["space"].get<int>()});
  }
  std::sort(plat.procs.begin(), plat.procs.end(), [](auto& a, auto& b) { return a.id < b.id; });
  if (pj.contains("links"))
    for (auto& l : pj["links"]) plat.links.push_back({l["src"].get<int>(), l["dst"].get<int>(), l["latency_s"].get<double>(), l["bandwidth_Bps"].get<double>()});
  port::Model mdl;
  if (!csv) {
    for (auto& e : nlohmann::json::parse(slurp(model)))
      mdl.entries.push_back({kind_of(e["kind"].get<std::string>()), e["proc_type"].get<std::string>(), e["peak_flops"].get<double>(), e["b_half"].get<double>()});
  } else {
    mdl.analytic = false;
    std::stringstream ss(slurp(model));
    std::string line;
    std::getline(ss, line);
    while (std::getline(ss, line)) {
      if (line.empty()) continue;
      std::stringstream ls(line);
      std::string a, b, c, d;
      std::getline(ls, a, ',');
      std::getline(ls, b, ',');
      std::getline(ls, c, ',');
      std::getline(ls, d, ',');
      mdl.rows.push_back({kind_of(a), b, std::stoll(c), std::stod(d)});
    }
  }
  // base tiling facts for the generator (partition of the root, graph.cpp:464-481)
  const long long s0 = hesp_snap_tiles(n, s_base, gen.min_block);
  const long long base_b = n / s0;
  const int n_base = hesp_member_count(HESP_CHOL, static_cast<int>(s0));
  std::vector<hesp_cand_desc> explicit_descs;
  if (!descs_path.empty()) {
    std::ifstream f(descs_path, std::ios::binary);
    hesp_cand_desc d;
    while (f.read(reinterpret_cast<char*>(&d), sizeof d)) explicit_descs.push_back(d);
    first = 0;
    count = static_cast<long long>(explicit_descs.size());
  }
  std::vector<Record> recs(count);
  std::vector<char> done(count, 0);
  std::atomic<long long> next{0};
  std::atomic<bool> stop{false};
  const auto t0 = std::chrono::steady_clock::now();
  auto work = [&]() {
    for (;;) {
      if (stop) return;
      const long long k = next++;
      if (k >= count) return;
      hesp_cand_desc d;
      if (!explicit_descs.empty()) d = explicit_descs[k];
      else hesp_generate(&gen, static_cast<int>(s0), n_base, base_b, first + k, &d);
      const port::Result r = port::evaluate(plat, mdl, sched, n, elem, s_base, d);
      recs[k] = Record{static_cast<uint64_t>(first + k), r.status, r.leaves, r.status ? 0.0 : r.makespan,
                       r.status ? 0 : r.ahash, r.status ? 0 : r.xhash};
      done[k] = 1;
      if (time_limit > 0 && std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > time_limit)
        stop = true;
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(work);
  for (auto& t : pool) t.join();
  const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::vector<Record> keep;
  long long ok = 0;
  for (long long k = 0; k < count; ++k)
    if (done[k]) {
      keep.push_back(recs[k]);
      ok += recs[k].status == 0;
    }
  if (!out.empty()) {
    FILE* f = std::fopen(out.c_str(), "wb");
    std::fwrite("HESPGLD1", 1, 8, f);
    const uint64_t m = keep.size();
    std::fwrite(&m, 8, 1, f);
    std::fwrite(keep.data(), sizeof(Record), keep.size(), f);
    std::fclose(f);
  }
  std::printf("{\"candidates\": %zu, \"ok\": %lld, \"failed\": %lld, \"wall_s\": %.6f, \"cand_per_s\": %.6f, \"threads\": %d}\n",
              keep.size(), ok, static_cast<long long>(keep.size()) - ok, wall, keep.size() / wall, threads);
  return 0;
}
