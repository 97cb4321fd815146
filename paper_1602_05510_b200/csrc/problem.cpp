// problem.cpp — validates the reference-shaped inputs and precomputes the
// read-only tables the device engine consumes:
//   * task_time(kind, b, type) for every block side a candidate can reach
//     (PerfModel::task_time restated, platform.cpp:347-390; log/exp of the
//     tabulated interpolation are evaluated here, never on the device);
//   * critical_times' per-task mean over processors (sim.cpp:96-106);
//   * transfer routes (transfer_time, platform.cpp:198-220);
//   * the base tiling partition_task(0, 1/s_base) (graph.cpp:456-513), built
//     once with the width-1 instantiation of the engine itself.
#include "problem.h"

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <map>
#include <set>
#include <stdexcept>

#include "engine.h"

namespace hx {

namespace {

double flops(int kind, long long b) {  // task_flops, platform.cpp:57-66
  const double bd = static_cast<double>(b);
  switch (kind) {
    case HESP_CHOL: return bd * bd * bd / 3.0;
    case HESP_TRSM: return bd * bd * bd;
    case HESP_SYRK: return bd * bd * bd;
    default: return 2.0 * bd * bd * bd;
  }
}

[[noreturn]] void bad(const std::string& m) { throw std::runtime_error(m); }

}  // namespace

double host_task_time(const hesp_perf_model& m, int kind, long long b, int type, bool* known) {
  *known = false;
  if (m.variant == HESP_MODEL_ANALYTIC) {
    for (int i = 0; i < m.n_entries; ++i) {
      const auto& e = m.entries[i];
      if (e.kind != kind || e.type != type) continue;
      *known = true;
      const double eff = static_cast<double>(b) / (static_cast<double>(b) + e.b_half);
      return flops(kind, b) / (e.peak_flops * eff);
    }
    return 0.0;
  }
  std::map<long long, double> per;  // b ascending
  for (int i = 0; i < m.n_rows; ++i) {
    const auto& r = m.rows[i];
    if (r.kind == kind && r.type == type) per[r.b] = r.seconds;
  }
  if (per.empty()) return 0.0;
  *known = true;
  auto ex = per.find(b);
  if (ex != per.end()) return ex->second;
  auto rate_at = [&](std::map<long long, double>::const_iterator it) {
    return flops(kind, it->first) / it->second;
  };
  auto hi = per.upper_bound(b);
  double rate;
  if (hi == per.begin()) {
    rate = rate_at(hi);
  } else if (hi == per.end()) {
    rate = rate_at(std::prev(hi));
  } else {
    auto lo = std::prev(hi);
    const double lb = std::log(static_cast<double>(lo->first));
    const double hb = std::log(static_cast<double>(hi->first));
    const double lr = std::log(rate_at(lo));
    const double hr = std::log(rate_at(hi));
    const double t = (std::log(static_cast<double>(b)) - lb) / (hb - lb);
    rate = std::exp(lr + t * (hr - lr));
  }
  return flops(kind, b) / rate;
}

HostProblem build_problem(const hesp_platform& plat, const hesp_perf_model& model,
                          const hesp_sched_config& sched, const hesp_workload& wl) {
  HostProblem hp;
  Problem& p = hp.p;
  // ---------------- platform (Platform::make / validate) ----------------
  if (plat.n_spaces < 1 || plat.n_spaces > MAXS) bad("platform: 1..8 memory spaces supported");
  if (plat.n_types < 1 || plat.n_types > MAXTYPES) bad("platform: 1..8 processor types supported");
  if (plat.n_procs < 1) bad("platform has no processors");
  if (plat.n_procs > MAXP) bad("platform: at most 32 processors (one warp lane each)");
  std::vector<int> ids;
  int mains = 0, main_id = 0;
  for (int i = 0; i < plat.n_spaces; ++i) {
    const auto& s = plat.spaces[i];
    if (s.capacity_bytes <= 0) bad("space has nonpositive capacity");
    if (std::find(ids.begin(), ids.end(), s.id) != ids.end()) bad("duplicate space id");
    ids.push_back(s.id);
    if (s.is_main) {
      ++mains;
      main_id = s.id;
    }
  }
  if (mains != 1) bad("platform must have exactly one main space");
  std::vector<int> sorted_ids = ids;
  std::sort(sorted_ids.begin(), sorted_ids.end());  // engine index = rank of the id (map order)
  auto sidx = [&](int id) {
    auto it = std::find(sorted_ids.begin(), sorted_ids.end(), id);
    if (it == sorted_ids.end()) bad("unknown space id");
    return static_cast<int>(it - sorted_ids.begin());
  };
  p.S = plat.n_spaces;
  p.main_space = sidx(main_id);
  for (int i = 0; i < plat.n_spaces; ++i) p.cap[sidx(plat.spaces[i].id)] = plat.spaces[i].capacity_bytes;
  {
    std::set<std::string> names;
    for (int i = 0; i < plat.n_types; ++i)
      if (!names.insert(plat.type_names[i]).second) bad("duplicate processor type");
  }
  p.n_types = plat.n_types;
  p.P = plat.n_procs;
  std::vector<hesp_processor> procs(plat.procs, plat.procs + plat.n_procs);
  std::sort(procs.begin(), procs.end(), [](auto& a, auto& b) { return a.id < b.id; });
  for (int i = 0; i < p.P; ++i) {
    if (procs[i].id != i) bad("processor ids must be dense 0..P-1");
    if (procs[i].type < 0 || procs[i].type >= p.n_types) bad("processor has unknown type");
    p.proc_type[i] = procs[i].type;
    p.proc_space[i] = sidx(procs[i].space);
  }
  if (plat.n_links > MAXL) bad("too many links");
  std::map<std::pair<int, int>, int> lidx;
  for (int i = 0; i < plat.n_links; ++i) {
    const auto& l = plat.links[i];
    const int a = sidx(l.src), b = sidx(l.dst);
    if (a == b) bad("link with src == dst");
    if (l.latency_s < 0) bad("negative link latency");
    if (l.bandwidth_bps <= 0) bad("nonpositive link bandwidth");
    if (lidx.count({a, b})) bad("duplicate link");
    lidx[{a, b}] = i;
    p.link_lat[i] = l.latency_s;
    p.link_bw[i] = l.bandwidth_bps;
    p.link_src[i] = a;
    p.link_dst[i] = b;
  }
  p.L = plat.n_links;
  for (int s = 0; s < p.S; ++s)
    if (s != p.main_space && (!lidx.count({s, p.main_space}) || !lidx.count({p.main_space, s})))
      bad("a space is missing a link to or from the main space");
  for (int a = 0; a < p.S; ++a)
    for (int b = 0; b < p.S; ++b) {
      int* r = p.route_l[a * MAXS + b];
      p.route_n[a * MAXS + b] = 0;
      if (a == b) continue;
      if (lidx.count({a, b})) {
        p.route_n[a * MAXS + b] = 1;
        r[0] = lidx[{a, b}];
      } else if (lidx.count({a, p.main_space}) && lidx.count({p.main_space, b})) {
        p.route_n[a * MAXS + b] = 2;
        r[0] = lidx[{a, p.main_space}];
        r[1] = lidx[{p.main_space, b}];
      }
    }

  // ---------------- model validation ----------------
  if (model.variant == HESP_MODEL_ANALYTIC) {
    std::set<std::pair<int, int>> seen;
    for (int i = 0; i < model.n_entries; ++i) {
      const auto& e = model.entries[i];
      if (e.peak_flops <= 0) bad("analytic model: peak_flops must be positive");
      if (e.b_half <= 0) bad("analytic model: b_half must be positive");
      if (!seen.insert({e.kind, e.type}).second) bad("analytic model: duplicate entry");
    }
  } else {
    std::set<std::tuple<int, int, long long>> seen;
    for (int i = 0; i < model.n_rows; ++i) {
      const auto& r = model.rows[i];
      if (r.b < 1) bad("perf table: b must be >= 1");
      if (r.seconds <= 0) bad("perf table: nonpositive time");
      if (!seen.insert({r.kind, r.type, r.b}).second) bad("perf table: duplicate entry");
    }
  }

  // ---------------- workload ----------------
  if (wl.n < 1) bad("matrix side must be >= 1");
  if (wl.elem_size < 1) bad("element size must be >= 1");
  if (wl.n >= (1LL << 30)) bad("matrix side must be < 2^30");
  if (wl.s_base < 2) bad("s_base must be >= 2");
  if (wl.gen.k_max < 0 || wl.gen.k_max > HESP_GEN_MAX_OPS) bad("k_max must lie in [0, 16]");
  if (wl.gen.n_s_choices < 1 || wl.gen.n_s_choices > 4) bad("1..4 s choices");
  if (sched.min_block != wl.gen.min_block) bad("sched.min_block must equal gen.min_block");
  p.n = wl.n;
  p.elem = wl.elem_size;
  p.s_base = wl.s_base;
  p.min_block = wl.gen.min_block;
  p.gen = wl.gen;
  p.ordering = sched.ordering;
  p.selection = sched.selection;
  p.caching = sched.caching;
  p.sched_seed = sched.seed;
  p.loop = 0;
  if (const char* lv = std::getenv("HESP_LOOP")) p.loop = std::atoi(lv);
  if (p.ordering < 0 || p.ordering > 1 || p.selection < 0 || p.selection > 3 || p.caching < 0 ||
      p.caching > 2)
    bad("unknown scheduling policy");

  // block sides reachable from n: the base tiling, then any requested split
  const long long s0 = hesp_snap_tiles(wl.n, wl.s_base, wl.gen.min_block);
  if (s0 == 0) bad("base tiling: no tiling of the root with tiles >= min_block");
  // Top-level tilings besides the base one (a candidate reaches them by
  // merging the base cluster and partitioning the root again): every tile
  // count the root snaps to whose tiling fits the slot next to the base's
  // share.  The base's caps follow below; the same K * smax^3 headroom holds.
  int smax_ = 2;
  for (int i = 0; i < wl.gen.n_s_choices; ++i) smax_ = std::max(smax_, wl.gen.s_choices[i]);
  smax_ += 1;
  const long long nbt0 = 1 + hesp_member_count(HESP_CHOL, static_cast<int>(s0));
  const long long maxt0 = nbt0 + std::max(1, wl.gen.k_max) * (long long)smax_ * smax_ * smax_ + 64;
  std::vector<int> extra_s;
  for (long long s = 2; s <= wl.n / std::max<long long>(1, wl.gen.min_block); ++s) {
    if (wl.n % s || s == s0) continue;
    if (1 + hesp_member_count(HESP_CHOL, static_cast<int>(std::min<long long>(s, 4096))) > std::max(nbt0, maxt0 / 2)) break;
    if ((int)extra_s.size() + 2 >= MAXTIL) break;
    extra_s.push_back(static_cast<int>(s));
  }
  std::vector<long long> bvals{wl.n};
  std::vector<long long> frontier;
  for (auto it = extra_s.rbegin(); it != extra_s.rend(); ++it) frontier.push_back(wl.n / *it);
  frontier.push_back(wl.n / s0);
  std::set<int> reqs{2, 3, 4, 5, 6, 7, 8};  // generator choices and the solver's choose_p range
  for (int i = 0; i < wl.gen.n_s_choices; ++i) reqs.insert(wl.gen.s_choices[i]);
  while (!frontier.empty()) {
    const long long b = frontier.back();
    frontier.pop_back();
    if (std::find(bvals.begin(), bvals.end(), b) != bvals.end()) continue;
    if ((int)bvals.size() >= MAXBV) break;
    bvals.push_back(b);
    for (int r : reqs) {
      if (r < 2) continue;
      const long long s = hesp_snap_tiles(b, r, wl.gen.min_block);
      if (s) frontier.push_back(b / s);
    }
  }
  p.nbv = static_cast<int>(bvals.size());
  for (int i = 0; i < p.nbv; ++i) {
    p.bval[i] = bvals[i];
    for (int k = 0; k < 4; ++k) {
      bool all_known = true;
      for (int ty = 0; ty < p.n_types; ++ty) {
        bool kn = false;
        p.ttime[k][i][ty] = host_task_time(model, k, bvals[i], ty, &kn);
        p.known[k][ty] = kn ? 1 : 0;
        all_known = all_known && kn;
      }
      // mean over processors in id order (sim.cpp:98-106)
      double sum = 0;
      for (int q = 0; q < p.P; ++q) sum += p.ttime[k][i][p.proc_type[q]];
      p.ctavg[k][i] = all_known ? sum / p.P : 0.0;
    }
  }

  for (int l = 0; l < p.L; ++l)
    for (int i = 0; i < p.nbv; ++i) {
      const long long bytes = p.bval[i] * p.bval[i] * wl.elem_size;
      p.hopq[l][i] = static_cast<double>(bytes) / p.link_bw[l];
      p.hopc[l][i] = p.link_lat[l] + static_cast<double>(bytes) / p.link_bw[l];
    }

  // ---------------- top-level tilings via the width-1 engine ----------------
  // Tiling = root_cholesky + partition_task(0, 1/s) run by the engine's own
  // build (graph.cpp:397-407, 456-513), then its predecessors (E5).
  TaskMeta root_t{};
  root_t.blk[0] = 0;
  root_t.blk[1] = 0;
  root_t.blk[2] = root_t.blk[3] = -1;
  root_t.b = static_cast<int32_t>(wl.n);
  root_t.kind = HESP_CHOL;
  root_t.nrd = 1;
  root_t.bidx = 0;
  BlockMeta root_b{};
  root_b.r = Region{0, 0, static_cast<int32_t>(wl.n), static_cast<int32_t>(wl.n)};
  root_b.tile = -1;
  root_b.next = -1;
  auto add_tiling = [&](int s) {
    std::vector<TaskMeta> tasks{root_t};
    std::vector<BlockMeta> blocks{root_b};
    if (s > 1) {
      Problem bp = p;
      bp.n_til = 0;  // the engine emits the root's partition instead of switching tilings
      bp.til[TIL_BASE] = BaseTiling{1, 1, 1, 0, wl.n, &root_t, &root_b, nullptr, nullptr};
      bp.base_tasks = &root_t;
      bp.base_blocks = &root_b;
      bp.n_base_tasks = 1;
      bp.n_base_blocks = 1;
      bp.max_nbb = 1;
      const int nsub = hesp_member_count(HESP_CHOL, s);
      bp.maxt = 1 + nsub + 8;
      bp.maxb = 1 + s * (s + 1) / 2 + 8;
      bp.maxbnd = 16;
      bp.maxcells = 16;
      bp.maxrn = 16;
      bp.maxedges = 16;
      bp.maxpb = 16;
      bp.maxgs = bp.maxb + 8;
      bp.maxgr = bp.maxb + 8;
      bp.lay = slot_layout(bp);
      std::vector<uint8_t> slot(bp.lay.total);
      Small sm{};
      Engine<HostWarp> eng(HostWarp{}, bp, slot.data(), &sm);
      eng.reset_to_base();
      eng.apply_op(0, s);
      if (eng.status) bad("top-level tiling s=" + std::to_string(s) + " failed with status " + std::to_string(eng.status));
      for (int id = 1; id < eng.ntasks; ++id) tasks.push_back(eng.tm()[id - 1]);
      for (int id = 1; id < eng.nblocks; ++id) blocks.push_back(eng.bm()[id - 1]);
    }
    // Predecessors (E5): the engine's per-cell last-writer/readers tracking
    // run once over the tiling, where every tile is a single cell.  Slot
    // order = the engine's processing order: read-only blocks in read order,
    // then the write.
    const int nt = static_cast<int>(tasks.size());
    const int nb = static_cast<int>(blocks.size());
    std::vector<int> writer(nb, -1);
    std::vector<std::vector<int>> readers(nb);
    std::vector<BasePreds> preds(nt, BasePreds{});
    std::vector<int32_t> plist;
    for (int j = 1; j < nt; ++j) {
      const TaskMeta& t = tasks[j];
      const int wb = t.blk[t.nrd];
      std::vector<int> uni;
      int slot = 0;
      BasePreds bp{};
      for (int k = 0; k <= t.nrd; ++k) {
        const int b = t.blk[k];
        if (k < t.nrd && b == wb) continue;
        bool dup = false;
        for (int q = 0; q < k; ++q)
          if (t.blk[q] == b && q < t.nrd) dup = true;
        if (dup && k < t.nrd) continue;
        const bool writes = k == t.nrd;
        std::vector<int> lst;
        if (writer[b] >= 0 && writer[b] != j) lst.push_back(writer[b]);
        if (!writes) {
          readers[b].push_back(j);
        } else {
          for (auto it = readers[b].rbegin(); it != readers[b].rend(); ++it)
            if (*it != j) lst.push_back(*it);
          writer[b] = j;
          readers[b].clear();
        }
        if (slot >= 3) bad("base task with more than 3 distinct blocks");
        bp.soff[slot] = static_cast<int>(plist.size());
        bp.scnt[slot] = static_cast<int>(lst.size());
        plist.insert(plist.end(), lst.begin(), lst.end());
        for (int x : lst)
          if (std::find(uni.begin(), uni.end(), x) == uni.end()) uni.push_back(x);
        ++slot;
      }
      bp.uoff = static_cast<int>(plist.size());
      bp.ucnt = static_cast<int>(uni.size());
      plist.insert(plist.end(), uni.begin(), uni.end());
      preds[j] = bp;
    }
    if (plist.empty()) plist.push_back(0);
    HostProblem::TilingOff o;
    o.s = s;
    o.tasks = hp.base_tasks.size();
    o.blocks = hp.base_blocks.size();
    o.preds = hp.base_preds.size();
    o.plist = hp.base_plist.size();
    o.n_tasks = nt;
    o.n_blocks = nb;
    o.base_b = wl.n / s;
    hp.til.push_back(o);
    hp.base_tasks.insert(hp.base_tasks.end(), tasks.begin(), tasks.end());
    hp.base_blocks.insert(hp.base_blocks.end(), blocks.begin(), blocks.end());
    hp.base_preds.insert(hp.base_preds.end(), preds.begin(), preds.end());
    hp.base_plist.insert(hp.base_plist.end(), plist.begin(), plist.end());
  };
  add_tiling(static_cast<int>(s0));  // TIL_BASE: arrays start at offset 0 (base_tasks & co.)
  add_tiling(1);                     // TIL_ROOT
  for (int s : extra_s) add_tiling(s);
  p.n_base_tasks = hp.til[TIL_BASE].n_tasks;
  p.n_base_blocks = hp.til[TIL_BASE].n_blocks;
  p.n_til = static_cast<int>(hp.til.size());
  p.max_nbb = 0;
  for (const auto& t : hp.til) p.max_nbb = std::max(p.max_nbb, t.n_blocks);
  p.n_base_leaves = p.n_base_tasks - 1;
  p.base_b = wl.n / s0;

  // ---------------- slot capacities ----------------
  int smax = 2;
  for (int i = 0; i < wl.gen.n_s_choices; ++i) smax = std::max(smax, wl.gen.s_choices[i]);
  smax += 1;  // snapping may move to a neighbouring divisor
  const int K = std::max(1, wl.gen.k_max);
  int max_nbt = 0;
  for (const auto& t : hp.til) max_nbt = std::max(max_nbt, t.n_tasks);
  p.maxt = max_nbt + K * smax * smax * smax + 64;
  p.maxb = p.max_nbb + K * 5 * smax * smax + 64;
  p.maxcells = p.max_nbb + K * 3 * 256 + 256;
  p.maxbnd = 4 * p.maxb + 4 * p.max_nbb + 64;
  // reader nodes and arena edges only arise for tasks touching subdivided
  // tiles (E5); overflow of any cap is reported as ST_ENGINE_LIMIT, never
  // silently truncated
  p.maxrn = 2 * p.maxt + p.maxcells;
  p.maxedges = 8 * p.maxt;
  p.maxpb = 4096;
  p.maxgs = std::max(p.maxt, 4 * p.maxb + 8);
  p.maxgr = p.maxb + 64;
  p.lay = slot_layout(p);
  bind_tilings(p, hp, hp.base_tasks.data(), hp.base_blocks.data(), hp.base_preds.data(), hp.base_plist.data());
  return hp;
}

void bind_tilings(Problem& p, const HostProblem& hp, const TaskMeta* tasks, const BlockMeta* blocks,
                  const BasePreds* preds, const int32_t* plist) {
  p.base_tasks = tasks;
  p.base_blocks = blocks;
  p.base_preds = preds;
  p.base_plist = plist;
  p.n_til = static_cast<int>(hp.til.size());
  for (int i = 0; i < p.n_til; ++i) {
    const auto& o = hp.til[i];
    p.til[i] = BaseTiling{o.s, o.n_tasks, o.n_blocks, 0, o.base_b, tasks + o.tasks, blocks + o.blocks,
                          preds + o.preds, plist + o.plist};
  }
}

}  // namespace hx
