// trace.cpp — host post-passes of the full-trace path (see trace.h).
//
// The schedule itself comes from the device (Engine<DevWarp, true>); this
// file only orders the device logs the way the reference orders its
// SimResult after the event loop:
//   ordering of events / residency log / transfers   sim.cpp:813-831
// The load post-passes (compute_idle_avgs sim.cpp:670-702, busy_time /
// LoadTrace::integral sim.cpp:71-87, compute_load_trace sim.cpp:975-991) run
// on the device (loadtrace.cu); verify_schedule (sim.cpp:857-973) too
// (verify.cu).
#include "trace.h"

#include <algorithm>
#include <cstdio>
#include <cstdint>
#include <map>
#include <string>
#include <unordered_map>

namespace hx {
namespace {

const char* kind_name(int k) {  // to_string(TaskKind), platform.cpp:39-47
  switch (k) {
    case 0: return "CHOL";
    case 1: return "TRSM";
    case 2: return "SYRK";
    case 3: return "GEMM";
  }
  return "?";
}

struct Ev {
  hesp_event e;
  std::string resource, subject;
};

void hop_link(const Problem& p, int src, int dst, int h, int32_t* hs, int32_t* hd) {
  const int l = p.route_l[src * MAXS + dst][h];
  *hs = p.link_src[l];
  *hd = p.link_dst[l];
}

}  // namespace

void to_reference_ids(TraceGraph& g, TraceLogs* logs, int off_t, int off_b, int off_c) {
  if (off_t == 0 && off_b == 0 && off_c == 0) return;
  auto xt = [&](int j) { return j > 0 ? j + off_t : j; };
  auto xb = [&](int b) { return b > 0 ? b + off_b : b; };
  auto meta = [&](TaskMeta m) {
    for (int k = 0; k < 4; ++k) m.blk[k] = xb(m.blk[k]);
    return m;
  };
  for (auto& j : g.leaves) j = xt(j);
  for (auto& j : g.preds) j = xt(j);
  for (auto& m : g.meta) m = meta(m);
  if (!g.bregion.empty()) {  // ids consumed before the top merge: erased blocks
    std::vector<Region> r(g.bregion.size() + off_b, Region{0, 0, 0, 0});
    std::vector<int32_t> in(g.bisint.size() + off_b, 0);
    for (size_t b = 0; b < g.bregion.size(); ++b) r[xb((int)b)] = g.bregion[b];
    for (size_t b = 0; b < g.bisint.size(); ++b) in[xb((int)b)] = g.bisint[b];
    g.bregion.swap(r);
    g.bisint.swap(in);
  }
  {
    TaskMeta gone{};
    gone.blk[0] = gone.blk[1] = gone.blk[2] = gone.blk[3] = -1;
    gone.nrd = -1;
    std::vector<TaskMeta> t(g.tmeta.size() + (g.tmeta.empty() ? 0 : off_t), gone);
    for (size_t j = 0; j < g.tmeta.size(); ++j) t[xt((int)j)] = meta(g.tmeta[j]);
    g.tmeta.swap(t);
  }
  {
    std::vector<PartEntry> c(g.parts.size() + off_c, PartEntry{-1, 0, 0, 0});  // merged before the top merge
    for (size_t i = 0; i < g.parts.size(); ++i) {
      PartEntry e = g.parts[i];
      if (e.task >= 0) e.task = xt(e.task);
      else e.task = -2 - xt(-2 - e.task);
      e.child0 = xt(e.child0);
      c[i + off_c] = e;
    }
    g.parts.swap(c);
  }
  if (logs) {
    for (auto& x : logs->xfers) x.block = xb(x.block);
    for (auto& r : logs->res) r.block = xb(r.block);
  }
}

int finish_trace(const Problem& p, const TraceGraph& g, const TraceLogs& logs, hesp_trace* tr, bool schedule_only) {
  // assignments in task-id order (std::map order of SimResult::assignments)
  int na = 0;
  for (size_t id = 0; id < logs.proc.size(); ++id) na += logs.proc[id] >= 0;
  // transfers: stable by (start, block) over emission order
  std::vector<XferLog> xs = schedule_only ? std::vector<XferLog>{} : logs.xfers;
  std::stable_sort(xs.begin(), xs.end(), [](const XferLog& a, const XferLog& b) {
    if (a.start != b.start) return a.start < b.start;
    return a.block < b.block;
  });
  std::vector<ResLog> rs = schedule_only ? std::vector<ResLog>{} : logs.res;
  std::stable_sort(rs.begin(), rs.end(), [](const ResLog& a, const ResLog& b) {
    if (a.time != b.time) return a.time < b.time;
    if (a.space != b.space) return a.space < b.space;
    if (a.delta != b.delta) return a.delta > b.delta;
    return a.block < b.block;
  });
  int nhops = 0;
  for (const auto& x : xs) nhops += x.nh;
  const int nev = schedule_only ? 0 : 2 * na + 2 * nhops;
  tr->n_assign = na;
  tr->n_xfer = (int32_t)xs.size();
  tr->n_res = (int32_t)rs.size();
  tr->n_events = nev;
  // load steps need the assignments first; their count is bounded by 2*na
  if (na > tr->cap_assign || (int)xs.size() > tr->cap_xfer || (int)rs.size() > tr->cap_res ||
      nev > tr->cap_events || 2 * na > tr->cap_steps) {
    tr->n_steps = 2 * na;
    return HESP_E_LIMIT;
  }
  {
    int k = 0;
    for (size_t id = 0; id < logs.proc.size(); ++id) {
      if (logs.proc[id] < 0) continue;
      hesp_assignment& a = tr->assignments[k++];
      a.task = (int32_t)id;
      a.proc = logs.proc[id];
      a.start = logs.start[id];
      a.end = logs.end[id];
      a.idle_avg = 0.0;
    }
  }
  for (size_t i = 0; i < xs.size(); ++i) {
    const XferLog& x = xs[i];
    hesp_transfer& t = tr->transfers[i];
    t.block = x.block;
    t.src_space = x.src;
    t.dst_space = x.dst;
    t.n_hops = x.nh;
    t.bytes = x.bytes;
    t.start = x.start;
    t.end = x.end;
    t.has_fragment = x.has_frag;
    t.frag_row = x.frow;
    t.frag_col = x.fcol;
    t.frag_rows = x.frows;
    t.frag_cols = x.fcols;
    t.pad = 0;
    for (int h = 0; h < 2; ++h) {
      t.hop_src[h] = t.hop_dst[h] = -1;
      t.hop_start[h] = t.hop_end[h] = 0.0;
      if (h < x.nh) {
        hop_link(p, x.src, x.dst, h, &t.hop_src[h], &t.hop_dst[h]);
        t.hop_start[h] = x.hs[h];
        t.hop_end[h] = x.he[h];
      }
    }
  }
  for (size_t i = 0; i < rs.size(); ++i) {
    tr->residency[i].time = rs[i].time;
    tr->residency[i].space = rs[i].space;
    tr->residency[i].block = rs[i].block;
    tr->residency[i].delta_bytes = rs[i].delta;
  }
  // events: every field is part of the sort key, so records that tie are
  // identical and the emission order does not matter
  if (!schedule_only) {
    std::vector<Ev> ev;
    ev.reserve(nev);
    std::unordered_map<int, int> li;  // task id -> leaf index
    for (size_t k = 0; k < g.leaves.size(); ++k) li[g.leaves[k]] = (int)k;
    for (int i = 0; i < na; ++i) {
      const hesp_assignment& a = tr->assignments[i];
      const auto it = li.find(a.task);
      const TaskMeta m = it != li.end() ? g.meta[it->second] : TaskMeta{};
      std::string subj = "T" + std::to_string(a.task) + ":" + kind_name(m.kind) + ":b" + std::to_string(m.b);
      std::string res = std::to_string(a.proc);
      for (int k = 0; k < 2; ++k) {
        Ev e{};
        e.e.kind = k == 0 ? HESP_EV_TASK_START : HESP_EV_TASK_END;
        e.e.id = a.task;
        e.e.task_kind = m.kind;
        e.e.res_a = a.proc;
        e.e.res_b = -1;
        e.e.b = m.b;
        e.e.time = k == 0 ? a.start : a.end;
        e.resource = res;
        e.subject = subj;
        ev.push_back(e);
      }
    }
    for (const auto& x : xs) {
      for (int h = 0; h < x.nh; ++h) {
        int32_t hs, hd;
        hop_link(p, x.src, x.dst, h, &hs, &hd);
        for (int k = 0; k < 2; ++k) {
          Ev e{};
          e.e.kind = k == 0 ? HESP_EV_XFER_START : HESP_EV_XFER_END;
          e.e.id = x.block;
          e.e.task_kind = -1;
          e.e.res_a = hs;
          e.e.res_b = hd;
          e.e.b = 0;
          e.e.time = k == 0 ? x.hs[h] : x.he[h];
          e.resource = std::to_string(hs) + "->" + std::to_string(hd);
          e.subject = "B" + std::to_string(x.block);
          ev.push_back(e);
        }
      }
    }
    std::stable_sort(ev.begin(), ev.end(), [](const Ev& a, const Ev& b) {
      if (a.e.time != b.e.time) return a.e.time < b.e.time;
      if (a.e.kind != b.e.kind) return a.e.kind < b.e.kind;
      if (a.resource != b.resource) return a.resource < b.resource;
      return a.subject < b.subject;
    });
    for (size_t i = 0; i < ev.size(); ++i) tr->events[i] = ev[i].e;
  }
  // load post-passes: computed on the device (loadtrace.cu)
  if (!logs.has_load || logs.idle.size() < logs.proc.size()) return HESP_E_INVALID;
  for (int i = 0; i < na; ++i) tr->assignments[i].idle_avg = logs.idle[tr->assignments[i].task];
  tr->n_steps = (int32_t)logs.steps_time.size();
  for (size_t i = 0; i < logs.steps_time.size(); ++i) {
    tr->steps[i].time = logs.steps_time[i];
    tr->steps[i].active = logs.steps_active[i];
    tr->steps[i].pad = 0;
  }
  tr->busy_time = logs.busy;
  const double mk = tr->outcome.makespan;
  const int P = p.P;
  tr->avg_load = (mk <= 0 || P < 1) ? 0.0 : logs.busy / (P * mk);  // SimResult::avg_load (sim.cpp:78-87)
  tr->load_integral = logs.integral;
  return HESP_OK;
}

void trace_bounds(const Problem& p, const TraceGraph& g, double* cp, double* work) {
  const int n = (int)g.leaves.size();
  std::unordered_map<int, int> li;
  for (int k = 0; k < n; ++k) li[g.leaves[k]] = k;
  std::vector<double> tmin(n, 0.0), fin(n, 0.0);
  double w = 0;
  for (int k = 0; k < n; ++k) {
    const TaskMeta& m = g.meta[k];
    double best = -1;
    for (int ty = 0; ty < p.n_types; ++ty) {
      const double t = p.ttime[m.kind][m.bidx][ty];
      if (p.known[m.kind][ty] && (best < 0 || t < best)) best = t;
    }
    tmin[k] = best < 0 ? 0.0 : best;
    w += tmin[k];
  }
  // leaves are in program order, so every predecessor precedes its task
  double longest = 0;
  for (int k = 0; k < n; ++k) {
    double ready = 0;
    for (int q = 0; q < g.pcnt[k]; ++q) {
      auto it = li.find(g.preds[g.poff[k] + q]);
      if (it != li.end() && fin[it->second] > ready) ready = fin[it->second];
    }
    fin[k] = ready + tmin[k];
    if (fin[k] > longest) longest = fin[k];
  }
  *cp = longest;
  *work = p.P > 0 ? w / p.P : 0.0;
}

}  // namespace hx
