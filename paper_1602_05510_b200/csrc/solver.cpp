// solver.cpp — hesp_solve: the iterative schedule/partition solver
// (SURVEY.md §8f row f1).  The reference declares it only (solver.hpp:57-86);
// its semantics are SPEC.md:410-461, restated here with the decisions the
// SPEC leaves open written down in DESIGN.md §10.
//
// Per iteration (SPEC solve):
//   simulate the state          device, full trace (hesp_eval_trace): idle_avg
//   record IterationRecord      makespan, DAG depth, flop-weighted side, load
//   collect_candidates          SPEC.md:420-427 (All / CP / Shallow + innermost clusters)
//   score_candidate, choose_p   SPEC.md:428-440, solver.hpp:51-66
//   validity filter             every candidate mutation in ONE device batch
//                               (hesp_eval_descs); failing graphs are dropped
//   select_candidate            SPEC.md:441-446 (Hard / Soft with hesp::Rng)
//   apply                       append the op(s) to the state's descriptor
// The host side only does the per-candidate arithmetic (one pass over the
// leaves); every schedule is simulated by the sm_100a engine.
#include <algorithm>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstring>
#include <map>
#include <vector>

#include "hesp_engine.h"
#include "trace.h"

namespace {

using hx::PartEntry;
using hx::Problem;
using hx::TaskMeta;
using hx::TraceGraph;

struct Rng {  // hesp::Rng (sim.cpp:59-69)
  uint64_t s;
  uint64_t next() { return hesp_splitmix_next(&s); }
  double uniform() { return (double)(next() >> 11) * 0x1.0p-53; }
};

struct Cand {
  int action;  // HESP_ACT_*
  int target;  // leaf task id / cluster id
  int parent;  // restored parent (merge / repartition)
  int k;       // tiles of the partition (0 for a merge)
  double score;
  int64_t d;
};

double task_flops(int kind, int64_t b) {  // platform.cpp:57-66
  const double bd = (double)b;
  switch (kind) {
    case HESP_CHOL: return bd * bd * bd / 3.0;
    case HESP_TRSM: return bd * bd * bd;
    case HESP_SYRK: return bd * bd * bd;
    default: return 2.0 * bd * bd * bd;
  }
}

// TaskGraph::snap_tiling (graph.cpp:450-454): largest s <= k dividing d with d/s >= min_block
int64_t snap_tiling(int64_t d, int64_t k, int64_t min_block) {
  for (int64_t s = k; s >= 2; --s)
    if (d % s == 0 && d / s >= min_block) return s;
  return 0;
}

// choose_p (solver.hpp:59-62) as a tile count: k = clamp(ceil(sqrt(I+1)) + 1,
// 2, min(k_max, d/min_block)), snapped down to a divisor grid; 0 = GrainTooSmall
int64_t choose_tiles(double idle, int64_t d, int64_t min_block, int64_t k_max) {
  if (d < 2 * min_block) return 0;
  const int64_t lim = std::min<int64_t>(k_max, d / min_block);
  int64_t k = (int64_t)std::ceil(std::sqrt(idle + 1.0)) + 1;
  k = std::max<int64_t>(2, std::min(k, lim));
  return snap_tiling(d, k, min_block);
}

struct Ctx {
  const Problem& p;
  const hesp_solver_config& cfg;
  // PerfModel::task_time through the engine's host table (every side the
  // engine can create is tabulated); false = no model for it
  bool ttime(int kind, int64_t b, int type, double* t) const {
    for (int i = 0; i < p.nbv; ++i)
      if (p.bval[i] == b) {
        if (!p.known[kind][type]) return false;
        *t = p.ttime[kind][i][type];
        return true;
      }
    return false;
  }
  int64_t choose_k(double idle, int64_t d) const { return choose_tiles(idle, d, cfg.min_block, cfg.k_max); }
  // W_sub: sum of the would-be sub-task times on one processor type, in emission order
  bool w_sub(int kind, int64_t d, int64_t k, int type, double* w) const {
    double sum = 0;
    const int cnt = hesp_member_count(kind, (int32_t)k);
    for (int m = 0; m < cnt; ++m) {
      double t;
      if (!ttime(hesp_member_kind(kind, (int32_t)k, m), d / k, type, &t)) return false;
      sum += t;
    }
    *w = sum;
    return true;
  }
};

// select_candidate over scores in candidate order (shared by hesp_solve).
// Hard: argmax score, ties to the lowest target id (a task id
// for partitions, a cluster id for merges/repartitions), then candidate order.
size_t select_index(const double* sc, const int32_t* tg, size_t n, int sampling, Rng& rng) {
  size_t pick = 0;
  if (sampling == HESP_SAMPLE_HARD) {
    for (size_t i = 1; i < n; ++i)
      if (sc[i] > sc[pick] || (sc[i] == sc[pick] && tg && tg[i] < tg[pick])) pick = i;
    return pick;
  }
  double total = 0;
  for (size_t i = 0; i < n; ++i) total += sc[i];
  const double u = rng.uniform() * total;
  double acc = 0;
  pick = n - 1;
  for (size_t i = 0; i < n; ++i) {
    acc += sc[i];
    if (u < acc) return i;
  }
  return pick;
}

}  // namespace

extern "C" double hesp_choose_p(double idle_avg, int64_t d, int64_t min_block, int32_t k_max) {
  if (k_max < 2 || min_block < 1) return 0.0;
  const int64_t k = choose_tiles(idle_avg, d, min_block, k_max);
  return k ? 1.0 / (double)k : 0.0;
}

extern "C" int32_t hesp_select_candidate(const double* scores, int32_t n, int32_t sampling, uint64_t* rng_state) {
  if (n <= 0 || !scores || !rng_state) return -1;
  Rng rng{*rng_state};
  const size_t i = select_index(scores, nullptr, (size_t)n, sampling, rng);
  *rng_state = rng.s;
  return (int32_t)i;
}

namespace {

// One solver chain (a state, its rng, its output record).
struct Chain {
  hesp_solver_config cfg;
  Rng rng;
  hesp_cand_desc cur;
  hesp_solver_result* out;
  std::vector<hesp_assignment> A;
  std::vector<hesp_load_step> S;
  hesp_solver_iteration rec;
  std::vector<Cand> cands;
  size_t first = 0;  // offset of this chain's mutations in the shared batch
};

bool valid_cfg(const hesp_solver_config* c) {
  return c && c->iterations >= 0 && c->k_max >= 2 && c->overhead_factor >= 1.0 && c->min_block >= 1 &&
         c->task_selection >= 0 && c->task_selection <= 2 && c->sampling >= 0 && c->sampling <= 2;
}

hesp_cand_desc mutate(const hesp_cand_desc& cur, const Cand& c) {
  hesp_cand_desc d = cur;
  if (c.action != HESP_ACT_PARTITION) d.ops[d.n_ops++] = hesp_op{c.target, HESP_OP_MERGE};
  if (c.action != HESP_ACT_MERGE) d.ops[d.n_ops++] = hesp_op{c.parent, c.k};
  return d;
}

// Metrics + candidate collection of one chain's traced state.
void collect(Chain& ch, const Problem& P, const TraceGraph& g, const hesp_trace& tr, int it) {
  const hesp_solver_config& cfg = ch.cfg;
  Ctx cx{P, cfg};
  hesp_solver_result* out = ch.out;
  const hesp_assignment* A = tr.assignments;
  const double makespan = tr.outcome.makespan;
    // ---- graph facts: clusters, membership, depth ----
    std::map<int, int> cluster_of;   // member task -> live cluster id
    std::map<int, int> parent_of;    // partitioned task -> live cluster id
    for (int c = 0; c < (int)g.parts.size(); ++c) {
      const PartEntry& pe = g.parts[c];
      if (pe.task < 0) continue;
      parent_of[pe.task] = c;
      for (int m = pe.child0; m < pe.child0 + pe.nchild; ++m) cluster_of[m] = c;
    }
    auto depth_of = [&](int t) {  // TaskGraph::task_depth (graph.cpp:564-572)
      int d = 0;
      for (auto it2 = cluster_of.find(t); it2 != cluster_of.end(); it2 = cluster_of.find(g.parts[it2->second].task))
        ++d;
      return d;
    };
    std::map<int, const hesp_assignment*> asg;  // leaf task id -> assignment
    for (int i = 0; i < tr.n_assign; ++i) asg[A[i].task] = &A[i];
    // ---- IterationRecord metrics ----
    hesp_solver_iteration rec{};
    rec.iteration = it;
    rec.action = HESP_ACT_NONE;
    rec.target = -1;
    rec.makespan = makespan;
    int depth = 0;
    double num = 0, den = 0;
    for (const auto& [id, a] : asg) {  // task-id order
      (void)a;
      depth = std::max(depth, depth_of(id));
      const TaskMeta& m = g.tmeta[id];
      const double f = task_flops(m.kind, m.b);
      num += f * (double)m.b;
      den += f;
    }
    rec.dag_depth = depth;
    rec.avg_block_side = den > 0 ? num / den : 0.0;
    rec.avg_load_pct = 100.0 * tr.avg_load;
    ch.rec = rec;
    if (out->best_iteration < 0 || makespan < out->best_makespan) {
      out->best_makespan = makespan;
      out->best_iteration = it;
      out->best = ch.cur;
    }
    ch.cands.clear();
    if (it + 1 == cfg.iterations) return;  // the last round's mutation could never be simulated
    std::vector<Cand>& cands = ch.cands;
    // ---- collect_candidates ----
    std::vector<int> tasks;  // selected leaves, id order
    if (cfg.task_selection == HESP_SEL_ALL) {
      for (const auto& [id, a] : asg) tasks.push_back(id);
    } else if (cfg.task_selection == HESP_SEL_SHALLOW) {
      int dmin = 1 << 30;
      for (const auto& [id, a] : asg) dmin = std::min(dmin, depth_of(id));
      for (const auto& [id, a] : asg)
        if (depth_of(id) == dmin) tasks.push_back(id);
    } else {  // CP: realized longest path, backtracked by latest-ending predecessor
      std::map<int, int> li;
      for (size_t k = 0; k < g.leaves.size(); ++k) li[g.leaves[k]] = (int)k;
      int curt = -1;
      for (const auto& [id, a] : asg)
        if (curt < 0 || a->end > asg[curt]->end) curt = id;
      while (curt >= 0) {
        tasks.push_back(curt);
        const int l = li[curt];
        int nxt = -1;
        for (int q = 0; q < g.pcnt[l]; ++q) {
          const int pr = g.preds[g.poff[l] + q];
          if (!asg.count(pr)) continue;
          if (nxt < 0 || asg[pr]->end > asg[nxt]->end || (asg[pr]->end == asg[nxt]->end && pr < nxt)) nxt = pr;
        }
        curt = nxt;
      }
      std::sort(tasks.begin(), tasks.end());
    }
    for (int id : tasks) {  // Partition(p) of a scheduled leaf
      const hesp_assignment& a = *asg[id];
      const TaskMeta& m = g.tmeta[id];
      const int64_t k = cx.choose_k(a.idle_avg, m.b);
      if (k == 0) continue;
      double w;
      if (!cx.w_sub(m.kind, m.b, k, P.proc_type[a.proc], &w)) continue;
      const double est = cfg.overhead_factor * w / std::min(a.idle_avg + 1.0, (double)k);
      const double score = std::max(0.0, (a.end - a.start) - est);
      if (score > 0) cands.push_back({HESP_ACT_PARTITION, id, id, (int)k, score, m.b});
    }
    for (int c = 0; c < (int)g.parts.size(); ++c) {  // innermost clusters (not the base one: the root's)
      const PartEntry& pe = g.parts[c];
      if (pe.task <= 0) continue;
      bool flat = true;
      double lo = 0, hi = 0, isum = 0;
      for (int mm = pe.child0; mm < pe.child0 + pe.nchild && flat; ++mm) {
        auto f = asg.find(mm);
        if (f == asg.end()) {
          flat = false;
          break;
        }
        const hesp_assignment& a = *f->second;
        if (mm == pe.child0 || a.start < lo) lo = a.start;
        if (mm == pe.child0 || a.end > hi) hi = a.end;
        isum += a.idle_avg;
      }
      if (!flat) continue;
      const TaskMeta& par = g.tmeta[pe.task];
      double tmin = 0;
      int tbest = -1;
      for (int ty = 0; ty < P.n_types; ++ty) {
        double t;
        if (!cx.ttime(par.kind, par.b, ty, &t)) continue;
        if (tbest < 0 || t < tmin) {
          tmin = t;
          tbest = ty;
        }
      }
      if (tbest < 0) continue;
      const double span = hi - lo;
      const double merge = std::max(0.0, span - tmin);
      if (merge > 0) cands.push_back({HESP_ACT_MERGE, c, pe.task, 0, merge, par.b});
      const double ic = isum / (double)pe.nchild;
      const int64_t k = cx.choose_k(ic, par.b);
      const int64_t kc = par.b / g.tmeta[pe.child0].b;
      double w;
      if (k == 0 || k == kc || !cx.w_sub(par.kind, par.b, k, tbest, &w)) continue;
      const double est = cfg.overhead_factor * w / std::min(ic + 1.0, (double)k);
      const double rep = merge + std::max(0.0, span - est);
      if (rep > 0) cands.push_back({HESP_ACT_REPARTITION, c, pe.task, (int)k, rep, par.b});
    }
    const hesp_cand_desc& cur = ch.cur;
    const size_t before = cands.size();
    cands.erase(std::remove_if(cands.begin(), cands.end(),
                               [&](const Cand& c) {
                                 return cur.n_ops + (c.action == HESP_ACT_REPARTITION ? 2 : 1) > HESP_MAX_OPS;
                               }),
                cands.end());
    if (cands.size() < before && out->budget_iteration < 0) out->budget_iteration = it;  // op budget reached
    ch.rec.n_candidates = (int32_t)cands.size();
}

// Runs n chains in lockstep: one batched schedule trace of every state and
// one device batch of every chain's candidate mutations per iteration.
int solve_chains(hesp_engine* e, int n, const hesp_cand_desc* initial, const hesp_solver_config* cfgs,
                 hesp_solver_result* outs) {
  const Problem& P = hesp_engine_problem(e);
  std::vector<Chain> chains(n);
  int iters = 0;
  for (int c = 0; c < n; ++c) {
    Chain& ch = chains[c];
    ch.cfg = cfgs[c];
    ch.rng = Rng{cfgs[c].seed};
    std::memset(&ch.cur, 0, sizeof ch.cur);
    if (initial) ch.cur = initial[c];
    ch.out = &outs[c];
    ch.out->n_history = 0;
    ch.out->best_makespan = 0;
    ch.out->best_iteration = -1;
    ch.out->budget_iteration = -1;
    ch.out->n_simulated = 0;
    std::memset(&ch.out->best, 0, sizeof ch.out->best);
    ch.A.resize((size_t)P.maxt);
    ch.S.resize(2 * (size_t)P.maxt + 2);
    iters = std::max(iters, ch.cfg.iterations);
  }
  std::vector<hesp_cand_desc> states;
  std::vector<hesp_neighbor> nbrs;
  std::vector<hesp_outcome> souts, outc;
  std::vector<TraceGraph> graphs;
  std::vector<hx::TraceLogs> logs;
  std::vector<int> live;
  for (int it = 0; it < iters; ++it) {
    live.clear();
    states.clear();
    for (int c = 0; c < n; ++c)
      if (it < chains[c].cfg.iterations) {
        live.push_back(c);
        states.push_back(chains[c].cur);
      }
    int r = hx::schedule_batch(e, states.data(), (int)states.size(), graphs, logs, souts);
    if (r != HESP_OK) return r;
    for (size_t q = 0; q < live.size(); ++q)
      if (souts[q].status != 0) return souts[q].status;  // only an initial state can fail
    // per-chain host work (post-passes, scoring) is independent: spread the
    // chains over the host threads
    std::atomic<size_t> next{0};
    std::atomic<int> err{0};
    auto work = [&]() {
      for (;;) {
        const size_t q = next.fetch_add(1);
        if (q >= live.size()) return;
        Chain& ch = chains[live[q]];
        ++ch.out->n_simulated;
        hesp_trace tr{};
        tr.cap_assign = (int32_t)ch.A.size();
        tr.cap_steps = (int32_t)ch.S.size();
        tr.assignments = ch.A.data();
        tr.steps = ch.S.data();
        tr.outcome = souts[q];
        const int rr = hx::finish_trace(P, graphs[q], logs[q], &tr, true);
        if (rr != HESP_OK) {
          err = rr;
          continue;
        }
        collect(ch, P, graphs[q], tr, it);
      }
    };
    const unsigned hw = std::thread::hardware_concurrency();
    const size_t nth = std::min<size_t>(live.size(), hw ? hw : 1);
    if (nth <= 1) {
      work();
    } else {
      std::vector<std::thread> pool;
      for (size_t t = 0; t < nth; ++t) pool.emplace_back(work);
      for (auto& t : pool) t.join();
    }
    if (err) return err;
    // ---- validity filter: every chain's mutations in one device batch, as
    // neighbours of the chain states (each state expanded once on the device)
    nbrs.clear();
    for (size_t q = 0; q < live.size(); ++q) {
      Chain& ch = chains[live[q]];
      ch.first = nbrs.size();
      for (const Cand& cd : ch.cands) {
        hesp_neighbor nb{};
        nb.base = (int32_t)q;
        if (cd.action != HESP_ACT_PARTITION) nb.ops[nb.n_ops++] = hesp_op{cd.target, HESP_OP_MERGE};
        if (cd.action != HESP_ACT_MERGE) nb.ops[nb.n_ops++] = hesp_op{cd.parent, cd.k};
        nbrs.push_back(nb);
      }
    }
    if (!nbrs.empty()) {
      outc.resize(nbrs.size());
      hesp_best b{};
      r = hesp_eval_neighbors(e, states.data(), (int32_t)states.size(), nbrs.data(), nbrs.size(), outc.data(), &b);
      if (r != 0) return r;
    }
    for (int c : live) {
      Chain& ch = chains[c];
      hesp_solver_iteration rec = ch.rec;
      std::vector<Cand> valid;
      ch.out->n_simulated += (int64_t)ch.cands.size();
      for (size_t i = 0; i < ch.cands.size(); ++i) {
        if (outc[ch.first + i].status == 0) {
          valid.push_back(ch.cands[i]);
          if (ch.cfg.sampling == HESP_SAMPLE_EXACT) valid.back().score = outc[ch.first + i].makespan;
        }
        // a mutation beyond the slot's capacity (ids consumed by merged
        // clusters count too): the chain has outgrown the engine's sizing
        if (outc[ch.first + i].status == HESP_ST_ENGINE_LIMIT && ch.out->budget_iteration < 0)
          ch.out->budget_iteration = rec.iteration;
      }
      rec.n_valid = (int32_t)valid.size();
      if (!valid.empty()) {
        // ---- select_candidate ----
        std::vector<double> sc(valid.size());
        std::vector<int32_t> tg(valid.size());
        for (size_t i = 0; i < valid.size(); ++i) {
          sc[i] = valid[i].score;
          tg[i] = valid[i].target;
        }
        size_t pick = 0;
        if (ch.cfg.sampling == HESP_SAMPLE_EXACT) {
          for (size_t i = 1; i < sc.size(); ++i)
            if (sc[i] < sc[pick]) pick = i;
        } else {
          pick = select_index(sc.data(), tg.data(), sc.size(), ch.cfg.sampling, ch.rng);
        }
        const Cand& cd = valid[pick];
        rec.action = cd.action;
        rec.target = cd.target;
        rec.d = cd.d;
        rec.p = cd.action == HESP_ACT_MERGE ? 1.0 : 1.0 / (double)cd.k;
        rec.score = cd.score;
        ch.cur = mutate(ch.cur, cd);
      }
      ch.out->history[ch.out->n_history++] = rec;
    }
  }
  return 0;
}

}  // namespace

extern "C" int hesp_solve(hesp_engine* e, const hesp_cand_desc* initial, const hesp_solver_config* cfgp,
                          hesp_solver_result* out) {
  if (!e || !valid_cfg(cfgp) || !out) return HESP_E_INVALID;
  if (out->cap_history < cfgp->iterations || (!out->history && cfgp->iterations > 0)) return HESP_E_INVALID;
  return solve_chains(e, 1, initial, cfgp, out);
}

extern "C" int hesp_solve_batch(hesp_engine* e, int32_t n_chains, const hesp_cand_desc* initial,
                                const hesp_solver_config* cfgs, hesp_solver_result* outs) {
  if (!e || n_chains < 1 || !cfgs || !outs) return HESP_E_INVALID;
  for (int c = 0; c < n_chains; ++c) {
    if (!valid_cfg(&cfgs[c])) return HESP_E_INVALID;
    if (outs[c].cap_history < cfgs[c].iterations || (!outs[c].history && cfgs[c].iterations > 0))
      return HESP_E_INVALID;
  }
  return solve_chains(e, n_chains, initial, cfgs, outs);
}
