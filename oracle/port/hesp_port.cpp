// hesp_port.cpp — CPU restatement of the reference hot path (see hesp_port.h).
// TEST INFRASTRUCTURE ONLY.  Each section cites the reference lines it
// restates (paths relative to /root/reference/proj).
#include "hesp_port.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <queue>
#include <set>
#include <tuple>

namespace port {
namespace {

using ll = long long;

// status codes = 1 + hesp::Err ordinal (errors.hpp:10-32)
enum { E_VALIDATION = 2, E_NOROUTE = 6, E_NOTLEAF = 8, E_INDIVISIBLE = 9, E_MODELMISS = 13,
       E_CAPACITY = 14, E_NOPROC = 15, E_COHERENCE = 20, E_INTERNAL = 21 };
struct Abort {
  int code;
};
[[noreturn]] void abort_with(int c) { throw Abort{c}; }

uint64_t bits_of(double x) {
  uint64_t u;
  std::memcpy(&u, &x, 8);
  return u;
}

// ---------------------------------------------------------------- geometry
// Region algebra, graph.cpp:25-84
struct Rect {
  ll r = 0, c = 0, h = 0, w = 0;
  auto key() const { return std::make_tuple(r, c, h, w); }
  bool operator==(const Rect& o) const { return key() == o.key(); }
};
bool holds(const Rect& o, const Rect& i) {  // non-strict containment
  return i.r >= o.r && i.c >= o.c && i.r + i.h <= o.r + o.h && i.c + i.w <= o.c + o.w;
}
bool touches(const Rect& a, const Rect& b) {
  return a.r < b.r + b.h && b.r < a.r + a.h && a.c < b.c + b.w && b.c < a.c + a.w;
}
// cells of `base` not inside any single cut, merged into horizontal runs per row strip
std::vector<Rect> minus(const Rect& base, const std::vector<Rect>& cuts) {
  std::vector<ll> xs{base.c, base.c + base.w}, ys{base.r, base.r + base.h};
  for (const Rect& k : cuts) {
    if (!touches(base, k)) continue;
    xs.push_back(std::clamp(k.c, base.c, base.c + base.w));
    xs.push_back(std::clamp(k.c + k.w, base.c, base.c + base.w));
    ys.push_back(std::clamp(k.r, base.r, base.r + base.h));
    ys.push_back(std::clamp(k.r + k.h, base.r, base.r + base.h));
  }
  std::sort(xs.begin(), xs.end());
  xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
  std::sort(ys.begin(), ys.end());
  ys.erase(std::unique(ys.begin(), ys.end()), ys.end());
  std::vector<Rect> out;
  for (size_t y = 0; y + 1 < ys.size(); ++y) {
    bool open = false;
    Rect run;
    for (size_t x = 0; x + 1 < xs.size(); ++x) {
      const Rect cell{ys[y], xs[x], ys[y + 1] - ys[y], xs[x + 1] - xs[x]};
      const bool hit = std::any_of(cuts.begin(), cuts.end(), [&](const Rect& k) { return holds(k, cell); });
      if (hit) {
        if (open) out.push_back(run);
        open = false;
      } else if (open) {
        run.w += cell.w;
      } else {
        run = cell;
        open = true;
      }
    }
    if (open) out.push_back(run);
  }
  return out;
}

// ---------------------------------------------------------------- data DAG
// DataDag, graph.cpp:89-212
struct Block {
  Rect g;
  std::vector<int> up, dn;
  bool isect = false;
};
struct Blocks {
  std::vector<Block> v;
  std::map<std::tuple<ll, ll, ll, ll>, int> at;

  static void add_unique(std::vector<int>& l, int x) {
    if (std::find(l.begin(), l.end(), x) == l.end()) l.push_back(x);
  }
  void connect(int a, int b) {
    add_unique(v[a].dn, b);
    add_unique(v[b].up, a);
  }
  void disconnect(int a, int b) {
    v[a].dn.erase(std::remove(v[a].dn.begin(), v[a].dn.end(), b), v[a].dn.end());
    v[b].up.erase(std::remove(v[b].up.begin(), v[b].up.end(), a), v[b].up.end());
  }
  int find(const Rect& g) const {
    auto it = at.find(g.key());
    return it == at.end() ? -1 : it->second;
  }
  bool strictly_in(int a, int b) const { return !(v[a].g == v[b].g) && holds(v[b].g, v[a].g); }
  int insert(const Rect& g, bool isect) {  // DataDag::create, graph.cpp:142-189
    const int id = static_cast<int>(v.size());
    std::vector<int> above, below;
    for (int j = 0; j < id; ++j) {
      if (v[j].g == g) continue;
      if (holds(v[j].g, g)) above.push_back(j);
      else if (holds(g, v[j].g)) below.push_back(j);
    }
    std::vector<int> ups, dns;
    for (int a : above)
      if (std::none_of(above.begin(), above.end(), [&](int q) { return q != a && strictly_in(q, a); }))
        ups.push_back(a);
    for (int d : below)
      if (std::none_of(below.begin(), below.end(), [&](int q) { return q != d && strictly_in(d, q); }))
        dns.push_back(d);
    v.push_back(Block{g, {}, {}, isect});
    at[g.key()] = id;
    for (int a : ups)
      for (int d : dns)
        if (std::find(v[a].dn.begin(), v[a].dn.end(), d) != v[a].dn.end()) disconnect(a, d);
    for (int a : ups) connect(a, id);
    for (int d : dns) connect(id, d);
    return id;
  }
  int obtain(const Rect& g) {  // DataDag::get_or_create, graph.cpp:191-212
    const int have = find(g);
    if (have >= 0) return have;
    const int id = insert(g, false);
    std::vector<std::pair<int, Rect>> overlaps;
    for (int j = 0; j < id; ++j) {
      if (v[j].isect || holds(v[j].g, g) || holds(g, v[j].g) || !touches(v[j].g, g)) continue;
      const Rect& o = v[j].g;
      const ll r0 = std::max(o.r, g.r), c0 = std::max(o.c, g.c);
      const ll r1 = std::min(o.r + o.h, g.r + g.h), c1 = std::min(o.c + o.w, g.c + g.w);
      overlaps.push_back({j, Rect{r0, c0, r1 - r0, c1 - c0}});
    }
    for (auto& [j, s] : overlaps) {
      const int e = find(s);
      if (e >= 0) {
        connect(id, e);
        connect(j, e);
      } else {
        insert(s, true);
      }
    }
    return id;
  }
  std::set<int> walk(int b, bool down) const {  // descendants / ancestors, graph.cpp:102-126
    std::set<int> seen;
    std::deque<int> q(down ? v[b].dn.begin() : v[b].up.begin(), down ? v[b].dn.end() : v[b].up.end());
    while (!q.empty()) {
      const int x = q.front();
      q.pop_front();
      if (!seen.insert(x).second) continue;
      const auto& nx = down ? v[x].dn : v[x].up;
      q.insert(q.end(), nx.begin(), nx.end());
    }
    return seen;
  }
};

// ---------------------------------------------------------------- task DAG
struct Task {
  int kind;
  ll b;
  std::vector<int> rd, wr;
  std::vector<int> seq;
  bool leaf = true;
};

struct Graph {
  Blocks blk;
  std::vector<Task> tk;
  ll elem = 4;
  Rect sub(const Rect& a, ll s, ll i, ll j) const {
    const ll tb = a.h / s;
    return Rect{a.r + i * tb, a.c + j * tb, tb, tb};
  }
  // partition_task, graph.cpp:456-513, with the loop nests of graph.cpp:313-389
  void split(int id, int s_req, ll min_block) {
    if (id < 0 || id >= static_cast<int>(tk.size())) abort_with(E_VALIDATION);
    if (!tk[id].leaf) abort_with(E_NOTLEAF);
    const double p = 1.0 / s_req;
    if (!(p > 0.0 && p < 1.0)) abort_with(E_VALIDATION);
    const ll d = tk[id].b;
    const ll s0 = std::max<ll>(2, std::llround(1.0 / p));
    const ll hi = d / std::max<ll>(1, min_block);
    ll s = 0;
    for (ll k = 0; k <= s0 + hi && !s; ++k)
      for (ll c : {s0 - k, s0 + k})
        if (c >= 2 && c <= hi && d % c == 0) {
          s = c;
          break;
        }
    if (!s) abort_with(E_INDIVISIBLE);
    std::vector<Rect> opnd;
    for (int r : tk[id].rd)
      if (std::find(tk[id].wr.begin(), tk[id].wr.end(), r) == tk[id].wr.end()) opnd.push_back(blk.v[r].g);
    const Rect a = blk.v[tk[id].wr.front()].g;
    struct Spec {
      int kind;
      std::vector<Rect> in;
      Rect out;
    };
    std::vector<Spec> specs;
    const int kind = tk[id].kind;
    if (kind == HESP_CHOL) {
      for (ll k = 0; k < s; ++k) {
        specs.push_back({HESP_CHOL, {sub(a, s, k, k)}, sub(a, s, k, k)});
        for (ll i = k + 1; i < s; ++i) specs.push_back({HESP_TRSM, {sub(a, s, k, k), sub(a, s, i, k)}, sub(a, s, i, k)});
        for (ll i = k + 1; i < s; ++i) {
          for (ll j = k + 1; j < i; ++j)
            specs.push_back({HESP_GEMM, {sub(a, s, i, k), sub(a, s, j, k), sub(a, s, i, j)}, sub(a, s, i, j)});
          specs.push_back({HESP_SYRK, {sub(a, s, i, k), sub(a, s, i, i)}, sub(a, s, i, i)});
        }
      }
    } else if (kind == HESP_TRSM) {
      if (opnd.size() != 1) abort_with(E_INTERNAL);
      const Rect l = opnd[0];
      for (ll j = 0; j < s; ++j)
        for (ll i = 0; i < s; ++i) {
          for (ll k = 0; k < j; ++k)
            specs.push_back({HESP_GEMM, {sub(a, s, i, k), sub(l, s, j, k), sub(a, s, i, j)}, sub(a, s, i, j)});
          specs.push_back({HESP_TRSM, {sub(l, s, j, j), sub(a, s, i, j)}, sub(a, s, i, j)});
        }
    } else if (kind == HESP_SYRK) {
      if (opnd.size() != 1) abort_with(E_INTERNAL);
      const Rect x = opnd[0];
      for (ll i = 0; i < s; ++i)
        for (ll j = 0; j <= i; ++j)
          for (ll k = 0; k < s; ++k) {
            if (i == j) specs.push_back({HESP_SYRK, {sub(x, s, i, k), sub(a, s, i, j)}, sub(a, s, i, j)});
            else specs.push_back({HESP_GEMM, {sub(x, s, i, k), sub(x, s, j, k), sub(a, s, i, j)}, sub(a, s, i, j)});
          }
    } else {
      if (opnd.size() != 2) abort_with(E_INTERNAL);
      for (ll i = 0; i < s; ++i)
        for (ll j = 0; j < s; ++j)
          for (ll k = 0; k < s; ++k)
            specs.push_back({HESP_GEMM, {sub(opnd[0], s, i, k), sub(opnd[1], s, j, k), sub(a, s, i, j)}, sub(a, s, i, j)});
    }
    for (size_t m = 0; m < specs.size(); ++m) {
      Task t;
      t.kind = specs[m].kind;
      for (const Rect& g : specs[m].in) t.rd.push_back(blk.obtain(g));
      t.wr.push_back(blk.obtain(specs[m].out));
      t.b = specs[m].out.h;
      t.seq = tk[id].seq;
      t.seq.push_back(static_cast<int>(m));
      tk.push_back(std::move(t));
    }
    tk[id].leaf = false;
  }
  std::vector<int> program_order() const {  // leaf_tasks, graph.cpp:552-562
    std::vector<int> l;
    for (int i = 0; i < static_cast<int>(tk.size()); ++i)
      if (tk[i].leaf) l.push_back(i);
    std::sort(l.begin(), l.end(), [&](int x, int y) { return tk[x].seq != tk[y].seq ? tk[x].seq < tk[y].seq : x < y; });
    return l;
  }
};

// ---------------------------------------------------------------- models
double flops_of(int kind, ll b) {  // task_flops, platform.cpp:57-66
  const double x = static_cast<double>(b);
  return kind == HESP_CHOL ? x * x * x / 3.0 : kind == HESP_GEMM ? 2.0 * x * x * x : x * x * x;
}
bool model_knows(const Model& m, int kind, const std::string& type) {
  if (m.analytic)
    return std::any_of(m.entries.begin(), m.entries.end(), [&](auto& e) { return e.kind == kind && e.type == type; });
  return std::any_of(m.rows.begin(), m.rows.end(), [&](auto& r) { return r.kind == kind && r.type == type; });
}
double model_time(const Model& m, int kind, ll b, const std::string& type) {  // platform.cpp:347-390
  if (m.analytic) {
    for (auto& e : m.entries)
      if (e.kind == kind && e.type == type) return flops_of(kind, b) / (e.peak * (static_cast<double>(b) / (static_cast<double>(b) + e.bhalf)));
    abort_with(4 + 1);
  }
  std::map<ll, double> pts;
  for (auto& r : m.rows)
    if (r.kind == kind && r.type == type) pts[r.b] = r.sec;
  if (pts.empty()) abort_with(4 + 1);
  if (pts.count(b)) return pts[b];
  auto rate = [&](std::map<ll, double>::iterator it) { return flops_of(kind, it->first) / it->second; };
  auto up = pts.upper_bound(b);
  double rt;
  if (up == pts.begin()) rt = rate(up);
  else if (up == pts.end()) rt = rate(std::prev(up));
  else {
    auto lo = std::prev(up);
    const double lb = std::log(static_cast<double>(lo->first)), hb = std::log(static_cast<double>(up->first));
    const double lr = std::log(rate(lo)), hr = std::log(rate(up));
    const double f = (std::log(static_cast<double>(b)) - lb) / (hb - lb);
    rt = std::exp(lr + f * (hr - lr));
  }
  return flops_of(kind, b) / rt;
}

// ---------------------------------------------------------------- simulation
// Engine, sim.cpp:257-834
struct Sim {
  const Platform& P;
  const Model& M;
  const Sched& C;
  const Graph& G;
  int mainsp = 0;
  struct Mem {
    std::map<int, double> valid;
    std::set<int> mat, dirty;
    ll used = 0;
  };
  std::map<int, Mem> mem;
  std::map<int, double> busy_until;
  std::map<std::pair<int, int>, double> link_free;
  std::map<std::pair<int, int>, double> stamp;
  std::map<std::pair<int, int>, int> pins;
  std::vector<std::tuple<double, int, int>> unpin;
  std::vector<Rect> written;
  std::vector<std::vector<int>> pred, succ;
  std::map<int, int> waiting;
  std::map<int, double> released;
  std::set<int> finished;
  std::map<int, double> crit;
  std::map<int, std::pair<double, double>> span;  // task -> (start, end)
  std::map<int, int> where;                       // task -> proc
  uint64_t ahash = 0, xhash = 0;
  uint64_t rng;

  Sim(const Platform& p, const Model& m, const Sched& c, const Graph& g) : P(p), M(m), C(c), G(g), rng(c.seed) {
    for (auto& s : P.spaces)
      if (s.main) mainsp = s.id;
  }
  const Space& space(int id) const {
    for (auto& s : P.spaces)
      if (s.id == id) return s;
    abort_with(E_VALIDATION);
  }
  const Link* link(int a, int b) const {
    for (auto& l : P.links)
      if (l.src == a && l.dst == b) return &l;
    return nullptr;
  }
  std::vector<const Link*> route(int a, int b) const {  // transfer_time, platform.cpp:198-220
    if (const Link* d = link(a, b)) return {d};
    const Link* u = link(a, mainsp);
    const Link* w = link(mainsp, b);
    if (!u || !w) abort_with(E_NOROUTE);
    return {u, w};
  }
  ll bytes_of(int b) const {
    const Rect& g = G.blk.v[b].g;
    return g.h * g.w * G.elem;
  }
  std::vector<int> holders(int b) const {  // source_spaces, sim.cpp:341-350
    std::vector<int> o;
    if (mem.at(mainsp).valid.count(b)) o.push_back(mainsp);
    for (auto& [sid, m] : mem)
      if (sid != mainsp && m.valid.count(b)) o.push_back(sid);
    return o;
  }
  bool is_pinned(int s, int b) const { return pins.count({s, b}) > 0; }
  void add_pin(int s, int b, double until) {
    ++pins[{s, b}];
    unpin.emplace_back(until, s, b);
  }
  double move(int b, const Rect* frag, int src, int dst, double ready, double now) {  // sim.cpp:468-499
    const ll n = frag ? frag->h * frag->w * G.elem : bytes_of(b);
    double t = std::max(ready, now), first = 0;
    bool firsthop = true;
    for (const Link* l : route(src, dst)) {
      double& f = link_free[{l->src, l->dst}];
      const double st = std::max(f, t);
      const double en = st + l->lat + static_cast<double>(n) / l->bw;
      f = en;
      t = en;
      if (firsthop) first = st;
      firsthop = false;
    }
    xhash += hesp_xfer_term(b, src, dst, n, bits_of(first), bits_of(t), frag ? frag->r : 0, frag ? frag->c : 0,
                            frag ? frag->h : 0, frag ? frag->w : 0);
    return t;
  }
  void make_room(int s, ll n, double at) {  // ensure_capacity, sim.cpp:374-439
    Mem& m = mem.at(s);
    const ll cap = space(s).cap;
    if (n > cap) abort_with(E_CAPACITY);
    while (m.used + n > cap) {
      int vic = -1;
      double vst = 0;
      for (int x : m.mat) {
        if (is_pinned(s, x)) continue;
        if (s == mainsp) {
          if (G.blk.v[x].up.empty()) continue;
          bool other = false;
          for (auto& [sid, mm] : mem)
            if (sid != s && mm.valid.count(x)) other = true;
          if (!other) continue;
        }
        const double st = stamp.at({s, x});
        if (vic < 0 || st < vst || (st == vst && x < vic)) {
          vic = x;
          vst = st;
        }
      }
      if (vic < 0) abort_with(E_CAPACITY);
      const ll vb = bytes_of(vic);
      if (m.dirty.count(vic)) {
        const double arr = move(vic, nullptr, s, mainsp, m.valid.at(vic), at);
        m.dirty.erase(vic);
        place(vic, mainsp, arr);
      }
      m.mat.erase(vic);
      m.valid.erase(vic);
      m.used -= vb;
      stamp.erase({s, vic});
      const Rect& vr = G.blk.v[vic].g;
      for (auto it = m.valid.begin(); it != m.valid.end();) {
        const int x = it->first;
        if (m.mat.count(x) || !touches(G.blk.v[x].g, vr)) {
          ++it;
          continue;
        }
        bool cov = false;
        for (int y : m.mat)
          if (holds(G.blk.v[y].g, G.blk.v[x].g)) {
            cov = true;
            break;
          }
        if (cov || s == mainsp) ++it;
        else it = m.valid.erase(it);
      }
    }
  }
  void claim(int b, int s, double at) {  // reserve_bytes, sim.cpp:441-450
    Mem& m = mem.at(s);
    if (m.mat.count(b)) return;
    make_room(s, bytes_of(b), at);
    m.mat.insert(b);
    m.used += bytes_of(b);
    stamp[{s, b}] = at;
  }
  void freshen(int b, int s, double at) {  // validate_from, sim.cpp:452-461
    Mem& m = mem.at(s);
    auto low = [&](int x) {
      auto it = m.valid.find(x);
      if (it == m.valid.end() || it->second > at) m.valid[x] = at;
    };
    low(b);
    for (int d : G.blk.walk(b, true)) low(d);
    stamp[{s, b}] = std::max(stamp[{s, b}], at);
  }
  void place(int b, int s, double at) {
    claim(b, s, at);
    freshen(b, s, at);
  }
  double fetch(int b, int s, double now) {  // acquire, sim.cpp:501-519
    Mem& m = mem.at(s);
    auto it = m.valid.find(b);
    if (it != m.valid.end()) {
      stamp[{s, b}] = std::max(stamp[{s, b}], now);
      return it->second;
    }
    auto src = holders(b);
    src.erase(std::remove(src.begin(), src.end(), s), src.end());
    if (!src.empty()) {
      const double arr = move(b, nullptr, src.front(), s, mem.at(src.front()).valid.at(b), now);
      add_pin(src.front(), b, arr);
      place(b, s, arr);
      return arr;
    }
    return assemble(b, s, now);
  }
  double assemble(int b, int s, double now) {  // gather, sim.cpp:521-572
    const Rect tgt = G.blk.v[b].g;
    struct Piece {
      int id;
      bool here;
      ll area;
    };
    std::vector<Piece> cand;
    for (int x = 0; x < static_cast<int>(G.blk.v.size()); ++x) {
      if (x == b || !holds(tgt, G.blk.v[x].g)) continue;
      const bool here = mem.at(s).valid.count(x) > 0;
      if (!here && holders(x).empty()) continue;
      cand.push_back({x, here, G.blk.v[x].g.h * G.blk.v[x].g.w});
    }
    std::sort(cand.begin(), cand.end(), [](const Piece& a, const Piece& c) {
      return a.here != c.here ? a.here : a.area != c.area ? a.area > c.area : a.id < c.id;
    });
    double arr = 0;
    std::vector<Rect> got;
    for (const Piece& pc : cand) {
      const Rect& g = G.blk.v[pc.id].g;
      if (minus(g, got).empty()) continue;
      arr = std::max(arr, fetch(pc.id, s, now));
      got.push_back(g);
    }
    const auto rest = minus(tgt, got);
    if (!rest.empty()) {
      for (const Rect& f : rest)
        for (const Rect& w : written)
          if (touches(f, w)) abort_with(E_COHERENCE);
      if (s != mainsp)
        for (const Rect& f : rest) arr = std::max(arr, move(b, &f, mainsp, s, 0.0, now));
    }
    auto& v = mem.at(s).valid;
    auto it = v.find(b);
    if (it == v.end() || it->second > arr) v[b] = arr;
    return arr;
  }
  void wipe_elsewhere(int b, int keep) {  // invalidate_elsewhere + invalidation_cone, sim.cpp:204-212, 574-590
    std::set<int> cone{b};
    for (int d : G.blk.walk(b, true)) cone.insert(d);
    for (int c : std::set<int>(cone))
      for (int a : G.blk.walk(c, false)) cone.insert(a);
    for (auto& [sid, m] : mem) {
      if (sid == keep) continue;
      for (int c : cone) {
        if (m.mat.count(c)) {
          m.mat.erase(c);
          m.used -= bytes_of(c);
          stamp.erase({sid, c});
        }
        m.valid.erase(c);
        m.dirty.erase(c);
      }
    }
  }
  const std::string& type_of(int p) const { return P.types[P.procs[p].type]; }
  void run_task(int t, int p, double now) {  // commit, sim.cpp:592-668
    const Task& T = G.tk[t];
    const int s = P.procs[p].space;
    std::set<int> ws(T.rd.begin(), T.rd.end());
    ws.insert(T.wr.begin(), T.wr.end());
    ll tot = 0;
    for (int b : ws) tot += bytes_of(b);
    if (tot > space(s).cap) abort_with(E_CAPACITY);
    double in = 0;
    for (int b : ws) {
      in = std::max(in, fetch(b, s, now));
      ++pins[{s, b}];
    }
    const int out = T.wr.front();
    claim(out, s, now);
    const double st = std::max({busy_until[p], released.at(t), in});
    const double en = st + model_time(M, T.kind, T.b, type_of(p));
    busy_until[p] = en;
    span[t] = {st, en};
    where[t] = p;
    ahash += hesp_assign_term(t, p, bits_of(st), bits_of(en));
    for (int b : ws) unpin.emplace_back(en, s, b);
    wipe_elsewhere(out, s);
    freshen(out, s, en);
    mem.at(s).valid[out] = en;
    written.push_back(G.blk.v[out].g);
    if (s != mainsp) {
      if (C.caching == 1) {
        mem.at(s).dirty.insert(out);
      } else {
        const double arr = move(out, nullptr, s, mainsp, en, now);
        add_pin(s, out, arr);
        place(out, mainsp, arr);
        if (C.caching == 2) {
          Mem& m = mem.at(s);
          m.mat.erase(out);
          m.used -= bytes_of(out);
          stamp.erase({s, out});
          m.valid.erase(out);
          for (int d : G.blk.walk(out, true)) m.valid.erase(d);
        }
      }
    }
    finished.insert(t);
    for (int x : succ[t])
      if (--waiting.at(x) == 0) {
        double r = 0;
        for (int y : pred[x]) r = std::max(r, span.at(y).second);
        released[x] = r;
      }
  }
  uint64_t draw() { return hesp_splitmix_next(&rng); }
  Result go() {  // Engine::run, sim.cpp:704-834
    const auto order = G.program_order();
    const int n = static_cast<int>(order.size());
    const int np = static_cast<int>(P.procs.size());
    Result res;
    res.leaves = n;
    for (int t : order)
      for (auto& ty : P.types)
        if (!model_knows(M, G.tk[t].kind, ty)) abort_with(E_MODELMISS);
    // dependences: the full conflict relation over program order (E2), graph.cpp:656-694
    pred.assign(G.tk.size(), {});
    succ.assign(G.tk.size(), {});
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        const Task& a = G.tk[order[i]];
        const Task& b = G.tk[order[j]];
        auto clash = [&](const std::vector<int>& x, const std::vector<int>& y) {
          for (int u : x)
            for (int w : y)
              if (touches(G.blk.v[u].g, G.blk.v[w].g)) return true;
          return false;
        };
        if (clash(a.wr, b.rd) || clash(a.wr, b.wr) || clash(a.rd, b.wr)) {
          pred[order[j]].push_back(order[i]);
          succ[order[i]].push_back(order[j]);
        }
      }
    // init_memory, sim.cpp:323-339
    for (auto& s : P.spaces) mem[s.id];
    for (int x = 0; x < static_cast<int>(G.blk.v.size()); ++x)
      if (G.blk.v[x].up.empty() && !G.blk.v[x].isect) {
        mem[mainsp].mat.insert(x);
        mem[mainsp].valid[x] = 0;
        mem[mainsp].used += bytes_of(x);
        stamp[{mainsp, x}] = 0;
      }
    if (mem[mainsp].used > space(mainsp).cap) abort_with(E_CAPACITY);
    for (int x = 0; x < static_cast<int>(G.blk.v.size()); ++x)
      if (!mem[mainsp].valid.count(x)) mem[mainsp].valid[x] = 0;
    for (int p = 0; p < np; ++p) busy_until[p] = 0;
    if (C.ordering == 1) {  // critical_times, sim.cpp:92-115
      std::map<int, double> avg;
      for (int t : order) {
        double sum = 0;
        for (int p = 0; p < np; ++p) sum += model_time(M, G.tk[t].kind, G.tk[t].b, type_of(p));
        avg[t] = sum / np;
      }
      for (int i = n - 1; i >= 0; --i) {
        double best = 0;
        for (int x : succ[order[i]]) best = std::max(best, crit.at(x));
        crit[order[i]] = avg[order[i]] + best;
      }
    }
    for (int t : order) {
      waiting[t] = static_cast<int>(pred[t].size());
      if (!waiting[t]) released[t] = 0;
    }
    std::priority_queue<double, std::vector<double>, std::greater<>> clock;
    clock.push(0.0);
    int done = 0;
    while (done < n) {
      if (clock.empty()) abort_with(E_INTERNAL);
      const double now = clock.top();
      while (!clock.empty() && clock.top() <= now) clock.pop();
      for (auto it = unpin.begin(); it != unpin.end();) {
        if (std::get<0>(*it) <= now) {
          const auto k = std::make_pair(std::get<1>(*it), std::get<2>(*it));
          if (--pins[k] <= 0) pins.erase(k);
          it = unpin.erase(it);
        } else {
          ++it;
        }
      }
      std::vector<std::pair<int, double>> rdy;
      for (auto& [t, r] : released)
        if (!finished.count(t) && r <= now) rdy.push_back({t, r});
      std::sort(rdy.begin(), rdy.end(), [&](auto& a, auto& b) {
        if (C.ordering == 0) return a.second != b.second ? a.second < b.second : a.first < b.first;
        const double x = crit.at(a.first), y = crit.at(b.first);
        return x != y ? x > y : a.first < b.first;
      });
      for (auto& [t, r] : rdy) {
        const Task& T = G.tk[t];
        std::vector<double> est(np, 0.0);
        std::vector<bool> idle(np);
        bool some = false;
        for (int p = 0; p < np; ++p) {
          idle[p] = busy_until[p] <= now;
          some = some || idle[p];
          if (C.selection != 3) continue;
          const int sp = P.procs[p].space;
          std::map<std::pair<int, int>, double> acc;
          std::set<int> bs(T.rd.begin(), T.rd.end());
          bs.insert(T.wr.begin(), T.wr.end());
          double e = 0;
          for (int b : bs) {
            auto it = mem.at(sp).valid.find(b);
            if (it != mem.at(sp).valid.end()) {
              e = std::max(e, it->second);
              continue;
            }
            auto src = holders(b);
            src.erase(std::remove(src.begin(), src.end(), sp), src.end());
            if (src.empty()) continue;
            double ta = std::max(now, mem.at(src.front()).valid.at(b));
            for (const Link* l : route(src.front(), sp)) {
              double& a = acc[{l->src, l->dst}];
              a += l->lat + static_cast<double>(bytes_of(b)) / l->bw;
              ta += a;
            }
            e = std::max(e, ta);
          }
          est[p] = e;
        }
        if ((C.selection == 0 || C.selection == 1) && !some) break;
        int pick = -1;  // select_processor, sim.cpp:136-192
        if (C.selection == 0) {
          std::vector<int> pool;
          for (int p = 0; p < np; ++p)
            if (idle[p]) pool.push_back(p);
          const double u = static_cast<double>(draw() >> 11) * 0x1.0p-53;
          pick = pool[static_cast<size_t>(u * static_cast<double>(pool.size())) % pool.size()];
        } else if (C.selection == 1) {
          double bt = 0;
          for (int p = 0; p < np; ++p) {
            if (!idle[p]) continue;
            const double x = model_time(M, T.kind, T.b, type_of(p));
            if (pick < 0 || x < bt) {
              pick = p;
              bt = x;
            }
          }
        } else if (C.selection == 2) {
          pick = 0;
          for (int p = 1; p < np; ++p)
            if (busy_until[p] < busy_until[pick]) pick = p;
        } else {
          double bf = 0, bi = 0;
          for (int p = 0; p < np; ++p) {
            const double f = std::max({busy_until[p], released.at(t), est[p]}) + model_time(M, T.kind, T.b, type_of(p));
            if (pick < 0 || f < bf || (f == bf && busy_until[p] < bi)) {
              pick = p;
              bf = f;
              bi = busy_until[p];
            }
          }
        }
        if (pick < 0) abort_with(E_NOPROC);
        run_task(t, pick, now);
        ++done;
        clock.push(span.at(t).second);
      }
    }
    for (auto& [t, se] : span) res.makespan = std::max(res.makespan, se.second);
    res.ahash = ahash;
    res.xhash = xhash;
    return res;
  }
};

}  // namespace

Result evaluate(const Platform& plat, const Model& model, const Sched& sched, ll n, int elem, int s_base,
                const hesp_cand_desc& desc) {
  Result r;
  int leaves = 0;
  try {
    Graph g;
    g.elem = elem;
    g.blk.obtain(Rect{0, 0, n, n});
    g.tk.push_back(Task{HESP_CHOL, n, {0}, {0}, {}, true});
    g.split(0, s_base, sched.min_block);
    for (int k = 0; k < desc.n_ops; ++k) g.split(desc.ops[k].task, desc.ops[k].s, sched.min_block);
    leaves = static_cast<int>(g.program_order().size());
    Sim sim(plat, model, sched, g);
    r = sim.go();
    r.leaves = leaves;
  } catch (const Abort& a) {
    r = Result{};
    r.status = a.code;
    r.leaves = leaves;
  }
  return r;
}

}  // namespace port
