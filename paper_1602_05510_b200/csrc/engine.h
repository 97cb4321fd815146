// engine.h — one candidate partitioning -> expanded task DAG -> simulated
// schedule -> makespan, executed cooperatively by one warp.
//
// The same source is instantiated twice:
//   * Engine<DevWarp>  (nvcc, sm_100a): the product — one warp per candidate,
//     lanes = processors / blocks / cells, ballots and shuffles for selection,
//     compaction and release;
//   * Engine<HostWarp> (g++): width-1 build used on the host to precompute
//     the shared base tiling and, in tests/tools, to debug the engine logic
//     on a CPU.  It is never called on the product path.
//
// Reference behaviour restated here (file:line under /root/reference/proj):
//   graph build      graph.cpp:142-212 (DataDag), 301-392 (partitioners),
//                    397-513 (root_cholesky / partition_task), 632-737 (deps)
//   simulation       sim.cpp:92-192 (ct, ordering, selection), 341-668
//                    (coherence, transfers, commit), 704-834 (event loop)
//
// Equivalences this engine relies on (DESIGN.md §3 proves each):
//   E1 DataDag links form the Hasse diagram of strict region containment, so
//      descendants/ancestors/invalidation cones are geometric queries.
//   E2 Only the transitive closure of the dependence relation affects a
//      schedule; per-cell last-writer/readers tracking generates it.
//   E3 Every commit and transfer ends strictly after the current epoch, so
//      epochs strictly increase, a pin is live iff its release time > now,
//      and epochs that release nothing can be skipped.  Checked at run time
//      (ST_ENGINE_INVARIANT if ever violated).
#pragma once

#include "engine_types.h"

#if defined(__CUDACC__)
#define HHD __host__ __device__ inline  // width-1 warp policy methods
#define HX __device__ __forceinline__   // tiny accessors
#define HXN __device__ __noinline__     // engine phases: one copy each keeps the kernel i-cache sized
#define NOUNROLL _Pragma("unroll 1")
#else
#include <cstring>
#define HHD inline
#define HX inline
#define HXN inline
#define NOUNROLL
#endif
// successor-CSR loops of build_deps: independent atomics per predecessor
#ifndef HESP_SUCC_UNROLL
#define HESP_SUCC_UNROLL 4
#endif
constexpr int kSuccUnroll = HESP_SUCC_UNROLL;

namespace hx {

#if !defined(__CUDACC__)
struct int4 {
  int x, y, z, w;
};
struct int2 {
  int x, y;
};
#endif

#if defined(__CUDACC__)
// The device problem lives in constant memory (engine_kernels.cu uploads it
// before every launch); device code names it statically so no lane ever
// loads a problem pointer from its local stack.
__constant__ Problem c_problem;
#define PB ::hx::c_problem
#else
#define PB (*pbp)
#endif

constexpr double ABSENT = 1.0e308;  // "no valid copy" / "no pin"
constexpr double NOPIN = -1.0;
constexpr double HOLD = 1.0e307;    // pinned for the commit in progress

// ---------------------------------------------------------------------------
// Warp policies

// Width-1 policy: the host build, and on the device the thread-per-candidate
// simulate kernel (every lane runs its own candidate).
struct HostWarp {
  static constexpr int W = 1;
  HHD int lane() const { return 0; }
  HHD unsigned ballot(bool p) const { return p ? 1u : 0u; }
  HHD unsigned lt() const { return 0u; }
  HHD void sync() const {}
  template <class T>
  HHD T bcast(T v, int) const { return v; }
  HHD bool any(bool p) const { return p; }
  HHD int sumi(int v) const { return v; }
  HHD long long suml(long long v) const { return v; }
  HHD double maxd(double v) const { return v; }
  HHD double mind(double v) const { return v; }
  HHD int mini(int v) const { return v; }
  HHD int maxi(int v) const { return v; }
  // lexicographic argmin of (a, b, id); lanes with id < 0 do not participate
  HHD void argmin3(double& a, double& b, int& id) const { (void)a; (void)b; (void)id; }
  HHD void argmin_lane(double& a, double& b, int& id) const { (void)a; (void)b; (void)id; }
  HHD int atomic_add(int* p, int v) const {
    int o = *p;
    *p += v;
    return o;
  }
  HHD int exch(int* p, int v) const {
    int o = *p;
    *p = v;
    return o;
  }
  // per-lane owned vectors (device: one register per lane; host: the array)
  struct LaneD {
    double a[32];
    HHD double get(int i) const { return a[i]; }
    HHD void set(int i, double x) { a[i] = x; }
    HHD double& own(int i) { return a[i]; }
    HHD void fill(double x) {
      for (double& v : a) v = x;
    }
    template <class I>
    HHD void gather(const LaneD& src, const I& idx) {  // a[i] = src[idx[i]]
      for (int i = 0; i < 32; ++i) a[i] = src.a[idx.a[i]];
    }
  };
  struct LaneI {
    int a[32];
    HHD int get(int i) const { return a[i]; }
    HHD int& own(int i) { return a[i]; }
  };
};

#if defined(__CUDACC__)
struct DevWarp {
  static constexpr int W = 32;
  static constexpr unsigned FULL = 0xffffffffu;
  __device__ __forceinline__ int lane() const { return (int)(threadIdx.x & 31u); }
  __device__ __forceinline__ unsigned ballot(bool p) const { return __ballot_sync(FULL, p); }
  __device__ __forceinline__ unsigned lt() const { return (1u << lane()) - 1u; }
  __device__ __forceinline__ void sync() const { __syncwarp(); }
  __device__ __forceinline__ int bcast(int v, int src) const { return __shfl_sync(FULL, v, src); }
  __device__ __forceinline__ double bcast(double v, int src) const { return __shfl_sync(FULL, v, src); }
  __device__ __forceinline__ bool any(bool p) const { return __any_sync(FULL, p); }
  __device__ __forceinline__ int sumi(int v) const { return __reduce_add_sync(FULL, (unsigned)v); }
  __device__ __forceinline__ long long suml(long long v) const {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
  }
  __device__ __forceinline__ double maxd(double v) const {
    for (int o = 16; o; o >>= 1) {
      double w = __shfl_xor_sync(FULL, v, o);
      v = v < w ? w : v;
    }
    return v;
  }
  __device__ __forceinline__ double mind(double v) const {
    for (int o = 16; o; o >>= 1) {
      double w = __shfl_xor_sync(FULL, v, o);
      v = w < v ? w : v;
    }
    return v;
  }
  __device__ __forceinline__ int mini(int v) const { return __reduce_min_sync(FULL, v); }
  __device__ __forceinline__ int maxi(int v) const { return __reduce_max_sync(FULL, v); }
  __device__ __forceinline__ void argmin3(double& a, double& b, int& id) const {
    for (int o = 16; o; o >>= 1) {
      const double a2 = __shfl_xor_sync(FULL, a, o);
      const double b2 = __shfl_xor_sync(FULL, b, o);
      const int i2 = __shfl_xor_sync(FULL, id, o);
      bool take;
      if (i2 < 0) take = false;
      else if (id < 0) take = true;
      else if (a2 != a) take = a2 < a;
      else if (b2 != b) take = b2 < b;
      else take = i2 < id;
      if (take) {
        a = a2;
        b = b2;
        id = i2;
      }
    }
  }
  // Lexicographic argmin of (a, b, lane) over lanes with id == lane >= 0,
  // for a, b >= 0: IEEE order of non-negative doubles is the unsigned order of
  // their bits, so two 32-bit redux.sync minima per key plus ballots replace
  // five rounds of three-key shuffles.
  __device__ __forceinline__ void argmin_lane(double& a, double& b, int& id) const {
    const bool v = id >= 0;
    const unsigned long long ka = v ? (unsigned long long)__double_as_longlong(a) : ~0ULL;
    const unsigned ha = (unsigned)(ka >> 32), la = (unsigned)ka;
    const unsigned mh = __reduce_min_sync(FULL, ha);
    const unsigned ml = __reduce_min_sync(FULL, ha == mh ? la : 0xffffffffu);
    unsigned cand = __ballot_sync(FULL, v && ha == mh && la == ml);
    if (cand & (cand - 1)) {  // tie on a: minimise b among the tied lanes
      const bool c = (cand >> lane()) & 1u;
      const unsigned long long kb = c ? (unsigned long long)__double_as_longlong(b) : ~0ULL;
      const unsigned hb = (unsigned)(kb >> 32), lb = (unsigned)kb;
      const unsigned mhb = __reduce_min_sync(FULL, hb);
      const unsigned mlb = __reduce_min_sync(FULL, hb == mhb ? lb : 0xffffffffu);
      cand = __ballot_sync(FULL, c && hb == mhb && lb == mlb);
    }
    if (cand == 0) {
      id = -1;
      return;
    }
    const int w = __ffs((int)cand) - 1;
    a = __shfl_sync(FULL, a, w);
    b = __shfl_sync(FULL, b, w);
    id = w;
  }
  __device__ __forceinline__ int atomic_add(int* p, int v) const { return atomicAdd(p, v); }
  __device__ __forceinline__ int exch(int* p, int v) const { return atomicExch(p, v); }
  struct LaneD {
    double v;
    __device__ __forceinline__ double get(int i) const { return __shfl_sync(FULL, v, i); }
    __device__ __forceinline__ void set(int i, double x) {
      if ((int)(threadIdx.x & 31u) == i) v = x;
    }
    __device__ __forceinline__ double& own(int) { return v; }
    __device__ __forceinline__ void fill(double x) { v = x; }
    template <class I>
    __device__ __forceinline__ void gather(const LaneD& src, const I& idx) {  // all lanes must call
      v = __shfl_sync(FULL, src.v, idx.v & 31);
    }
  };
  struct LaneI {
    int v;
    __device__ __forceinline__ int get(int i) const { return __shfl_sync(FULL, v, i); }
    __device__ __forceinline__ int& own(int) { return v; }
  };
};
#endif

HX double dmax(double a, double b) { return a < b ? b : a; }  // == std::max
HX double dmin(double a, double b) { return b < a ? b : a; }
#if defined(__CUDACC__)
HX int ctz32(unsigned m) { return __ffs((int)m) - 1; }
HX int popc32(unsigned m) { return __popc(m); }
#else
HX int ctz32(unsigned m) { return __builtin_ctz(m); }
HX int popc32(unsigned m) { return __builtin_popcount(m); }
#endif
HX bool rcontains(const Region& o, const Region& i) {           // graph.cpp:34-38
  return i.row >= o.row && i.col >= o.col && i.row + i.rows <= o.row + o.rows &&
         i.col + i.cols <= o.col + o.cols;
}
HX bool roverlap(const Region& a, const Region& b) {  // graph.cpp:40-43
  return a.row < b.row + b.rows && b.row < a.row + a.rows && a.col < b.col + b.cols &&
         b.col < a.col + a.cols;
}
HX bool rsame(const Region& a, const Region& b) {
  return a.row == b.row && a.col == b.col && a.rows == b.rows && a.cols == b.cols;
}
HX uint64_t dbits(double x) {
  uint64_t u;
#if defined(__CUDACC__)
  u = (uint64_t)__double_as_longlong(x);
#else
  std::memcpy(&u, &x, 8);
#endif
  return u;
}

// A/B switches (-D at build time): 16-byte record loads in the lean loop.
#ifndef HESP_VEC_LOADS
#define HESP_VEC_LOADS 1
#endif
#ifndef HESP_MATCH_DEDUP
#define HESP_MATCH_DEDUP 1
#endif
#ifndef HESP_XPAR  // A/B only: 0 drops the intersection-link emulation (E7)
#define HESP_XPAR 1
#endif

// Folding a hash term into the warp's shared copy: a read-modify-write by
// every lane is only correct while the warp is converged, so (1) one lane
// folds, or (2) the warp reconverges first; (0) the unguarded form (A/B only).
#ifndef HESP_HASH_FOLD
#define HESP_HASH_FOLD 1
#endif
#if HESP_HASH_FOLD == 1
#define HASH_FOLD(acc, t)                   \
  do {                                      \
    if (wp.lane() == 0) (acc) += (t);       \
  } while (0)
#elif HESP_HASH_FOLD == 2
#define HASH_FOLD(acc, t) \
  do {                    \
    wp.sync();            \
    (acc) += (t);         \
  } while (0)
#else
#define HASH_FOLD(acc, t) ((acc) += (t))
#endif

// 32-byte records in two 16-byte loads (the generic path otherwise splits
// them field by field).
HX STask ld_stask(const STask* p) {
#if defined(__CUDACC__) && HESP_VEC_LOADS
  const int4 a = reinterpret_cast<const int4*>(p)[0], b = reinterpret_cast<const int4*>(p)[1];
  STask t;
  t.ws0 = a.x; t.ws1 = a.y; t.ws2 = a.z; t.nw = a.w;
  t.out = b.x; t.kb = b.y; t.b = b.z; t.pad = b.w;
  return t;
#else
  return *p;
#endif
}
HX TState ld_tstate(const TState* p) {
#if defined(__CUDACC__) && HESP_VEC_LOADS
  const double2 a = reinterpret_cast<const double2*>(p)[0];
  const int4 b = reinterpret_cast<const int4*>(p)[1];
  TState t;
  t.rel = a.x; t.ct = a.y;
  t.missing = b.x; t.soff = b.y; t.scnt = b.z; t.pad = b.w;
  return t;
#else
  return *p;
#endif
}

// Small per-warp state (shared memory on the device).
// State of the lean event loop across its cold exits (sim_lean): the loop
// returns to its driver for every call-requiring step, so no value is live
// across a call inside the hot loop and nothing spills.
struct LeanState {
  double tnow, mk, pmin;
  int32_t pool_n, committed, done, nr, first;
  int32_t phase;                  // resume point of the task in progress: 0 none, 1 acquire, 2 coherence done, 3 write-back done
  int32_t r_k, r_p, r_s;          // block being acquired, processor, space
  double r_inputs, r_start, r_end;
  int32_t op, op_b, op_s, pad_;   // cold request
  double op_at, op_at2, op_result;
};

struct Small {
  double proc_free[MAXP];
  double link_free[MAXL];
  long long used[MAXS];
  uint64_t ah, xh;  // event-loop result hashes (one copy per warp)
  int32_t ptype[MAXP], pspace[MAXP];
  BaseView bv;  // the candidate's top-level tiling and reference-id offsets
  int32_t nxp;  // candidate intersection descriptors holding extra (non-Hasse) DataDag parent links
  int32_t nxp_pad;
  double* vstage;  // the lean loop's valid-time table in shared memory (HESP_VSTAGE experiment), else null
  double* vst_base;  // this warp's staging area and its capacity in doubles (set by sim_kernel)
  int32_t vst_cap, vst_pad;
  LeanState L;
};
static_assert(sizeof(Small) <= SMALL_BYTES, "slot reserve for Small");

#if defined(__CUDACC__)
// One Small per warp of a CTA (<= 4 warps), declared at namespace scope so
// every access compiles to LDS/STS (a Small* parameter would be a generic
// pointer: LD/ST through the generic path).  Each kernel that touches it gets
// its own per-CTA allocation.
constexpr int SMALL_WARPS = 4;
__shared__ Small g_small[SMALL_WARPS];
// The candidate's top-level tiling view and link counter, apart from Small so
// the build kernels (which need only these) do not carve Small's ~1 KB per
// warp of event-loop state out of their L1.
__shared__ BaseView g_bview[SMALL_WARPS];
__shared__ int32_t g_nxp[SMALL_WARPS];
#endif

// ---------------------------------------------------------------------------
// Engine

template <class WP, bool TRACE = false>
struct Engine {
  WP wp;
  const Problem* pbp;
  Small* sm;
  // slot arrays: offsets from the (constant-memory) problem, no per-lane pointer copies
  uint8_t* slot;
  HX SlotHeader* hdr() const { return (SlotHeader*)(slot + PB.lay.hdr); }
  HX TaskMeta* tm() const { return (TaskMeta*)(slot + PB.lay.tm); }
  HX TState* ts() const { return (TState*)(slot + PB.lay.ts); }
  HX int32_t* t_poff() const { return (int32_t*)(slot + PB.lay.t_poff); }
  HX int32_t* t_pcnt() const { return (int32_t*)(slot + PB.lay.t_pcnt); }
  HX int32_t* leaf() const { return (int32_t*)(slot + PB.lay.leaf); }
  // per-task event-loop record (built in build_deps)
  HX STask* wsb() const { return (STask*)(slot + PB.lay.wsb); }
  HX int4* bcell() const { return (int4*)(slot + PB.lay.bcell); }      // cell range per block
  HX uint16_t* rht() const { return (uint16_t*)(slot + PB.lay.rht); }  // region hash of new blocks
  HX uint8_t* pmark() const { return (uint8_t*)(slot + PB.lay.pmark); }  // 1 + partition entry per task id
  HX int32_t* bref() const { return (int32_t*)(slot + PB.lay.bref); }     // by candidate block id - n_bb()
  HX int32_t* xpar() const { return (int32_t*)(slot + PB.lay.xpar); }     // [candidate block - n_bb()][XPAR]
  HX PartEntry* part() const { return (PartEntry*)(slot + PB.lay.part); }  // clusters, by id
  HX int32_t* dstack() const { return (int32_t*)(slot + PB.lay.dstack); }
  HX uint8_t* tmis() const { return (uint8_t*)(slot + PB.lay.tmis); }
  HX uint8_t* wrt() const { return (uint8_t*)(slot + PB.lay.wrt); }
  HX int32_t* pmk() const { return (int32_t*)(slot + PB.lay.pmk); }
  HX BlockMeta* bm() const { return (BlockMeta*)(slot + PB.lay.bm); }
  HX uint32_t* bflags() const { return (uint32_t*)(slot + PB.lay.bflags); }
  HX double* valid() const {
#if defined(__CUDACC__)
    if constexpr (WP::W > 1) {
      double* vs = SM().vstage;  // SMEM-staging experiment (sim_kernel, HESP_VSTAGE > 0)
      if (vs) return vs;
    }
#endif
    return (double*)(slot + PB.lay.valid);
  }
  HX double* lastu() const { return (double*)(slot + PB.lay.lastu); }
  HX double* pinu() const { return (double*)(slot + PB.lay.pinu); }
  HX int32_t* tl_head() const { return (int32_t*)(slot + PB.lay.tl_head); }
  HX int32_t* tl_cnt() const { return (int32_t*)(slot + PB.lay.tl_cnt); }
  HX int32_t* tl_boff() const { return (int32_t*)(slot + PB.lay.tl_boff); }
  HX int32_t* tl_nrb() const { return (int32_t*)(slot + PB.lay.tl_nrb); }
  HX int32_t* tl_ncb() const { return (int32_t*)(slot + PB.lay.tl_ncb); }
  HX int32_t* tl_coff() const { return (int32_t*)(slot + PB.lay.tl_coff); }
  HX int32_t* tl_ids() const { return (int32_t*)(slot + PB.lay.tl_ids); }
  HX int32_t* bnd() const { return (int32_t*)(slot + PB.lay.bnd); }
  HX int32_t* c_writer() const { return (int32_t*)(slot + PB.lay.c_writer); }
  HX int32_t* c_rhead() const { return (int32_t*)(slot + PB.lay.c_rhead); }
  HX int32_t* rnode() const { return (int32_t*)(slot + PB.lay.rnode); }
  HX int32_t* preds() const { return (int32_t*)(slot + PB.lay.preds); }
  HX int32_t* succs() const { return (int32_t*)(slot + PB.lay.succs); }
  HX int32_t* pool() const { return (int32_t*)(slot + PB.lay.pool); }
  HX double* pool_rel() const { return (double*)(slot + PB.lay.pool_rel); }
  HX double* pool_key() const { return (double*)(slot + PB.lay.pool_key); }
  HX double* ready_key() const { return (double*)(slot + PB.lay.ready_key); }
  HX int32_t* ready() const { return (int32_t*)(slot + PB.lay.ready); }
  HX int32_t* pbuf() const { return (int32_t*)(slot + PB.lay.pbuf); }
  // build_deps' per-task access records (4 x int2 per task id), over the
  // simulate-only pool/ready arrays (written only once the event loop starts;
  // slot_layout checks the span)
  HX int2* dacc() const { return (int2*)(slot + PB.lay.pool); }
  HX int32_t* gs_a() const { return (int32_t*)(slot + PB.lay.gs_a); }
  HX int32_t* gs_b() const { return (int32_t*)(slot + PB.lay.gs_b); }
  HX Region* gs_reg() const { return (Region*)(slot + PB.lay.gs_reg); }
  HX Region* gs_reg2() const { return (Region*)(slot + PB.lay.gs_reg2); }
  // scalars (uniform across lanes)
  int32_t status = 0;
  // base task / block counts (overlay boundary), space count, main space:
  // read from the problem (constant memory), never from `this` (the engine
  // object lives in local memory on the device)
  HX int n_bt() const {
    return BV().nbt;
  }
  HX int n_bb() const {
    return BV().nbb;
  }
  HX const TaskMeta* bt_() const {
    return BV().bt;
  }
  HX const BlockMeta* bb_() const {
    return BV().bb;
  }
  HX const BasePreds* bp_() const {
    return BV().bp;
  }
  HX const int32_t* bpl_() const {
    return BV().bpl;
  }
  HX long long base_b_() const {
    return BV().base_b;
  }
  // reference ids of internal task / block ids (BaseView)
  HX int xtask(int j) const {
    return j ? j + BV().off_t : 0;
  }
  HX int xblock(int b) const {
    return b ? b + BV().off_b : 0;
  }
  HX int n_sp() const { return PB.S; }
  HX int msp() const { return PB.main_space; }
  int32_t ntasks, nblocks;  // next ids
  int32_t npart = 0;
  int32_t nleaves = 0;
  int32_t n_tl_ids = 0;
  int32_t nedges = 0;
  int32_t sum_k = 0;  // sum over leaves of distinct blocks accessed (k_t)
  int32_t pool_n = 0;
  double now = 0.0;
  double makespan = 0.0;
  uint64_t ahash = 0, xhash = 0;
  uint64_t rng = 0;
  // No-eviction fast path (DESIGN.md §3 E4): when every block but the root
  // fits in every space (plus the root in main), ensure_capacity can never
  // evict, so LRU stamps, pins, mat/dirty flags and `used` -- read only by
  // eviction -- need not be maintained.
  bool fast = false;
  // optional per-task schedule trace (hesp_eval_detail): proc/start/end by task id
  int32_t* tr_proc = nullptr;
  double *tr_start = nullptr, *tr_end = nullptr;
  int32_t tr_cap = 0;
  TraceBufs* tb = nullptr;  // full-trace sinks (TRACE only)

  // ---- full-trace logging (compiled out unless TRACE) ----
  HX void log_res(double t, int s, long long delta, int b) {  // one lane calls
    if constexpr (TRACE) {
      if (!tb || tb->lite) return;
      const int k = atomic_slot(&tb->nr);
      if (k < tb->rcap) {
        ResLog r;
        r.time = t;
        r.space = s;
        r.block = b;
        r.delta = delta;
        tb->r[k] = r;
      } else {
        tb->overflow = 1;
      }
    }
  }
  HX void log_xfer(int blk, const Region* frag, long long bytes, int src, int dst, double start0, double end,
                   int nh, const double* hs, const double* he) {  // uniform: lane 0 writes
    if constexpr (TRACE) {
      if (!tb || tb->lite) return;
      if (wp.lane() == 0) {
        const int k = tb->nx++;
        if (k < tb->xcap) {
          XferLog x;
          x.block = blk;
          x.src = src;
          x.dst = dst;
          x.nh = nh;
          x.bytes = bytes;
          x.start = start0;
          x.end = end;
          x.has_frag = frag ? 1 : 0;
          x.frow = frag ? frag->row : 0;
          x.fcol = frag ? frag->col : 0;
          x.frows = frag ? frag->rows : 0;
          x.fcols = frag ? frag->cols : 0;
          x.pad = 0;
          for (int h = 0; h < 2; ++h) {
            x.hs[h] = h < nh ? hs[h] : 0.0;
            x.he[h] = h < nh ? he[h] : 0.0;
          }
          tb->x[k] = x;
        } else {
          tb->overflow = 1;
        }
      }
      wp.sync();
    }
  }
  HX int atomic_slot(int32_t* c) const {
#if defined(__CUDACC__)
    return atomicAdd(c, 1);
#else
    return (*c)++;
#endif
  }

  HX Engine(WP w, const Problem& p, uint8_t* slot_, Small* s) : wp(w), pbp(&p), sm(s), slot(slot_) {
  }

  HX void fail(int32_t code) {
    if (status == 0) status = code;
  }

  // The warp's Small: real shared memory on the device (warp-wide engine),
  // the caller's buffer for the width-1 instantiations.
  HX Small& SM() const {
#if defined(__CUDACC__)
    if constexpr (WP::W > 1) return g_small[threadIdx.x >> 5];
#endif
    return *sm;
  }
  HX BaseView& BV() const {
#if defined(__CUDACC__)
    if constexpr (WP::W > 1) return g_bview[threadIdx.x >> 5];
#endif
    return sm->bv;
  }
  HX int32_t& NXP() const {
#if defined(__CUDACC__)
    if constexpr (WP::W > 1) return g_nxp[threadIdx.x >> 5];
#endif
    return sm->nxp;
  }

  // ---- overlay accessors (base graph shared, candidate deltas private) ----
  HX TaskMeta task(int id) const { return id < n_bt() ? bt_()[id] : tm()[id - n_bt()]; }
  HX const BlockMeta& bmeta(int b) const { return b < n_bb() ? bb_()[b] : bm()[b - n_bb()]; }
  HX Region reg(int b) const { return bmeta(b).r; }
  HX int tile_of(int b) const { return bmeta(b).tile; }
  HX long long rbytes(const Region& r) const { return (long long)r.rows * r.cols * PB.elem; }
  HX long long bbytes(int b) const { return rbytes(reg(b)); }
  HX double& V(int b, int s) { return valid()[(size_t)b * n_sp() + s]; }
  HX double& LU(int b, int s) { return lastu()[(size_t)b * n_sp() + s]; }
  HX double& PIN(int b, int s) { return pinu()[(size_t)b * n_sp() + s]; }
  HX bool is_mat(int b, int s) const { return (bflags()[b] >> s) & 1u; }
  HX bool is_dirty(int b, int s) const { return (bflags()[b] >> (8 + s)) & 1u; }
  HX int part_index(int task) const {
    NOUNROLL for (int i = 0; i < npart; ++i)
      if (part()[i].task == task) return i;
    return -1;
  }
  // O(1) variant once pmark() is filled (build_order onwards)
  HX int part_of(int task) const { return (int)pmark()[task] - 1; }
  // base tile with no sub-blocks: its invalidation cone is {root, itself}
  // and it has no descendants (E1)
  HX bool simple_tile(int b) const {
    const int tt = b == 0 ? -1 : tile_of(b);
    return tt > 0 && tl_cnt()[tt] == 0;
  }
  HX int bidx_of(long long b) const {
    NOUNROLL for (int i = 0; i < PB.nbv; ++i)
      if (PB.bval[i] == b) return i;
    return -1;
  }

  // =========================================================================
  // Graph build: DataDag::get_or_create / partition_task
  // =========================================================================

  // Existing block with exactly region r (DataDag::find_by_region).  t >= 0:
  // r lies inside base tile t, so only the root, the tile and the tile's
  // blocks can match.  t < 0 (base build): every block.
  static HX unsigned rhash(const Region& r) {
    unsigned h = (unsigned)r.row * 0x9E3779B1u ^ (unsigned)r.col * 0x85EBCA77u ^ (unsigned)r.rows * 0xC2B2AE3Du;
    h ^= h >> 15;
    return h * 0x27D4EB2Fu;
  }
  HX bool rht_usable() const { return nblocks - n_bb() < RHT / 2; }

  HXN int find_block(const Region& r, int t) {
    if (t < 0) {
      int found = -1;
      NOUNROLL for (int base = 0; base < nblocks; base += WP::W) {
        const int b = base + wp.lane();
        const bool hit = b < nblocks && rsame(reg(b), r);
        const unsigned m = wp.ballot(hit);
        if (m) {
          found = base + ctz32(m);
          break;
        }
      }
      return found;
    }
    if (r.rows >= base_b_() || r.cols >= base_b_()) {  // only a tile- or root-sized region can be either
      if (rsame(reg(0), r)) return 0;
      if (rsame(reg(t), r)) return t;
    }
    if (rht_usable()) {  // open addressing over the candidate's own blocks
      unsigned i = rhash(r) & (RHT - 1);
      NOUNROLL for (;;) {
        const int e = rht()[i];
        if (e == 0xffff) return -1;
        if (rsame(bm()[e].r, r)) return n_bb() + e;
        i = (i + 1) & (RHT - 1);
      }
    }
    NOUNROLL for (int base = n_bb(); base < nblocks; base += WP::W) {
      const int b = base + wp.lane();
      const bool hit = b < nblocks && bm()[b - n_bb()].tile == t && rsame(bm()[b - n_bb()].r, r);
      const unsigned m = wp.ballot(hit);
      if (m) return base + ctz32(m);
    }
    return -1;
  }

  HXN int create_block(const Region& r, bool isint, int t) {  // DataDag::create, graph.cpp:142-189
    if (nblocks >= PB.maxb) {
      fail(ST_ENGINE_LIMIT);
      return -1;
    }
    const int id = nblocks++;
    BlockMeta m;
    m.r = r;
    m.tile = t < 0 ? id : t;  // base build: every new block is a base tile
    m.next = -1;
    m.isint = isint ? 1 : 0;
    m.pad = 0;
    if (wp.lane() == 0) {
      bm()[id - n_bb()] = m;
      bref()[id - n_bb()] = 0;
      if (isint)  // extra parent links are only ever read for intersection descriptors
        NOUNROLL for (int k = 0; k < XPAR; ++k) xpar()[(id - n_bb()) * XPAR + k] = -1;
    }
    if (t >= 0 && id - n_bb() < RHT / 2) {
      unsigned i = rhash(r) & (RHT - 1);
      while (rht()[i] != 0xffff) i = (i + 1) & (RHT - 1);
      if (wp.lane() == 0) rht()[i] = (uint16_t)(id - n_bb());
    }
    wp.sync();
#if HESP_XPAR
    if (t >= 0 && NXP() > 0) xpar_on_create(id, t);  // (shared memory: no local-memory load per block)
#endif
    return id;
  }

  // ---- DataDag parent links of intersection descriptors (graph.cpp:142-266) ----
  // A prune erases an intersection descriptor when any of its *parents* dies
  // (graph.cpp:221-228).  Its parents are its minimal strict containers (E1:
  // create() links a block to them and unlinks the pairs it bridges,
  // graph.cpp:142-189) plus the links get_or_create adds when a partial
  // overlap's intersection already exists (graph.cpp:203-206), which need
  // not be minimal.  Those extra links are kept per intersection (xpar) and
  // dropped exactly when create() would unlink them.

  // Minimal strict containers of region r among the live blocks of tile t
  // (root and tile included), excluding block `self`; into out[], count
  // returned (-1: more than cap).
  HXN int min_containers(const Region& r, int t, int self, int* out, int cap) {
    int n = 0;
    auto consider = [&](int x) {
      if (x == self) return;
      const Region rx = reg(x);
      if (dead_region(rx) || rsame(rx, r) || !rcontains(rx, r)) return;
      // minimal: no other live container strictly inside x
      bool minimal = true;
      NOUNROLL for (int y = n_bb(); y < nblocks && minimal; ++y) {
        if (y == self || y == x || tile_of(y) != t) continue;
        const Region ry = reg(y);
        if (!dead_region(ry) && !rsame(ry, r) && rcontains(ry, r) && !rsame(ry, rx) && rcontains(rx, ry))
          minimal = false;
      }
      if (x == 0 && minimal && !rsame(reg(t), r) && rcontains(reg(t), r)) minimal = false;  // the tile is inside the root
      if (minimal) {
        if (n < cap) out[n] = x;
        ++n;
      }
    };
    consider(0);
    consider(t);
    NOUNROLL for (int x = n_bb(); x < nblocks; ++x)
      if (tile_of(x) == t) consider(x);
    return n <= cap ? n : -1;
  }
  HX int32_t& XP(int b, int k) const { return xpar()[(b - n_bb()) * XPAR + k]; }
  HX void xpar_remove(int b, int v) {
    int w = 0;
    for (int k = 0; k < XPAR; ++k) {
      const int e = XP(b, k);
      if (e >= 0 && e != v) XP(b, w++) = e;
    }
    for (; w < XPAR; ++w) XP(b, w) = -1;
  }
  HX bool xpar_add(int b, int v) {  // false: no room
    for (int k = 0; k < XPAR; ++k) {
      const int e = XP(b, k);
      if (e == v) return true;
      if (e < 0) {
        if (k == 0) ++NXP();
        XP(b, k) = v;
        return true;
      }
    }
    return false;
  }
  // create(N) unlinks (p, c) for p in parents(N), c in children(N) (the
  // maximal blocks strictly inside N): an intersection's extra parent p goes
  // when N now sits between them.  Lane 0 works, the warp waits (rare path:
  // only candidates with extra links).
  // scratch for the rare link paths below (lane 0): the gather region
  // buffer, unused while a candidate is being built
  HX int32_t* lscratch() const { return (int32_t*)gs_reg(); }
  HXN void xpar_on_create(int nid, int t) {
    if (wp.lane() == 0) {
      const Region rn = reg(nid);
      int* par = lscratch();
      const int np = min_containers(rn, t, nid, par, 8);
      if (np < 0) {
        fail(ST_ENGINE_LIMIT);
      } else {
        NOUNROLL for (int i = n_bb(); i < nblocks; ++i) {
          if (i == nid || !bmeta(i).isint || XP(i, 0) < 0 || tile_of(i) != t) continue;
          const Region ri = reg(i);
          if (dead_region(ri) || rsame(ri, rn) || !rcontains(rn, ri)) continue;
          bool maximal = true;  // no live block strictly between i and N
          NOUNROLL for (int y = n_bb(); y < nblocks && maximal; ++y) {
            if (y == i || y == nid || tile_of(y) != t) continue;
            const Region ry = reg(y);
            if (!dead_region(ry) && !rsame(ry, ri) && !rsame(ry, rn) && rcontains(ry, ri) && rcontains(rn, ry))
              maximal = false;
          }
          if (!maximal) continue;
          NOUNROLL for (int k = 0; k < np; ++k) xpar_remove(i, par[k]);
          if (XP(i, 0) < 0) --NXP();
        }
      }
    }
    status = wp.bcast(status, 0);
    wp.sync();
  }
  // prune_unreferenced's treatment of intersection descriptors (graph.cpp:
  // 216-228, 256-262) before the non-intersection blocks of a merge die:
  // in id order, an intersection dies when any parent is dead.  `top`: the
  // merge of the top cluster (every block but the root dies).  A survivor
  // left with a dead parent would be relinked (graph.cpp:229-255): 201.  A
  // dying intersection a live task still references makes the reference's
  // own infer_dependences throw std::out_of_range from map::at: status 100.
  HXN void prune_intersections(bool top) {
    if (wp.lane() == 0) {
      int32_t* dead = gs_b();  // scratch: candidate block -> 1 if dead
      NOUNROLL for (int b = n_bb(); b < nblocks; ++b) {
        const BlockMeta& o = bm()[b - n_bb()];
        dead[b - n_bb()] = !dead_region(o.r) && !o.isint && (top || bref()[b - n_bb()] == 0);
      }
      auto is_dead = [&](int p) -> bool { return p >= n_bb() ? dead[p - n_bb()] != 0 : (top && p != 0); };
      bool limit = false;
      for (int pass = 0; pass < 2 && !limit; ++pass) {
        NOUNROLL for (int i = n_bb(); i < nblocks && !limit; ++i) {
          const BlockMeta& o = bm()[i - n_bb()];
          if (!o.isint || dead_region(o.r) || (pass == 0 && dead[i - n_bb()])) continue;
          if (pass == 1 && dead[i - n_bb()]) continue;
          int* par = lscratch();
          const int np = min_containers(o.r, o.tile, i, par, 8);
          if (np < 0) {
            limit = true;
            break;
          }
          bool d = false;
          NOUNROLL for (int k = 0; k < np; ++k) d |= is_dead(par[k]);
          NOUNROLL for (int k = 0; k < XPAR; ++k) d |= XP(i, k) >= 0 && is_dead(XP(i, k));
          if (pass == 0) {
            dead[i - n_bb()] = d ? 1 : 0;
          } else if (d) {
            // survived with a dead parent (a higher-id intersection died
            // after it was checked): it inherits links to its nearest alive
            // ancestors through dead blocks (alive_ancestors, graph.cpp:229-255)
            if (top) {
              limit = true;
              break;
            }
            int* work = lscratch() + 16;
            int nw = 0;
            auto push_dead_parents = [&](int b) {
              int* pp = lscratch() + 8;
              const Region rb = reg(b);
              const int n2 = min_containers(rb, tile_of(b), b, pp, 8);
              if (n2 < 0) {
                limit = true;
                return;
              }
              auto visit = [&](int q) {
                if (is_dead(q)) {
                  bool seen = false;
                  for (int z = 0; z < nw; ++z) seen |= work[z] == q;
                  if (!seen) {
                    if (nw < 16) work[nw++] = q;
                    else limit = true;
                  }
                } else if (!xpar_add(i, q)) {
                  limit = true;
                }
              };
              NOUNROLL for (int k = 0; k < n2; ++k) visit(pp[k]);
              if (b >= n_bb() && bmeta(b).isint)
                NOUNROLL for (int k = 0; k < XPAR; ++k)
                  if (XP(b, k) >= 0) visit(XP(b, k));
            };
            push_dead_parents(i);
            NOUNROLL for (int z = 0; z < nw && !limit; ++z) push_dead_parents(work[z]);
            NOUNROLL for (int z = 0; z < nw; ++z) xpar_remove(i, work[z]);  // the dead ones go with the erase
          }
        }
      }
      if (limit) {
        fail(ST_ENGINE_LIMIT);
      } else {
        NOUNROLL for (int i = n_bb(); i < nblocks; ++i) {
          BlockMeta& o = bm()[i - n_bb()];
          if (!o.isint || !dead[i - n_bb()]) continue;
          if (!top && bref()[i - n_bb()] > 0) {
            // erased while a task still references it: the reference's
            // infer_dependences throws at once if that task is a leaf; a
            // dangling reference from a partitioned task is not modelled
            bool leaf_ref = false;
            NOUNROLL for (int m = n_bt(); m < ntasks; ++m) {
              if (dead_task(m)) continue;
              const TaskMeta tmm = tm()[m - n_bt()];
              bool refs = false;
              NOUNROLL for (int k = 0; k <= tmm.nrd; ++k) refs |= tmm.blk[k] == i;
              if (refs && part_index(m) < 0) leaf_ref = true;
            }
            fail(leaf_ref ? ST_FOREIGN : ST_ENGINE_LIMIT);
          }
          if (XP(i, 0) >= 0) --NXP();
          NOUNROLL for (int k = 0; k < XPAR; ++k) XP(i, k) = -1;
          o.r.row = -1;
          o.r.col = -1;
          o.r.rows = 0;
          o.r.cols = 0;
        }
      }
    }
    status = wp.bcast(status, 0);
    wp.sync();
  }

  // r is a dyadic square of base tile t: side = tile side / 2^k at an offset
  // that is a multiple of the side.  Two dyadic squares of one tile are
  // nested or disjoint, never partially overlapping.
  HX bool dyadic(const Region& r, int t) const {
    const Region T = reg(t);
    if (r.rows != r.cols || r.rows <= 0 || T.rows % r.rows) return false;
    const int q = T.rows / r.rows;
    return (q & (q - 1)) == 0 && (r.row - T.row) % r.rows == 0 && (r.col - T.col) % r.cols == 0;
  }

  HXN int get_or_create(const Region& r, int t) {  // graph.cpp:191-212
    const int ex = find_block(r, t);
    if (ex >= 0) return ex;
    const int id = create_block(r, false, t);
    if (id < 0) return -1;
    // Partial overlaps with existing non-intersection blocks get an
    // intersection descriptor (id order).  Inside tile t only the tile's own
    // blocks can partially overlap r (root and tile contain it), and none can
    // while every block of the tile (r included) is dyadic: skip the scan.
    if (t >= 0) {
      if (dyadic(r, t) && !tmis()[t]) return id;
      if (wp.lane() == 0) tmis()[t] = 1;
      wp.sync();
    }
    int nsect = 0;
    const int lo = t < 0 ? 0 : n_bb();
    NOUNROLL for (int base = lo; base < id; base += WP::W) {
      const int b = base + wp.lane();
      bool hit = false;
      if (b < id) {
        const BlockMeta& o = bmeta(b);
        hit = (t < 0 || o.tile == t) && !o.isint && !rcontains(o.r, r) && !rcontains(r, o.r) &&
              roverlap(o.r, r);
      }
      const unsigned m = wp.ballot(hit);
      if (hit) {
        const int slot = nsect + popc32(m & wp.lt());
        if (slot < PB.maxgs) gs_a()[slot] = b;
      }
      nsect += popc32(m);
    }
    wp.sync();
    if (nsect > PB.maxgs) {
      fail(ST_ENGINE_LIMIT);
      return -1;
    }
    if (nsect > 0 && t < 0) {
      fail(ST_ENGINE_LIMIT);  // the base tiling never overlaps partially
      return -1;
    }
    NOUNROLL for (int k = 0; k < nsect; ++k) {
      const Region o = reg(gs_a()[k]);
      Region sct;
      sct.row = o.row > r.row ? o.row : r.row;
      sct.col = o.col > r.col ? o.col : r.col;
      const int r1 = (o.row + o.rows < r.row + r.rows) ? o.row + o.rows : r.row + r.rows;
      const int c1 = (o.col + o.cols < r.col + r.cols) ? o.col + o.cols : r.col + r.cols;
      sct.rows = r1 - sct.row;
      sct.cols = c1 - sct.col;
      const int ex = find_block(sct, t);
      if (ex < 0) {
        if (create_block(sct, true, t) < 0) return -1;
      } else if (HESP_XPAR && bmeta(ex).isint) {
        // link(id, ex), link(other, ex) (graph.cpp:203-206): not necessarily Hasse
        bool ok = true;
        if (wp.lane() == 0) ok = xpar_add(ex, id) && xpar_add(ex, gs_a()[k]);
        wp.sync();
        if (wp.any(!ok)) {
          fail(ST_ENGINE_LIMIT);
          return -1;
        }
      }
    }
    return id;
  }

  // Region of tile (i, j) of an s x s tiling of r (graph.cpp:294-297).
  static HX Region sub(const Region& r, int s, int i, int j) {
    const int tb = r.rows / s;
    Region o;
    o.row = r.row + i * tb;
    o.col = r.col + j * tb;
    o.rows = tb;
    o.cols = tb;
    return o;
  }

  // One emitted sub-task: resolve its regions to blocks (reads in spec order,
  // then the write: graph.cpp:500-501) and append it with the next task id.
  HXN void emit(int kind, int nr, const Region* rr, const int* rt, const Region& w, int wt) {
    if (ntasks >= PB.maxt) {
      fail(ST_ENGINE_LIMIT);
      return;
    }
    TaskMeta m;
    m.pad = 0;
    // the 4 block slots with constant indices (the record stays in registers)
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      if (k >= nr) break;
      m.blk[k] = get_or_create(rr[k], rt[k]);
      if (status) return;
    }
    const int wblk = get_or_create(w, wt);
    if (status) return;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k == nr) m.blk[k] = wblk;
      else if (k > nr) m.blk[k] = -1;
    }
    m.kind = (int8_t)kind;
    m.nrd = (int8_t)nr;
    m.b = w.rows;
    const int bi = bidx_of(w.rows);
    if (bi < 0) {
      fail(ST_ENGINE_LIMIT);  // block side missing from the host time table
      return;
    }
    m.bidx = (int8_t)bi;
    const int id = ntasks++;
    if (wp.lane() == 0) {
      tm()[id - n_bt()] = m;
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if (k <= nr && m.blk[k] >= n_bb()) ++bref()[m.blk[k] - n_bb()];
    }
    wp.sync();
  }

  // merged-away task (member of a dead cluster): no longer in tasks_
  HX bool dead_task(int id) const {
    NOUNROLL for (int i = 0; i < npart; ++i) {
      const PartEntry pe = part()[i];
      if (pe.task < 0 && id >= pe.child0 && id < pe.child0 + pe.nchild) return true;
    }
    return false;
  }
  static HX bool dead_region(const Region& r) { return r.rows == 0; }

  // TaskGraph::merge_cluster (graph.cpp:521-534) with
  // DataDag::prune_unreferenced (graph.cpp:214-266): the members leave the
  // graph (their ids stay consumed), the parent is a leaf again, and every
  // candidate block no remaining task references is removed -- here by
  // giving it an empty region, which no geometric query (find, overlap,
  // containment, scopes) can match.  Intersection descriptors are pruned by
  // their DataDag parent links, which E1 does not model after a prune; a
  // merge while any intersection block exists reports ST_ENGINE_LIMIT.
  // Merging the top cluster returns the candidate to the unpartitioned root
  // (BaseView TIL_ROOT); a later partition of the root moves it onto another
  // shared top-level tiling.
  HXN void apply_merge(int c) {
    if (c < 0 || c >= npart || part()[c].task < 0) return fail(ST_UNKNOWN_CLUSTER);
    const PartEntry pe = part()[c];
    NOUNROLL for (int m = pe.child0; m < pe.child0 + pe.nchild; ++m)
      if (part_index(m) >= 0) return fail(ST_NESTED_CLUSTER);
    bool sect = false;
    NOUNROLL for (int b = n_bb() + wp.lane(); b < nblocks; b += WP::W) {
      const BlockMeta& o = bm()[b - n_bb()];
      if (o.isint && !dead_region(o.r)) sect = true;
    }
    const bool with_sect = wp.any(sect);
    if (c == 0) {
      if (with_sect) {
        prune_intersections(true);
        if (status) return;
      }
      // The top cluster (the root's): every other cluster is already merged
      // (its members are leaves), so the prune leaves the root alone -- the
      // unpartitioned root, with every id consumed so far staying consumed.
      if (pe.task != 0 || pe.child0 != 1) return fail(ST_INTERNAL);
      const BaseView& v = BV();
      const int nt = ntasks + v.off_t, nb = nblocks + v.off_b, nc = npart + v.off_c;
      reset_to_base(TIL_ROOT, nt - 1, nb - 1, nc);
      return;
    }
    NOUNROLL for (int m = pe.child0 + wp.lane(); m < pe.child0 + pe.nchild; m += WP::W) {
      const TaskMeta t = tm()[m - n_bt()];
      NOUNROLL for (int k = 0; k <= t.nrd; ++k)
        if (t.blk[k] >= n_bb()) wp.atomic_add(&bref()[t.blk[k] - n_bb()], -1);
    }
    wp.sync();
    if (with_sect) {
      prune_intersections(false);
      if (status) return;
    }
    NOUNROLL for (int b = n_bb() + wp.lane(); b < nblocks; b += WP::W) {
      BlockMeta& o = bm()[b - n_bb()];
      if (!o.isint && bref()[b - n_bb()] == 0 && !dead_region(o.r)) {
        o.r.row = -1;
        o.r.col = -1;
        o.r.rows = 0;
        o.r.cols = 0;
      }
    }
    if (wp.lane() == 0) part()[c].task = -2 - pe.task;
    wp.sync();
  }

  // TaskGraph::partition_task (graph.cpp:456-513) followed by the
  // enumerate_partition loop nests (graph.cpp:301-392).
  HXN void apply_op(int task_id, int s_req) {
    if (task_id < 0 || task_id >= ntasks) return fail(ST_VALIDATION);
    if (task_id >= n_bt() && dead_task(task_id)) return fail(ST_VALIDATION);  // merged away: unknown task
    if (part_index(task_id) >= 0) return fail(ST_NOT_A_LEAF);
    const double p = 1.0 / (double)s_req;
    if (!(p > 0.0 && p < 1.0)) return fail(ST_VALIDATION);
    const TaskMeta t = task(task_id);
    const int s = (int)hesp_snap_tiles(t.b, s_req, PB.min_block);
    if (s == 0) return fail(ST_INDIVISIBLE);
    if (task_id == 0 && PB.n_til > 0) {
      // partitioning the unpartitioned root: the candidate moves onto the
      // shared top-level tiling with that tile count, ids continuing from the
      // ones consumed so far (n_til == 0: the host is building the tilings)
      int k = -1;
      NOUNROLL for (int i = 0; i < PB.n_til; ++i)
        if (i != TIL_ROOT && PB.til[i].s == s) k = i;
      if (k < 0) return fail(ST_ENGINE_LIMIT);  // a tiling larger than the slot holds
      const BaseView v = BV();
      reset_to_base(k, v.off_t, v.off_b, v.off_c);
      return;
    }
    if (npart >= MAXPART) return fail(ST_ENGINE_LIMIT);
    // operands = reads minus writes, in read order; write = writes.front()
    const int wb = t.blk[t.nrd];
    Region opr[3];
    int opt[3];
    int nop = 0;
    NOUNROLL for (int k = 0; k < t.nrd; ++k)
      if (t.blk[k] != wb) {
        opr[nop] = reg(t.blk[k]);
        opt[nop] = tile_of(t.blk[k]);
        ++nop;
      }
    const Region a = reg(wb);
    const int at = tile_of(wb);
    const int child0 = ntasks;
    Region rr[3];
    int rt[3];
    switch (t.kind) {
      case HESP_CHOL:
        NOUNROLL for (int k = 0; k < s && !status; ++k) {
          const Region akk = sub(a, s, k, k);
          rr[0] = akk;
          rt[0] = at;
          emit(HESP_CHOL, 1, rr, rt, akk, at);
          NOUNROLL for (int i = k + 1; i < s && !status; ++i) {
            rr[0] = akk;
            rr[1] = sub(a, s, i, k);
            rt[0] = rt[1] = at;
            emit(HESP_TRSM, 2, rr, rt, rr[1], at);
          }
          NOUNROLL for (int i = k + 1; i < s && !status; ++i) {
            const Region aik = sub(a, s, i, k);
            NOUNROLL for (int j = k + 1; j < i && !status; ++j) {
              rr[0] = aik;
              rr[1] = sub(a, s, j, k);
              rr[2] = sub(a, s, i, j);
              rt[0] = rt[1] = rt[2] = at;
              emit(HESP_GEMM, 3, rr, rt, rr[2], at);
            }
            if (status) break;
            rr[0] = aik;
            rr[1] = sub(a, s, i, i);
            rt[0] = rt[1] = at;
            emit(HESP_SYRK, 2, rr, rt, rr[1], at);
          }
        }
        break;
      case HESP_TRSM: {
        if (nop != 1) return fail(ST_INTERNAL);
        const Region l = opr[0];
        const int lt = opt[0];
        NOUNROLL for (int j = 0; j < s && !status; ++j) {
          const Region ljj = sub(l, s, j, j);
          NOUNROLL for (int i = 0; i < s && !status; ++i) {
            const Region bij = sub(a, s, i, j);
            NOUNROLL for (int k = 0; k < j && !status; ++k) {
              rr[0] = sub(a, s, i, k);
              rr[1] = sub(l, s, j, k);
              rr[2] = bij;
              rt[0] = at;
              rt[1] = lt;
              rt[2] = at;
              emit(HESP_GEMM, 3, rr, rt, bij, at);
            }
            if (status) break;
            rr[0] = ljj;
            rr[1] = bij;
            rt[0] = lt;
            rt[1] = at;
            emit(HESP_TRSM, 2, rr, rt, bij, at);
          }
        }
        break;
      }
      case HESP_SYRK: {
        if (nop != 1) return fail(ST_INTERNAL);
        const Region src = opr[0];
        const int st = opt[0];
        NOUNROLL for (int i = 0; i < s && !status; ++i)
          NOUNROLL for (int j = 0; j <= i && !status; ++j) {
            const Region cij = sub(a, s, i, j);
            NOUNROLL for (int k = 0; k < s && !status; ++k) {
              rr[0] = sub(src, s, i, k);
              rt[0] = st;
              if (i == j) {
                rr[1] = cij;
                rt[1] = at;
                emit(HESP_SYRK, 2, rr, rt, cij, at);
              } else {
                rr[1] = sub(src, s, j, k);
                rr[2] = cij;
                rt[1] = st;
                rt[2] = at;
                emit(HESP_GEMM, 3, rr, rt, cij, at);
              }
            }
          }
        break;
      }
      default: {
        if (nop != 2) return fail(ST_INTERNAL);
        const Region ma = opr[0], mb = opr[1];
        NOUNROLL for (int i = 0; i < s && !status; ++i)
          NOUNROLL for (int j = 0; j < s && !status; ++j) {
            const Region cij = sub(a, s, i, j);
            NOUNROLL for (int k = 0; k < s && !status; ++k) {
              rr[0] = sub(ma, s, i, k);
              rr[1] = sub(mb, s, j, k);
              rr[2] = cij;
              rt[0] = opt[0];
              rt[1] = opt[1];
              rt[2] = at;
              emit(HESP_GEMM, 3, rr, rt, cij, at);
            }
          }
        break;
      }
    }
    if (status) return;
    if (wp.lane() == 0) {
      part()[npart].task = task_id;
      part()[npart].child0 = child0;
      part()[npart].nchild = ntasks - child0;
      part()[npart].leaves = 0;
    }
    wp.sync();
    ++npart;
  }

  // =========================================================================
  // Post-build indexing: per-tile block lists, leaf() program order, deps
  // =========================================================================

  // Per-tile CSR of the candidate's own blocks (order inside a tile is
  // irrelevant: every consumer is order-independent or sorts).
  HXN void build_tiles() {
    NOUNROLL for (int i = wp.lane(); i < n_bb(); i += WP::W) tl_cnt()[i] = 0;
    wp.sync();
    NOUNROLL for (int b = n_bb() + wp.lane(); b < nblocks; b += WP::W)
      if (!dead_region(bm()[b - n_bb()].r)) wp.atomic_add(&tl_cnt()[bm()[b - n_bb()].tile], 1);
    wp.sync();
    // exclusive scan over base tiles
    int run = 0;
    NOUNROLL for (int base = 0; base < n_bb(); base += WP::W) {
      const int i = base + wp.lane();
      const int c = i < n_bb() ? tl_cnt()[i] : 0;
      int incl = c;
#if defined(__CUDACC__)
      if constexpr (WP::W > 1) {
        NOUNROLL for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (wp.lane() >= o) incl += v;
        }
      }
#endif
      if (i < n_bb()) tl_head()[i] = run + incl - c;
      run += wp.bcast(incl, WP::W - 1);
    }
    wp.sync();
    NOUNROLL for (int i = wp.lane(); i < n_bb(); i += WP::W) tl_ncb()[i] = 0;  // fill cursor
    wp.sync();
    NOUNROLL for (int b = n_bb() + wp.lane(); b < nblocks; b += WP::W) {
      if (dead_region(bm()[b - n_bb()].r)) continue;
      const int t = bm()[b - n_bb()].tile;
      const int pos = wp.atomic_add(&tl_ncb()[t], 1);
      tl_ids()[tl_head()[t] + pos] = b;
    }
    wp.sync();
    n_tl_ids = run;
  }

  // Leaf program order: lexicographic seq, i.e. depth-first over clusters
  // with members in emission order (graph.cpp:552-562).
  HXN void build_order() {
    NOUNROLL for (int i = wp.lane(); i < ntasks; i += WP::W) pmark()[i] = 0;
    wp.sync();
    if (wp.lane() == 0)
      for (int i = 0; i < npart; ++i)
        if (part()[i].task >= 0) pmark()[part()[i].task] = (uint8_t)(i + 1);
    wp.sync();
    // subtree leaf() counts, innermost partitions last in op order
    NOUNROLL for (int i = npart - 1; i >= 0; --i) {
      const PartEntry pe = part()[i];
      if (pe.task < 0) continue;  // merged away
      int cnt = 0;
      NOUNROLL for (int c = pe.child0; c < pe.child0 + pe.nchild; ++c) {
        const int pi = part_of(c);
        cnt += pi >= 0 ? part()[pi].leaves : 1;
      }
      if (wp.lane() == 0) part()[i].leaves = cnt;
      wp.sync();
    }
    // explicit stack of (first child, count, output position)
    // pending sibling subtrees: at most one entry per cluster (slot scratch)
    int* const sf = dstack();
    int* const sc = sf + MAXPART;
    int* const sp = sc + MAXPART;
    int top = 0;
    const int r = part_of(0);
    if (r < 0) {  // unpartitioned root: a single leaf()
      if (wp.lane() == 0) leaf()[0] = 0;
      wp.sync();
      nleaves = 1;
      return;
    }
    if (wp.lane() == 0) {
      sf[0] = part()[r].child0;
      sc[0] = part()[r].nchild;
      sp[0] = 0;
    }
    top = 1;
    nleaves = part()[r].leaves;
    while (top > 0) {
      wp.sync();
      --top;
      const int f = sf[top], c = sc[top];
      int pos = sp[top];
      NOUNROLL for (int base = 0; base < c; base += WP::W) {
        const int k = base + wp.lane();
        int pi = -1, sz = 0;
        if (k < c) {
          pi = part_of(f + k);
          sz = pi >= 0 ? part()[pi].leaves : 1;
        }
        int incl = sz;
#if defined(__CUDACC__)
        if constexpr (WP::W > 1) {
          NOUNROLL for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (wp.lane() >= o) incl += v;
          }
        }
#endif
        const int my = pos + incl - sz;
        if (k < c && pi < 0) leaf()[my] = f + k;
        const unsigned m = wp.ballot(k < c && pi >= 0);
        NOUNROLL for (unsigned mm = m; mm; mm &= mm - 1) {
          const int ln = ctz32(mm);
          const int q = wp.bcast(pi, ln);
          const int qp = wp.bcast(my, ln);
          if (top < MAXPART && wp.lane() == 0) {
            sf[top] = part()[q].child0;
            sc[top] = part()[q].nchild;
            sp[top] = qp;
          }
          ++top;
        }
        pos += wp.bcast(incl, WP::W - 1);
      }
    }
    wp.sync();
  }

  // Column/row boundaries of every tile's blocks -> cell grids.
  HXN void build_cells() {
    int nb_used = 0, nc_used = 0;
    NOUNROLL for (int t = 1; t < n_bb() && !status; ++t) {
      const int cnt = tl_cnt()[t];
      if (cnt == 0) {
        if (wp.lane() == 0) {
          tl_boff()[t] = -1;
          tl_nrb()[t] = 2;
          tl_ncb()[t] = 2;
          tl_coff()[t] = nc_used;
          c_writer()[nc_used] = -1;
          c_rhead()[nc_used] = -1;
        }
        wp.sync();
        ++nc_used;
        continue;
      }
      const Region tr = reg(t);
      // candidate boundaries: tile edges + every member's edges (rows, then cols)
      const int nraw = 2 * cnt + 2;
      if (nb_used + 2 * nraw > PB.maxbnd) return fail(ST_ENGINE_LIMIT);
      int* rows = bnd() + nb_used;
      int* cols = rows + nraw;
      // raw values into gs_a() / gs_reg() scratch, then rank-unique into place
      int* raw_r = gs_a();
      int* raw_c = gs_a() + nraw;
      if (2 * nraw > PB.maxgs) return fail(ST_ENGINE_LIMIT);
      NOUNROLL for (int k = wp.lane(); k < nraw; k += WP::W) {
        int vr, vc;
        if (k < 2) {
          vr = k == 0 ? tr.row : tr.row + tr.rows;
          vc = k == 0 ? tr.col : tr.col + tr.cols;
        } else {
          const Region m = reg(tl_ids()[tl_head()[t] + (k - 2) / 2]);
          vr = (k & 1) ? m.row + m.rows : m.row;
          vc = (k & 1) ? m.col + m.cols : m.col;
        }
        raw_r[k] = vr;
        raw_c[k] = vc;
      }
      wp.sync();
      // sort (value, index) then keep first occurrences: rows -> rows[], cols -> cols[]
      NOUNROLL for (int k = wp.lane(); k < nraw; k += WP::W) {
        const int vr = raw_r[k], vc = raw_c[k];
        int rr = 0, rc = 0;
        NOUNROLL for (int q = 0; q < nraw; ++q) {
          const int ur = raw_r[q], uc = raw_c[q];
          rr += (ur < vr) || (ur == vr && q < k);
          rc += (uc < vc) || (uc == vc && q < k);
        }
        rows[rr] = vr;
        cols[rc] = vc;
      }
      wp.sync();
      int nr = 0, nc = 0;
      NOUNROLL for (int base = 0; base < nraw; base += WP::W) {
        const int k = base + wp.lane();
        int vr = 0, vc = 0;
        bool kr = false, kc = false;
        if (k < nraw) {
          vr = rows[k];
          vc = cols[k];
          kr = k == 0 || rows[k - 1] != vr;
          kc = k == 0 || cols[k - 1] != vc;
        }
        const unsigned mr = wp.ballot(kr), mc = wp.ballot(kc);
        wp.sync();
        if (kr) gs_a()[nr + popc32(mr & wp.lt())] = vr;
        if (kc) gs_a()[nraw + nc + popc32(mc & wp.lt())] = vc;
        nr += popc32(mr);
        nc += popc32(mc);
      }
      wp.sync();
      NOUNROLL for (int k = wp.lane(); k < nr; k += WP::W) rows[k] = gs_a()[k];
      wp.sync();
      // cols right after the nr distinct rows
      NOUNROLL for (int k = wp.lane(); k < nc; k += WP::W) rows[nr + k] = gs_a()[nraw + k];
      wp.sync();
      const int ncell = (nr - 1) * (nc - 1);
      if (nc_used + ncell > PB.maxcells) return fail(ST_ENGINE_LIMIT);
      NOUNROLL for (int k = wp.lane(); k < ncell; k += WP::W) {
        c_writer()[nc_used + k] = -1;
        c_rhead()[nc_used + k] = -1;
      }
      if (wp.lane() == 0) {
        tl_boff()[t] = nb_used;
        tl_nrb()[t] = nr;
        tl_ncb()[t] = nc;
        tl_coff()[t] = nc_used;
      }
      wp.sync();
      // cell rectangle of the tile and of each of its blocks, once
      NOUNROLL for (int k = wp.lane(); k < cnt + 1; k += WP::W) {
        const int b = k == 0 ? t : tl_ids()[tl_head()[t] + k - 1];
        const Region rg = reg(b);
        int4 cr;
        cr.x = cr.y = cr.z = cr.w = 0;
        NOUNROLL for (int q = 0; q < nr; ++q) {
          if (rows[q] == rg.row) cr.x = q;
          if (rows[q] == rg.row + rg.rows) cr.y = q;
        }
        NOUNROLL for (int q = 0; q < nc; ++q) {
          if (rows[nr + q] == rg.col) cr.z = q;
          if (rows[nr + q] == rg.col + rg.cols) cr.w = q;
        }
        bcell()[b] = cr;
      }
      wp.sync();
      nb_used += nr + nc;
      nc_used += ncell;
    }
  }

  // Cell rectangle [r0,r1) x [c0,c1) of block b inside its tile.
  HX void cell_range(int b, int& t, int& r0, int& r1, int& c0, int& c1) {
    t = tile_of(b);
    const int off = tl_boff()[t];
    if (off < 0) {
      r0 = c0 = 0;
      r1 = c1 = 1;
      return;
    }
    const int4 cr = bcell()[b];  // precomputed in build_cells
    r0 = cr.x;
    r1 = cr.y;
    c0 = cr.z;
    c1 = cr.w;
  }

  // Predecessor list of leaf j: candidate arena (off >= 0) or, for base tasks
  // whose tiles have no sub-blocks, the shared base table (off = ~index).
  HX const int32_t* pred_list(int j) const {
    const int off = t_poff()[j];
    return off >= 0 ? preds() + off : bpl_() + ~off;
  }

  // Dependences (E2): per cell, last writer + readers since that write.
  // E5: a base task whose tiles all lack sub-blocks sees the
  // base tiling's exact accessor history on them (a partitioned accessor
  // would have created sub-blocks), so its predecessors are the base
  // predecessors precomputed on the host; only tasks touching subdivided
  // tiles run the cell tracking, in program order.
  HXN void build_deps() {
    int rn_used = 0;
    nedges = 0;
    NOUNROLL for (int i = wp.lane(); i < ntasks; i += WP::W) pmk()[i] = -1;
    wp.sync();
    // ---- pass 0 (parallel): classify leaves, take base preds for the fast ones
    int nslow = 0;
    int sk = 0;  // this lane's share of sum_k (a register, not the engine object in local memory)
    int* const slow = gs_b();
    NOUNROLL for (int base = 0; base < nleaves; base += WP::W) {
      const int li = base + wp.lane();
      bool isslow = false;
      int j = -1;
      if (li < nleaves) {
        j = leaf()[li];
        const TaskMeta t = task(j);
        {
          int w[4];
          const int nw = working_set(t, w);
          STask ws;
          ws.ws0 = w[0];
          ws.ws1 = nw > 1 ? w[1] : -1;
          ws.ws2 = nw > 2 ? w[2] : -1;
          ws.nw = nw;
          ws.out = t.nrd == 0 ? t.blk[0] : (t.nrd == 1 ? t.blk[1] : (t.nrd == 2 ? t.blk[2] : t.blk[3]));
          ws.kb = (int)t.kind | ((int)t.bidx << 8);
          ws.b = t.b;
          // static per-block facts the event loop would otherwise look up per
          // commit: bit k = working-set block k is a base tile with no
          // sub-blocks (no descendants, no intersections), bit 3 = the same
          // for the output block (tile membership is fixed after the build)
          int fl = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k)
            if (k < nw && simple_tile(w[k])) fl |= 1 << k;
          if (simple_tile(ws.out)) fl |= 8;
          // bit 4: the working-set blocks are pairwise disjoint, so acquiring
          // one never changes another's validity (the lean loop reads all of
          // them in one round); bit 5: the output's coherence cone needs the
          // general scan (the root, or a tile holding partial overlaps)
          bool disj = true;
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int c = a + 1; c < 4; ++c)
              if (c < nw && roverlap(reg(w[a]), reg(w[c]))) disj = false;
          if (disj) fl |= 16;
          if (ws.out == 0 || tmis()[tile_of(ws.out)]) fl |= 32;
          ws.pad = fl;
          wsb()[j] = ws;
        }
        int kt = 0;
        bool fastj = j < n_bt();
        // (loops over the <= 4 block slots unrolled: constant indices keep
        // the task record in registers instead of a local-memory copy)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (k > t.nrd) break;
          bool dup = false;
#pragma unroll
          for (int q = 0; q < k; ++q) dup |= t.blk[q] == t.blk[k];
          kt += !dup;
          // (the root block has no tile: a leaf root -- the unpartitioned
          // root's only task -- has no predecessors at all)
          const int tt = tile_of(t.blk[k]);
          if (fastj && tt >= 0 && tl_cnt()[tt] != 0) fastj = false;
        }
        sk += kt;
        if (fastj) {
          const BasePreds& bp = bp_()[j];
          t_poff()[j] = ~bp.uoff;
          t_pcnt()[j] = bp.ucnt;
          ts()[j].missing = bp.ucnt;
        } else {
          // the serial pass's per-access facts, resolved here in parallel:
          // distinct blocks (read-only ones in read order, then the write),
          // each either a base contribution (x = -1 - slot, E5) or its cell
          // rectangle (x = first cell, y = w | rows << 11 | row stride << 22);
          // nacc = 0 leaves the task to the serial pass's own derivation
          const int wb = t.nrd == 0 ? t.blk[0] : (t.nrd == 1 ? t.blk[1] : (t.nrd == 2 ? t.blk[2] : t.blk[3]));
          int2* rec = dacc() + 4 * j;
          int na = 0;
          bool packed = true;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            if (k > t.nrd) break;
            const int b = t.blk[k];
            if (k < t.nrd && b == wb) continue;  // in-place read: covered by the write
            bool dup = false;
#pragma unroll
            for (int q = 0; q < k; ++q)
              if (t.blk[q] == b && q < t.nrd) dup = true;
            if (dup && k < t.nrd) continue;
            int2 r;
            if (j < n_bt() && tl_cnt()[tile_of(b)] == 0) {
              r.x = -1 - na;
              r.y = 0;
            } else {
              int tt, r0, r1, c0, c1;
              cell_range(b, tt, r0, r1, c0, c1);
              const int nc = tl_ncb()[tt] - 1;
              const int w = c1 - c0, rows = r1 - r0;
              if (w >= 2048 || rows >= 2048 || nc >= 1024) packed = false;
              r.x = tl_coff()[tt] + r0 * nc + c0;
              r.y = w | (rows << 11) | (nc << 22);
            }
            if (na < 4) rec[na] = r;
            ++na;
          }
          if (na > 4) packed = false;
          j |= (packed ? na : 0) << 28;
        }
        isslow = !fastj;
      }
      const unsigned m = wp.ballot(isslow);
      if (isslow) slow[nslow + popc32(m & wp.lt())] = j;
      nslow += popc32(m);
    }
    wp.sync();
    sum_k = wp.sumi(sum_k + sk);
    // ---- pass A (serial in program order): cell tracking for the slow leaves
    // (the edge count lives in a register for the pass; only a fail() ends
    // the pass early, so status is checked once)
    if (status) return;
    int ne = nedges;
    auto bail = [&](int code) {
      nedges = ne;
      fail(code);
    };
    NOUNROLL for (int si = 0; si < nslow; ++si) {
      const int j = slow[si] & 0x0fffffff;
      const int nacc = (int)((unsigned)slow[si] >> 28);
      const int2* rec = dacc() + 4 * j;
      TaskMeta t;
      int nsteps;
      if (nacc) {
        nsteps = nacc;
      } else {
        t = task(j);
        nsteps = t.nrd + 1;
      }
      int npb = 0;
      int slot = 0;
      // distinct blocks, read-only ones first in read order, then the write
      NOUNROLL for (int k = 0; k < nsteps; ++k) {
        bool writes;
        int2 r;
        int w, nc, rows;
        if (nacc) {
          r = rec[k];
          writes = k == nacc - 1;
          w = r.y & 2047;
          rows = (r.y >> 11) & 2047;
          nc = (int)((unsigned)r.y >> 22);
        } else {
          const int wb = t.blk[t.nrd];
          const int b = t.blk[k];
          if (k < t.nrd && b == wb) continue;  // in-place read: covered by the write
          bool dup = false;
          NOUNROLL for (int q = 0; q < k; ++q)
            if (t.blk[q] == b && q < t.nrd) dup = true;
          if (dup && k < t.nrd) continue;
          writes = (k == t.nrd);
          if (j < n_bt() && tl_cnt()[tile_of(b)] == 0) {
            r.x = -1 - slot;
            r.y = 0;
          } else {
            int tt, r0, r1, c0, c1;
            cell_range(b, tt, r0, r1, c0, c1);
            nc = tl_ncb()[tt] - 1;
            r.x = tl_coff()[tt] + r0 * nc + c0;
            r.y = 0;
            rows = r1 - r0;
            w = c1 - c0;
          }
        }
        ++slot;
        if (r.x < 0) {
          // unsubdivided tile of a base task: its base contribution (E5)
          const BasePreds& bp = bp_()[j];
          const int myslot = -1 - r.x;
          const int off = bp.soff[myslot], cnt = bp.scnt[myslot];
          NOUNROLL for (int q = wp.lane(); q < cnt; q += WP::W)
            if (npb + q < PB.maxpb) pbuf()[npb + q] = bpl_()[off + q];
          npb += cnt;
          wp.sync();
          if (npb > PB.maxpb) return bail(ST_ENGINE_LIMIT);
          continue;
        }
        const int ncells = rows * w;
        const int cfirst = r.x;
        const float rw = 1.0f / (float)w;  // q / w via a corrected float reciprocal (q < 2^20)
        NOUNROLL for (int base = 0; base < ncells; base += WP::W) {
          const int q = base + wp.lane();
          int cell = -1;
          if (q < ncells) {
            int rq = (int)((float)q * rw);
            if (rq * w > q) --rq;
            else if ((rq + 1) * w <= q) ++rq;
            cell = cfirst + rq * nc + (q - rq * w);
          }
          // last writer
          int wr = cell >= 0 ? c_writer()[cell] : -1;
          bool e = wr >= 0 && wr != j;
          unsigned m = wp.ballot(e);
          if (e) {
            const int at = npb + popc32(m & wp.lt());
            if (at < PB.maxpb) pbuf()[at] = wr;
          }
          npb += popc32(m);
          if (!writes) {
            // join readers
            unsigned mr = wp.ballot(cell >= 0);
            if (cell >= 0) {
              const int at = rn_used + popc32(mr & wp.lt());
              if (at < PB.maxrn) {
                rnode()[2 * at] = j;
                rnode()[2 * at + 1] = c_rhead()[cell];
                c_rhead()[cell] = at;
              }
            }
            rn_used += popc32(mr);
          } else {
            // consume readers (per-lane list walks, lock-stepped emission)
            int node = cell >= 0 ? c_rhead()[cell] : -1;
            while (wp.any(node >= 0)) {
              int rd = -1;
              if (node >= 0) {
                rd = rnode()[2 * node];
                node = rnode()[2 * node + 1];
              }
              const bool ee = rd >= 0 && rd != j;
              const unsigned me = wp.ballot(ee);
              if (ee) {
                const int at = npb + popc32(me & wp.lt());
                if (at < PB.maxpb) pbuf()[at] = rd;
              }
              npb += popc32(me);
            }
            if (cell >= 0) {
              c_writer()[cell] = j;
              c_rhead()[cell] = -1;
            }
          }
          wp.sync();
        }
        if (rn_used > PB.maxrn || npb > PB.maxpb) return bail(ST_ENGINE_LIMIT);
      }
      // dedup -> preds arena
      int m = 0;
#if defined(__CUDACC__)
      if (WP::W > 1 && HESP_MATCH_DEDUP && npb <= WP::W) {
        // one round, no memory atomics: a candidate is kept by the lowest
        // lane holding its value (first occurrence, the same order as below)
        const int q = wp.lane();
        const int v = q < npb ? pbuf()[q] : -1 - q;  // distinct fillers
        const unsigned same = __match_any_sync(0xffffffffu, v);
        const bool keep = q < npb && (same & ((1u << q) - 1u)) == 0u;
        const unsigned mk = wp.ballot(keep);
        if (keep) {
          const int at = ne + popc32(mk & wp.lt());
          if (at < PB.maxedges) preds()[at] = v;
        }
        m = popc32(mk);
      } else
#endif
      NOUNROLL for (int base = 0; base < npb; base += WP::W) {
        const int q = base + wp.lane();
        bool keep = false;
        int v = -1;
        if (q < npb) {
          v = pbuf()[q];
          // first claimant of predecessor v for task j keeps it (marks were
          // cleared at the start of build_deps, so a stale j cannot match)
          keep = wp.exch(&pmk()[v], j) != j;
        }
        const unsigned mk = wp.ballot(keep);
        if (keep) {
          const int at = ne + m + popc32(mk & wp.lt());
          if (at < PB.maxedges) preds()[at] = v;
        }
        m += popc32(mk);
      }
      if (ne + m > PB.maxedges) return bail(ST_ENGINE_LIMIT);
      if (wp.lane() == 0) {
        t_poff()[j] = ne;
        t_pcnt()[j] = m;
        ts()[j].missing = m;
      }
      wp.sync();
      ne += m;
    }
    nedges = ne;
    // ---- pass B (parallel): successors CSR from all predecessor lists
    NOUNROLL for (int li = wp.lane(); li < nleaves; li += WP::W) ts()[leaf()[li]].scnt = 0;
    wp.sync();
    int total = 0;
    NOUNROLL for (int li = wp.lane(); li < nleaves; li += WP::W) {
      const int j = leaf()[li];
      const int32_t* pl_ = pred_list(j);
      const int cnt = t_pcnt()[j];
      total += cnt;
      _Pragma("unroll kSuccUnroll") for (int q = 0; q < cnt; ++q) wp.atomic_add(&ts()[pl_[q]].scnt, 1);
    }
    wp.sync();
    total = wp.sumi(total);
    nedges = total;  // all edges, base-table and arena alike
    int run = 0;
    NOUNROLL for (int base = 0; base < nleaves; base += WP::W) {
      const int li = base + wp.lane();
      const int c = li < nleaves ? ts()[leaf()[li]].scnt : 0;
      int incl = c;
#if defined(__CUDACC__)
      if constexpr (WP::W > 1) {
        NOUNROLL for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (wp.lane() >= o) incl += v;
        }
      }
#endif
      if (li < nleaves) {
        ts()[leaf()[li]].soff = run + incl - c;
        ts()[leaf()[li]].scnt = 0;  // reused as fill cursor
      }
      run += wp.bcast(incl, WP::W - 1);
    }
    wp.sync();
    if (run > PB.maxedges) return fail(ST_ENGINE_LIMIT);
    NOUNROLL for (int li = wp.lane(); li < nleaves; li += WP::W) {  // order within a list is irrelevant
      const int j = leaf()[li];
      const int32_t* pl_ = pred_list(j);
      const int cnt = t_pcnt()[j];
      _Pragma("unroll kSuccUnroll") for (int q = 0; q < cnt; ++q) {
        const int p = pl_[q];
        const int pos = wp.atomic_add(&ts()[p].scnt, 1);
        succs()[ts()[p].soff + pos] = j;
      }
    }
    wp.sync();
  }

  // critical_times (sim.cpp:92-115): ct = avg + max(0, max_succ ct), reverse
  // program order; pushed to preds() so each pred sees all its successors.
  HXN void build_ct() {
    // ct(j) = avg(j) + max(0, max over successors ct(s)); successors lie later
    // in program order.  Chunks of 32 leaves from the end: a lane finalises
    // its task once every successor's ct is known (-1 = not yet), so a chunk
    // needs as many rounds as its longest internal successor chain.
    NOUNROLL for (int li = wp.lane(); li < nleaves; li += WP::W) ts()[leaf()[li]].ct = -1.0;
    wp.sync();
    NOUNROLL for (int hi = nleaves; hi > 0; hi -= WP::W) {
      const int li = hi - WP::W + wp.lane();
      bool todo = li >= 0;
      int j = -1;
      double avg = 0.0;
      if (todo) {
        j = leaf()[li];
        const int kb = wsb()[j].kb;
        avg = PB.ctavg[kb & 0xff][kb >> 8];
      }
      NOUNROLL while (wp.any(todo)) {
        if (todo) {
          const TState& tj = ts()[j];
          double best = 0.0;
          bool ready = true;
          NOUNROLL for (int q = 0; q < tj.scnt; ++q) {
            const double c = ts()[succs()[tj.soff + q]].ct;
            if (c < 0.0) ready = false;
            best = dmax(best, c);
          }
          if (ready) {
            ts()[j].ct = avg + best;
            todo = false;
          }
        }
        wp.sync();
      }
    }
  }

  // =========================================================================
  // Coherence / memory model (sim.cpp:323-590)
  // =========================================================================

  // Blocks that can overlap a block of tile t: root, the tile, its CSR list.
  // Visit order is irrelevant for every caller.
  template <class F>
  HX void for_scope(int t, F&& f) {
    if (t < 0) {  // the root: everything
      NOUNROLL for (int b = wp.lane(); b < nblocks; b += WP::W) f(b);
      wp.sync();
      return;
    }
    const int cnt = 2 + tl_cnt()[t];
    const int head = tl_head()[t];
    NOUNROLL for (int k = wp.lane(); k < cnt; k += WP::W) {
      const int b = k == 0 ? 0 : (k == 1 ? t : tl_ids()[head + k - 2]);
      f(b);
    }
    wp.sync();
  }

  HX int source_space(int b, int exclude) {  // source_spaces().front() minus `exclude` (sim.cpp:341-350)
    if (msp() != exclude && V(b, msp()) != ABSENT) return msp();
    NOUNROLL for (int s = 0; s < n_sp(); ++s)
      if (s != msp() && s != exclude && V(b, s) != ABSENT) return s;
    return -1;
  }

  // Engine::plan_transfer (sim.cpp:468-499): FIFO per directed link.
  HXN double plan_transfer(int blk, const Region* frag, long long bytes, int src, int dst,
                          double data_ready, double tnow) {
    const int nh = PB.route_n[src * MAXS + dst];
    if (nh == 0) {
      fail(ST_NO_ROUTE);
      return 0.0;
    }
    double rdy = dmax(data_ready, tnow);
    double start0 = 0.0;
    double hs[2] = {0.0, 0.0}, he[2] = {0.0, 0.0};
    NOUNROLL for (int h = 0; h < nh; ++h) {
      const int l = PB.route_l[src * MAXS + dst][h];
      const double st = dmax(SM().link_free[l], rdy);
      const double en = st + PB.link_lat[l] + (double)bytes / PB.link_bw[l];
      SM().link_free[l] = en;
      rdy = en;
      if (h == 0) start0 = st;
      if (TRACE && h < 2) {
        hs[h] = st;
        he[h] = en;
      }
    }
    if (!(rdy > now)) fail(ST_ENGINE_INVARIANT);
    log_xfer(blk, frag, bytes, src, dst, start0, rdy, nh, hs, he);
    if (frag)
      xhash += hesp_xfer_term(xblock(blk), src, dst, bytes, dbits(start0), dbits(rdy), frag->row, frag->col,
                              frag->rows, frag->cols);
    else
      xhash += hesp_xfer_term(xblock(blk), src, dst, bytes, dbits(start0), dbits(rdy), 0, 0, 0, 0);
    return rdy;
  }

  // Scalar state is replicated in every lane: uniform code stores the same
  // value from all lanes (idempotent), so no lane-0 store + __syncwarp.
  HX void set_flag(int b, uint32_t bit, bool on) {
    const uint32_t f = bflags()[b];
    bflags()[b] = on ? (f | bit) : (f & ~bit);
  }
  HX void setV(int b, int s, double v) { V(b, s) = v; }
  HX void setLU(int b, int s, double v) { LU(b, s) = v; }
  HX void setPIN(int b, int s, double v) { PIN(b, s) = v; }
  HX void add_used(int s, long long d) {
    if (wp.lane() == 0) SM().used[s] += d;
    wp.sync();
  }

  // x strictly inside b (== DataDag::descendants by E1), for x in b's scope
  HX bool inside(int x, int b, int t, const Region& rb) const {
    if (b == 0) return x != 0;
    return x != 0 && x != t && x != b && rcontains(rb, reg(x));
  }

  // validate_from (sim.cpp:452-461): block and descendants valid() at min(., at)
  HXN void validate_from(int b, int s, double at) {
    const int t = b == 0 ? -1 : tile_of(b);
    const Region rb = reg(b);
    for_scope(t, [&](int x) {
      if (x == b || inside(x, b, t, rb)) {
        double& v = V(x, s);
        if (v > at) v = at;
      }
    });
    if (!fast) LU(b, s) = dmax(LU(b, s), at);
  }

  // ensure_capacity (sim.cpp:374-439).  The only recursion in the reference
  // is a dirty flush from an accelerator into main (materialize in main),
  // and main never holds dirty blocks, so FLUSH=false is the flush's own
  // instance: no device recursion, no call stack.
  template <bool FLUSH>
  HXN void ensure_capacity(int s, long long bytes, double at) {
    const long long cap = PB.cap[s];
    if (bytes > cap) return fail(ST_CAPACITY);
    while (SM().used[s] + bytes > cap) {
      // LRU victim: min (stamp, id) among unpinned materialised blocks
      double bst = ABSENT;
      double dummy = 0.0;
      int bid = -1;
      NOUNROLL for (int base = 0; base < nblocks; base += WP::W) {
        const int b = base + wp.lane();
        if (b < nblocks && is_mat(b, s) && !(PIN(b, s) > now)) {
          bool ok = true;
          if (s == msp()) {
            if (b == 0) ok = false;  // roots are never evicted from main
            else {
              bool elsewhere = false;
              NOUNROLL for (int s2 = 0; s2 < n_sp(); ++s2)
                if (s2 != s && V(b, s2) != ABSENT) elsewhere = true;
              ok = elsewhere;
            }
          }
          if (ok) {
            const double st = LU(b, s);
            if (bid < 0 || st < bst || (st == bst && b < bid)) {
              bst = st;
              bid = b;
            }
          }
        }
      }
      wp.argmin3(bst, dummy, bid);
      if (bid < 0) return fail(ST_CAPACITY);
      const int victim = bid;
      const long long vbytes = bbytes(victim);
      if (is_dirty(victim, s)) {
        if (!FLUSH) return fail(ST_ENGINE_INVARIANT);
        const double rdy = V(victim, s);
        const double arr = plan_transfer(victim, nullptr, vbytes, s, msp(), rdy, at);  // sim.cpp:408-409 passes `at`
        if (status) return;
        set_flag(victim, 1u << (8 + s), false);
        reserve_bytes<false>(victim, msp(), arr);
        if (status) return;
        validate_from(victim, msp(), arr);
      }
      set_flag(victim, 1u << s, false);
      setV(victim, s, ABSENT);
      add_used(s, -vbytes);
      if (TRACE && wp.lane() == 0) log_res(at, s, -vbytes, victim);
      setLU(victim, s, 0.0);
      if (s != msp()) {
        // views lose their backing when no materialised block covers them
        const Region vr = reg(victim);
        NOUNROLL for (int base = 0; base < nblocks; base += WP::W) {
          const int x = base + wp.lane();
          bool drop = false;
          if (x < nblocks && V(x, s) != ABSENT && !is_mat(x, s)) {
            const Region xr = reg(x);
            if (roverlap(xr, vr)) {
              bool covered = false;
              NOUNROLL for (int m = 0; m < nblocks && !covered; ++m)
                if (is_mat(m, s) && rcontains(reg(m), xr)) covered = true;
              drop = !covered;
            }
          }
          wp.sync();
          if (drop) V(x, s) = ABSENT;
        }
        wp.sync();
      }
    }
  }

  template <bool FLUSH = true>
  HX void reserve_bytes(int b, int s, double at) {  // sim.cpp:441-450
    if (fast || is_mat(b, s)) return;
    const long long bytes = bbytes(b);
    ensure_capacity<FLUSH>(s, bytes, at);
    if (status) return;
    set_flag(b, 1u << s, true);
    add_used(s, bytes);
    if (TRACE && wp.lane() == 0) log_res(at, s, bytes, b);
    setLU(b, s, at);
  }

  template <bool FLUSH = true>
  HX void materialize(int b, int s, double at) {  // sim.cpp:463-466
    reserve_bytes<FLUSH>(b, s, at);
    if (status) return;
    validate_from(b, s, at);
  }

  HX void pin(int s, int b, double until) {  // sim.cpp:352-355 (E3 representation)
    if (fast) return;
    PIN(b, s) = dmax(PIN(b, s), until);
  }

  // acquire (sim.cpp:501-519) without the gather fallback.
  HXN double acquire_direct(int b, int s, bool& need_gather) {
    need_gather = false;
    const double v = V(b, s);
    if (v != ABSENT) {
      if (!fast) LU(b, s) = dmax(LU(b, s), now);
      return v;
    }
    const int src = source_space(b, s);
    if (src >= 0) {
      const double rdy = V(b, src);
      const double arr = plan_transfer(b, nullptr, bbytes(b), src, s, rdy, now);
      if (status) return 0.0;
      pin(src, b, arr);
      materialize(b, s, arr);
      return arr;
    }
    need_gather = true;
    return 0.0;
  }

  HX double acquire(int b, int s) {
    bool g;
    const double r = acquire_direct(b, s, g);
    if (!g || status) return r;
    return gather(b, s);
  }

  // subtract_regions (graph.cpp:45-84) restricted to what callers need:
  // mode 0 -> returns 1 if base minus cuts is non-empty; mode 1 -> writes the
  // row-sweep fragments into out[] and returns their count.
  HXN int subtract(const Region& base, const Region* cuts, int ncut, Region* out, int mode) {
    int nx = 0, ny = 0;
    // computed redundantly by every lane (uniform), stored by lane 0
    int lx[32], ly[32];
    auto insl = [&](int* arr, int& n, int v) {
      NOUNROLL for (int k = 0; k < n; ++k)
        if (arr[k] == v) return true;
      if (n >= 32) return false;
      int k = n++;
      while (k > 0 && arr[k - 1] > v) {
        arr[k] = arr[k - 1];
        --k;
      }
      arr[k] = v;
      return true;
    };
    bool ok = insl(lx, nx, base.col) && insl(lx, nx, base.col + base.cols) && insl(ly, ny, base.row) &&
              insl(ly, ny, base.row + base.rows);
    NOUNROLL for (int c = 0; c < ncut && ok; ++c) {
      const Region& cr = cuts[c];
      if (!roverlap(base, cr)) continue;
      auto clampi = [](int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); };
      ok = insl(lx, nx, clampi(cr.col, base.col, base.col + base.cols)) &&
           insl(lx, nx, clampi(cr.col + cr.cols, base.col, base.col + base.cols)) &&
           insl(ly, ny, clampi(cr.row, base.row, base.row + base.rows)) &&
           insl(ly, ny, clampi(cr.row + cr.rows, base.row, base.row + base.rows));
    }
    if (!ok) {
      fail(ST_ENGINE_LIMIT);
      return 0;
    }
    int nout = 0;
    NOUNROLL for (int yi = 0; yi + 1 < ny; ++yi) {
      bool have = false;
      Region run;
      run.row = run.col = run.rows = run.cols = 0;
      NOUNROLL for (int xi = 0; xi + 1 < nx; ++xi) {
        Region cell;
        cell.row = ly[yi];
        cell.col = lx[xi];
        cell.rows = ly[yi + 1] - ly[yi];
        cell.cols = lx[xi + 1] - lx[xi];
        bool covered = false;
        NOUNROLL for (int c = 0; c < ncut; ++c)
          if (rcontains(cuts[c], cell)) {
            covered = true;
            break;
          }
        if (covered) {
          if (have) {
            if (mode == 0) return 1;
            if (nout >= PB.maxgr) {
              fail(ST_ENGINE_LIMIT);
              return 0;
            }
            if (wp.lane() == 0) out[nout] = run;
            ++nout;
          }
          have = false;
        } else if (have) {
          run.cols += cell.cols;
        } else {
          run = cell;
          have = true;
        }
      }
      if (have) {
        if (mode == 0) return 1;
        if (nout >= PB.maxgr) {
          fail(ST_ENGINE_LIMIT);
          return 0;
        }
        if (wp.lane() == 0) out[nout] = run;
        ++nout;
      }
    }
    wp.sync();
    return nout;
  }

  // gather (sim.cpp:521-572): assemble a block with no whole valid() copy.
  HXN double gather(int blk, int s) {
    const Region target = reg(blk);
    const int t = blk == 0 ? -1 : tile_of(blk);
    // candidate pieces: contained blocks valid() here or anywhere
    int np = 0;
    {
      const int cnt = t < 0 ? nblocks : 2 + tl_cnt()[t];
      const int head = t < 0 ? 0 : tl_head()[t];
      NOUNROLL for (int base = 0; base < cnt; base += WP::W) {
        const int k = base + wp.lane();
        int b = -1;
        bool hit = false;
        if (k < cnt) {
          b = t < 0 ? k : (k == 0 ? 0 : (k == 1 ? t : tl_ids()[head + k - 2]));
          if (b != blk && rcontains(target, reg(b))) {
            bool any = false;
            NOUNROLL for (int q = 0; q < n_sp(); ++q)
              if (V(b, q) != ABSENT) any = true;
            hit = any;
          }
        }
        const unsigned m = wp.ballot(hit);
        if (hit) {
          const int at = np + popc32(m & wp.lt());
          if (at < PB.maxgs) gs_a()[at] = b;
        }
        np += popc32(m);
      }
      wp.sync();
      if (np > PB.maxgs) {
        fail(ST_ENGINE_LIMIT);
        return 0.0;
      }
    }
    // sort pieces: local first, then area descending, then id (sim.cpp:540-544)
    NOUNROLL for (int k = wp.lane(); k < np; k += WP::W) {
      const int a = gs_a()[k];
      const bool la = V(a, s) != ABSENT;
      const Region ra = reg(a);
      const long long aa = (long long)ra.rows * ra.cols;
      int rank = 0;
      NOUNROLL for (int q = 0; q < np; ++q) {
        const int c = gs_a()[q];
        if (c == a) continue;
        const bool lc = V(c, s) != ABSENT;
        const Region rc = reg(c);
        const long long ac = (long long)rc.rows * rc.cols;
        bool before;
        if (lc != la) before = lc;
        else if (ac != aa) before = ac > aa;
        else before = c < a;
        rank += before;
      }
      gs_reg2()[rank].row = a;  // stash sorted ids in gs_reg2()[].row
    }
    wp.sync();
    double arrival = 0.0;
    int ncov = 0;
    if (np > PB.maxgr) {
      fail(ST_ENGINE_LIMIT);
      return 0.0;
    }
    NOUNROLL for (int k = 0; k < np; ++k) {
      const int piece = gs_reg2()[k].row;
      const Region pr = reg(piece);
      if (subtract(pr, gs_reg(), ncov, nullptr, 0) == 0) {
        if (status) return 0.0;
        continue;  // adds nothing
      }
      bool g;
      const double a = acquire_direct(piece, s, g);
      if (status) return 0.0;
      if (g) {  // a listed piece is valid() somewhere, so this cannot happen
        fail(ST_ENGINE_INVARIANT);
        return 0.0;
      }
      arrival = dmax(arrival, a);
      if (wp.lane() == 0) gs_reg()[ncov] = pr;
      wp.sync();
      ++ncov;
    }
    // residue from main, unless it overlaps data written since the start
    const int nfr = subtract(target, gs_reg(), ncov, gs_reg2(), 1);
    if (status) return 0.0;
    if (nfr > 0) {
      bool bad = false;
      NOUNROLL for (int f = 0; f < nfr && !bad; ++f) {
        const Region fr = gs_reg2()[f];
        bool hit = false;
        for_scope(t, [&](int x) {
          if (wrt()[x])
            if (roverlap(fr, reg(x))) hit = true;
        });
        bad = wp.any(hit);
      }
      if (bad) {
        fail(ST_COHERENCE);
        return 0.0;
      }
      if (s != msp())
        NOUNROLL for (int f = 0; f < nfr; ++f) {
          const Region fr = gs_reg2()[f];
          arrival = dmax(arrival, plan_transfer(blk, &fr, rbytes(fr), msp(), s, 0.0, now));
          if (status) return 0.0;
        }
    }
    if (V(blk, s) > arrival) setV(blk, s, arrival);
    return arrival;
  }

  // invalidate_elsewhere (sim.cpp:574-590) over the invalidation cone
  // (sim.cpp:204-212), which by E1 is: blocks inside b, plus blocks strictly
  // containing some block inside b.
  HXN void invalidate_elsewhere(int b, int ws, double at) {
    const int t = b == 0 ? -1 : tile_of(b);
    const Region rb = reg(b);
    long long freed[MAXS];
    NOUNROLL for (int q = 0; q < MAXS; ++q) freed[q] = 0;
    const int cnt = t < 0 ? nblocks : 2 + tl_cnt()[t];
    const int head = t < 0 ? 0 : tl_head()[t];
    NOUNROLL for (int k = wp.lane(); k < cnt; k += WP::W) {
      const int x = t < 0 ? k : (k == 0 ? 0 : (k == 1 ? t : tl_ids()[head + k - 2]));
      const Region rx = reg(x);
      bool in = false;
      if (rcontains(rb, rx) || rcontains(rx, rb)) in = true;
      else if (roverlap(rx, rb)) {
        // partial overlap: in the cone iff some block inside b is strictly inside x
        NOUNROLL for (int q = 0; q < cnt && !in; ++q) {
          const int c = t < 0 ? q : (q == 0 ? 0 : (q == 1 ? t : tl_ids()[head + q - 2]));
          const Region rc = reg(c);
          if (c != x && rcontains(rb, rc) && rcontains(rx, rc) && !rsame(rx, rc)) in = true;
        }
      }
      if (!in) continue;
      if (fast) {
        NOUNROLL for (int q = 0; q < n_sp(); ++q)
          if (q != ws) V(x, q) = ABSENT;
        continue;
      }
      uint32_t f = bflags()[x];
      NOUNROLL for (int q = 0; q < n_sp(); ++q) {
        if (q == ws) continue;
        if ((f >> q) & 1u) {
          freed[q] += rbytes(rx);
          LU(x, q) = 0.0;
          if (TRACE) log_res(at, q, -rbytes(rx), x);
        }
        V(x, q) = ABSENT;
      }
      const uint32_t keep = (1u << ws) | (1u << (8 + ws)) | (1u << 16);
      bflags()[x] = f & keep;
    }
    wp.sync();
    if (fast) return;
    NOUNROLL for (int q = 0; q < n_sp(); ++q) {
      if (q == ws) continue;
      const long long fr = wp.suml(freed[q]);
      if (fr) add_used(q, -fr);
    }
  }

  // =========================================================================
  // Scheduling (sim.cpp:704-834)
  // =========================================================================

  // Working set of a task: distinct blocks of reads u writes in id order
  // (the std::set iteration of sim.cpp:597-598 and sim.cpp:768-769).
  static HX int working_set(const TaskMeta& t, int* w) {
    // the task's distinct blocks, ascending; the <= 4 block slots unrolled
    // with constant indices so the caller's w[] can stay in registers
    int nw = 0;
    w[0] = w[1] = w[2] = w[3] = 0x7fffffff;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k > t.nrd) break;
      const int b = t.blk[k];
      bool dup = false;
      int ins = 0;  // insertion point: the entries below b
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        dup |= q < nw && w[q] == b;
        ins += q < nw && w[q] < b;
      }
      if (dup) continue;
#pragma unroll
      for (int q = 3; q > 0; --q)
        if (q > ins) w[q] = w[q - 1];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q == ins) w[q] = b;
      ++nw;
    }
    return nw;
  }

  using LaneD = typename WP::LaneD;
  using LaneI = typename WP::LaneI;

  HX uint64_t rng_next() { return hesp_splitmix_next(&rng); }

  // WT / WA write-back of a task's output to main (sim.cpp:631-656).
  HXN void write_back(int out, int s, double end) {
    const double arr = plan_transfer(out, nullptr, bbytes(out), s, msp(), end, now);
    if (status) return;
    pin(s, out, arr);
    materialize<false>(out, msp(), arr);
    if (status) return;
    if (PB.caching == CACHE_WA) {  // write-around: drop the local copy (sim.cpp:643-655)
      if (!fast) {
        set_flag(out, 1u << s, false);
        add_used(s, -bbytes(out));
        if (TRACE && wp.lane() == 0) log_res(arr, s, -bbytes(out), out);
        setLU(out, s, 0.0);
      }
      V(out, s) = ABSENT;
      const int tt = out == 0 ? -1 : tile_of(out);
      if (!(tt > 0 && tl_cnt()[tt] == 0)) {
        const Region ro = reg(out);
        for_scope(tt, [&](int x) {
          if (inside(x, out, tt, ro)) V(x, s) = ABSENT;
        });
      }
    }
  }

  // The event loop (sim.cpp:704-834) with Engine::commit (sim.cpp:592-668)
  // inlined.  Everything the loop touches per task -- array bases, clocks,
  // pool size, hashes, makespan -- is copied into registers first (lanes own
  // processor and link clocks); `this` is only touched by the cold paths
  // (gather, eviction bookkeeping, coherence over subdivided tiles).
  HXN void simulate() {
    const int P = PB.P;
#if defined(__CUDACC__)
    if constexpr (WP::W > 1) {
      SM().vstage = nullptr;  // only sim_lean stages
      wp.sync();
    }
#endif
    if (nleaves == 0) return fail(ST_VALIDATION);
    if (P < 1) return fail(ST_NO_PROCESSORS);
    // check_models (sim.cpp:312-321)
    bool miss = false;
    NOUNROLL for (int li = wp.lane(); li < nleaves; li += WP::W) {
      const TaskMeta t = task(leaf()[li]);
      NOUNROLL for (int ty = 0; ty < PB.n_types; ++ty)
        if (!PB.known[t.kind][ty]) miss = true;
    }
    if (wp.any(miss)) return fail(ST_MODEL_MISS);
    // E4: can any space ever need to evict?  (root only ever lives in main)
    {
      long long nonroot = 0;
      NOUNROLL for (int x = 1 + wp.lane(); x < nblocks; x += WP::W) nonroot += bbytes(x);
      nonroot = wp.suml(nonroot);
      bool ok = true;
      const bool root_leaf = BV().til == TIL_ROOT;  // the root task itself is scheduled: its block goes anywhere
      NOUNROLL for (int q = 0; q < n_sp(); ++q)
        if (nonroot + ((q == msp() || root_leaf) ? bbytes(0) : 0) > PB.cap[q]) ok = false;
      fast = ok && (!TRACE || (tb && tb->lite));  // the full trace keeps residency bookkeeping
    }
    if (fast && !TRACE && PB.loop == 0) {  // the batch kernels' lean loop
      switch (PB.selection) {
        case SEL_EFTP: return sim_lean<SEL_EFTP>();
        case SEL_EITP: return sim_lean<SEL_EITP>();
        case SEL_FP: return sim_lean<SEL_FP>();
        default: return sim_lean<SEL_RP>();
      }
    }
    switch (PB.selection) {
      case SEL_EFTP: return fast ? sim_loop<SEL_EFTP, true>() : sim_loop<SEL_EFTP, false>();
      case SEL_EITP: return fast ? sim_loop<SEL_EITP, true>() : sim_loop<SEL_EITP, false>();
      case SEL_FP: return fast ? sim_loop<SEL_FP, true>() : sim_loop<SEL_FP, false>();
      default: return fast ? sim_loop<SEL_RP, true>() : sim_loop<SEL_RP, false>();
    }
  }

  // The loop proper, specialised on the selection policy and on E4 (no
  // eviction possible) so one batch executes one compact instantiation.
  template <int SELT, bool FASTT>
  HXN void sim_loop() {
    const int P = PB.P;
    // init_memory (sim.cpp:323-339): root materialised in main, every block
    // valid in main at t=0 (views into the root data)
    NOUNROLL for (int x = wp.lane(); x < nblocks; x += WP::W) {
      NOUNROLL for (int q = 0; q < n_sp(); ++q) {
        V(x, q) = q == msp() ? 0.0 : ABSENT;
        if (!fast) {
          LU(x, q) = 0.0;
          PIN(x, q) = NOPIN;
        }
      }
      if (!fast) bflags()[x] = x == 0 ? (1u << msp()) : 0u;  // read only by eviction bookkeeping
      wrt()[x] = 0;
    }
    NOUNROLL for (int q = wp.lane(); q < MAXS; q += WP::W) SM().used[q] = q == msp() ? bbytes(0) : 0;
    if (TRACE && wp.lane() == 0) log_res(0.0, msp(), bbytes(0), 0);  // init_memory (sim.cpp:333)
    wp.sync();
    if (SM().used[msp()] > PB.cap[msp()]) return fail(ST_CAPACITY);
    if (PB.ordering == ORD_PL) build_ct();
    if (status) return;

    // ---------------- register copies for the hot loop ----------------
    // Only the slot base stays live; every array base is rematerialised from
    // it and a constant-memory offset at the point of use (one IADD), which
    // keeps ~30 registers of pointers out of the spill set.
    uint8_t* const sl = slot;
#define HOT_ARR(type, field) ((type*)(sl + PB.lay.field))
#define VV HOT_ARR(double, valid)
#define T HOT_ARR(TState, ts)
#define SU HOT_ARR(const int, succs)
#define LF HOT_ARR(const int, leaf)
#define PO HOT_ARR(int, pool)
#define PR HOT_ARR(double, pool_rel)
#define PK HOT_ARR(double, pool_key)
#define RI HOT_ARR(int, gs_a)
#define RK HOT_ARR(double, ready_key)
#define RS HOT_ARR(int, ready)
#define TLC HOT_ARR(const int, tl_cnt)
#define BF HOT_ARR(uint32_t, bflags)
#define TM HOT_ARR(const TaskMeta, tm)
#define BM HOT_ARR(const BlockMeta, bm)
#define BT (bt_())
#define BB (bb_())
    // problem-wide scalars are read from constant memory at each use
#define nbt_ n_bt()
#define nbb_ n_bb()
#define S_ PB.S
#define ms PB.main_space
#define elem PB.elem
#define sel SELT
#define waits (SELT == SEL_RP || SELT == SEL_FP)
#define pl (PB.ordering == ORD_PL)
    const int nl = nleaves;
    constexpr bool fst = FASTT;
    auto Vr = [&](int b, int s) -> double& { return VV[b * S_ + s]; };
    auto taskm = [&](int id) -> TaskMeta { return id < nbt_ ? BT[id] : TM[id - nbt_]; };
    auto tileof = [&](int b) -> int { return b < nbb_ ? BB[b].tile : BM[b - nbb_].tile; };
    auto bytesof = [&](int b) -> long long {
      const Region r = b < nbb_ ? BB[b].r : BM[b - nbb_].r;
      return (long long)r.rows * r.cols * elem;
    };
    // source_spaces().front() minus `excl` (sim.cpp:341-350): main first, then id order
    auto srcsp = [&](int b, int excl) -> int {
      if (ms != excl && Vr(b, ms) != ABSENT) return ms;
      NOUNROLL for (int q = 0; q < S_; ++q)
        if (q != ms && q != excl && Vr(b, q) != ABSENT) return q;
      return -1;
    };

    // initial pool: leaves without predecessors, release 0
    int pool_n = 0;
    NOUNROLL for (int base = 0; base < nl; base += WP::W) {
      const int li = base + wp.lane();
      bool z = false;
      int j = -1;
      double key = 0.0;
      if (li < nl) {
        j = LF[li];
        TState& st = T[j];
        st.rel = 0.0;
        z = st.missing == 0;
        key = pl ? st.ct : 0.0;
      }
      const unsigned m = wp.ballot(z);
      if (z) {
        const int at = pool_n + popc32(m & wp.lt());
        PO[at] = j;
        PR[at] = 0.0;
        PK[at] = key;
      }
      pool_n += popc32(m);
    }
    wp.sync();
    // lane-owned clocks and processor attributes
    LaneD est, estp;
    // processor clocks and attributes in the warp's Small, like the link clocks
#define PF_OWN(q) SM().proc_free[q]
#define PF_GET(p) SM().proc_free[p]
#define PF_SET(p, v) (SM().proc_free[p] = (v))
#define PTYPE(q) SM().ptype[q]
#define PSPACE_OWN SM().pspace[wp.lane()]
    NOUNROLL for (int q = wp.lane(); q < MAXP; q += WP::W) SM().proc_free[q] = 0.0;
    est.fill(0.0);
    estp.fill(0.0);
    NOUNROLL for (int q = wp.lane(); q < MAXP; q += WP::W) {
      PTYPE(q) = q < P ? PB.proc_type[q] : 0;
      SM().pspace[q] = q < P ? PB.proc_space[q] : 0;
    }
#if defined(__CUDACC__)
    const int eft_k = wp.lane() / S_, eft_sp = wp.lane() - (wp.lane() / S_) * S_;  // lane = (block, space)
    (void)eft_k;
    (void)eft_sp;
#endif
    rng = PB.sched_seed;
    double tnow = 0.0, mk = 0.0;
    // link clocks and the result hashes live in the warp's shared Small
    // (uniform values: every lane stores the same value and reads its own
    // store), which keeps them out of the register file the loop spills from
    Small& smw = SM();
    smw.ah = 0;
    smw.xh = 0;
#define HAH smw.ah
#define HXH smw.xh
    NOUNROLL for (int i = wp.lane(); i < MAXL; i += WP::W) smw.link_free[i] = 0.0;
    wp.sync();
    int st = 0;  // status mirror for the hot loop
    now = 0.0;

    // plan_transfer (sim.cpp:468-499) on lane-owned link clocks
    auto xfer = [&](int blk, long long nbytes, int bi, int src, int dst, double data_ready) -> double {
      const int nh = PB.route_n[src * MAXS + dst];
      if (nh == 0) {
        st = ST_NO_ROUTE;
        return 0.0;
      }
      double rdy = dmax(data_ready, tnow), start0 = 0.0;
      double hs[2] = {0.0, 0.0}, he[2] = {0.0, 0.0};
      NOUNROLL for (int h = 0; h < nh; ++h) {
        const int l = PB.route_l[src * MAXS + dst][h];
        const double s0 = dmax(smw.link_free[l], rdy);
        const double en = s0 + PB.link_lat[l] + PB.hopq[l][bi];  // (s0 + lat) + bytes/bw
        smw.link_free[l] = en;  // uniform: every lane stores the same value and reads its own store
        rdy = en;
        if (h == 0) start0 = s0;
        if (TRACE && h < 2) {
          hs[h] = s0;
          he[h] = en;
        }
      }
      if (!(rdy > tnow)) st = ST_ENGINE_INVARIANT;
      if (TRACE) log_xfer(blk, nullptr, nbytes, src, dst, start0, rdy, nh, hs, he);
      {  // one lane folds the term (only lane 0's copy of the hashes is reported)
        const uint64_t xt_ = hesp_xfer_term(xblock(blk), src, dst, nbytes, dbits(start0), dbits(rdy), 0, 0, 0, 0);
        if (wp.lane() == 0) HXH += xt_;
      }
      return rdy;
    };
    // cold-call bracket: hand the uniform hot state to the member paths and back
    auto cold_in = [&]() {
      now = tnow;
      wp.sync();
      if (wp.lane() == 0) {
        xhash += HXH;
        HXH = 0;
      }
      status = st;
    };
    auto cold_out = [&]() {
      wp.sync();
      st = status;
    };
    // validate_from on the hot path: an unsubdivided tile has no descendants
    auto validate = [&](int b, int s, double at, bool simple) {
      if (fst && simple) {
        double& v = Vr(b, s);
        if (v > at) v = at;
      } else {
        validate_from(b, s, at);
      }
    };
    // acquire (sim.cpp:501-519)
    auto acquire_h = [&](int b, int s, int bi, long long nbytes, bool simple) -> double {
      const double v = Vr(b, s);
      if (v != ABSENT) {
        if (!fst) LU(b, s) = dmax(LU(b, s), tnow);
        return v;
      }
      const int src = srcsp(b, s);
      if (src >= 0) {
        const double arr = xfer(b, nbytes, bi, src, s, Vr(b, src));
        if (st) return 0.0;
        if (!fst) {
          pin(src, b, arr);
          cold_in();
          reserve_bytes(b, s, arr);  // may evict and flush
          cold_out();
          if (st) return 0.0;
        }
        validate(b, s, arr, simple);
        return arr;
      }
      cold_in();
      const double r = gather(b, s);  // assemble from pieces + residue from main
      cold_out();
      return r;
    };
    // est_transfer_ready of space sp (sim.cpp:762-793).  The per-link
    // accumulators (`acc` map, fresh per processor) have at most 3 blocks x
    // 2 hops = 6 distinct keys: kept in unrolled register slots.
    auto eft_space_h = [&](int sp, const int* w, int nw, bool& noroute) -> double {
      double est_ = 0.0;
      int al[6] = {-1, -1, -1, -1, -1, -1};
      double av[6] = {0, 0, 0, 0, 0, 0};
      NOUNROLL for (int k = 0; k < nw; ++k) {
        const int b = w[k];
        const double v = Vr(b, sp);
        if (v != ABSENT) {
          est_ = dmax(est_, v);
          continue;
        }
        const int src = srcsp(b, sp);
        if (src < 0) continue;
        const int nh = PB.route_n[src * MAXS + sp];
        if (nh == 0) {
          noroute = true;
          continue;
        }
        const double nbytes = (double)bytesof(b);
        double tarr = dmax(tnow, Vr(b, src));
        NOUNROLL for (int h = 0; h < nh; ++h) {
          const int l = PB.route_l[src * MAXS + sp][h];
          const double hop = PB.link_lat[l] + nbytes / PB.link_bw[l];
          double acc = 0.0;
          bool placed = false;
#pragma unroll
          for (int z = 0; z < 6; ++z) {
            if (!placed && (al[z] == l || al[z] < 0)) {
              al[z] = l;
              av[z] += hop;
              acc = av[z];
              placed = true;
            }
          }
          tarr += acc;
        }
        est_ = dmax(est_, tarr);
      }
      return est_;
    };

    int committed = 0;
    bool first = true;
    NOUNROLL while (committed < nl) {
      if (!first) {
        // next epoch (E3): smallest pending release / processor-free time > now
        double nx = ABSENT;
        NOUNROLL for (int k = wp.lane(); k < pool_n; k += WP::W) {
          const double r = PR[k];
          if (r > tnow && r < nx) nx = r;
        }
        if (waits) {
          NOUNROLL for (int q = wp.lane(); q < P; q += WP::W) {
            const double f = PF_OWN(q);
            if (f > tnow && f < nx) nx = f;
          }
        }
        nx = wp.mind(nx);
        if (nx == ABSENT) return fail(ST_INTERNAL);  // scheduler stalled
        tnow = nx;  // the member `now` is only read by the cold paths: set in cold_in
      }
      first = false;
      // ready = released, uncommitted, rel <= now, ordered FCFS (rel asc, id
      // asc) or PL (ct desc, id asc) (sim.cpp:117-134); non-ready entries are
      // compacted to the pool front on the way.
      int nr = 0, keep = 0;
      NOUNROLL for (int base = 0; base < pool_n; base += WP::W) {
        const int k = base + wp.lane();
        bool r = false, kp = false;
        int j = -1;
        double rl = 0.0, key = 0.0;
        if (k < pool_n) {
          j = PO[k];
          rl = PR[k];
          key = PK[k];
          r = rl <= tnow;
          kp = !r;
        }
        const unsigned m = wp.ballot(r), mk2 = wp.ballot(kp);
        if (r) {
          const int at = nr + popc32(m & wp.lt());
          RI[at] = j;
          RK[at] = key;
        }
        if (kp) {
          const int at = keep + popc32(mk2 & wp.lt());
          PO[at] = j;
          PR[at] = rl;
          PK[at] = key;
        }
        nr += popc32(m);
        keep += popc32(mk2);
        wp.sync();
      }
      pool_n = keep;
      if (nr == 0) continue;
      if (nr == 1) {
        RS[0] = RI[0];
      } else {
        NOUNROLL for (int k = wp.lane(); k < nr; k += WP::W) {
          const int a = RI[k];
          const double ka = RK[k];
          int rank = 0;
          NOUNROLL for (int q = 0; q < nr; ++q) {
            const int c = RI[q];
            const double kc = RK[q];
            rank += (kc != ka) ? (pl ? kc > ka : kc < ka) : (c < a);
          }
          RS[rank] = a;
        }
        wp.sync();
      }
      int done = 0;
      NOUNROLL for (; done < nr; ++done) {
        const int j = RS[done];
        const STask tk = HOT_ARR(const STask, wsb)[j];
        const double rel = T[j].rel;
        const int tkind = tk.kb & 0xff, tbidx = tk.kb >> 8;
        const int w[4] = {tk.ws0, tk.ws1, tk.ws2, -1};
        const int nw = tk.nw;
        const long long tbytes = (long long)tk.b * tk.b * elem;  // every block of a task has its side
        int p = -1;
        // ---------------- processor selection (sim.cpp:136-192) ----------------
        if (waits) {
          unsigned idle_mask = 0;
          NOUNROLL for (int q = wp.lane(); q < P; q += WP::W)
            if (PF_OWN(q) <= tnow) idle_mask |= 1u << q;
#if defined(__CUDACC__)
          if constexpr (WP::W > 1) idle_mask = __reduce_or_sync(0xffffffffu, idle_mask);
#endif
          if (idle_mask == 0) break;  // R-P/F-P wait for a processor (sim.cpp:800-801)
          if (sel == SEL_RP) {
            const int n = popc32(idle_mask);
            const double u = (double)(rng_next() >> 11) * 0x1.0p-53;
            const int k = (int)((unsigned long long)(u * (double)n) % (unsigned long long)n);
            unsigned mmm = idle_mask;
            for (int q = 0; q < k; ++q) mmm &= mmm - 1;
            p = ctz32(mmm);
          } else {  // F-P: fastest idle processor, lowest id
            double a = ABSENT, b2 = 0.0;
            int id = -1;
            NOUNROLL for (int q = wp.lane(); q < P; q += WP::W) {
              if (!((idle_mask >> q) & 1u)) continue;
              const double tt = PB.ttime[tkind][tbidx][PTYPE(q)];
              if (id < 0 || tt < a) {
                a = tt;
                id = q;
              }
            }
            wp.argmin_lane(a, b2, id);
            p = id;
          }
        } else {
          if (sel == SEL_EFTP) {
            bool noroute = false;
#if defined(__CUDACC__)
            if constexpr (WP::W > 1) {
            // Warp-parallel est_transfer_ready (sim.cpp:762-793): lane (k, sp)
            // owns block k of the working set in space sp.  One round trip
            // loads every V(b_k, sp); ballots give each block's valid-space
            // mask; the per-link accumulators of the reference's `acc` map are
            // rebuilt in order from the (<= 2) earlier blocks of the same space
            // by shuffles; a segmented max gives the estimate per space.
            {
              const unsigned FULL = 0xffffffffu;
              const int lane = wp.lane();
              const int Sx = S_;
              const int k = eft_k, sp = eft_sp;
              const bool act = k < nw;
              const int b = k == 0 ? tk.ws0 : (k == 1 ? tk.ws1 : tk.ws2);
              const double v = act ? Vr(b, sp) : ABSENT;
              const unsigned vm = __ballot_sync(FULL, act && v != ABSENT);
              const unsigned mymask = act ? (vm >> (k * Sx)) & ((1u << Sx) - 1u) : 0u;
              int src = -1;
              if (act && v == ABSENT) {
                if (ms != sp && ((mymask >> ms) & 1u)) {
                  src = ms;
                } else {
                  const unsigned o = mymask & ~(1u << ms) & ~(1u << sp);
                  if (o) src = ctz32(o);
                }
              }
              const double vsrc = __shfl_sync(FULL, v, src >= 0 ? k * Sx + src : lane);
              int l0 = -1, l1 = -1, nh = 0;
              double c0 = 0.0, c1 = 0.0;
              if (src >= 0) {
                nh = PB.route_n[src * MAXS + sp];
                if (nh == 0) noroute = true;
                // every block of a task has the task's side (graph.cpp:303-307):
                // hop cost lat + bytes/bw precomputed per (link, side)
                if (nh >= 1) {
                  l0 = PB.route_l[src * MAXS + sp][0];
                  c0 = PB.hopc[l0][tbidx];
                }
                if (nh >= 2) {
                  l1 = PB.route_l[src * MAXS + sp][1];
                  c1 = PB.hopc[l1][tbidx];
                }
              }
              double acc0 = 0.0, acc1 = 0.0;
              // rebuild only if some lane transfers; only nw-1 earlier blocks exist
              const int rounds = __any_sync(FULL, src >= 0) ? nw - 1 : 0;
#pragma unroll
              for (int kp = 0; kp < 2; ++kp) {  // earlier blocks of this space, in order
                if (kp >= rounds) break;
                const int from = kp * Sx + sp < 32 ? kp * Sx + sp : lane;
                const int pl0 = __shfl_sync(FULL, l0, from), pl1 = __shfl_sync(FULL, l1, from);
                const double pc0 = __shfl_sync(FULL, c0, from), pc1 = __shfl_sync(FULL, c1, from);
                if (kp < k) {
                  if (l0 >= 0 && pl0 == l0) acc0 += pc0;
                  if (l0 >= 0 && pl1 == l0) acc0 += pc1;
                  if (l1 >= 0 && pl0 == l1) acc1 += pc0;
                  if (l1 >= 0 && pl1 == l1) acc1 += pc1;
                }
              }
              double val = 0.0;
              if (act) {
                if (v != ABSENT) {
                  val = v;
                } else if (src >= 0 && nh > 0) {
                  double tarr = dmax(tnow, vsrc);
                  acc0 += c0;
                  tarr += acc0;
                  if (nh == 2) {
                    acc1 += c1;
                    tarr += acc1;
                  }
                  val = tarr;
                }
              }
              double e = val;  // est(sp) = max(0, max_k val(k, sp)), held by lane sp
#pragma unroll
              for (int kp = 1; kp < 3; ++kp) {
                const int from = kp * Sx + lane < 32 ? kp * Sx + lane : lane;
                const double o = __shfl_sync(FULL, val, from);
                if (lane < Sx && kp < nw) e = dmax(e, o);
              }
              estp.own(0) = __shfl_sync(FULL, e, PSPACE_OWN);
            }
            if (wp.any(noroute)) return fail(ST_NO_ROUTE);
            } else
#endif
            {  // one lane: the reference's loop, space by space
            NOUNROLL for (int sp = wp.lane(); sp < S_; sp += WP::W) est.own(sp) = eft_space_h(sp, w, nw, noroute);
            if (wp.any(noroute)) return fail(ST_NO_ROUTE);
            NOUNROLL for (int q = 0; q < P; ++q) estp.own(q) = est.get(SM().pspace[q]);  // estimate of each processor's space
            }
          }
          double a = ABSENT, b2 = 0.0;
          int id = -1;
          NOUNROLL for (int q = wp.lane(); q < P; q += WP::W) {
            const double nf = PF_OWN(q);
            double qa, qb = 0.0;
            if (sel == SEL_EFTP) {
              qa = dmax(dmax(nf, rel), estp.own(q)) + PB.ttime[tkind][tbidx][PTYPE(q)];
              qb = nf;
            } else {
              qa = nf;  // EIT-P
            }
            if (id < 0 || qa < a || (qa == a && qb < b2)) {
              a = qa;
              b2 = qb;
              id = q;
            }
          }
          wp.argmin_lane(a, b2, id);
          p = id;
        }
        if (p < 0) return fail(ST_NO_PROCESSORS);
        // ---------------- commit (sim.cpp:592-668) ----------------
        const int s = SM().pspace[p];
        const int type = PTYPE(p);
        if (!fst) {
          long long wset = 0;
          NOUNROLL for (int k = 0; k < nw; ++k) wset += bytesof(w[k]);
          if (wset > PB.cap[s]) return fail(ST_CAPACITY);
        }
        double inputs = 0.0;
        double saved[3] = {0.0, 0.0, 0.0};
        NOUNROLL for (int k = 0; k < nw; ++k) {  // working set in id order (<= 3 blocks, registers)
          const int wb = k == 0 ? tk.ws0 : (k == 1 ? tk.ws1 : tk.ws2);
          const double a = acquire_h(wb, s, tbidx, tbytes, (tk.pad >> k) & 1);
          if (st) return fail(st);
          inputs = dmax(inputs, a);
          if (!fst) {
            saved[k] = PIN(wb, s);
            setPIN(wb, s, HOLD);
          }
        }
        const int out = tk.out;
        if (!fst) {
          cold_in();
          reserve_bytes(out, s, tnow);
          cold_out();
          if (st) return fail(st);
        }
        const double start = dmax(dmax(PF_GET(p), rel), inputs);
        const double end = start + PB.ttime[tkind][tbidx][type];
        if (!(end > tnow) || start < tnow) return fail(ST_ENGINE_INVARIANT);
        PF_SET(p, end);
        {
          const uint64_t at_ = hesp_assign_term(xtask(j), p, dbits(start), dbits(end));
          if (wp.lane() == 0) HAH += at_;
        }
        if (TRACE && xtask(j) < tr_cap && wp.lane() == 0) {
          tr_proc[xtask(j)] = p;
          tr_start[xtask(j)] = start;
          tr_end[xtask(j)] = end;
        }
        mk = dmax(mk, end);
        if (!fst) {
#pragma unroll
          for (int k = 0; k < 3; ++k)
            if (k < nw) setPIN(k == 0 ? tk.ws0 : (k == 1 ? tk.ws1 : tk.ws2), s, dmax(saved[k], end));
        }
        // write coherence (sim.cpp:625-628): invalidate the cone elsewhere,
        // validate out and its descendants here, valid[out] = end
        {
          if (fst && (tk.pad & 8)) {  // cone = {root, tile}, no descendants
            NOUNROLL for (int q = wp.lane(); q < S_; q += WP::W)
              if (q != s) {
                Vr(0, q) = ABSENT;
                Vr(out, q) = ABSENT;
              }
            wp.sync();
          } else {
            invalidate_elsewhere(out, s, start);
            validate_from(out, s, end);
          }
          Vr(out, s) = end;
        }
        HOT_ARR(uint8_t, wrt)[out] = 1;  // written (gather's coherence check): a plain store
        if (s != ms) {
          if (PB.caching == CACHE_WB) {
            if (!fst) set_flag(out, 1u << (8 + s), true);
          } else {
            cold_in();
            write_back(out, s, end);  // WT / WA (cold: the headline policy is WB)
            cold_out();
            if (st) return fail(st);
          }
        }
        // release successors (sim.cpp:660-667): running max of pred ends;
        // released tasks enter the pool with release time and key inline
        const int off = T[j].soff, cnt = T[j].scnt;
        int added = 0;
        NOUNROLL for (int base = 0; base < cnt; base += WP::W) {
          const int q = base + wp.lane();
          bool rl = false;
          int sj = -1;
          double r = 0.0, key = 0.0;
          if (q < cnt) {
            sj = SU[off + q];
            TState& ts_ = T[sj];
            const int left = --ts_.missing;
            r = dmax(ts_.rel, end);
            ts_.rel = r;
            rl = left == 0;
            if (rl) key = pl ? ts_.ct : r;
          }
          const unsigned m = wp.ballot(rl);
          if (rl) {
            const int at = pool_n + added + popc32(m & wp.lt());
            PO[at] = sj;
            PR[at] = r;
            PK[at] = key;
          }
          added += popc32(m);
        }
        wp.sync();
        pool_n += added;
        ++committed;
      }
      // R-P/F-P: ready tasks that found no idle processor return to the pool
      if (done < nr) {
        NOUNROLL for (int k = done + wp.lane(); k < nr; k += WP::W) {
          const int j = RS[k];
          const int at = pool_n + (k - done);
          PO[at] = j;
          PR[at] = T[j].rel;
          PK[at] = pl ? T[j].ct : T[j].rel;
        }
        wp.sync();
        pool_n += nr - done;
      }
    }
    makespan = mk;
    wp.sync();
    ahash += HAH;
    xhash += HXH;
#undef HAH
#undef HXH
#undef PF_OWN
#undef PF_GET
#undef PF_SET
#undef PTYPE
#undef PSPACE_OWN
#undef HOT_ARR
#undef nbt_
#undef nbb_
#undef S_
#undef ms
#undef elem
#undef sel
#undef waits
#undef pl
#undef VV
#undef T
#undef SU
#undef LF
#undef PO
#undef PR
#undef PK
#undef RI
#undef RK
#undef RS
#undef TLC
#undef BF
#undef TM
#undef BM
#undef BT
#undef BB
  }

  // =========================================================================
  // Lean event loop: the batch kernels' instance of sim.cpp:704-834 on the
  // E4 fast path (no eviction possible).  Same decisions as sim_loop; built
  // so the hot loop contains no call and keeps no value in local memory:
  //   * the loop (lean_run, inlined into its driver) returns to the driver
  //     for every step that needs a member call -- gather (sim.cpp:521-572),
  //     the WT/WA write-back, coherence over the root or over a tile holding
  //     partial overlaps -- with its state in the warp's Small (LeanState),
  //     and resumes the task in progress where it left it;
  //   * coherence over a subdivided tile is one lane-parallel pass over the
  //     tile's scope (root, tile, its blocks): the invalidation cone
  //     (sim.cpp:204-212) of a block in a tile without partial overlaps is
  //     exactly the blocks containing it or inside it (E1), and
  //     validate_from (sim.cpp:452-461) the blocks inside it;
  //   * acquire (sim.cpp:501-519) reads V(b_k, q) of the whole working set
  //     in one round, lane (k, q); a task's working-set blocks are pairwise
  //     disjoint (STask flag bit 4, checked at build time), so acquiring one
  //     never changes another, and only the transfers run in id order (the
  //     per-link FIFO of plan_transfer, sim.cpp:468-499);
  //   * EFT-P/EIT-P commit every ready task of an epoch, so the ready set is
  //     the pool entries at the pool's minimum release time, kept
  //     incrementally (no separate next-epoch scan);
  //   * clocks, attributes and hashes live in the warp's Small (LDS/STS).
  // =========================================================================
  enum : int32_t { LEAN_DONE = 0, LEAN_GATHER = 1, LEAN_VALIDATE = 2, LEAN_COHERENCE = 3, LEAN_WRITEBACK = 4 };


  template <int SELT>
  HXN void sim_lean() {
    const int P = PB.P;
    Small& W = SM();
    const int nl = nleaves;
#if defined(__CUDACC__)
    if constexpr (WP::W > 1) {  // SMEM-staging experiment: the valid-time table in shared memory when it fits
      W.vstage = (W.vst_cap > 0 && nblocks * PB.S <= W.vst_cap) ? W.vst_base : nullptr;
      wp.sync();
    }
#endif
    // init_memory (sim.cpp:323-339): every block valid in main at t=0
    NOUNROLL for (int x = wp.lane(); x < nblocks; x += WP::W) {
      NOUNROLL for (int q = 0; q < n_sp(); ++q) V(x, q) = q == msp() ? 0.0 : ABSENT;
      wrt()[x] = 0;
    }
    wp.sync();
    if (bbytes(0) > PB.cap[msp()]) return fail(ST_CAPACITY);  // the root materialised in main (sim.cpp:335-336)
    if (PB.ordering == ORD_PL) build_ct();
    if (status) return;
    // initial pool: leaves without predecessors, release 0
    int pool_n = 0;
    NOUNROLL for (int base = 0; base < nl; base += WP::W) {
      const int li = base + wp.lane();
      bool z = false;
      int j = -1;
      double key = 0.0;
      if (li < nl) {
        j = leaf()[li];
        TState& st_ = ts()[j];
        st_.rel = 0.0;
        z = st_.missing == 0;
        key = PB.ordering == ORD_PL ? st_.ct : 0.0;
      }
      const unsigned m = wp.ballot(z);
      if (z) {
        const int at = pool_n + popc32(m & wp.lt());
        pool()[at] = j;
        pool_rel()[at] = 0.0;
        pool_key()[at] = key;
      }
      pool_n += popc32(m);
    }
    NOUNROLL for (int q = wp.lane(); q < MAXP; q += WP::W) {
      W.proc_free[q] = 0.0;
      W.ptype[q] = q < P ? PB.proc_type[q] : 0;
      W.pspace[q] = q < P ? PB.proc_space[q] : 0;
    }
    NOUNROLL for (int i = wp.lane(); i < MAXL; i += WP::W) W.link_free[i] = 0.0;
    wp.sync();
    W.ah = 0;
    W.xh = 0;
    W.L.tnow = 0.0;
    W.L.mk = 0.0;
    W.L.pmin = 0.0;
    W.L.pool_n = pool_n;
    W.L.committed = 0;
    W.L.done = 0;
    W.L.nr = 0;
    W.L.first = 1;
    W.L.phase = 0;
    rng = PB.sched_seed;
    wp.sync();
    // driver: run the hot loop; serve its cold requests with the member paths
    NOUNROLL for (;;) {
      const int op = lean_run<SELT>();
      if (op == LEAN_DONE) break;
      wp.sync();
      now = W.L.tnow;
      const int b = W.L.op_b, s = W.L.op_s;
      const double at = W.L.op_at, at2 = W.L.op_at2;
      if (op == LEAN_GATHER) {
        const double r = gather(b, s);
        wp.sync();
        W.L.op_result = r;
      } else if (op == LEAN_VALIDATE) {
        validate_from(b, s, at);
      } else if (op == LEAN_COHERENCE) {
        invalidate_elsewhere(b, s, at);
        validate_from(b, s, at2);
      } else {
        write_back(b, s, at);
      }
      wp.sync();
      if (status) return;
    }
    if (status) return;
    wp.sync();
    makespan = W.L.mk;
    ahash += W.ah;
    xhash += W.xh;
  }

  // The hot loop.  Returns LEAN_DONE (finished or failed: `status`) or a cold
  // request in W.L (op, op_b, op_s, op_at, op_at2) with the loop state saved.
  template <int SELT>
  HX int lean_run() {
    const int P = PB.P;
    uint8_t* const sl = slot;
#define LA(type, field) ((type*)(sl + PB.lay.field))
#define LV(b, q) (vbase_[(b) * PB.S + (q)])
#define LS PB.S
#define LMS PB.main_space
#define LPL (PB.ordering == ORD_PL)
    constexpr bool waits = (SELT == SEL_RP || SELT == SEL_FP);
    Small& W = SM();
    double* const vbase_ = (WP::W > 1 && W.vstage) ? W.vstage : LA(double, valid);
    const int nl = nleaves;
    double tnow = W.L.tnow, mk = W.L.mk, pmin = W.L.pmin;
    int pool_n = W.L.pool_n, committed = W.L.committed, done = W.L.done, nr = W.L.nr;
    bool first = W.L.first != 0;
    int phase = W.L.phase;
#if defined(__CUDACC__)
    const int lk = wp.lane() / LS, lq = wp.lane() - (wp.lane() / LS) * LS;  // lane = (block k, space q)
#else
    const int lk = 0, lq = 0;
#endif
    (void)lk;
    (void)lq;
    int st = 0;
    // block regions through the local slot base, never through `this`
    auto lreg = [&](int b) -> Region {
      return b < n_bb() ? bb_()[b].r : LA(const BlockMeta, bm)[b - n_bb()].r;
    };
    auto ltile = [&](int b) -> int {
      return b < n_bb() ? bb_()[b].tile : LA(const BlockMeta, bm)[b - n_bb()].tile;
    };
    // leave the loop: state into W.L (uniform stores), then a cold request
    auto save = [&]() {
      W.L.tnow = tnow;
      W.L.mk = mk;
      W.L.pmin = pmin;
      W.L.pool_n = pool_n;
      W.L.committed = committed;
      W.L.done = done;
      W.L.nr = nr;
      W.L.first = first ? 1 : 0;
    };
    auto request = [&](int op, int b, int s, double at, double at2) -> int {
      save();
      W.L.op = op;
      W.L.op_b = b;
      W.L.op_s = s;
      W.L.op_at = at;
      W.L.op_at2 = at2;
      wp.sync();
      return op;
    };
    auto failed = [&](int code) -> int {
      fail(code);
      return LEAN_DONE;
    };
    // plan_transfer (sim.cpp:468-499) on the warp's link clocks
    auto xfer = [&](int blk, long long nbytes, int bi, int src, int dst, double data_ready) -> double {
      const int nh = PB.route_n[src * MAXS + dst];
      if (nh == 0) {
        st = ST_NO_ROUTE;
        return 0.0;
      }
      double rdy = dmax(data_ready, tnow), start0 = 0.0;
      NOUNROLL for (int h = 0; h < nh; ++h) {
        const int l = PB.route_l[src * MAXS + dst][h];
        const double s0 = dmax(W.link_free[l], rdy);
        const double en = s0 + PB.link_lat[l] + PB.hopq[l][bi];  // (s0 + lat) + bytes/bw
        W.link_free[l] = en;
        rdy = en;
        if (h == 0) start0 = s0;
      }
      if (!(rdy > tnow)) st = ST_ENGINE_INVARIANT;
      // one lane folds the term: a read-modify-write of shared state by every
      // lane is only safe while the warp stays converged
      const uint64_t xt_ = hesp_xfer_term(xblock(blk), src, dst, nbytes, dbits(start0), dbits(rdy), 0, 0, 0, 0);
      HASH_FOLD(W.xh, xt_);
      return rdy;
    };
    // validate_from (sim.cpp:452-461), b != 0: b and every block inside it
    auto validate = [&](int b, int s, double at, bool simple) {
      if (simple) {
        double& v = LV(b, s);
        if (v > at) v = at;
        return;
      }
      const int t = ltile(b);
      const Region rb = lreg(b);
      const int cnt = 2 + LA(const int, tl_cnt)[t];
      const int head = LA(const int, tl_head)[t];
      NOUNROLL for (int k = wp.lane(); k < cnt; k += WP::W) {
        const int x = k == 0 ? 0 : (k == 1 ? t : LA(const int, tl_ids)[head + k - 2]);
        if (x == b || (x != 0 && x != t && rcontains(rb, lreg(x)))) {
          double& v = LV(x, s);
          if (v > at) v = at;
        }
      }
      wp.sync();
    };

    NOUNROLL for (;;) {
      if (phase == 0 && done >= nr) {
        if (committed >= nl) {
          save();
          return LEAN_DONE;
        }
        // ---------------- epoch (E3) and ready set (sim.cpp:742-752) ----------------
        nr = 0;
        done = 0;
        if (!waits) {
          // every ready task commits in its epoch: ready = pool entries at the
          // pool minimum; the remaining entries' minimum is the next epoch
          if (!first && pool_n == 0) return failed(ST_INTERNAL);  // scheduler stalled
          tnow = first ? 0.0 : pmin;
          double nmin = ABSENT;
          int keep = 0;
          NOUNROLL for (int base = 0; base < pool_n; base += WP::W) {
            const int k = base + wp.lane();
            bool r = false, kp = false;
            int j = -1;
            double rl = 0.0, key = 0.0;
            if (k < pool_n) {
              j = LA(const int, pool)[k];
              rl = LA(const double, pool_rel)[k];
              key = LA(const double, pool_key)[k];
              r = rl <= tnow;
              kp = !r;
              if (kp && rl < nmin) nmin = rl;
            }
            const unsigned m = wp.ballot(r), mk2 = wp.ballot(kp);
            if (r) {
              const int at = nr + popc32(m & wp.lt());
              LA(int, gs_a)[at] = j;
              LA(double, ready_key)[at] = key;
            }
            if (kp) {
              const int at = keep + popc32(mk2 & wp.lt());
              LA(int, pool)[at] = j;
              LA(double, pool_rel)[at] = rl;
              LA(double, pool_key)[at] = key;
            }
            nr += popc32(m);
            keep += popc32(mk2);
            wp.sync();
          }
          pmin = wp.mind(nmin);  // ABSENT when nothing stays behind
          pool_n = keep;
        } else {
          if (!first) {
            double nx = ABSENT;
            NOUNROLL for (int k = wp.lane(); k < pool_n; k += WP::W) {
              const double r = LA(const double, pool_rel)[k];
              if (r > tnow && r < nx) nx = r;
            }
            NOUNROLL for (int q = wp.lane(); q < P; q += WP::W) {
              const double f = W.proc_free[q];
              if (f > tnow && f < nx) nx = f;
            }
            nx = wp.mind(nx);
            if (nx == ABSENT) return failed(ST_INTERNAL);
            tnow = nx;
          }
          int keep = 0;
          NOUNROLL for (int base = 0; base < pool_n; base += WP::W) {
            const int k = base + wp.lane();
            bool r = false, kp = false;
            int j = -1;
            double rl = 0.0, key = 0.0;
            if (k < pool_n) {
              j = LA(const int, pool)[k];
              rl = LA(const double, pool_rel)[k];
              key = LA(const double, pool_key)[k];
              r = rl <= tnow;
              kp = !r;
            }
            const unsigned m = wp.ballot(r), mk2 = wp.ballot(kp);
            if (r) {
              const int at = nr + popc32(m & wp.lt());
              LA(int, gs_a)[at] = j;
              LA(double, ready_key)[at] = key;
            }
            if (kp) {
              const int at = keep + popc32(mk2 & wp.lt());
              LA(int, pool)[at] = j;
              LA(double, pool_rel)[at] = rl;
              LA(double, pool_key)[at] = key;
            }
            nr += popc32(m);
            keep += popc32(mk2);
            wp.sync();
          }
          pool_n = keep;
        }
        first = false;
        if (nr == 0) continue;
        // order_ready (sim.cpp:117-134): FCFS (release asc, id asc) / PL (ct desc, id asc)
        if (nr == 1) {
          LA(int, ready)[0] = LA(const int, gs_a)[0];
        } else {
          NOUNROLL for (int k = wp.lane(); k < nr; k += WP::W) {
            const int a = LA(const int, gs_a)[k];
            const double ka = LA(const double, ready_key)[k];
            int rank = 0;
            NOUNROLL for (int q = 0; q < nr; ++q) {
              const int c = LA(const int, gs_a)[q];
              const double kc = LA(const double, ready_key)[q];
              rank += (kc != ka) ? (LPL ? kc > ka : kc < ka) : (c < a);
            }
            LA(int, ready)[rank] = a;
          }
        }
        wp.sync();
      }
      // ---------------- one ready task ----------------
      const int j = LA(const int, ready)[done];
      const STask tk = ld_stask(LA(const STask, wsb) + j);
      const TState tj = ld_tstate(LA(const TState, ts) + j);  // j's own record: no commit writes it before j's release
      const int tkind = tk.kb & 0xff, tbidx = tk.kb >> 8;
      const int nw = tk.nw;
      const long long tbytes = (long long)tk.b * tk.b * PB.elem;  // every block of a task has its side
      int p = -1, s = 0, k0 = 0;
      double inputs = 0.0, start = 0.0, end = 0.0;
      if (phase != 0) {  // resuming after a cold step
        p = W.L.r_p;
        s = W.L.r_s;
        start = W.L.r_start;
        end = W.L.r_end;
        if (phase == 1) {
          k0 = W.L.r_k + 1;
          inputs = W.L.r_inputs;
          if (W.L.op == LEAN_GATHER) inputs = dmax(inputs, W.L.op_result);
        }
      } else {
        const double rel = tj.rel;
        // ---------------- select_processor (sim.cpp:136-192) ----------------
        if (waits) {
          unsigned idle_mask = 0;
          NOUNROLL for (int q = wp.lane(); q < P; q += WP::W)
            if (W.proc_free[q] <= tnow) idle_mask |= 1u << q;
#if defined(__CUDACC__)
          if constexpr (WP::W > 1) idle_mask = __reduce_or_sync(0xffffffffu, idle_mask);
#endif
          if (idle_mask == 0) {  // R-P/F-P wait for a processor (sim.cpp:800-801): the rest return to the pool
            NOUNROLL for (int k = done + wp.lane(); k < nr; k += WP::W) {
              const int jj = LA(const int, ready)[k];
              const int at = pool_n + (k - done);
              const TState tt = LA(const TState, ts)[jj];
              LA(int, pool)[at] = jj;
              LA(double, pool_rel)[at] = tt.rel;
              LA(double, pool_key)[at] = LPL ? tt.ct : tt.rel;
            }
            wp.sync();
            pool_n += nr - done;
            done = nr;
            continue;
          }
          if (SELT == SEL_RP) {
            const int n = popc32(idle_mask);
            const double u = (double)(rng_next() >> 11) * 0x1.0p-53;
            const int k = (int)((unsigned long long)(u * (double)n) % (unsigned long long)n);
            unsigned mmm = idle_mask;
            for (int q = 0; q < k; ++q) mmm &= mmm - 1;
            p = ctz32(mmm);
          } else {  // F-P: fastest idle processor, lowest id
            double a = ABSENT, b2 = 0.0;
            int id = -1;
            NOUNROLL for (int q = wp.lane(); q < P; q += WP::W) {
              if (!((idle_mask >> q) & 1u)) continue;
              const double tt = PB.ttime[tkind][tbidx][W.ptype[q]];
              if (id < 0 || tt < a) {
                a = tt;
                id = q;
              }
            }
            wp.argmin_lane(a, b2, id);
            p = id;
          }
        } else if (SELT == SEL_EFTP && WP::W == 1) {
          // width 1: the reference's loop, space by space, then processor by processor
          bool noroute = false;
          double est[MAXS];
          const int w[3] = {tk.ws0, tk.ws1, tk.ws2};
          NOUNROLL for (int sp = 0; sp < LS; ++sp) {
            double est_ = 0.0;
            int al[6] = {-1, -1, -1, -1, -1, -1};
            double av[6] = {0, 0, 0, 0, 0, 0};
            NOUNROLL for (int k = 0; k < nw; ++k) {
              const int b = w[k];
              const double v = LV(b, sp);
              if (v != ABSENT) {
                est_ = dmax(est_, v);
                continue;
              }
              int src = -1;
              if (LMS != sp && LV(b, LMS) != ABSENT) src = LMS;
              else
                NOUNROLL for (int q = 0; q < LS; ++q)
                  if (q != LMS && q != sp && LV(b, q) != ABSENT) {
                    src = q;
                    break;
                  }
              if (src < 0) continue;
              const int nh = PB.route_n[src * MAXS + sp];
              if (nh == 0) {
                noroute = true;
                continue;
              }
              double tarr = dmax(tnow, LV(b, src));
              NOUNROLL for (int h = 0; h < nh; ++h) {
                const int l = PB.route_l[src * MAXS + sp][h];
                const double hop = PB.link_lat[l] + (double)tbytes / PB.link_bw[l];
                double acc = 0.0;
                bool placed = false;
                for (int z = 0; z < 6; ++z) {
                  if (!placed && (al[z] == l || al[z] < 0)) {
                    al[z] = l;
                    av[z] += hop;
                    acc = av[z];
                    placed = true;
                  }
                }
                tarr += acc;
              }
              est_ = dmax(est_, tarr);
            }
            est[sp] = est_;
          }
          if (noroute) return failed(ST_NO_ROUTE);
          double a = ABSENT, b2 = 0.0;
          NOUNROLL for (int q = 0; q < P; ++q) {
            const double nf = W.proc_free[q];
            const double qa = dmax(dmax(nf, rel), est[W.pspace[q]]) + PB.ttime[tkind][tbidx][W.ptype[q]];
            if (p < 0 || qa < a || (qa == a && nf < b2)) {
              a = qa;
              b2 = nf;
              p = q;
            }
          }
        } else {
          double est_own = 0.0;  // EFT estimate of the lane's processor's space
#if defined(__CUDACC__)
          if (SELT == SEL_EFTP && WP::W > 1) {
            // est_transfer_ready (sim.cpp:762-793), lane (k, sp): one round
            // loads every V(b_k, sp); ballots give each block's valid-space
            // mask; the reference's ordered per-link accumulators are rebuilt
            // from the (<= 2) earlier blocks of the same space by shuffles;
            // a segmented max gives the estimate per space
            const unsigned FULL = 0xffffffffu;
            const int lane = wp.lane();
            const int Sx = LS;
            const int k = lk, sp = lq;
            const bool act = k < nw;
            const int b = k == 0 ? tk.ws0 : (k == 1 ? tk.ws1 : tk.ws2);
            const double v = act ? LV(b, sp) : ABSENT;
            const unsigned vm = __ballot_sync(FULL, act && v != ABSENT);
            const unsigned mymask = act ? (vm >> (k * Sx)) & ((1u << Sx) - 1u) : 0u;
            int src = -1;
            if (act && v == ABSENT) {
              if (LMS != sp && ((mymask >> LMS) & 1u)) {
                src = LMS;
              } else {
                const unsigned o = mymask & ~(1u << LMS) & ~(1u << sp);
                if (o) src = ctz32(o);
              }
            }
            const double vsrc = __shfl_sync(FULL, v, src >= 0 ? k * Sx + src : lane);
            int l0 = -1, l1 = -1, nh = 0;
            double c0 = 0.0, c1 = 0.0;
            if (src >= 0) {
              nh = PB.route_n[src * MAXS + sp];
              if (nh >= 1) {
                l0 = PB.route_l[src * MAXS + sp][0];
                c0 = PB.hopc[l0][tbidx];
              }
              if (nh >= 2) {
                l1 = PB.route_l[src * MAXS + sp][1];
                c1 = PB.hopc[l1][tbidx];
              }
            }
            if (__any_sync(FULL, src >= 0 && nh == 0)) return failed(ST_NO_ROUTE);
            double acc0 = 0.0, acc1 = 0.0;
            const int rounds = __any_sync(FULL, src >= 0) ? nw - 1 : 0;
#pragma unroll
            for (int kp = 0; kp < 2; ++kp) {
              if (kp >= rounds) break;
              const int from = kp * Sx + sp < 32 ? kp * Sx + sp : lane;
              const int pl0 = __shfl_sync(FULL, l0, from), pl1 = __shfl_sync(FULL, l1, from);
              const double pc0 = __shfl_sync(FULL, c0, from), pc1 = __shfl_sync(FULL, c1, from);
              if (kp < k) {
                if (l0 >= 0 && pl0 == l0) acc0 += pc0;
                if (l0 >= 0 && pl1 == l0) acc0 += pc1;
                if (l1 >= 0 && pl0 == l1) acc1 += pc0;
                if (l1 >= 0 && pl1 == l1) acc1 += pc1;
              }
            }
            double val = 0.0;
            if (act) {
              if (v != ABSENT) {
                val = v;
              } else if (src >= 0) {
                double tarr = dmax(tnow, vsrc);
                acc0 += c0;
                tarr += acc0;
                if (nh == 2) {
                  acc1 += c1;
                  tarr += acc1;
                }
                val = tarr;
              }
            }
            double e = val;
#pragma unroll
            for (int kp = 1; kp < 3; ++kp) {
              const int from = kp * Sx + lane < 32 ? kp * Sx + lane : lane;
              const double o = __shfl_sync(FULL, val, from);
              if (lane < Sx && kp < nw) e = dmax(e, o);
            }
            est_own = __shfl_sync(FULL, e, W.pspace[lane]);
          }
#endif
          double a = ABSENT, b2 = 0.0;
          int id = -1;
          NOUNROLL for (int q = wp.lane(); q < P; q += WP::W) {
            const double nf = W.proc_free[q];
            double qa, qb = 0.0;
            if (SELT == SEL_EFTP) {
              qa = dmax(dmax(nf, rel), est_own) + PB.ttime[tkind][tbidx][W.ptype[q]];
              qb = nf;
            } else {
              qa = nf;  // EIT-P
            }
            if (id < 0 || qa < a || (qa == a && qb < b2)) {
              a = qa;
              b2 = qb;
              id = q;
            }
          }
          wp.argmin_lane(a, b2, id);
          p = id;
        }
        if (p < 0) return failed(ST_NO_PROCESSORS);
        s = W.pspace[p];
      }
      // ---------------- commit (sim.cpp:592-668) ----------------
      if (phase <= 1) {
        // acquire the working set in id order (std::set iteration, sim.cpp:597-611)
#if defined(__CUDACC__)
        if (WP::W > 1 && (tk.pad & 16)) {
          const unsigned FULL = 0xffffffffu;
          const bool act = lk >= k0 && lk < nw;
          const int b = lk == 0 ? tk.ws0 : (lk == 1 ? tk.ws1 : tk.ws2);
          const double v = act ? LV(b, lq) : ABSENT;
          const unsigned vm = __ballot_sync(FULL, act && v != ABSENT);
          NOUNROLL for (int k = k0; k < nw; ++k) {
            const unsigned msk = (vm >> (k * LS)) & ((1u << LS) - 1u);
            const double vk = __shfl_sync(FULL, v, k * LS + s);
            if ((msk >> s) & 1u) {
              inputs = dmax(inputs, vk);
              continue;
            }
            const int bk = k == 0 ? tk.ws0 : (k == 1 ? tk.ws1 : tk.ws2);
            int src = -1;
            if (LMS != s && ((msk >> LMS) & 1u)) {
              src = LMS;
            } else {
              const unsigned o = msk & ~(1u << LMS) & ~(1u << s);
              if (o) src = ctz32(o);
            }
            W.L.r_k = k;
            W.L.r_p = p;
            W.L.r_s = s;
            W.L.phase = 1;
            if (src < 0) {
              W.L.r_inputs = inputs;
              return request(LEAN_GATHER, bk, s, 0.0, 0.0);  // assemble from pieces (sim.cpp:521-572)
            }
            const double vs = __shfl_sync(FULL, v, k * LS + src);
            const double arr = xfer(bk, tbytes, tbidx, src, s, vs);
            if (st) return failed(st);
            inputs = dmax(inputs, arr);
            if (bk == 0) {
              W.L.r_inputs = inputs;
              return request(LEAN_VALIDATE, bk, s, arr, 0.0);
            }
            validate(bk, s, arr, (tk.pad >> k) & 1);
          }
        } else
#endif
        {
          NOUNROLL for (int k = k0; k < nw; ++k) {
            const int bk = k == 0 ? tk.ws0 : (k == 1 ? tk.ws1 : tk.ws2);
            const double v = LV(bk, s);
            if (v != ABSENT) {
              inputs = dmax(inputs, v);
              continue;
            }
            int src = -1;
            if (LMS != s && LV(bk, LMS) != ABSENT) src = LMS;
            else
              NOUNROLL for (int q = 0; q < LS; ++q)
                if (q != LMS && q != s && LV(bk, q) != ABSENT) {
                  src = q;
                  break;
                }
            W.L.r_k = k;
            W.L.r_p = p;
            W.L.r_s = s;
            W.L.phase = 1;
            if (src < 0) {
              W.L.r_inputs = inputs;
              return request(LEAN_GATHER, bk, s, 0.0, 0.0);
            }
            const double arr = xfer(bk, tbytes, tbidx, src, s, LV(bk, src));
            if (st) return failed(st);
            inputs = dmax(inputs, arr);
            if (bk == 0) {
              W.L.r_inputs = inputs;
              return request(LEAN_VALIDATE, bk, s, arr, 0.0);
            }
            validate(bk, s, arr, (tk.pad >> k) & 1);
          }
        }
        const double rel = tj.rel;
        start = dmax(dmax(W.proc_free[p], rel), inputs);
        end = start + PB.ttime[tkind][tbidx][W.ptype[p]];
        if (!(end > tnow) || start < tnow) return failed(ST_ENGINE_INVARIANT);
        W.proc_free[p] = end;
        {
          const uint64_t at_ = hesp_assign_term(xtask(j), p, dbits(start), dbits(end));
          HASH_FOLD(W.ah, at_);
        }
        mk = dmax(mk, end);
        // write coherence (sim.cpp:625-628): invalidate the cone elsewhere,
        // validate out and the blocks inside it here, valid[out] = end
        const int out = tk.out;
        if (tk.pad & 8) {  // unsubdivided tile: cone = {root, tile}, nothing inside
          NOUNROLL for (int q = wp.lane(); q < LS; q += WP::W)
            if (q != s) {
              LV(0, q) = ABSENT;
              LV(out, q) = ABSENT;
            }
          wp.sync();
        } else if (tk.pad & 32) {  // the root, or partial overlaps in the tile: the general scans
          W.L.r_p = p;
          W.L.r_s = s;
          W.L.r_start = start;
          W.L.r_end = end;
          W.L.phase = 2;
          return request(LEAN_COHERENCE, out, s, start, end);
        } else {
          const int t = ltile(out);
          const Region rb = lreg(out);
          const int cnt = 2 + LA(const int, tl_cnt)[t];
          const int head = LA(const int, tl_head)[t];
          NOUNROLL for (int k = wp.lane(); k < cnt; k += WP::W) {
            const int x = k == 0 ? 0 : (k == 1 ? t : LA(const int, tl_ids)[head + k - 2]);
            const Region rx = lreg(x);
            const bool inside_ = rcontains(rb, rx);
            if (inside_ || rcontains(rx, rb)) {
              NOUNROLL for (int q = 0; q < LS; ++q)
                if (q != s) LV(x, q) = ABSENT;
            }
            if (inside_ && x != 0 && x != t) {
              double& v = LV(x, s);
              if (v > end) v = end;
            }
          }
          wp.sync();
        }
      }
      if (phase <= 2) {
        const int out = tk.out;
        LV(out, s) = end;
        LA(uint8_t, wrt)[out] = 1;  // written since t=0 (gather's coherence check)
        if (s != LMS && PB.caching != CACHE_WB) {  // WT / WA (sim.cpp:631-656); the headline policy is WB
          W.L.r_p = p;
          W.L.r_s = s;
          W.L.r_start = start;
          W.L.r_end = end;
          W.L.phase = 3;
          return request(LEAN_WRITEBACK, out, s, end, 0.0);
        }
      }
      phase = 0;
      W.L.phase = 0;
      // release successors (sim.cpp:660-667): running max of predecessor
      // ends; released tasks enter the pool with release time and key
      {
        int added = 0;
        double amin = ABSENT;
        NOUNROLL for (int base = 0; base < tj.scnt; base += WP::W) {
          const int q = base + wp.lane();
          bool rl = false;
          int sj = -1;
          double r = 0.0, key = 0.0;
          if (q < tj.scnt) {
            sj = LA(const int, succs)[tj.soff + q];
            TState& ts_ = LA(TState, ts)[sj];
            const int left = --ts_.missing;
            r = dmax(ts_.rel, end);
            ts_.rel = r;
            rl = left == 0;
            if (rl) {
              key = LPL ? ts_.ct : r;
              if (r < amin) amin = r;
            }
          }
          const unsigned m = wp.ballot(rl);
          if (rl) {
            const int at = pool_n + added + popc32(m & wp.lt());
            LA(int, pool)[at] = sj;
            LA(double, pool_rel)[at] = r;
            LA(double, pool_key)[at] = key;
          }
          added += popc32(m);
        }
        if (!waits && added) pmin = dmin(pmin, wp.mind(amin));
        wp.sync();
        pool_n += added;
      }
      ++committed;
      ++done;
    }
#undef LA
#undef LV
#undef LS
#undef LMS
#undef LPL
  }

  // =========================================================================
  // One candidate, end to end
  // =========================================================================

  // The warp's view of top-level tiling `til` with reference-id offsets.
  HX void set_view(int til, int off_t, int off_b, int off_c) {
    const BaseTiling& T = PB.til[til];
    BaseView& v = BV();
    v.nbt = T.n_tasks;
    v.nbb = T.n_blocks;
    v.til = til;
    v.pad = 0;
    v.base_b = T.base_b;
    v.bt = T.tasks;
    v.bb = T.blocks;
    v.bp = T.preds;
    v.bpl = T.plist;
    v.off_t = off_t;
    v.off_b = off_b;
    v.off_c = off_c;
    v.pad2 = 0;
    wp.sync();
  }

  // Starts from a top-level tiling (root + its cluster, shared tables); the
  // workload's base tiling with reference ids unshifted by default.
  HXN void reset_to_base(int til = TIL_BASE, int off_t = 0, int off_b = 0, int off_c = 0) {
    set_view(til, off_t, off_b, off_c);
    NOUNROLL for (int i = wp.lane(); i < n_bb(); i += WP::W) tmis()[i] = 0;
    NOUNROLL for (int i = wp.lane(); i < RHT / 2; i += WP::W) ((uint32_t*)rht())[i] = 0xffffffffu;
    wp.sync();
    status = 0;
    ntasks = n_bt();
    nblocks = n_bb();
    npart = 0;
    NXP() = 0;
    makespan = 0.0;
    ahash = xhash = 0;
    if (n_bt() > 1) {  // the top op partitioned the root into tasks 1..n_bt()-1
      if (wp.lane() == 0) {
        part()[0].task = 0;
        part()[0].child0 = 1;
        part()[0].nchild = n_bt() - 1;
        part()[0].leaves = 0;
      }
      wp.sync();
      npart = 1;
    }
  }

  // One descriptor op in reference ids (partition_task / merge_cluster).
  HX void apply_ext(const hesp_op& o) {
    const BaseView& v = BV();
    if (o.s == HESP_OP_MERGE) {
      if (o.task < v.off_c) return fail(ST_UNKNOWN_CLUSTER);  // merged with an earlier top cluster
      return apply_merge(o.task - v.off_c);
    }
    if (o.task != 0 && o.task <= v.off_t) return fail(ST_VALIDATION);  // merged away: unknown task
    apply_op(o.task == 0 ? 0 : o.task - v.off_t, o.s);
  }

  // Build phase: base tiling + ops -> leaves, dependences; state left in the slot.
  HXN void build(const hesp_cand_desc& d) {
    reset_to_base();
    if (d.n_ops < 0 || d.n_ops > HESP_MAX_OPS) fail(ST_ENGINE_LIMIT);  // never read past ops[]
    NOUNROLL for (int k = 0; k < d.n_ops && !status; ++k) apply_ext(d.ops[k]);
    finish_build();
  }

  // Neighbour evaluation (hesp_eval_neighbors): a base state's op sequence is
  // applied once into a template slot (build_template); each neighbour copies
  // the template's graph arrays and applies only its own extra ops.  Same
  // ids, blocks and hash-table contents as replaying every op.
  HXN void build_template(const hesp_cand_desc& d) {
    reset_to_base();
    if (d.n_ops < 0 || d.n_ops > HESP_MAX_OPS) fail(ST_ENGINE_LIMIT);
    NOUNROLL for (int k = 0; k < d.n_ops && !status; ++k) apply_ext(d.ops[k]);
    if (wp.lane() == 0) {
      SlotHeader h{};
      h.status = status;
      h.ntasks = ntasks;
      h.nblocks = nblocks;
      h.npart = npart;
      h.nxp = NXP();
      put_view(h);
      *hdr() = h;
    }
    wp.sync();
  }
  HX void put_view(SlotHeader& h) const {
    const BaseView& v = BV();
    h.til = v.til;
    h.off_t = v.off_t;
    h.off_b = v.off_b;
    h.off_c = v.off_c;
  }
  HXN void build_neighbor(const uint8_t* tslot, int n_extra, const hesp_op* extra) {
    const SlotHeader th = *(const SlotHeader*)(tslot + PB.lay.hdr);
    set_view(th.til, th.off_t, th.off_b, th.off_c);
    auto copy = [&](size_t off, size_t bytes) {  // 4-byte words, lane-strided
      const uint32_t* src = (const uint32_t*)(tslot + off);
      uint32_t* dst = (uint32_t*)(slot + off);
      NOUNROLL for (size_t i = wp.lane(); i < bytes / 4; i += WP::W) dst[i] = src[i];
    };
    const int nt = th.ntasks - n_bt(), nb = th.nblocks - n_bb();
    copy(PB.lay.tm, sizeof(TaskMeta) * (size_t)(nt > 0 ? nt : 0));
    copy(PB.lay.bm, sizeof(BlockMeta) * (size_t)(nb > 0 ? nb : 0));
    copy(PB.lay.bref, 4 * (size_t)(nb > 0 ? nb : 0));
    copy(PB.lay.xpar, 4 * (size_t)XPAR * (size_t)(nb > 0 ? nb : 0));
    copy(PB.lay.rht, 2 * (size_t)RHT);
    copy(PB.lay.part, sizeof(PartEntry) * (size_t)th.npart);
    copy(PB.lay.tmis, ((size_t)n_bb() + 3) & ~(size_t)3);
    wp.sync();
    status = th.status;
    ntasks = th.ntasks;
    nblocks = th.nblocks;
    npart = th.npart;
    NXP() = th.nxp;
    makespan = 0.0;
    ahash = xhash = 0;
    NOUNROLL for (int k = 0; k < n_extra && !status; ++k) apply_ext(extra[k]);
    finish_build();
  }

  HXN void finish_build() {
    sum_k = 0;
    nleaves = 0;
    nedges = 0;
    if (!status) build_tiles();
    if (!status) build_order();
    const int n_out = status ? 0 : nleaves;
    if (!status) build_cells();
    if (!status) build_deps();
    if (wp.lane() == 0) {
      SlotHeader h{};
      h.status = status;
      h.ntasks = ntasks;
      h.nblocks = nblocks;
      h.nleaves = nleaves;
      h.nedges = nedges;
      h.sum_k = sum_k;
      h.n_leaves_out = n_out;
      h.npart = npart;
      h.nxp = NXP();
      put_view(h);
      *hdr() = h;
    }
    wp.sync();
  }

  // Simulate phase on a slot left by build().
  HXN Outcome sim_slot() {
    const SlotHeader h = *hdr();
    set_view(h.til, h.off_t, h.off_b, h.off_c);
    status = h.status;
    ntasks = h.ntasks;
    nblocks = h.nblocks;
    nleaves = h.nleaves;
    nedges = h.nedges;
    sum_k = h.sum_k;
    makespan = 0.0;
    ahash = xhash = 0;
    if (!status) simulate();
    Outcome o;
    o.n_leaves = h.n_leaves_out;
    o.status = status;
    o.makespan = status ? 0.0 : makespan;
    o.assign_hash = status ? 0 : ahash;
    o.xfer_hash = status ? 0 : xhash;
    o.sum_k = sum_k;
    o.n_edges = nedges;
    return o;
  }

  HXN Outcome run(const hesp_cand_desc& d) {
    build(d);
    if constexpr (TRACE) export_graph();
    return sim_slot();
  }

  // Trace mode: the candidate's leaves (program order), their reads/writes,
  // predecessor lists and every block's region, for verify_schedule.
  HXN void export_graph() {
    if (!tb || status) return;
    const int nl = nleaves, nb = nblocks;
    if (nl > tb->leaf_cap || nb > tb->block_cap) {
      if (wp.lane() == 0) tb->overflow = 1;
      wp.sync();
      return;
    }
    int np = 0;
    NOUNROLL for (int li = 0; li < nl; ++li) np += t_pcnt()[leaf()[li]];
    if (np > tb->pred_cap) {
      if (wp.lane() == 0) tb->overflow = 1;
      wp.sync();
      return;
    }
    int off = 0;
    NOUNROLL for (int li = 0; li < nl; ++li) {
      const int j = leaf()[li];
      const int cnt = t_pcnt()[j];
      const int32_t* pl_ = pred_list(j);
      NOUNROLL for (int q = wp.lane(); q < cnt; q += WP::W) tb->lpreds[off + q] = pl_[q];
      if (wp.lane() == 0) {
        tb->leaves[li] = j;
        tb->lmeta[li] = task(j);
        tb->lpoff[li] = off;
        tb->lpcnt[li] = cnt;
      }
      off += cnt;
    }
    NOUNROLL for (int b = wp.lane(); b < nb; b += WP::W) {
      tb->bregion[b] = reg(b);
      tb->bisint[b] = bmeta(b).isint;
    }
    NOUNROLL for (int c = wp.lane(); c < npart; c += WP::W) tb->parts[c] = part()[c];
    if (ntasks <= tb->task_cap)
      NOUNROLL for (int j = wp.lane(); j < ntasks; j += WP::W) tb->tmeta[j] = task(j);
    if (wp.lane() == 0) {
      tb->off_t = BV().off_t;
      tb->off_b = BV().off_b;
      tb->off_c = BV().off_c;
      tb->nleaves = nl;
      tb->npreds = np;
      tb->nblocks = nb;
      tb->nparts = npart;
      tb->ntasks = ntasks;
      if (ntasks > tb->task_cap) tb->overflow = 1;
    }
    wp.sync();
  }
};

}  // namespace hx
