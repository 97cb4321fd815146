// engine_kernels.cu — sm_100a kernels and the C ABI (include/hesp_engine.h).
//
// K1 per chunk of candidates, two persistent kernels (one warp per candidate,
//    indices pulled from a global atomic counter over a longest-first order:
//    candidates vary ~10x in cost, early CoherenceError vs a full 1.3k-task
//    schedule; order_keys* + a CUB radix sort build the order):
//    build_kernel: generate/load the descriptor, expand the DAG, dependences;
//    sim_kernel:   the event loop, 32-byte outcome, per-warp best.
//    Splitting the phases keeps every resident warp in the same code
//    (instruction-fetch stalls 52% -> ~25%) and lets each phase have its own
//    register budget.  sim_thread_kernel (HESP_SIM_THREAD=1) is the measured
//    thread-per-candidate alternative (profiles/README.md).
// K2 reduce_best: grid-level argmin of (makespan, index) over status == 0.
// K3 hesp_min_reduce: the cross-GPU winner, two int64 MIN all-reduces over
//    the caller's NCCL communicator (NVLink / NVSwitch), NCCL dlopen'ed.
// detail_kernel: one candidate with the full trace (Engine<DevWarp, true>).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "engine.h"
#include "hesp_engine.h"
#include "problem.h"
#include "trace.h"

using namespace hx;

namespace {

thread_local std::string g_last_error;

// Host threads for the per-candidate host loops of the end-to-end path
// (descriptor packing, outcome copy-out): one below 16k candidates, else up
// to 8 (HESP_HOST_THREADS overrides).
int host_threads(uint64_t count) {
  int n = 1;
  if (count >= 16384) {
    const unsigned hc = std::thread::hardware_concurrency();
    n = (int)std::min<unsigned>(8u, hc > 1 ? hc : 1u);
  }
  if (const char* v = getenv("HESP_HOST_THREADS")) n = std::max(1, atoi(v));
  return n;
}

// fn(t, a, b) over nthr contiguous ranges [a, b) of [0, count); range 0 on the caller.
template <class F>
void host_ranges(uint64_t count, int nthr, F&& fn) {
  auto lo = [&](int t) { return count * (uint64_t)t / (uint64_t)nthr; };
  if (nthr <= 1) {
    fn(0, 0, count);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(nthr - 1);
  int t = 1;
  try {
    for (; t < nthr; ++t) th.emplace_back([&fn, &lo, t] { fn(t, lo(t), lo(t + 1)); });
  } catch (...) {  // no thread for range t: the caller runs the remaining ranges itself
  }
  for (int r = t; r < nthr; ++r) fn(r, lo(r), lo(r + 1));
  fn(0, lo(0), lo(1));
  for (auto& x : th) x.join();
}

struct WarpBest {
  double makespan;
  long long index;
  long long n_ok;
  long long n_eval;
  long long leaves, k, edges;
};

constexpr int WARPS_PER_BLOCK = 4;
static_assert(WARPS_PER_BLOCK <= hx::SMALL_WARPS, "one Small per warp");
// Register budgets (min resident CTAs of 4 warps per SM): the build phase
// is latency-bound with a small live set (16 CTAs = 64 warps, 32 regs); the
// event loop keeps ~60 values live and spills below 64 registers.
#ifndef HESP_BUILD_MIN_BLOCKS
#define HESP_BUILD_MIN_BLOCKS 16
#endif
#ifndef HESP_SIM_MIN_BLOCKS
#define HESP_SIM_MIN_BLOCKS 8
#endif

// The problem tables live in constant memory (hx::c_problem, engine.h):
// every access is warp-uniform, so they are broadcast from the constant cache
// instead of occupying L1 next to the per-warp state.

__device__ __noinline__ void generate_desc(unsigned long long index, hesp_cand_desc* d) {
  hesp_generate(&c_problem.gen, (int)(c_problem.n / c_problem.base_b), c_problem.n_base_leaves, c_problem.base_b,
                index, d);
}

// Phase-split evaluation (chunked): every resident warp of a launch runs the
// same phase, so the instruction working set is one phase's code.
__global__ void __launch_bounds__(WARPS_PER_BLOCK * 32, HESP_BUILD_MIN_BLOCKS)
    build_kernel(const hesp_cand_desc* __restrict__ descs, unsigned long long first_index,
                 unsigned long long count, uint8_t* slots, unsigned long long* counter,
                 const uint32_t* __restrict__ order) {
  const int lane = threadIdx.x & 31;
  const Problem& pb = c_problem;
  for (;;) {
    unsigned long long k = 0;
    if (lane == 0) k = atomicAdd(counter, 1ULL);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= count) break;
    if (order) k = order[k];
    uint8_t* slot = slots + (size_t)k * pb.lay.total;
    // The descriptor is read in place (a handful of uniform loads per op);
    // a generated one is written into the slot's gather scratch (unused
    // until the simulate phase).  No shared-memory staging: the build
    // kernel's shared memory stays small, leaving its L1 the larger split.
    const hesp_cand_desc* d = descs ? descs + k : nullptr;
    if (!descs) {
      hesp_cand_desc* g = (hesp_cand_desc*)(slot + pb.lay.gs_reg2);
      if (lane == 0) generate_desc(first_index + k, g);
      __syncwarp();
      d = g;
    }
    Engine<DevWarp> eng(DevWarp{}, pb, slot, nullptr);
    eng.build(*d);
    __syncwarp();
  }
}

// Build-phase cost proxy from the descriptor alone: sum of s^3 over its
// partition ops (the sub-task count of a GEMM split; merges add nothing).
__global__ void order_keys_desc(const hesp_cand_desc* __restrict__ descs, unsigned long long count,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const hesp_cand_desc* d = descs + k;
  const int n = d->n_ops < HESP_MAX_OPS ? d->n_ops : HESP_MAX_OPS;
  uint32_t c = 0;
  for (int i = 0; i < n; ++i) {
    const int s = d->ops[i].s;
    if (s > 1 && s <= 64) c += (uint32_t)(s * s * s);
  }
  keys[k] = c;
  vals[k] = (uint32_t)k;
}

// Longest-processing-time-first order for the simulate kernel: candidates
// vary ~10x in cost, and a persistent kernel's tail is the last long
// candidates; starting the largest expanded DAGs first shrinks it.  Key =
// leaf count (0 for candidates whose build already failed).
__global__ void order_keys(const uint8_t* __restrict__ slots, unsigned long long count, uint32_t* __restrict__ keys,
                           uint32_t* __restrict__ vals) {
  const unsigned long long k = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (k >= count) return;
  const SlotHeader h = *(const SlotHeader*)(slots + k * c_problem.lay.total + c_problem.lay.hdr);
  keys[k] = h.status ? 0u : (uint32_t)h.nleaves;
  vals[k] = (uint32_t)k;
}

__global__ void template_kernel(const hesp_cand_desc* __restrict__ bases, uint8_t* tslots) {
  __shared__ hesp_cand_desc sd;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) sd = bases[b];
  __syncwarp();
  Engine<DevWarp> eng(DevWarp{}, c_problem, tslots + (size_t)b * c_problem.lay.total, nullptr);
  eng.build_template(sd);
}

__global__ void __launch_bounds__(WARPS_PER_BLOCK * 32, HESP_BUILD_MIN_BLOCKS)
    neighbor_build_kernel(const hesp_neighbor* __restrict__ nbrs, const uint8_t* __restrict__ tslots,
                          unsigned long long count, uint8_t* slots, unsigned long long* counter) {
  __shared__ hesp_neighbor snb[WARPS_PER_BLOCK];
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const Problem& pb = c_problem;
  for (;;) {
    unsigned long long k = 0;
    if (lane == 0) k = atomicAdd(counter, 1ULL);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= count) break;
    if (lane < 6) ((int32_t*)&snb[wib])[lane] = ((const int32_t*)(nbrs + k))[lane];
    __syncwarp();
    const hesp_neighbor& nb = snb[wib];
    const int n_ops = nb.n_ops < 0 ? 0 : (nb.n_ops > 2 ? 2 : nb.n_ops);
    Engine<DevWarp> eng(DevWarp{}, pb, slots + (size_t)k * pb.lay.total, nullptr);
    eng.build_neighbor(tslots + (size_t)nb.base * pb.lay.total, n_ops, nb.ops);
    __syncwarp();
  }
}

__global__ void __launch_bounds__(WARPS_PER_BLOCK * 32, HESP_SIM_MIN_BLOCKS)
    sim_kernel(unsigned long long first_index, unsigned long long count, hesp_outcome* __restrict__ out,
               WarpBest* __restrict__ wbest, int accumulate, uint8_t* slots, unsigned long long* counter,
               const uint32_t* __restrict__ order, int vst_cap) {
  extern __shared__ double g_vst[];  // SMEM-staging experiment (HESP_VSTAGE): vst_cap doubles per warp
  const int wib = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * WARPS_PER_BLOCK + wib;
  const Problem& pb = c_problem;
  g_small[wib].vst_base = g_vst + (size_t)wib * vst_cap;
  g_small[wib].vst_cap = vst_cap;
  __syncwarp();
  WarpBest b{0.0, -1, 0, 0, 0, 0, 0};
  if (accumulate) b = wbest[gw];
  for (;;) {
    unsigned long long k = 0;
    if (lane == 0) k = atomicAdd(counter, 1ULL);
    k = __shfl_sync(0xffffffffu, k, 0);
    if (k >= count) break;
    if (order) k = order[k];
    Engine<DevWarp> eng(DevWarp{}, pb, slots + (size_t)k * pb.lay.total, &g_small[wib]);
    const Outcome o = eng.sim_slot();
    if (lane == 0 && out) {
      hesp_outcome r;
      r.status = o.status;
      r.n_leaves = o.n_leaves;
      r.makespan = o.makespan;
      r.assign_hash = o.assign_hash;
      r.xfer_hash = o.xfer_hash;
      out[k] = r;
    }
    ++b.n_eval;
    b.leaves += o.n_leaves;
    b.k += o.sum_k;
    b.edges += o.n_edges;
    if (o.status == 0) {
      ++b.n_ok;
      const long long gi = (long long)(first_index + k);
      if (b.index < 0 || o.makespan < b.makespan || (o.makespan == b.makespan && gi < b.index)) {
        b.makespan = o.makespan;
        b.index = gi;
      }
    }
    __syncwarp();
  }
  if (lane == 0) wbest[gw] = b;
}

// Thread-per-candidate simulate kernel (HESP_SIM_THREAD=1): the same event
// loop instantiated at width 1 (Engine<HostWarp>, the source the host build
// verifies), one candidate per thread, the longest-first order keeping a
// warp's candidates of similar size.  Small lives in the candidate's slot.
#ifndef HESP_SIMT_MIN_BLOCKS
#define HESP_SIMT_MIN_BLOCKS 8
#endif
constexpr int SIMT_THREADS = 128;

__global__ void __launch_bounds__(SIMT_THREADS, HESP_SIMT_MIN_BLOCKS)
    sim_thread_kernel(unsigned long long first_index, unsigned long long count, hesp_outcome* __restrict__ out,
                      WarpBest* __restrict__ wbest, uint8_t* slots, const uint32_t* __restrict__ order) {
  const Problem& pb = c_problem;
  const unsigned long long tid = blockIdx.x * (unsigned long long)SIMT_THREADS + threadIdx.x;
  const unsigned long long nthreads = (unsigned long long)gridDim.x * SIMT_THREADS;
  const long long gw = (long long)(tid >> 5);
  WarpBest b{0.0, -1, 0, 0, 0, 0, 0};
  for (unsigned long long i = tid; i < count; i += nthreads) {
    const unsigned long long k = order ? order[i] : i;
    uint8_t* slot = slots + (size_t)k * pb.lay.total;
    Engine<HostWarp> eng(HostWarp{}, pb, slot, (Small*)(slot + pb.lay.small));
    const Outcome o = eng.sim_slot();
    if (out) {
      hesp_outcome r;
      r.status = o.status;
      r.n_leaves = o.n_leaves;
      r.makespan = o.makespan;
      r.assign_hash = o.assign_hash;
      r.xfer_hash = o.xfer_hash;
      out[k] = r;
    }
    ++b.n_eval;
    b.leaves += o.n_leaves;
    b.k += o.sum_k;
    b.edges += o.n_edges;
    if (o.status == 0) {
      ++b.n_ok;
      const long long gi = (long long)(first_index + k);
      if (b.index < 0 || o.makespan < b.makespan || (o.makespan == b.makespan && gi < b.index)) {
        b.makespan = o.makespan;
        b.index = gi;
      }
    }
  }
  // warp merge of the lanes' bests, folded into this warp's accumulator
  for (int off = 16; off; off >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, b.makespan, off);
    const long long i2 = __shfl_xor_sync(0xffffffffu, b.index, off);
    b.n_ok += __shfl_xor_sync(0xffffffffu, b.n_ok, off);
    b.n_eval += __shfl_xor_sync(0xffffffffu, b.n_eval, off);
    b.leaves += __shfl_xor_sync(0xffffffffu, b.leaves, off);
    b.k += __shfl_xor_sync(0xffffffffu, b.k, off);
    b.edges += __shfl_xor_sync(0xffffffffu, b.edges, off);
    if (i2 >= 0 && (b.index < 0 || m2 < b.makespan || (m2 == b.makespan && i2 < b.index))) {
      b.makespan = m2;
      b.index = i2;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    WarpBest a = wbest[gw];
    a.n_ok += b.n_ok;
    a.n_eval += b.n_eval;
    a.leaves += b.leaves;
    a.k += b.k;
    a.edges += b.edges;
    if (b.index >= 0 && (a.index < 0 || b.makespan < a.makespan || (b.makespan == a.makespan && b.index < a.index))) {
      a.makespan = b.makespan;
      a.index = b.index;
    }
    wbest[gw] = a;
  }
}

// Host descriptors travel packed (offsets + the used ops only: a C2
// descriptor averages ~40 of its 520 bytes); this expands them in HBM.
__global__ void unpack_descs(const uint32_t* __restrict__ off, const hesp_op* __restrict__ ops,
                             unsigned long long count, hesp_cand_desc* __restrict__ out) {
  const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint32_t o = off[i], n = off[i + 1] - o;
  hesp_cand_desc* d = out + i;
  d->n_ops = (int32_t)n;
  d->reserved = 0;
  for (uint32_t k = 0; k < n; ++k) d->ops[k] = ops[o + k];
}

__global__ void init_best(WarpBest* __restrict__ wb, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) wb[i] = WarpBest{0.0, -1, 0, 0, 0, 0, 0};
}

__global__ void reduce_best(const WarpBest* __restrict__ wb, int n, hesp_best* __restrict__ best) {
  __shared__ double smk[32];
  __shared__ long long sidx[32], sok[32], sev[32], sl[32], sk[32], se[32];
  double mk = 0.0;
  long long idx = -1, ok = 0, ev = 0, lv = 0, kk = 0, ed = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const WarpBest b = wb[i];
    ok += b.n_ok;
    ev += b.n_eval;
    lv += b.leaves;
    kk += b.k;
    ed += b.edges;
    if (b.index >= 0 && (idx < 0 || b.makespan < mk || (b.makespan == mk && b.index < idx))) {
      mk = b.makespan;
      idx = b.index;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const double m2 = __shfl_xor_sync(0xffffffffu, mk, o);
    const long long i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    ok += __shfl_xor_sync(0xffffffffu, ok, o);
    ev += __shfl_xor_sync(0xffffffffu, ev, o);
    lv += __shfl_xor_sync(0xffffffffu, lv, o);
    kk += __shfl_xor_sync(0xffffffffu, kk, o);
    ed += __shfl_xor_sync(0xffffffffu, ed, o);
    if (i2 >= 0 && (idx < 0 || m2 < mk || (m2 == mk && i2 < idx))) {
      mk = m2;
      idx = i2;
    }
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    smk[w] = mk;
    sidx[w] = idx;
    sok[w] = ok;
    sev[w] = ev;
    sl[w] = lv;
    sk[w] = kk;
    se[w] = ed;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    hesp_best r{0.0, -1, 0, 0, 0, 0, 0, 0.0, 0.0, 0.0};
    for (int i = 0; i < nw; ++i) {
      r.n_ok += sok[i];
      r.n_evaluated += sev[i];
      r.sum_leaves += sl[i];
      r.sum_k += sk[i];
      r.sum_edges += se[i];
      if (sidx[i] >= 0 && (r.index < 0 || smk[i] < r.makespan ||
                           (smk[i] == r.makespan && sidx[i] < r.index))) {
        r.makespan = smk[i];
        r.index = sidx[i];
      }
    }
    *best = r;
  }
}

__global__ void gen_kernel(unsigned long long first, unsigned long long count, hesp_cand_desc* __restrict__ out) {
  const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const Problem& pb = c_problem;
  hesp_cand_desc d;
  hesp_generate(&pb.gen, (int)(pb.n / pb.base_b), pb.n_base_leaves, pb.base_b, first + i, &d);
  out[i] = d;
}

__global__ void detail_kernel(const hesp_cand_desc* __restrict__ desc, uint8_t* slot, int32_t cap, int32_t* proc,
                              double* start, double* end, hesp_outcome* out, TraceBufs* tb) {
  __shared__ hesp_cand_desc sd;
  if (threadIdx.x == 0) sd = *desc;
  __syncwarp();
  Engine<DevWarp, true> eng(DevWarp{}, c_problem, slot, &g_small[0]);
  eng.tr_proc = proc;
  eng.tr_start = start;
  eng.tr_end = end;
  eng.tr_cap = cap;
  eng.tb = tb;
  const Outcome o = eng.run(sd);
  if (threadIdx.x == 0) {
    out->status = o.status;
    out->n_leaves = o.n_leaves;
    out->makespan = o.makespan;
    out->assign_hash = o.assign_hash;
    out->xfer_hash = o.xfer_hash;
  }
}

// Many candidates' schedules at once (the batched solver): one warp per
// candidate, the trace engine in schedule-only mode (E4 fast path, no logs),
// per-candidate output regions.
__global__ void schedule_kernel(const hesp_cand_desc* __restrict__ descs, uint8_t* slots, int32_t cap,
                                int32_t* proc, double* start, double* end, hesp_outcome* out, TraceBufs* tbs) {
  __shared__ hesp_cand_desc sd;
  const int b = blockIdx.x;
  if (threadIdx.x == 0) sd = descs[b];
  __syncwarp();
  uint8_t* slot = slots + (size_t)b * c_problem.lay.total;
  Engine<DevWarp, true> eng(DevWarp{}, c_problem, slot, &g_small[0]);
  eng.tr_proc = proc + (size_t)b * cap;
  eng.tr_start = start + (size_t)b * cap;
  eng.tr_end = end + (size_t)b * cap;
  eng.tr_cap = cap;
  eng.tb = tbs + b;
  const Outcome o = eng.run(sd);
  if (threadIdx.x == 0) {
    hesp_outcome r;
    r.status = o.status;
    r.n_leaves = o.n_leaves;
    r.makespan = o.makespan;
    r.assign_hash = o.assign_hash;
    r.xfer_hash = o.xfer_hash;
    out[b] = r;
  }
}

}  // namespace

struct hesp_engine {
  int device = 0;
  HostProblem hp;
  Problem* d_problem = nullptr;
  TaskMeta* d_base_tasks = nullptr;
  BasePreds* d_base_preds = nullptr;
  int32_t* d_base_plist = nullptr;
  BlockMeta* d_base_blocks = nullptr;
  SlotLayout L{};
  uint8_t* d_scratch = nullptr;
  int n_slots = 0, n_blocks = 0, sm_count = 0, blocks_per_sm = 0;  // sim kernel grid
  int n_build_blocks = 0;
  WarpBest* d_wbest = nullptr;
  hesp_best* d_best = nullptr;
  hesp_best* h_best = nullptr;  // pinned
  unsigned long long* d_counter = nullptr;
  hesp_outcome* d_out = nullptr;
  size_t out_cap = 0;
  hesp_cand_desc* d_descs = nullptr;
  size_t desc_cap = 0;
  hesp_cand_desc* h_descs = nullptr;  // pinned staging
  hesp_outcome* h_out = nullptr;      // pinned staging
  size_t h_cap = 0;
  cudaStream_t stream = nullptr;
  long long launches = 0;
  // per-candidate slots of one chunk (build -> simulate hand-off)
  bool split = true;
  uint8_t* d_cslots = nullptr;
  unsigned long long chunk = 0;      // max candidates per chunk (memory budget)
  unsigned long long cslots_n = 0;   // slots currently allocated
  uint32_t* d_order = nullptr;       // LPT order: keys/vals in, keys/vals out (4 x cslots_n)
  uint8_t* d_tslots = nullptr;       // template slots of hesp_eval_neighbors' bases
  int tslots_n = 0;
  hesp_neighbor* d_nbrs = nullptr;
  size_t nbr_cap = 0;
  uint8_t* d_pack = nullptr;         // packed host descriptors (hesp_eval_descs)
  void* d_lt = nullptr;              // load post-pass scratch (loadtrace.cu)
  size_t lt_cap = 0;
  size_t pack_cap = 0;
  size_t last_h2d_bytes = 0;
  hesp_cand_desc* d_gen = nullptr;   // generated descriptors of one chunk (LPT on generated batches)
  void* d_sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  bool lpt = true;
  bool sim_thread = false;           // HESP_SIM_THREAD=1: thread-per-candidate simulate kernel
  int vst_cap = 0;                   // HESP_VSTAGE=<bytes per warp>: valid times staged in shared memory (experiment)
  int n_simt_blocks = 0;
  int n_wbest = 0;                   // entries of d_wbest (max of both simulate grids, in warps)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  static constexpr int NEV = 64;     // per-chunk kernel timing (build, sim)
  cudaEvent_t evc[NEV][4] = {};
  int nev_used = 0;
  hx::TraceGraph last_graph;  // candidate of the last hesp_eval_trace (for hesp_verify_trace)
  std::vector<void*> trace_bufs;  // device buffers of hesp_eval_trace, allocated on first use
  TraceBufs trace_tb{};
  TraceBufs* d_trace_tb = nullptr;
  hesp_cand_desc* d_trace_desc = nullptr;
  int32_t* d_trace_proc = nullptr;
  double *d_trace_start = nullptr, *d_trace_end = nullptr;
  hesp_outcome* d_trace_out = nullptr;
  // batched schedule-only traces (hx::schedule_batch), grown on demand
  std::vector<void*> sched_bufs;
  int sched_cap = 0;
  uint8_t* d_sslots = nullptr;
  int32_t *d_sproc = nullptr, *d_sleaves = nullptr, *d_slpoff = nullptr, *d_slpcnt = nullptr, *d_slpreds = nullptr;
  double *d_sstart = nullptr, *d_send = nullptr;
  TaskMeta *d_slmeta = nullptr, *d_stmeta = nullptr;
  Region* d_sbregion = nullptr;
  int32_t* d_sbisint = nullptr;
  PartEntry* d_sparts = nullptr;
  TraceBufs* d_stbs = nullptr;
  hesp_outcome* d_sout = nullptr;
  // hesp_min_reduce's exchange words (allocated on first use, kept)
  long long* d_reduce = nullptr;
  long long* h_reduce = nullptr;
  long long min_reduces = 0;
};

namespace {

bool ck(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return false;
}

// Buffers grow geometrically (x1.5, at least 1024 entries): callers such as
// the solver issue batches of slowly varying size, and every reallocation is
// a synchronising cudaFree + cudaMalloc(Host).
size_t grown(size_t need, size_t have) {
  const size_t g = have + have / 2;
  return need > g ? (need > 1024 ? need : 1024) : g;
}

bool grow_out(hesp_engine* e, size_t n) {
  if (n <= e->out_cap) return true;
  n = grown(n, e->out_cap);
  if (e->d_out) cudaFree(e->d_out);
  e->d_out = nullptr;
  if (!ck(cudaMalloc(&e->d_out, n * sizeof(hesp_outcome)), "cudaMalloc outcomes")) return false;
  e->out_cap = n;
  return true;
}

bool grow_host(hesp_engine* e, size_t n) {
  if (n <= e->h_cap) return true;
  n = grown(n, e->h_cap);
  if (e->h_descs) cudaFreeHost(e->h_descs);
  if (e->h_out) cudaFreeHost(e->h_out);
  e->h_descs = nullptr;
  e->h_out = nullptr;
  if (!ck(cudaMallocHost(&e->h_descs, n * sizeof(hesp_cand_desc)), "cudaMallocHost descs")) return false;
  if (!ck(cudaMallocHost(&e->h_out, n * sizeof(hesp_outcome)), "cudaMallocHost outcomes")) return false;
  e->h_cap = n;
  return true;
}

int launch_split(hesp_engine* e, const hesp_cand_desc* d_descs, uint64_t first, uint64_t count,
                 hesp_outcome* d_out, cudaStream_t st, const hesp_neighbor* d_nbrs = nullptr,
                 const uint8_t* d_tslots = nullptr) {
  // equal-size chunks under the memory cap: each chunk pays one load-balance tail
  const unsigned long long nchunks = count ? (count + e->chunk - 1) / e->chunk : 1;
  const unsigned long long per = count ? (count + nchunks - 1) / nchunks : 1;  // equal-size chunks
  unsigned long long need = per;
  if (need > e->cslots_n) {
    need = grown(need, e->cslots_n);
    if (need > e->chunk) need = e->chunk > per ? e->chunk : per;
    if (e->d_cslots) cudaFree(e->d_cslots);
    e->d_cslots = nullptr;
    e->cslots_n = 0;
    if (!ck(cudaMalloc(&e->d_cslots, (size_t)need * e->L.total), "malloc chunk slots")) return HESP_E_CUDA;
    e->cslots_n = need;
    if (e->d_order) cudaFree(e->d_order);
    if (e->d_sort_tmp) cudaFree(e->d_sort_tmp);
    if (e->d_gen) cudaFree(e->d_gen);
    e->d_gen = nullptr;
    e->d_order = nullptr;
    e->d_sort_tmp = nullptr;
    if (!ck(cudaMalloc(&e->d_order, 4 * sizeof(uint32_t) * need), "malloc order")) return HESP_E_CUDA;
    e->sort_tmp_bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, e->sort_tmp_bytes, e->d_order, e->d_order + need,
                                              e->d_order + 2 * need, e->d_order + 3 * need, (int)need, 0, 32, st);
    if (!ck(cudaMalloc(&e->d_sort_tmp, e->sort_tmp_bytes ? e->sort_tmp_bytes : 1), "malloc sort tmp"))
      return HESP_E_CUDA;
  }
  const unsigned long long chunk = per;
  if (!ck(cudaMemcpyToSymbolAsync(c_problem, &e->hp.p, sizeof(Problem), 0, cudaMemcpyHostToDevice, st),
          "problem -> constant"))
    return HESP_E_CUDA;
  cudaEventRecord(e->ev0, st);
  e->nev_used = 0;
  int acc = 0;
  if (e->sim_thread) {  // the thread kernel always accumulates: start from empty per-warp bests
    init_best<<<(e->n_wbest + 255) / 256, 256, 0, st>>>(e->d_wbest, e->n_wbest);
    e->launches += 1;
  }
  for (uint64_t c0 = 0; c0 < count || (count == 0 && c0 == 0); c0 += chunk) {
    const uint64_t n = count - c0 < chunk ? count - c0 : chunk;
    cudaMemsetAsync(e->d_counter, 0, 2 * sizeof(unsigned long long), st);
    const int ci = (int)(c0 / chunk);
    const bool timed = ci < hesp_engine::NEV;
    if (timed) cudaEventRecord(e->evc[ci][0], st);
    const hesp_cand_desc* cd = d_descs ? d_descs + c0 : nullptr;
    if (e->lpt && !cd && !d_nbrs && n > 1) {  // generated candidates: materialise the descriptors to order them
      if (!e->d_gen) {
        if (!ck(cudaMalloc(&e->d_gen, e->cslots_n * sizeof(hesp_cand_desc)), "malloc gen descs")) return HESP_E_CUDA;
      }
      gen_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(first + c0, n, e->d_gen);
      e->launches += 1;
      cd = e->d_gen;
    }
    const uint32_t* border = nullptr;
    if (e->lpt && cd && n > 1) {
      uint32_t* kin = e->d_order;
      uint32_t* kout = e->d_order + chunk;
      uint32_t* vin = e->d_order + 2 * chunk;
      uint32_t* vout = e->d_order + 3 * chunk;
      order_keys_desc<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(cd, n, kin, vin);
      size_t tb = e->sort_tmp_bytes;
      cub::DeviceRadixSort::SortPairsDescending(e->d_sort_tmp, tb, kin, kout, vin, vout, (int)n, 0, 32, st);
      border = vout;
      e->launches += 1;
    }
    if (d_nbrs)
      neighbor_build_kernel<<<e->n_build_blocks, WARPS_PER_BLOCK * 32, 0, st>>>(d_nbrs + c0, d_tslots, n,
                                                                            e->d_cslots, e->d_counter);
    else
      build_kernel<<<e->n_build_blocks, WARPS_PER_BLOCK * 32, 0, st>>>(cd, first + c0, n, e->d_cslots,
                                                                   e->d_counter, border);
    const uint32_t* order = nullptr;
    if (e->lpt && n > 1) {
      uint32_t* kin = e->d_order;
      uint32_t* kout = e->d_order + chunk;
      uint32_t* vin = e->d_order + 2 * chunk;
      uint32_t* vout = e->d_order + 3 * chunk;
      order_keys<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(e->d_cslots, n, kin, vin);
      size_t tb = e->sort_tmp_bytes;
      cub::DeviceRadixSort::SortPairsDescending(e->d_sort_tmp, tb, kin, kout, vin, vout, (int)n, 0, 32, st);
      order = vout;
      e->launches += 1;
    }
    if (timed) cudaEventRecord(e->evc[ci][1], st);
    if (e->sim_thread)
      sim_thread_kernel<<<e->n_simt_blocks, SIMT_THREADS, 0, st>>>(first + c0, n, d_out ? d_out + c0 : nullptr,
                                                                   e->d_wbest, e->d_cslots, order);
    else
      sim_kernel<<<e->n_blocks, WARPS_PER_BLOCK * 32, (size_t)WARPS_PER_BLOCK * e->vst_cap * 8, st>>>(
          first + c0, n, d_out ? d_out + c0 : nullptr, e->d_wbest, acc, e->d_cslots, e->d_counter + 1, order,
          e->vst_cap);
    if (timed) cudaEventRecord(e->evc[ci][2], st);
    e->nev_used = ci + 1 < hesp_engine::NEV ? ci + 1 : hesp_engine::NEV;
    e->launches += 2;
    acc = 1;
    if (count == 0) break;
  }
  cudaEventRecord(e->ev1, st);
  // only the entries this call's simulate grid wrote (the array is sized for
  // the larger of the two grids)
  reduce_best<<<1, 1024, 0, st>>>(e->d_wbest, e->sim_thread ? e->n_wbest : e->n_slots, e->d_best);
  e->launches += 1;
  if (!ck(cudaGetLastError(), "split launch")) return HESP_E_CUDA;
  return HESP_OK;
}

int launch_eval(hesp_engine* e, const hesp_cand_desc* d_descs, uint64_t first, uint64_t count,
                hesp_outcome* d_out, cudaStream_t st) {
  return launch_split(e, d_descs, first, count, d_out, st);
}

int finish_best(hesp_engine* e, hesp_best* best, cudaStream_t st) {
  if (!best) return HESP_OK;
  if (!ck(cudaMemcpyAsync(e->h_best, e->d_best, sizeof(hesp_best), cudaMemcpyDeviceToHost, st), "best D2H"))
    return HESP_E_CUDA;
  if (!ck(cudaStreamSynchronize(st), "sync")) return HESP_E_CUDA;
  *best = *e->h_best;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e->ev0, e->ev1);
  best->kernel_ms = ms;
  best->build_ms = 0.0;
  best->sim_ms = 0.0;
  if (e->split) {
    for (int i = 0; i < e->nev_used; ++i) {
      float b = 0.f, m = 0.f;
      cudaEventElapsedTime(&b, e->evc[i][0], e->evc[i][1]);
      cudaEventElapsedTime(&m, e->evc[i][1], e->evc[i][2]);
      best->build_ms += b;
      best->sim_ms += m;
    }
  }
  return HESP_OK;
}

}  // namespace

namespace {
template <class T>
bool dalloc(T** p, size_t n, std::vector<void*>& owned) {
  if (!ck(cudaMalloc((void**)p, (n ? n : 1) * sizeof(T)), "cudaMalloc trace")) return false;
  owned.push_back(*p);
  return true;
}

// Load post-passes of B traces (by-task-id arrays of nid entries each) on the
// engine's stream, into logs[b] (null entries skipped).
int load_traces(hesp_engine* e, const int32_t* proc, const double* start, const double* end, int nid, int B,
                std::vector<hx::TraceLogs*>& logs) {
  const size_t need = hx::load_trace_scratch_bytes(nid, B);
  if (need > e->lt_cap) {
    if (e->d_lt) cudaFree(e->d_lt);
    e->d_lt = nullptr;
    e->lt_cap = 0;
    if (!ck(cudaMalloc(&e->d_lt, need), "malloc load-trace scratch")) return HESP_E_CUDA;
    e->lt_cap = need;
  }
  const int r = hx::load_trace_device(proc, start, end, nid, B, e->hp.p.P, e->d_lt, e->stream, logs);
  if (r != HESP_OK) g_last_error = "load-trace post-pass failed";
  return r;
}
template <class T>
bool d2h(std::vector<T>& v, const T* d, size_t n) {
  v.resize(n);
  return !n || ck(cudaMemcpy(v.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost), "trace D2H");
}
}  // namespace

extern "C" {

const char* hesp_last_error(void) { return g_last_error.c_str(); }

const char* hesp_status_name(int32_t s) {
  static const char* names[] = {"ok",
                                "ParseError",
                                "ValidationError",
                                "DuplicateEntry",
                                "UnknownKindOrType",
                                "EmptyModel",
                                "NoRoute",
                                "InvalidSize",
                                "NotALeaf",
                                "IndivisibleGrain",
                                "UnknownPartitioner",
                                "NestedCluster",
                                "UnknownCluster",
                                "ModelMiss",
                                "CapacityInfeasible",
                                "NoProcessors",
                                "GrainTooSmall",
                                "EmptyCandidates",
                                "MissingTrace",
                                "ConfigError",
                                "CoherenceError",
                                "InternalError"};
  if (s >= 0 && s <= 21) return names[s];
  if (s == 100) return "ForeignException";
  if (s == ST_ENGINE_LIMIT) return "EngineLimit";
  if (s == ST_ENGINE_INVARIANT) return "EngineInvariant";
  if (s == HESP_ST_UNREPRODUCIBLE) return "Unreproducible";
  return "Unknown";
}

hesp_engine* hesp_engine_create(int device, const hesp_platform* platform, const hesp_perf_model* model,
                                const hesp_sched_config* sched, const hesp_workload* workload) {
  if (!platform || !model || !sched || !workload) {
    g_last_error = "null argument";
    return nullptr;
  }
  auto* e = new hesp_engine();
  e->device = device;
  try {
    e->hp = build_problem(*platform, *model, *sched, *workload);
  } catch (const std::exception& ex) {
    g_last_error = ex.what();
    delete e;
    return nullptr;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    g_last_error = "no CUDA device " + std::to_string(device);
    delete e;
    return nullptr;
  }
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10) {
    g_last_error = "engine is built for sm_100a; device is sm_" + std::to_string(prop.major * 10 + prop.minor);
    delete e;
    return nullptr;
  }
  auto fail = [&](cudaError_t c, const char* what) -> hesp_engine* {
    ck(c, what);
    hesp_engine_destroy(e);
    return nullptr;
  };
  cudaError_t c;
  if ((c = cudaSetDevice(device)) != cudaSuccess) return fail(c, "cudaSetDevice");
  if ((c = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking)) != cudaSuccess)
    return fail(c, "stream");
  e->sm_count = prop.multiProcessorCount;
  int bps = 0;
  // A/B knob: the unified L1/SMEM split (percent of the maximum carveout)
  {
    // The simulate kernel needs ~50 KB of shared memory at 8 CTAs/SM; the
    // driver's default split gives it a 100 KB carve-out.  The smallest split
    // that holds it (64 KB) leaves 192 KB of L1 for the per-candidate state:
    // L1 hit 71 % -> 79 %, +1-2 % (profiles/README.md).  Kept only when the
    // occupancy stays the same.
    int before = 0, after = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&before, sim_kernel, WARPS_PER_BLOCK * 32, 0);
    const char* v = getenv("HESP_CARVEOUT_SIM");
    cudaFuncSetAttribute(sim_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, v ? atoi(v) : 22);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&after, sim_kernel, WARPS_PER_BLOCK * 32, 0);
    if (!v && after < before)
      cudaFuncSetAttribute(sim_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, -1);  // driver default
  }
  // The build kernel keeps the driver's split: with ~2.3 KB of shared memory
  // per CTA (no descriptor staging, the view apart from Small) the driver
  // already picks the 64 KB configuration (L1 hit 51 % -> 56 %); an explicit
  // preference only made it pick larger ones (profiles/README.md).
  if (const char* v = getenv("HESP_CARVEOUT_BUILD"))
    cudaFuncSetAttribute(build_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(v));
  if (const char* v = getenv("HESP_VSTAGE")) {
    e->vst_cap = std::max(0, atoi(v)) / 8;
    cudaFuncSetAttribute(sim_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         WARPS_PER_BLOCK * e->vst_cap * 8);
  }
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, sim_kernel, WARPS_PER_BLOCK * 32,
                                                (size_t)WARPS_PER_BLOCK * e->vst_cap * 8);
  int bbps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bbps, build_kernel, WARPS_PER_BLOCK * 32, 0);
  if (bbps < 1) bbps = 1;
  // A/B knobs: resident CTAs per SM below the occupancy limit (fewer warps
  // in flight, a smaller concurrent working set)
  if (const char* v = getenv("HESP_BUILD_CTAS")) bbps = std::max(1, std::min(bbps, atoi(v)));
  if (const char* v = getenv("HESP_SIM_CTAS")) bps = std::max(1, std::min(bps, atoi(v)));
  e->n_build_blocks = prop.multiProcessorCount * bbps;
  if (bps < 1) bps = 1;
  e->blocks_per_sm = bps;
  e->n_blocks = e->sm_count * bps;
  e->n_slots = e->n_blocks * WARPS_PER_BLOCK;
  Problem p = e->hp.p;
  const size_t nt = e->hp.base_tasks.size(), nb = e->hp.base_blocks.size();
  if ((c = cudaMalloc(&e->d_base_tasks, nt * sizeof(TaskMeta))) != cudaSuccess) return fail(c, "malloc");
  if ((c = cudaMalloc(&e->d_base_blocks, nb * sizeof(BlockMeta))) != cudaSuccess) return fail(c, "malloc");
  cudaMemcpy(e->d_base_tasks, e->hp.base_tasks.data(), nt * sizeof(TaskMeta), cudaMemcpyHostToDevice);
  cudaMemcpy(e->d_base_blocks, e->hp.base_blocks.data(), nb * sizeof(BlockMeta), cudaMemcpyHostToDevice);
  const size_t npr = e->hp.base_preds.size(), npl = e->hp.base_plist.size();
  if ((c = cudaMalloc(&e->d_base_preds, npr * sizeof(BasePreds))) != cudaSuccess) return fail(c, "malloc");
  if ((c = cudaMalloc(&e->d_base_plist, npl * sizeof(int32_t))) != cudaSuccess) return fail(c, "malloc");
  cudaMemcpy(e->d_base_preds, e->hp.base_preds.data(), npr * sizeof(BasePreds), cudaMemcpyHostToDevice);
  cudaMemcpy(e->d_base_plist, e->hp.base_plist.data(), npl * sizeof(int32_t), cudaMemcpyHostToDevice);
  bind_tilings(p, e->hp, e->d_base_tasks, e->d_base_blocks, e->d_base_preds, e->d_base_plist);
  p.lay = slot_layout(p);
  e->L = p.lay;
  if ((c = cudaMalloc(&e->d_problem, sizeof(Problem))) != cudaSuccess) return fail(c, "malloc");
  cudaMemcpy(e->d_problem, &p, sizeof(Problem), cudaMemcpyHostToDevice);
  {
    if (const char* t = getenv("HESP_SIM_THREAD")) e->sim_thread = atoi(t) != 0;
    int tb = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb, sim_thread_kernel, SIMT_THREADS, 0);
    if (tb < 1) tb = 1;
    e->n_simt_blocks = e->sm_count * tb;
    const int simt_warps = e->n_simt_blocks * (SIMT_THREADS / 32);
    e->n_wbest = e->n_slots > simt_warps ? e->n_slots : simt_warps;
  }
  if ((c = cudaMalloc(&e->d_wbest, (size_t)e->n_wbest * sizeof(WarpBest))) != cudaSuccess) return fail(c, "malloc");
  if ((c = cudaMalloc(&e->d_best, sizeof(hesp_best))) != cudaSuccess) return fail(c, "malloc");
  if ((c = cudaMalloc(&e->d_counter, 2 * sizeof(unsigned long long))) != cudaSuccess) return fail(c, "malloc");
  {
    e->split = true;
    // Chunk = candidates whose slots are resident at once: up to 131072
    // (HESP_CHUNK), bounded by 60% of free device memory (HESP_MEM_FRAC).
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const char* mf = getenv("HESP_MEM_FRAC");
    const double frac = mf ? atof(mf) : 0.6;
    if (const char* l = getenv("HESP_LPT")) e->lpt = atoi(l) != 0;
    unsigned long long cap = (unsigned long long)(frac * (double)free_b) / (unsigned long long)e->L.total;
    const char* ch = getenv("HESP_CHUNK");
    unsigned long long want = ch ? strtoull(ch, nullptr, 10) : 131072ULL;
    if (cap < 1024) cap = 1024;
    e->chunk = want < cap ? want : cap;
  }
  // one slot for the single-candidate detail / trace kernel
  if ((c = cudaMalloc(&e->d_scratch, (size_t)(e->split ? 1 : e->n_slots) * e->L.total)) != cudaSuccess)
    return fail(c, "malloc scratch");
  if ((c = cudaMallocHost(&e->h_best, sizeof(hesp_best))) != cudaSuccess) return fail(c, "malloc host");
  if ((c = cudaEventCreate(&e->ev0)) != cudaSuccess) return fail(c, "event");
  if ((c = cudaEventCreate(&e->ev1)) != cudaSuccess) return fail(c, "event");
  for (int i = 0; i < hesp_engine::NEV; ++i)
    for (int j = 0; j < 3; ++j)
      if ((c = cudaEventCreate(&e->evc[i][j])) != cudaSuccess) return fail(c, "event");
  e->hp.p = p;
  return e;
}

void hesp_engine_destroy(hesp_engine* e) {
  if (!e) return;
  cudaFree(e->d_problem);
  cudaFree(e->d_base_tasks);
  cudaFree(e->d_base_blocks);
  cudaFree(e->d_base_preds);
  cudaFree(e->d_base_plist);
  cudaFree(e->d_scratch);
  cudaFree(e->d_cslots);
  cudaFree(e->d_order);
  cudaFree(e->d_pack);
  cudaFree(e->d_lt);
  cudaFree(e->d_tslots);
  cudaFree(e->d_nbrs);
  cudaFree(e->d_sort_tmp);
  cudaFree(e->d_gen);
  for (void* q : e->trace_bufs) cudaFree(q);
  for (void* q : e->sched_bufs) cudaFree(q);
  cudaFree(e->d_wbest);
  cudaFree(e->d_best);
  cudaFree(e->d_counter);
  cudaFree(e->d_out);
  cudaFree(e->d_descs);
  cudaFree(e->d_reduce);
  if (e->h_reduce) cudaFreeHost(e->h_reduce);
  if (e->h_best) cudaFreeHost(e->h_best);
  if (e->h_descs) cudaFreeHost(e->h_descs);
  if (e->h_out) cudaFreeHost(e->h_out);
  if (e->ev0) cudaEventDestroy(e->ev0);
  if (e->ev1) cudaEventDestroy(e->ev1);
  for (int i = 0; i < hesp_engine::NEV; ++i)
    for (int j = 0; j < 3; ++j)
      if (e->evc[i][j]) cudaEventDestroy(e->evc[i][j]);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
}

int hesp_engine_get_info(const hesp_engine* e, hesp_engine_info* info) {
  if (!e || !info) return HESP_E_INVALID;
  info->kernel_launches = e->launches;
  info->n_base_tasks = e->hp.p.n_base_tasks;
  info->n_base_blocks = e->hp.p.n_base_blocks;
  info->n_slots = e->n_slots;
  info->sm_count = e->sm_count;
  info->slot_bytes = (int64_t)e->L.total;
  info->warps_per_block = WARPS_PER_BLOCK;
  info->blocks_per_sm = e->blocks_per_sm;
  info->chunk = e->split ? (int64_t)e->chunk : 0;
  info->last_h2d_bytes = (int64_t)e->last_h2d_bytes;
  info->min_reduces = e->min_reduces;
  return HESP_OK;
}

int hesp_eval_generated(hesp_engine* e, uint64_t first_index, uint64_t count, hesp_outcome* out,
                        hesp_best* best) {
  if (!e) return HESP_E_INVALID;
  cudaSetDevice(e->device);
  hesp_outcome* dout = nullptr;
  if (out) {
    if (!grow_out(e, count)) return HESP_E_CUDA;
    dout = e->d_out;
  }
  int r = launch_eval(e, nullptr, first_index, count, dout, e->stream);
  if (r) return r;
  if (out && !ck(cudaMemcpyAsync(out, dout, count * sizeof(hesp_outcome), cudaMemcpyDeviceToHost, e->stream),
                 "outcomes D2H"))
    return HESP_E_CUDA;
  if (best) return finish_best(e, best, e->stream);
  return ck(cudaStreamSynchronize(e->stream), "sync") ? HESP_OK : HESP_E_CUDA;
}

int hesp_eval_descs(hesp_engine* e, const hesp_cand_desc* descs, uint64_t count, uint64_t first_index,
                    hesp_outcome* out, hesp_best* best) {
  if (!e || !descs) return HESP_E_INVALID;
  cudaSetDevice(e->device);
  if (count > e->desc_cap) {
    if (e->d_descs) cudaFree(e->d_descs);
    e->d_descs = nullptr;
    const size_t cap = grown(count, e->desc_cap);
    if (!ck(cudaMalloc(&e->d_descs, cap * sizeof(hesp_cand_desc)), "malloc descs")) return HESP_E_CUDA;
    e->desc_cap = cap;
  }
  if (!grow_out(e, count) || !grow_host(e, count)) return HESP_E_CUDA;
  // pack into the pinned staging buffer: offsets[count + 1], then the used ops
  // (always fits: 4 (count + 1) + 8 * sum(n_ops) <= 520 * count)
  // (host threads over index ranges: a count pass, a scan of the per-range
  // totals, then each range writes its offsets and ops -- the same bytes as
  // one serial pass; it is host time inside every end-to-end call)
  uint32_t* hoff = reinterpret_cast<uint32_t*>(e->h_descs);
  hesp_op* hops = reinterpret_cast<hesp_op*>(reinterpret_cast<uint8_t*>(e->h_descs) + ((4 * (count + 1) + 7) & ~7ULL));
  auto nops = [&](uint64_t i) {
    const int n = descs[i].n_ops;
    return (uint32_t)(n < 0 ? 0 : (n > HESP_MAX_OPS ? HESP_MAX_OPS : n));
  };
  const int nthr = host_threads(count);
  std::vector<uint32_t> part(nthr + 1, 0);
  host_ranges(count, nthr, [&](int t, uint64_t a, uint64_t b) {
    uint32_t s = 0;
    for (uint64_t i = a; i < b; ++i) s += nops(i);
    part[t + 1] = s;
  });
  for (int t = 0; t < nthr; ++t) part[t + 1] += part[t];
  host_ranges(count, nthr, [&](int t, uint64_t a, uint64_t b) {
    uint32_t tot = part[t];
    for (uint64_t i = a; i < b; ++i) {
      hoff[i] = tot;
      const uint32_t n = nops(i);
      std::memcpy(hops + tot, descs[i].ops, (size_t)n * sizeof(hesp_op));
      tot += n;
    }
  });
  const uint32_t tot = part[nthr];
  hoff[count] = tot;
  const size_t ops_at = (4 * (count + 1) + 7) & ~7ULL;
  const size_t bytes = ops_at + (size_t)tot * sizeof(hesp_op);
  if (bytes > e->pack_cap) {
    if (e->d_pack) cudaFree(e->d_pack);
    e->d_pack = nullptr;
    const size_t cap = grown(bytes, e->pack_cap);
    if (!ck(cudaMalloc(&e->d_pack, cap), "malloc pack")) return HESP_E_CUDA;
    e->pack_cap = cap;
  }
  if (!ck(cudaMemcpyAsync(e->d_pack, e->h_descs, bytes, cudaMemcpyHostToDevice, e->stream), "descs H2D"))
    return HESP_E_CUDA;
  e->last_h2d_bytes = bytes;
  if (count) {
    unpack_descs<<<(unsigned)((count + 255) / 256), 256, 0, e->stream>>>(
        reinterpret_cast<const uint32_t*>(e->d_pack), reinterpret_cast<const hesp_op*>(e->d_pack + ops_at), count,
        e->d_descs);
    e->launches += 1;
  }
  int r = launch_eval(e, e->d_descs, first_index, count, e->d_out, e->stream);
  if (r) return r;
  if (!ck(cudaMemcpyAsync(e->h_out, e->d_out, count * sizeof(hesp_outcome), cudaMemcpyDeviceToHost, e->stream),
          "outcomes D2H"))
    return HESP_E_CUDA;
  r = finish_best(e, best, e->stream);
  if (r) return r;
  if (!ck(cudaStreamSynchronize(e->stream), "sync")) return HESP_E_CUDA;
  if (out)
    host_ranges(count, nthr, [&](int, uint64_t a, uint64_t b) {
      std::memcpy(out + a, e->h_out + a, (b - a) * sizeof(hesp_outcome));
    });
  return HESP_OK;
}

int hesp_eval_neighbors(hesp_engine* e, const hesp_cand_desc* bases, int32_t n_bases, const hesp_neighbor* nbrs,
                        uint64_t count, hesp_outcome* out, hesp_best* best) {
  if (!e || !bases || n_bases < 1 || (!nbrs && count)) return HESP_E_INVALID;
  for (uint64_t k = 0; k < count; ++k)
    if (nbrs[k].base < 0 || nbrs[k].base >= n_bases) {
      g_last_error = "hesp_eval_neighbors: base index out of range";
      return HESP_E_INVALID;
    }
  cudaSetDevice(e->device);
  cudaStream_t st = e->stream;
  if (n_bases > e->tslots_n) {
    if (e->d_tslots) cudaFree(e->d_tslots);
    e->d_tslots = nullptr;
    e->tslots_n = 0;
    if (!ck(cudaMalloc(&e->d_tslots, (size_t)n_bases * e->L.total), "malloc template slots")) return HESP_E_CUDA;
    e->tslots_n = n_bases;
  }
  if (count > e->nbr_cap) {
    if (e->d_nbrs) cudaFree(e->d_nbrs);
    e->d_nbrs = nullptr;
    const size_t cap = grown(count, e->nbr_cap);
    if (!ck(cudaMalloc(&e->d_nbrs, cap * sizeof(hesp_neighbor)), "malloc neighbours")) return HESP_E_CUDA;
    e->nbr_cap = cap;
  }
  if ((size_t)n_bases > e->desc_cap) {
    if (e->d_descs) cudaFree(e->d_descs);
    e->d_descs = nullptr;
    const size_t cap = grown((size_t)n_bases, e->desc_cap);
    if (!ck(cudaMalloc(&e->d_descs, cap * sizeof(hesp_cand_desc)), "malloc descs")) return HESP_E_CUDA;
    e->desc_cap = cap;
  }
  if (!grow_out(e, count) || !grow_host(e, count)) return HESP_E_CUDA;
  bool ok = ck(cudaMemcpyAsync(e->d_descs, bases, (size_t)n_bases * sizeof(hesp_cand_desc), cudaMemcpyHostToDevice,
                               st), "bases H2D") &&
            (!count || ck(cudaMemcpyAsync(e->d_nbrs, nbrs, count * sizeof(hesp_neighbor), cudaMemcpyHostToDevice, st),
                          "neighbours H2D")) &&
            ck(cudaMemcpyToSymbolAsync(c_problem, &e->hp.p, sizeof(Problem), 0, cudaMemcpyHostToDevice, st),
               "problem -> constant");
  if (!ok) return HESP_E_CUDA;
  template_kernel<<<n_bases, 32, 0, st>>>(e->d_descs, e->d_tslots);
  e->launches += 1;
  int r = launch_split(e, nullptr, 0, count, e->d_out, st, e->d_nbrs, e->d_tslots);
  if (r) return r;
  if (!ck(cudaMemcpyAsync(e->h_out, e->d_out, count * sizeof(hesp_outcome), cudaMemcpyDeviceToHost, st),
          "outcomes D2H"))
    return HESP_E_CUDA;
  r = finish_best(e, best, st);
  if (r) return r;
  if (!ck(cudaStreamSynchronize(st), "sync")) return HESP_E_CUDA;
  if (out) std::memcpy(out, e->h_out, count * sizeof(hesp_outcome));
  return HESP_OK;
}

int hesp_eval_descs_device(hesp_engine* e, const hesp_cand_desc* descs_dev, uint64_t count, uint64_t first_index,
                           hesp_outcome* out_dev, hesp_best* best, void* stream) {
  if (!e || !descs_dev) return HESP_E_INVALID;
  cudaSetDevice(e->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
  int r = launch_eval(e, descs_dev, first_index, count, out_dev, st);
  if (r) return r;
  return finish_best(e, best, st);
}

int hesp_generate_device(hesp_engine* e, uint64_t first_index, uint64_t count, hesp_cand_desc* descs_dev,
                         void* stream) {
  if (!e || !descs_dev) return HESP_E_INVALID;
  cudaSetDevice(e->device);
  cudaStream_t st = stream ? (cudaStream_t)stream : e->stream;
  const unsigned blocks = (unsigned)((count + 255) / 256);
  if (!ck(cudaMemcpyToSymbolAsync(c_problem, &e->hp.p, sizeof(Problem), 0, cudaMemcpyHostToDevice, st),
          "problem -> constant"))
    return HESP_E_CUDA;
  if (blocks) gen_kernel<<<blocks, 256, 0, st>>>(first_index, count, descs_dev);
  e->launches += blocks ? 1 : 0;
  return ck(cudaGetLastError(), "gen launch") ? HESP_OK : HESP_E_CUDA;
}

int hesp_eval_detail(hesp_engine* e, const hesp_cand_desc* desc, int32_t cap, int32_t* proc, double* start,
                     double* end, hesp_outcome* out) {
  if (!e || !desc || cap < 0) return HESP_E_INVALID;
  cudaSetDevice(e->device);
  hesp_cand_desc* dd = nullptr;
  int32_t* dp = nullptr;
  double *ds = nullptr, *de = nullptr;
  hesp_outcome* dout = nullptr;
  const size_t n = cap > 0 ? (size_t)cap : 1;
  bool ok = ck(cudaMalloc(&dd, sizeof(hesp_cand_desc)), "malloc") && ck(cudaMalloc(&dp, n * 4), "malloc") &&
            ck(cudaMalloc(&ds, n * 8), "malloc") && ck(cudaMalloc(&de, n * 8), "malloc") &&
            ck(cudaMalloc(&dout, sizeof(hesp_outcome)), "malloc");
  // every copy and fill is ordered on the engine's (non-blocking) stream,
  // ahead of and behind the kernel
  cudaStream_t st = e->stream;
  hesp_outcome o{};
  if (ok) {
    ok = ck(cudaMemcpyAsync(dd, desc, sizeof(hesp_cand_desc), cudaMemcpyHostToDevice, st), "detail H2D") &&
         ck(cudaMemsetAsync(dp, 0xff, n * 4, st), "detail memset") && ck(cudaMemsetAsync(ds, 0, n * 8, st), "detail memset") &&
         ck(cudaMemsetAsync(de, 0, n * 8, st), "detail memset") &&
         ck(cudaMemcpyToSymbolAsync(c_problem, &e->hp.p, sizeof(Problem), 0, cudaMemcpyHostToDevice, st), "problem");
  }
  if (ok) {
    detail_kernel<<<1, 32, 0, st>>>(dd, e->d_scratch, cap, dp, ds, de, dout, nullptr);
    e->launches += 1;
    ok = ck(cudaGetLastError(), "detail launch") &&
         ck(cudaMemcpyAsync(&o, dout, sizeof(o), cudaMemcpyDeviceToHost, st), "detail D2H") &&
         (!proc || !cap || ck(cudaMemcpyAsync(proc, dp, (size_t)cap * 4, cudaMemcpyDeviceToHost, st), "detail D2H")) &&
         (!start || !cap || ck(cudaMemcpyAsync(start, ds, (size_t)cap * 8, cudaMemcpyDeviceToHost, st), "detail D2H")) &&
         (!end || !cap || ck(cudaMemcpyAsync(end, de, (size_t)cap * 8, cudaMemcpyDeviceToHost, st), "detail D2H")) &&
         ck(cudaStreamSynchronize(st), "detail");
    if (ok && out) *out = o;
  }
  cudaFree(dd);
  cudaFree(dp);
  cudaFree(ds);
  cudaFree(de);
  cudaFree(dout);
  return ok ? o.status : HESP_E_CUDA;
}

int hesp_eval_trace(hesp_engine* e, const hesp_cand_desc* desc, hesp_trace* tr) {
  if (!e || !desc || !tr) return HESP_E_INVALID;
  if (tr->cap_assign < 0 || tr->cap_xfer < 0 || tr->cap_res < 0 || tr->cap_events < 0 || tr->cap_steps < 0)
    return HESP_E_INVALID;
  cudaSetDevice(e->device);
  e->last_graph = hx::TraceGraph{};
  const Problem& P = e->hp.p;
  const int T = P.maxt, B = P.maxb;
  // device log capacities: transfers and residency changes per task are few
  // (<= 3 acquires + write-back + flushes); gathers add fragments
  const int xcap = 16 * T + 1024, rcap = 32 * T + 1024;
  bool ok = true;
  if (!e->d_trace_tb) {  // first trace on this handle: allocate once, reuse after
    std::vector<void*>& owned = e->trace_bufs;
    TraceBufs& tb0 = e->trace_tb;
    ok = dalloc(&e->d_trace_desc, 1, owned) && dalloc(&e->d_trace_proc, 2 * T, owned) &&
         dalloc(&e->d_trace_start, 2 * T, owned) && dalloc(&e->d_trace_end, 2 * T, owned) &&
         dalloc(&e->d_trace_out, 1, owned) && dalloc(&tb0.x, xcap, owned) && dalloc(&tb0.r, rcap, owned) &&
         dalloc(&tb0.leaves, T, owned) && dalloc(&tb0.lmeta, T, owned) && dalloc(&tb0.lpoff, T, owned) &&
         dalloc(&tb0.lpcnt, T, owned) && dalloc(&tb0.lpreds, P.maxedges, owned) && dalloc(&tb0.bregion, B, owned) &&
         dalloc(&tb0.bisint, B, owned) && dalloc(&tb0.parts, MAXPART, owned) && dalloc(&tb0.tmeta, T, owned) &&
         dalloc(&e->d_trace_tb, 1, owned);
    tb0.xcap = xcap;
    tb0.rcap = rcap;
    tb0.leaf_cap = T;
    tb0.pred_cap = P.maxedges;
    tb0.block_cap = B;
    tb0.task_cap = T;
    if (!ok) {
      for (void* q : owned) cudaFree(q);
      owned.clear();
      e->d_trace_tb = nullptr;
      return HESP_E_CUDA;
    }
  }
  hesp_cand_desc* dd = e->d_trace_desc;
  int32_t* dp = e->d_trace_proc;
  double *ds = e->d_trace_start, *de = e->d_trace_end;
  hesp_outcome* dout = e->d_trace_out;
  TraceBufs* dtb = e->d_trace_tb;
  TraceBufs tb = e->trace_tb;  // counters zero
  tb.lite = (tr->flags & HESP_TRACE_SCHEDULE_ONLY) ? 1 : 0;
  XferLog* dx = tb.x;
  ResLog* dr = tb.r;
  hesp_outcome o{};
  hx::TraceLogs logs;
  TraceBufs hb{};
  if (ok) {
    // host -> device inputs, fills, the kernel and the read-back all on the
    // engine's stream (tb/hb are pageable: the final synchronize orders them)
    cudaStream_t st = e->stream;
    ok = ck(cudaMemcpyAsync(dtb, &tb, sizeof(tb), cudaMemcpyHostToDevice, st), "trace H2D") &&
         ck(cudaMemcpyAsync(dd, desc, sizeof(hesp_cand_desc), cudaMemcpyHostToDevice, st), "trace H2D") &&
         ck(cudaMemsetAsync(dp, 0xff, (size_t)T * 8, st), "trace memset") &&
         ck(cudaMemcpyToSymbolAsync(c_problem, &P, sizeof(Problem), 0, cudaMemcpyHostToDevice, st), "problem");
    if (ok) {
      // per-task arrays by reference task id: below 2 * maxt (ids consumed
      // before a merge of the top cluster stay below the slot's task cap)
      detail_kernel<<<1, 32, 0, st>>>(dd, e->d_scratch, 2 * T, dp, ds, de, dout, dtb);
      e->launches += 1;
      ok = ck(cudaGetLastError(), "trace launch") &&
           ck(cudaMemcpyAsync(&o, dout, sizeof(o), cudaMemcpyDeviceToHost, st), "trace D2H") &&
           ck(cudaMemcpyAsync(&hb, dtb, sizeof(hb), cudaMemcpyDeviceToHost, st), "trace D2H") &&
           ck(cudaStreamSynchronize(st), "trace kernel");
    }
  }
  if (ok && hb.overflow) {
    g_last_error = "trace buffers overflowed";
    ok = false;
  }
  if (ok && o.status == 0) {
    hx::TraceGraph& g = e->last_graph;
    ok = d2h(logs.proc, dp, 2 * (size_t)T) && d2h(logs.start, ds, 2 * (size_t)T) && d2h(logs.end, de, 2 * (size_t)T) &&
         d2h(logs.xfers, dx, (size_t)hb.nx) && d2h(logs.res, dr, (size_t)hb.nr) &&
         d2h(g.leaves, tb.leaves, (size_t)hb.nleaves) && d2h(g.meta, tb.lmeta, (size_t)hb.nleaves) &&
         d2h(g.poff, tb.lpoff, (size_t)hb.nleaves) && d2h(g.pcnt, tb.lpcnt, (size_t)hb.nleaves) &&
         d2h(g.preds, tb.lpreds, (size_t)hb.npreds) && d2h(g.bregion, tb.bregion, (size_t)hb.nblocks) &&
         d2h(g.bisint, tb.bisint, (size_t)hb.nblocks) && d2h(g.parts, tb.parts, (size_t)hb.nparts) &&
         d2h(g.tmeta, tb.tmeta, (size_t)hb.ntasks);
    if (ok) hx::to_reference_ids(g, &logs, hb.off_t, hb.off_b, hb.off_c);
    g.valid = ok;
    if (ok) {
      std::vector<hx::TraceLogs*> one{&logs};
      const int r = load_traces(e, dp, ds, de, 2 * T, 1, one);
      if (r != HESP_OK) return r;
    }
  }
  if (!ok) return o.status ? o.status : HESP_E_CUDA;
  tr->outcome = o;
  tr->n_assign = tr->n_xfer = tr->n_res = tr->n_events = tr->n_steps = 0;
  tr->busy_time = tr->avg_load = tr->load_integral = 0.0;
  if (o.status != 0) return o.status;
  const int r = hx::finish_trace(P, e->last_graph, logs, tr, tb.lite != 0);
  if (r != HESP_OK) {
    g_last_error = "trace arrays too small (see the hesp_trace counts)";
    return r;
  }
  return 0;
}

}  // extern "C"

const hx::Problem& hesp_engine_problem(const hesp_engine* e) { return e->hp.p; }

int hx::schedule_batch(hesp_engine* e, const hesp_cand_desc* descs, int B, std::vector<TraceGraph>& graphs,
                       std::vector<TraceLogs>& logs, std::vector<hesp_outcome>& outs) {
  if (!e || !descs || B < 1) return HESP_E_INVALID;
  cudaSetDevice(e->device);
  const Problem& P = e->hp.p;
  const size_t T = P.maxt, E = P.maxedges, NB = P.maxb;
  if (B > e->sched_cap) {
    for (void* q : e->sched_bufs) cudaFree(q);
    e->sched_bufs.clear();
    e->sched_cap = 0;
    std::vector<void*>& o = e->sched_bufs;
    const size_t b = (size_t)B;
    const bool ok = dalloc(&e->d_sslots, b * e->L.total, o) && dalloc(&e->d_sproc, b * 2 * T, o) &&
                    dalloc(&e->d_sstart, b * 2 * T, o) && dalloc(&e->d_send, b * 2 * T, o) &&
                    dalloc(&e->d_sleaves, b * T, o) && dalloc(&e->d_slmeta, b * T, o) &&
                    dalloc(&e->d_slpoff, b * T, o) && dalloc(&e->d_slpcnt, b * T, o) &&
                    dalloc(&e->d_slpreds, b * E, o) && dalloc(&e->d_sbregion, b * NB, o) &&
                    dalloc(&e->d_sbisint, b * NB, o) && dalloc(&e->d_sparts, b * MAXPART, o) &&
                    dalloc(&e->d_stmeta, b * T, o) && dalloc(&e->d_stbs, b, o) && dalloc(&e->d_sout, b, o);
    if (!ok) {
      for (void* q : o) cudaFree(q);
      o.clear();
      return HESP_E_CUDA;
    }
    e->sched_cap = B;
  }
  std::vector<TraceBufs> tbs(B);
  for (int b = 0; b < B; ++b) {
    TraceBufs& t = tbs[b];
    t = TraceBufs{};
    t.lite = 1;
    t.leaves = e->d_sleaves + b * T;
    t.lmeta = e->d_slmeta + b * T;
    t.lpoff = e->d_slpoff + b * T;
    t.lpcnt = e->d_slpcnt + b * T;
    t.lpreds = e->d_slpreds + b * E;
    t.bregion = e->d_sbregion + b * NB;
    t.bisint = e->d_sbisint + b * NB;
    t.parts = e->d_sparts + (size_t)b * MAXPART;
    t.tmeta = e->d_stmeta + b * T;
    t.leaf_cap = (int)T;
    t.pred_cap = (int)E;
    t.block_cap = (int)NB;
    t.task_cap = (int)T;
  }
  hesp_cand_desc* dd = nullptr;
  if (!ck(cudaMalloc(&dd, (size_t)B * sizeof(hesp_cand_desc)), "malloc descs")) return HESP_E_CUDA;
  cudaStream_t st = e->stream;
  bool ok = ck(cudaMemcpyAsync(dd, descs, (size_t)B * sizeof(hesp_cand_desc), cudaMemcpyHostToDevice, st), "H2D") &&
            ck(cudaMemcpyAsync(e->d_stbs, tbs.data(), (size_t)B * sizeof(TraceBufs), cudaMemcpyHostToDevice, st),
               "H2D") &&
            ck(cudaMemsetAsync(e->d_sproc, 0xff, (size_t)B * T * 8, st), "memset") &&
            ck(cudaMemcpyToSymbolAsync(c_problem, &P, sizeof(Problem), 0, cudaMemcpyHostToDevice, st), "problem");
  if (ok) {
    schedule_kernel<<<B, 32, 0, st>>>(dd, e->d_sslots, (int32_t)(2 * T), e->d_sproc, e->d_sstart, e->d_send, e->d_sout,
                                      e->d_stbs);
    e->launches += 1;
    ok = ck(cudaStreamSynchronize(st), "schedule kernel");
  }
  std::vector<TraceBufs> hb(B);
  outs.assign(B, hesp_outcome{});
  ok = ok && d2h(hb, e->d_stbs, B) && ck(cudaMemcpy(outs.data(), e->d_sout, B * sizeof(hesp_outcome),
                                                   cudaMemcpyDeviceToHost), "D2H");
  cudaFree(dd);
  if (!ok) return HESP_E_CUDA;
  std::vector<int32_t> proc;
  std::vector<double> s0, s1;
  const size_t TX = 2 * T;  // per-task arrays by reference task id
  ok = d2h(proc, e->d_sproc, (size_t)B * TX) && d2h(s0, e->d_sstart, (size_t)B * TX) && d2h(s1, e->d_send, (size_t)B * TX);
  if (!ok) return HESP_E_CUDA;
  graphs.assign(B, TraceGraph{});
  logs.assign(B, TraceLogs{});
  for (int b = 0; b < B; ++b) {
    if (hb[b].overflow) {
      g_last_error = "schedule batch: trace buffers overflowed";
      return HESP_E_CUDA;
    }
    if (outs[b].status != 0) continue;
    TraceGraph& g = graphs[b];
    TraceLogs& L = logs[b];
    L.proc.assign(proc.begin() + b * TX, proc.begin() + (b + 1) * TX);
    L.start.assign(s0.begin() + b * TX, s0.begin() + (b + 1) * TX);
    L.end.assign(s1.begin() + b * TX, s1.begin() + (b + 1) * TX);
    const TraceBufs& t = tbs[b];
    ok = d2h(g.leaves, t.leaves, (size_t)hb[b].nleaves) && d2h(g.meta, t.lmeta, (size_t)hb[b].nleaves) &&
         d2h(g.poff, t.lpoff, (size_t)hb[b].nleaves) && d2h(g.pcnt, t.lpcnt, (size_t)hb[b].nleaves) &&
         d2h(g.preds, t.lpreds, (size_t)hb[b].npreds) && d2h(g.parts, t.parts, (size_t)hb[b].nparts) &&
         d2h(g.tmeta, t.tmeta, (size_t)hb[b].ntasks);
    if (!ok) return HESP_E_CUDA;
    hx::to_reference_ids(g, nullptr, hb[b].off_t, hb[b].off_b, hb[b].off_c);
    g.valid = true;
  }
  {
    std::vector<hx::TraceLogs*> lp(B, nullptr);
    for (int b = 0; b < B; ++b)
      if (outs[b].status == 0) lp[b] = &logs[b];
    const int r = load_traces(e, e->d_sproc, e->d_sstart, e->d_send, (int)TX, B, lp);
    if (r != HESP_OK) return r;
  }
  return HESP_OK;
}
void hx::set_last_error(const std::string& msg) { g_last_error = msg; }
const hx::TraceGraph& hesp_engine_last_graph(const hesp_engine* e) { return e->last_graph; }

extern "C" {

int hesp_trace_blocks(const hesp_engine* e, hesp_block_info* out, int32_t cap, int32_t* n) {
  if (!e || !n || cap < 0 || (cap > 0 && !out) || !e->last_graph.valid) {
    g_last_error = "hesp_trace_blocks needs a successful hesp_eval_trace first";
    return HESP_E_INVALID;
  }
  const hx::TraceGraph& g = e->last_graph;
  *n = (int32_t)g.bregion.size();
  for (int32_t b = 0; b < *n && b < cap; ++b) {
    const Region& r = g.bregion[b];
    out[b] = hesp_block_info{r.row, r.col, r.rows, r.cols, b < (int32_t)g.bisint.size() ? g.bisint[b] : 0, 0};
  }
  return HESP_OK;
}

int hesp_trace_bounds(const hesp_engine* e, double* cp, double* work) {
  if (!e || !cp || !work || !e->last_graph.valid) {
    g_last_error = "hesp_trace_bounds needs a successful hesp_eval_trace first";
    return HESP_E_INVALID;
  }
  hx::trace_bounds(e->hp.p, e->last_graph, cp, work);
  return HESP_OK;
}

int hesp_verify_trace(const hesp_engine* e, const hesp_trace* tr, char* buf, size_t cap, int32_t* n_violations) {
  if (!e || !tr || !e->last_graph.valid) {
    g_last_error = "hesp_verify_trace needs a successful hesp_eval_trace first";
    return HESP_E_INVALID;
  }
  cudaSetDevice(e->device);
  std::vector<std::string> v;
  const int rc = hx::verify_trace_device(e->hp.p, e->last_graph, *tr, e->stream, v);
  if (rc != HESP_OK) return rc;
  if (n_violations) *n_violations = (int32_t)v.size();
  if (buf && cap) {
    std::string all;
    for (size_t i = 0; i < v.size(); ++i) {
      if (i) all += '\n';
      all += v[i];
    }
    const size_t n = all.size() < cap - 1 ? all.size() : cap - 1;
    std::memcpy(buf, all.data(), n);
    buf[n] = 0;
  }
  return HESP_OK;
}

}  // extern "C"

namespace {
// NCCL entry points resolved at run time: the process's libnccl.so.2 (the one
// that created the caller's communicator) or the system one.
typedef int (*nccl_allreduce_fn)(const void*, void*, size_t, int, int, void*, cudaStream_t);
typedef const char* (*nccl_errstr_fn)(int);
struct NcclApi {
  nccl_allreduce_fn allreduce = nullptr;
  nccl_errstr_fn errstr = nullptr;
  bool ok = false;
};
NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    // HESP_NCCL_LIB names an explicit library (the two-process test's
    // ncclAllReduce shim); otherwise the process's own libnccl.so.2
    void* h = nullptr;
    if (const char* lib = getenv("HESP_NCCL_LIB")) h = dlopen(lib, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (h) {
      a.allreduce = (nccl_allreduce_fn)dlsym(h, "ncclAllReduce");
      a.errstr = (nccl_errstr_fn)dlsym(h, "ncclGetErrorString");
    }
    a.ok = a.allreduce != nullptr;
    return a;
  }();
  return api;
}
constexpr int NCCL_INT64 = 4, NCCL_SUM = 0, NCCL_MIN = 3;  // nccl.h ncclDataType_t / ncclRedOp_t

__global__ void winner_keys(long long* buf) {  // buf[0] = makespan key, buf[1] = index (in/out)
  // second round: keep the index only where this rank holds the global key
  if (threadIdx.x == 0 && buf[2] != buf[0]) buf[1] = 0x7fffffffffffffffLL;
}
}  // namespace

extern "C" {

int hesp_min_reduce(hesp_engine* e, void* comm, hesp_best* best) {
  if (!e || !comm || !best) return HESP_E_INVALID;
  NcclApi& api = nccl_api();
  if (!api.ok) {
    g_last_error = "hesp_min_reduce: libnccl.so.2 not found";
    return HESP_E_INVALID;
  }
  cudaSetDevice(e->device);
  const long long NONE = 0x7fffffffffffffffLL;
  long long h[10];
  long long key;
  std::memcpy(&key, &best->makespan, 8);
  h[0] = best->index >= 0 ? key : NONE;   // global min key goes here
  h[1] = best->index >= 0 ? best->index : NONE;
  h[2] = h[0];                            // this rank's key (kept)
  h[3] = best->n_ok;
  h[4] = best->n_evaluated;
  h[5] = best->sum_leaves;
  h[6] = best->sum_k;
  h[7] = best->sum_edges;
  // persistent device / pinned host words: no allocation (and no
  // synchronising cudaFree) inside a caller's timed region
  if (!e->d_reduce && !ck(cudaMalloc(&e->d_reduce, sizeof h), "malloc reduce")) return HESP_E_CUDA;
  if (!e->h_reduce && !ck(cudaMallocHost(&e->h_reduce, sizeof h), "malloc reduce host")) return HESP_E_CUDA;
  long long* d = e->d_reduce;
  std::memcpy(e->h_reduce, h, sizeof h);
  cudaStream_t st = e->stream;
  int r = 0;
  bool ok = ck(cudaMemcpyAsync(d, e->h_reduce, sizeof h, cudaMemcpyHostToDevice, st), "reduce H2D");
  if (ok) r = api.allreduce(d, d, 1, NCCL_INT64, NCCL_MIN, comm, st);           // 1: min key
  if (ok && r == 0) {
    winner_keys<<<1, 32, 0, st>>>(d);                                         // index only on the holders
    e->launches += 1;
    r = api.allreduce(d + 1, d + 1, 1, NCCL_INT64, NCCL_MIN, comm, st);         // 2: lowest index
  }
  if (ok && r == 0) r = api.allreduce(d + 3, d + 3, 5, NCCL_INT64, NCCL_SUM, comm, st);  // counters
  if (ok && r != 0) {
    g_last_error = std::string("ncclAllReduce: ") + (api.errstr ? api.errstr(r) : "error");
    ok = false;
  }
  ok = ok && ck(cudaMemcpyAsync(e->h_reduce, d, sizeof h, cudaMemcpyDeviceToHost, st), "reduce D2H") &&
       ck(cudaStreamSynchronize(st), "reduce sync");
  if (!ok) return r ? HESP_E_INVALID : HESP_E_CUDA;
  std::memcpy(h, e->h_reduce, sizeof h);
  ++e->min_reduces;
  if (h[0] == NONE) {
    best->index = -1;
    best->makespan = 0.0;
  } else {
    std::memcpy(&best->makespan, &h[0], 8);
    best->index = h[1];
  }
  best->n_ok = h[3];
  best->n_evaluated = h[4];
  best->sum_leaves = h[5];
  best->sum_k = h[6];
  best->sum_edges = h[7];
  return HESP_OK;
}

int hesp_generate_batch(const hesp_gen_config* gen, int32_t s_base_snapped, int32_t n_base, int64_t base_b,
                        uint64_t first_index, uint64_t count, hesp_cand_desc* descs) {
  if (!gen || !descs) return HESP_E_INVALID;
  for (uint64_t i = 0; i < count; ++i) hesp_generate(gen, s_base_snapped, n_base, base_b, first_index + i, &descs[i]);
  return HESP_OK;
}

int hesp_generate_host(const hesp_engine* e, uint64_t first_index, uint64_t count, hesp_cand_desc* descs) {
  if (!e || !descs) return HESP_E_INVALID;
  const Problem& p = e->hp.p;
  for (uint64_t i = 0; i < count; ++i)
    hesp_generate(&p.gen, (int)(p.n / p.base_b), p.n_base_leaves, p.base_b, first_index + i, &descs[i]);
  return HESP_OK;
}

}  // extern "C"
