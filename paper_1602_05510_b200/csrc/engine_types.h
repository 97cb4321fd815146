// engine_types.h — device-resident problem tables and per-candidate slot
// layout of the batched candidate-schedule engine.  Plain structs, no torch.
#pragma once

#include <stddef.h>
#include <stdint.h>

#include "hesp_workload.h"

namespace hx {

constexpr int MAXP = 32;      // processors (one warp lane each)
constexpr int MAXS = 8;       // memory spaces
constexpr int MAXL = 32;      // directed links
constexpr int MAXTYPES = 8;   // processor types
constexpr int MAXBV = 48;     // distinct block sides with tabulated times
constexpr int MAXPART = HESP_MAX_OPS + 2;  // clusters per candidate (slot array)
constexpr size_t SMALL_BYTES = 2048;       // >= sizeof(hx::Small) (engine.h asserts)
constexpr int RHT = 2048;  // per-candidate region hash (new blocks), 16-bit ids
constexpr int MAXTIL = 8;  // top-level tilings of the root a candidate can sit on
constexpr int XPAR = 4;    // extra DataDag parent links kept per intersection descriptor
constexpr int TIL_BASE = 0, TIL_ROOT = 1;  // the workload's base tiling; the unpartitioned root

// Status codes: 0 ok, 1 + hesp::Err ordinal (errors.hpp:10-32), engine codes >= 200.
enum : int32_t {
  ST_OK = 0,
  ST_VALIDATION = 1 + 1,
  ST_NO_ROUTE = 1 + 5,
  ST_NOT_A_LEAF = 1 + 7,
  ST_INDIVISIBLE = 1 + 8,
  ST_NESTED_CLUSTER = 1 + 10,
  ST_UNKNOWN_CLUSTER = 1 + 11,
  ST_MODEL_MISS = 1 + 12,
  ST_CAPACITY = 1 + 13,
  ST_NO_PROCESSORS = 1 + 14,
  ST_COHERENCE = 1 + 19,
  ST_INTERNAL = 1 + 20,
  ST_FOREIGN = 100,           // the reference throws a non-hesp exception (std::out_of_range) here
  ST_ENGINE_LIMIT = 201,      // a per-candidate buffer of the engine overflowed
  ST_ENGINE_INVARIANT = 202,  // an equivalence assumption of the engine was violated
};

enum : int32_t { ORD_FCFS = 0, ORD_PL = 1 };
enum : int32_t { SEL_RP = 0, SEL_FP = 1, SEL_EITP = 2, SEL_EFTP = 3 };
enum : int32_t { CACHE_WT = 0, CACHE_WB = 1, CACHE_WA = 2 };

struct Region {
  int32_t row, col, rows, cols;
};

// Static description of one task: blk[0..nrd) are its reads in spec order,
// blk[nrd] its single write (reference Task::reads/writes, graph.hpp:90-102).
struct TaskMeta {
  int32_t blk[4];
  int32_t b;
  int8_t kind, nrd, bidx, pad;
};

struct BlockMeta {
  Region r;
  int32_t tile;    // base tile containing the block (itself for a tile, -1 for the root)
  int32_t next;    // next block of the same tile, creation (= id) order
  int32_t isint;   // intersection descriptor (DataBlock::is_intersection)
  int32_t pad;
};

// Per-task simulation state, one 32-byte record (a single sector).
struct TState {
  double rel;       // release time = running max of predecessor ends
  double ct;        // critical time (PL) / best successor ct while building
  int32_t missing;  // predecessors not yet committed
  int32_t soff, scnt;  // successor list (CSR)
  int32_t pad;      // (a committed flag here cost a store per commit; nothing read it)
};

// Host-precomputed predecessors of a base task (E5): the deduplicated union
// and the per-block-slot contributions, as offsets into Problem::base_plist.
struct BasePreds {
  int32_t uoff, ucnt;
  int32_t soff[3], scnt[3];
};

// Per-task record of the event loop (built once per candidate): sorted
// working set, output block, kind | bidx << 8, block side.
struct STask {
  int32_t ws0, ws1, ws2, nw;
  int32_t out, kb, b, pad;
};

// Per-candidate state carried from the build kernel to the simulate kernel.
struct SlotHeader {
  int32_t status, ntasks, nblocks, nleaves, nedges, sum_k, n_leaves_out, npart;
  // top-level tiling the candidate sits on and its id offsets (BaseView)
  int32_t til, off_t, off_b, off_c;
  int32_t nxp;  // intersection descriptors holding extra parent links (Engine::nxp)
  int32_t pad1, pad2, pad3;
};



// One top-level tiling of the root, shared by every candidate on it: the root
// (task 0, block 0) plus the tasks and blocks TaskGraph::partition_task(0, 1/s)
// creates, in creation order, and their host-precomputed predecessors (E5).
// s == 1: the unpartitioned root (root_cholesky alone, or after the base
// cluster was merged away: graph.cpp:397-407, 521-534).
struct BaseTiling {
  int32_t s, n_tasks, n_blocks, pad;
  int64_t base_b;  // tile side (n for the unpartitioned root)
  const TaskMeta* tasks;
  const BlockMeta* blocks;
  const BasePreds* preds;
  const int32_t* plist;
};

// A candidate's view of its top-level tiling (per warp, in the warp's Small).
// Reference ids are offset once the base cluster has been merged away: task
// ids, block ids and cluster ids keep counting (graph.cpp:438, DataDag
// next_id_), so internal id i > 0 is reference id i + off.  Internal ids keep
// the reference's relative order, which is all the schedule depends on.
struct BaseView {
  int32_t nbt, nbb, til, pad;
  int64_t base_b;
  const TaskMeta* bt;
  const BlockMeta* bb;
  const BasePreds* bp;
  const int32_t* bpl;
  int32_t off_t, off_b, off_c, pad2;
};

// Byte layout of one per-warp slot (all arrays in global memory).
struct SlotLayout {
  size_t hdr, tm, ts, t_poff, t_pcnt, leaf, wsb;
  size_t bm, bflags, valid, lastu, pinu, bcell, rht, pmark, bref, xpar, part, dstack, small, tmis, wrt, pmk;
  size_t tl_head, tl_cnt, tl_boff, tl_nrb, tl_ncb, tl_coff, tl_ids;
  size_t bnd, c_writer, c_rhead, rnode, preds, succs, pool, pool_rel, pool_key, ready, ready_key, pbuf;
  size_t gs_a, gs_b, gs_reg, gs_reg2;  // gs_reg* sized maxgr
  size_t total;
};

struct Problem {
  // ---- platform (platform.hpp:24-86) ----
  int32_t P, S, main_space, n_types, L;
  int32_t proc_type[MAXP], proc_space[MAXP];
  int64_t cap[MAXS];
  int32_t route_n[MAXS * MAXS];  // hops of transfer_time's route (0 = NoRoute)
  int32_t route_l[MAXS * MAXS][2];
  double link_lat[MAXL], link_bw[MAXL];
  int32_t link_src[MAXL], link_dst[MAXL];
  // ---- performance model, precomputed on the host (platform.cpp:347-390) ----
  int32_t nbv;
  int64_t bval[MAXBV];
  double ttime[4][MAXBV][MAXTYPES];  // task_time(kind, b, type)
  double ctavg[4][MAXBV];            // critical_times' per-task mean over processors (sim.cpp:96-106)
  uint8_t known[4][MAXTYPES];        // PerfModel::knows
  // per (link, block side): bytes/bw and lat + bytes/bw of moving one block,
  // the same IEEE operations as transfer_time/plan_transfer (platform.cpp:207,
  // sim.cpp:486, 785-787), so the device never divides on the hot path
  double hopq[MAXL][MAXBV];
  double hopc[MAXL][MAXBV];
  // ---- workload ----
  int64_t n;
  int32_t elem;
  int32_t s_base;
  int64_t min_block;
  int32_t n_base_tasks;   // ids 0..n_base_tasks-1 (root + base tiling)
  int32_t n_base_blocks;  // ids 0..n_base_blocks-1 (root + base tiles)
  int32_t n_base_leaves;  // = n_base_tasks - 1
  int64_t base_b;
  hesp_gen_config gen;
  // ---- scheduling policy (SchedConfig, sim.hpp:26-32) ----
  int32_t ordering, selection, caching;
  int32_t loop;  // event-loop variant of the batch kernels: 0 lean (default), 1 general (A/B: HESP_LOOP=1)
  uint64_t sched_seed;
  // ---- capacities of the per-candidate slot ----
  int32_t maxt, maxb, maxbnd, maxcells, maxrn, maxedges, maxpb, maxgs, maxgr;
  // ---- base graph (shared by every candidate) ----
  const TaskMeta* base_tasks;    // [n_base_tasks]
  const BlockMeta* base_blocks;  // [n_base_blocks]
  const BasePreds* base_preds;   // [n_base_tasks]
  const int32_t* base_plist;
  // every top-level tiling: [TIL_BASE] = the base tiling above, [TIL_ROOT] =
  // the unpartitioned root, then the other tilings of the root that fit a slot
  BaseTiling til[MAXTIL];
  int32_t n_til;
  int32_t max_nbb;  // blocks of the largest tiling (per-tile slot arrays)
  // ---- per-candidate slot layout (byte offsets, identical for every slot) ----
  SlotLayout lay;
};

// One cluster (TaskCluster, graph.hpp:103-108); index = cluster id.  A merged
// cluster keeps its entry (ids are never reused) with task = -2 - parent.
struct PartEntry {
  int32_t task, child0, nchild, leaves;
};

// ---- full-trace mode (Engine<..., TRACE = true>, hesp_eval_trace) ----
// One transfer as plan_transfer records it (sim.cpp:468-499), in emission
// order, with the per-hop times the reference turns into Xfer events.
struct XferLog {
  int32_t block, src, dst, nh;
  int64_t bytes;
  double start, end;
  int32_t has_frag, frow, fcol, frows, fcols, pad;
  double hs[2], he[2];
};
// One residency change (sim.cpp ResidencyChange), in emission order.
struct ResLog {
  double time;
  int32_t space, block;
  int64_t delta;
};
// Device-side sinks of the trace kernel (one candidate).  Counters are
// advanced by the owning warp; overflow is reported, never written past.
struct TraceBufs {
  XferLog* x;
  ResLog* r;
  int32_t xcap, rcap;
  int32_t nx, nr;
  // graph of the traced candidate (for verify_schedule on the host)
  int32_t* leaves;   // program order
  TaskMeta* lmeta;   // per leaf
  int32_t* lpoff;    // per leaf: offset/count into lpreds
  int32_t* lpcnt;
  int32_t* lpreds;
  Region* bregion;   // per block id
  int32_t* bisint;
  PartEntry* parts;  // clusters by id (MAXPART)
  TaskMeta* tmeta;   // every task id < ntasks (leaf or not; merged-away ones too)
  int32_t nparts, ntasks, task_cap, pad_;
  int32_t leaf_cap, pred_cap, block_cap;
  int32_t nleaves, npreds, nblocks;
  int32_t overflow;
  int32_t lite;  // schedule only: keep the E4 fast path, no logs
  // reference-id offsets of the candidate (BaseView); the exported graph and
  // the logs carry internal ids, the per-task arrays reference ids
  int32_t off_t, off_b, off_c, pad2;
};

// Per-candidate result record (also the golden-record payload).
struct Outcome {
  int32_t status;
  int32_t n_leaves;
  double makespan;
  uint64_t assign_hash;
  uint64_t xfer_hash;
  int32_t sum_k;    // work counters for the roofline accounting (not part of parity)
  int32_t n_edges;
};

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

inline SlotLayout slot_layout(const Problem& p) {
  SlotLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    o = align_up(o, 16);
    size_t at = o;
    o += bytes;
    return at;
  };
  const size_t T = (size_t)p.maxt, B = (size_t)p.maxb, S = (size_t)p.S,
               NB = (size_t)(p.max_nbb > p.n_base_blocks ? p.max_nbb : p.n_base_blocks);
  L.hdr = take(sizeof(SlotHeader));
  L.tm = take(sizeof(TaskMeta) * T);
  L.ts = take(sizeof(TState) * T);
  L.t_poff = take(4 * T);
  L.t_pcnt = take(4 * T);
  L.leaf = take(4 * T);
  L.wsb = take(sizeof(STask) * T);
  L.bm = take(sizeof(BlockMeta) * B);
  L.bflags = take(4 * B);
  L.bcell = take(16 * B);
  L.rht = take(2 * (size_t)RHT);
  L.pmark = take(T);
  L.bref = take(4 * B);  // task references per candidate block (merge pruning)
  L.xpar = take(4 * (size_t)XPAR * B);  // per candidate intersection: non-Hasse DataDag parents
  L.part = take(sizeof(PartEntry) * MAXPART);
  L.dstack = take(3 * 4 * (size_t)MAXPART);
  L.small = take(SMALL_BYTES);  // per-candidate Small of the thread-per-candidate simulate kernel
  L.tmis = take((NB + 3) & ~(size_t)3);  // per base tile: holds a non-dyadic block (partial overlaps possible)
  L.wrt = take(B);              // per block: written since t=0 (gather's coherence check)
  L.pmk = take(4 * T);          // per task: last task whose predecessor list took it (dedup)
  L.valid = take(8 * B * S);
  L.lastu = take(8 * B * S);
  L.pinu = take(8 * B * S);
  L.tl_head = take(4 * NB);
  L.tl_cnt = take(4 * NB);
  L.tl_boff = take(4 * NB);
  L.tl_nrb = take(4 * NB);
  L.tl_ncb = take(4 * NB);
  L.tl_coff = take(4 * NB);
  L.tl_ids = take(4 * B);
  L.bnd = take(4 * (size_t)p.maxbnd);
  L.c_writer = take(4 * (size_t)p.maxcells);
  L.c_rhead = take(4 * (size_t)p.maxcells);
  L.rnode = take(8 * (size_t)p.maxrn);
  L.preds = take(4 * (size_t)p.maxedges);
  L.succs = take(4 * (size_t)p.maxedges);
  // pool .. ready_key stay back to back: build_deps keeps 4 int2 access
  // records per task over their 4+8+8+4+8 = 32 bytes per task (Engine::dacc)
  L.pool = take(4 * T);
  L.pool_rel = take(8 * T);
  L.pool_key = take(8 * T);
  L.ready = take(4 * T);
  L.ready_key = take(8 * T);
  L.pbuf = take(4 * (size_t)p.maxpb);
  L.gs_a = take(4 * (size_t)p.maxgs);
  L.gs_b = take(4 * (size_t)p.maxgs);
  L.gs_reg = take(sizeof(Region) * (size_t)p.maxgr);
  L.gs_reg2 = take(sizeof(Region) * (size_t)p.maxgr);
  L.total = align_up(o, 256);
  return L;
}

}  // namespace hx
