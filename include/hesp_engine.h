/* hesp_engine.h — C ABI of the B200 batched candidate-schedule engine.
 *
 * Drop-in for the reference path:
 *   TaskGraph::root_cholesky + partition_task      graph.hpp:119,136  (graph.cpp:397-513)
 *   simulate(graph, platform, model, cfg)          sim.hpp:150-151    (sim.cpp:838-842)
 *   the batch caller solve()/collect_candidates    solver.hpp:74-84   (declared only)
 * Inputs mirror the reference's value types field for field:
 *   hesp_platform      <- hesp::Platform::make(spaces, types, processors, links)  platform.hpp:57
 *   hesp_perf_model    <- PerfModel::analytic / PerfModel::tabulated             platform.hpp:118-121
 *   hesp_sched_config  <- hesp::SchedConfig                                       sim.hpp:26-32
 *   hesp_workload      <- root_cholesky(n, elem) + partition_task(0, 1/s_base)    graph.hpp:119,136
 * Errors never cross the ABI as exceptions: calls return 0 or a negative
 * HESP_E_* code (message via hesp_last_error), and every candidate carries a
 * status = 0 (ok) or 1 + hesp::Err ordinal (errors.hpp:10-32) of the error
 * the reference would have thrown for it; >= 200 are engine limits.
 *
 * One engine handle per GPU; a handle is not thread-safe.  No torch types.
 */
#ifndef HESP_ENGINE_H
#define HESP_ENGINE_H

#include <stddef.h>
#include <stdint.h>

#include "hesp_workload.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- reference value types ------------------------------------------- */
/* (hesp_fixture_load below fills these from the reference's own files.) */
typedef struct {
  int32_t id;
  int64_t capacity_bytes;
  int32_t is_main;
} hesp_space; /* MemorySpace, platform.hpp:29-33 */

typedef struct {
  int32_t id;
  int32_t type;  /* index into type_names */
  int32_t space; /* memory space id */
} hesp_processor; /* Processor, platform.hpp:35-39 */

typedef struct {
  int32_t src, dst;
  double latency_s;
  double bandwidth_bps;
} hesp_link; /* Link, platform.hpp:41-46 */

typedef struct {
  int32_t n_spaces;
  const hesp_space* spaces;
  int32_t n_types;
  const char* const* type_names; /* ProcessorType::name, platform.hpp:24-27 */
  int32_t n_procs;
  const hesp_processor* procs;
  int32_t n_links;
  const hesp_link* links;
} hesp_platform;

typedef struct {
  int32_t kind; /* HESP_CHOL .. HESP_GEMM */
  int32_t type; /* index into hesp_platform.type_names */
  double peak_flops;
  double b_half;
} hesp_analytic_entry; /* PerfModel::analytic tuple, platform.hpp:118-119 */

typedef struct {
  int32_t kind;
  int32_t type;
  int64_t b;
  double seconds;
} hesp_table_row; /* PerfModel::tabulated tuple, platform.hpp:120-121 */

enum { HESP_MODEL_TABULATED = 0, HESP_MODEL_ANALYTIC = 1 }; /* PerfModel::Variant */

typedef struct {
  int32_t variant;
  int32_t n_entries;
  const hesp_analytic_entry* entries;
  int32_t n_rows;
  const hesp_table_row* rows;
} hesp_perf_model;

enum { HESP_FCFS = 0, HESP_PL = 1 };                              /* Ordering  */
enum { HESP_RP = 0, HESP_FP = 1, HESP_EITP = 2, HESP_EFTP = 3 };  /* Selection */
enum { HESP_WT = 0, HESP_WB = 1, HESP_WA = 2 };                   /* Caching   */

typedef struct {
  int32_t ordering, selection, caching;
  int32_t reserved;
  uint64_t seed;
  int64_t min_block;
} hesp_sched_config; /* SchedConfig, sim.hpp:26-32 */

typedef struct {
  int64_t n;          /* matrix side (root_cholesky) */
  int32_t elem_size;  /* bytes per element */
  int32_t s_base;     /* base tiling applied to task 0: partition_task(0, 1.0/s_base) */
  hesp_gen_config gen; /* candidate generator (include/hesp_workload.h) */
} hesp_workload;

/* ---- results ---------------------------------------------------------- */
typedef struct {
  int32_t status;      /* 0 ok; 1 + hesp::Err ordinal; >= 200 engine limit */
  int32_t n_leaves;    /* leaf tasks of the expanded DAG (0 if the build failed) */
  double makespan;     /* SimResult::makespan (0 when status != 0) */
  uint64_t assign_hash; /* sum of hesp_assign_term over SimResult::assignments */
  uint64_t xfer_hash;   /* sum of hesp_xfer_term over SimResult::transfers */
} hesp_outcome;

typedef struct {
  double makespan;    /* best makespan over status == 0 candidates */
  int64_t index;      /* lowest global candidate index achieving it (-1 if none) */
  int64_t n_ok;       /* candidates with status == 0 */
  int64_t n_evaluated;
  /* work actually done by the batch (roofline accounting) */
  int64_t sum_leaves; /* leaf tasks of all expanded DAGs */
  int64_t sum_k;      /* sum over leaves of distinct blocks accessed */
  int64_t sum_edges;  /* dependence edges generated */
  double kernel_ms;   /* CUDA-event duration of all evaluation kernels of the call (same stream) */
  double build_ms;    /* of which build kernels (phase-split mode) */
  double sim_ms;      /* of which simulate kernels (phase-split mode) */
} hesp_best;

enum {
  HESP_OK = 0,
  HESP_E_INVALID = -1, /* bad argument / platform / model (message in hesp_last_error) */
  HESP_E_CUDA = -2,    /* CUDA runtime failure */
  HESP_E_NODEV = -3,   /* no usable sm_100 device */
  HESP_E_LIMIT = -4    /* a caller-provided trace array is too small (counts report the need) */
};
/* Per-candidate engine statuses (>= 200; below 200 a status is 1 + hesp::Err). */
enum {
  HESP_ST_ENGINE_LIMIT = 201,      /* a per-candidate buffer of the engine would overflow */
  HESP_ST_ENGINE_INVARIANT = 202,  /* an equivalence the engine relies on was violated (never seen) */
  HESP_ST_UNREPRODUCIBLE = 203     /* bridge: a TaskGraph whose history its replay cannot reproduce */
};

typedef struct hesp_engine hesp_engine;

/* The reference's fixture files read in C:
 * Platform::from_json (platform.cpp:157-196) and PerfModel::from_analytic_json
 * / from_table_csv (platform.cpp:238-320; a path ending in .csv is a table).
 * Model entries of types the platform does not declare are dropped.  NULL on
 * a parse error (message in hesp_last_error); the returned views stay valid
 * until hesp_fixture_free. */
typedef struct hesp_fixture hesp_fixture;
hesp_fixture* hesp_fixture_load(const char* platform_path, const char* model_path);
const hesp_platform* hesp_fixture_platform(const hesp_fixture* f);
const hesp_perf_model* hesp_fixture_model(const hesp_fixture* f);
void hesp_fixture_free(hesp_fixture* f);

/* Validate inputs, precompute the model tables and the base tiling, upload
 * them and size the per-warp scratch.  Returns NULL on error. */
hesp_engine* hesp_engine_create(int device, const hesp_platform* platform,
                                const hesp_perf_model* model, const hesp_sched_config* sched,
                                const hesp_workload* workload);

/* Candidates first_index .. first_index+count-1 generated on the device from
 * workload.gen (no H2D traffic).  out (host, may be NULL) receives one
 * outcome per candidate; best (host, may be NULL) the argmin. */
int hesp_eval_generated(hesp_engine* e, uint64_t first_index, uint64_t count, hesp_outcome* out,
                        hesp_best* best);

/* Explicit candidate descriptors from HOST memory (copied in through pinned
 * staging; outcomes copied back).  Candidate k is reported as index first_index+k. */
int hesp_eval_descs(hesp_engine* e, const hesp_cand_desc* descs, uint64_t count,
                    uint64_t first_index, hesp_outcome* out, hesp_best* best);

/* Device-resident variant: descs_dev / out_dev are device pointers (out_dev
 * may be NULL), stream is a cudaStream_t (NULL = the engine's stream).
 * best (host, may be NULL) is synchronised before return. */
int hesp_eval_descs_device(hesp_engine* e, const hesp_cand_desc* descs_dev, uint64_t count,
                           uint64_t first_index, hesp_outcome* out_dev, hesp_best* best,
                           void* stream);

/* Write descriptors for candidates first..first+count-1 (device generator)
 * into a device buffer. */
int hesp_generate_device(hesp_engine* e, uint64_t first_index, uint64_t count,
                         hesp_cand_desc* descs_dev, void* stream);

/* Host copy of the device generator (same function), for callers that want
 * descriptors in host memory. */
int hesp_generate_host(const hesp_engine* e, uint64_t first_index, uint64_t count,
                       hesp_cand_desc* descs);

/* Pure host generator (no engine, no device): descriptors of candidates
 * first..first+count-1 for a workload whose base tiling has n_base leaves
 * of side base_b (s_base_snapped = n / base_b).  Same code as the device
 * generator (include/hesp_workload.h). */
int hesp_generate_batch(const hesp_gen_config* gen, int32_t s_base_snapped, int32_t n_base, int64_t base_b,
                        uint64_t first_index, uint64_t count, hesp_cand_desc* descs);

/* Per-task schedule of one candidate: for every (reference) task id < cap,
 * proc/start/end (proc = -1 for non-leaf, merged-away or unscheduled ids; ids
 * keep counting across merges of the base cluster, so size cap by the ids the
 * descriptor's ops consume).  Returns the outcome status. */
int hesp_eval_detail(hesp_engine* e, const hesp_cand_desc* desc, int32_t cap, int32_t* proc,
                     double* start, double* end, hesp_outcome* out);

/* ---------------------------------------------------------------------------
 * Full trace of one candidate: the complete
 * hesp::SimResult of simulate() (sim.hpp:77-88) -- assignments, transfers
 * with their routes, time-ordered events, residency log, idle_avg -- plus
 * compute_load_trace (sim.cpp:975-991) and the SimResult summary metrics.
 * The schedule is simulated on the device (one warp, full residency
 * bookkeeping); the host only orders the device logs the way Engine::run
 * does (sim.cpp:813-831) and derives the reference's post-passes
 * (compute_idle_avgs sim.cpp:670-702, busy_time/avg_load sim.cpp:78-87,
 * LoadTrace::integral sim.cpp:71-76). */
typedef struct {
  int32_t task, proc;
  double start, end;
  double idle_avg;   /* SimResult::idle_avg[task] */
} hesp_assignment;

typedef struct {
  int32_t block, src_space, dst_space, n_hops;
  int64_t bytes;
  double start, end;
  int32_t has_fragment, frag_row, frag_col, frag_rows, frag_cols, pad;
  int32_t hop_src[2], hop_dst[2];  /* TransferRec::route */
  double hop_start[2], hop_end[2]; /* per-hop times (the Xfer events) */
} hesp_transfer;

typedef struct {
  double time;
  int32_t space, block;
  int64_t delta_bytes;
} hesp_residency;

/* hesp_trace.flags: skip the transfer / residency / event logs (and their
 * bookkeeping), e.g. for the solver, which reads only the assignments */
#define HESP_TRACE_SCHEDULE_ONLY 1

enum { HESP_EV_TASK_START = 0, HESP_EV_TASK_END = 1, HESP_EV_XFER_START = 2, HESP_EV_XFER_END = 3 };
/* EventRec (sim.hpp:34-39) with its strings kept structured: subject is
 * "T<id>:<KIND>:b<b>" (task events) or "B<id>" (transfer events); resource is
 * the processor id or the link "src->dst". */
typedef struct {
  int32_t kind;
  int32_t id;         /* task id or block id */
  int32_t task_kind;  /* hesp TaskKind ordinal (task events) */
  int32_t res_a;      /* processor id, or link source space */
  int32_t res_b;      /* link destination space (transfer events), else -1 */
  int32_t pad;
  int64_t b;          /* task block side (task events) */
  double time;
} hesp_event;

typedef struct {
  double time;
  int32_t active, pad;
} hesp_load_step;

typedef struct {
  /* in: caller arrays and their capacities (entries) */
  int32_t cap_assign, cap_xfer, cap_res, cap_events, cap_steps;
  int32_t flags;                /* HESP_TRACE_SCHEDULE_ONLY: assignments + idle_avg + load only */
  hesp_assignment* assignments; /* task-id order (SimResult::assignments map order) */
  hesp_transfer* transfers;     /* Engine::run order: (start, block), stable */
  hesp_residency* residency;    /* (time, space, delta desc, block), stable */
  hesp_event* events;           /* (time, kind, resource, subject), stable */
  hesp_load_step* steps;        /* LoadTrace::steps */
  /* out: counts (also set, with HESP_E_LIMIT, when an array is too small) */
  int32_t n_assign, n_xfer, n_res, n_events, n_steps;
  int32_t pad1;
  hesp_outcome outcome;         /* status, leaves, makespan, the two hashes */
  double busy_time, avg_load, load_integral;
} hesp_trace;

/* Simulates one candidate with full tracing.  Returns the candidate status
 * (0 = ok, else 1 + Err ordinal; the arrays are filled only when 0), or a
 * negative HESP_E_* code.  The candidate's graph is kept in the handle for
 * hesp_verify_trace. */
int hesp_eval_trace(hesp_engine* e, const hesp_cand_desc* desc, hesp_trace* trace);

/* verify_schedule (sim.cpp:857-973) of a trace (possibly edited by the
 * caller) against the graph of the candidate last passed to
 * hesp_eval_trace: per-processor overlap, dependence order over the reduced
 * edge list, read coherence, capacity.  Writes the violation messages,
 * '\n'-separated and NUL-terminated, into buf (truncated to cap bytes) and
 * their count into *n_violations.  Returns HESP_OK or HESP_E_INVALID. */
int hesp_verify_trace(const hesp_engine* e, const hesp_trace* trace, char* buf, size_t cap,
                      int32_t* n_violations);

/* Makespan lower bounds of the candidate last passed to hesp_eval_trace
 * (SPEC.md acceptance 5): *cp = longest dependence path with every task at
 * its fastest processor type's time; *work = sum of those times / processors. */
int hesp_trace_bounds(const hesp_engine* e, double* cp, double* work);

/* The data blocks of the candidate last passed to hesp_eval_trace, indexed by
 * reference block id (DataDag::blocks(), graph.hpp:48-79): block k's region
 * and is_intersection flag; ids consumed by blocks the candidate's merges
 * erased have rows = cols = 0.  *n = the id count; writes min(n, cap)
 * entries.  Returns HESP_OK or HESP_E_INVALID (no successful trace yet).
 * (The reference-side bridge maps a caller's TaskGraph onto the engine's
 * ids with it: include/hesp_b200_bridge.hpp.) */
typedef struct {
  int64_t row, col, rows, cols;
  int32_t is_intersection, pad;
} hesp_block_info;
int hesp_trace_blocks(const hesp_engine* e, hesp_block_info* out, int32_t cap, int32_t* n);

/* ---------------------------------------------------------------------------
 * Iterative schedule/partition solver (the reference
 * declares it only: solver.hpp:57-86, semantics SPEC.md:410-461).  A chain
 * state is a candidate descriptor (base tiling + partition/merge ops).  Each
 * iteration simulates the state on the device with the full trace (idle_avg
 * per task), records its metrics, collects and scores candidates exactly as
 * SPEC's collect_candidates / score_candidate / choose_p define them, then
 * evaluates EVERY candidate mutation in one device batch and keeps only the
 * ones whose graph simulates (status 0) before select_candidate (Hard: max
 * score, lowest target id on ties, then candidate order; Soft:
 * score-proportional draw from hesp::Rng).  A chain state holds at most
 * HESP_MAX_OPS ops (merges append, they do not cancel): once candidates would
 * exceed it they are dropped and budget_iteration records where that began.
 * DESIGN.md §10 states the decisions the SPEC leaves open. */
enum { HESP_SEL_ALL = 0, HESP_SEL_CP = 1, HESP_SEL_SHALLOW = 2 };
/* HESP_SAMPLE_EXACT (an extension, not in SPEC): the validity batch already
 * simulated every candidate mutation, so pick the one with the smallest
 * simulated makespan (first in candidate order on ties); `score` then
 * records that makespan. */
enum { HESP_SAMPLE_HARD = 0, HESP_SAMPLE_SOFT = 1, HESP_SAMPLE_EXACT = 2 };
enum { HESP_ACT_NONE = -1, HESP_ACT_PARTITION = 0, HESP_ACT_MERGE = 1, HESP_ACT_REPARTITION = 2 };

typedef struct {              /* SolverConfig, solver.hpp:20-28 */
  int32_t iterations;
  int32_t task_selection;     /* HESP_SEL_* */
  int32_t sampling;           /* HESP_SAMPLE_* */
  int32_t k_max;
  uint64_t seed;
  int64_t min_block;
  double overhead_factor;
} hesp_solver_config;

typedef struct {              /* IterationRecord, solver.hpp:42-49 */
  int32_t iteration;
  int32_t action;             /* HESP_ACT_* applied at the end of the round */
  int32_t target;             /* leaf task id or cluster id */
  int32_t n_candidates;       /* collected (score > 0, within the op budget) */
  int32_t n_valid;            /* of which simulate on the device */
  int32_t dag_depth;
  int64_t d;                  /* characteristic block side of the target */
  double p;                   /* partition parameter of the applied candidate (1 = merge) */
  double score;
  double makespan;
  double avg_block_side;      /* flop-weighted mean leaf block side */
  double avg_load_pct;
} hesp_solver_iteration;

typedef struct {
  int32_t cap_history;        /* in: entries of history (>= iterations) */
  int32_t n_history;
  hesp_solver_iteration* history;
  hesp_cand_desc best;        /* best state found (min makespan, earliest iteration) */
  double best_makespan;
  int32_t best_iteration;
  int32_t budget_iteration;   /* first iteration whose candidates were cut because the state
                                 descriptor would exceed HESP_MAX_OPS ops, or overflowed the
                                 engine's per-candidate slot (ids consumed by merged clusters
                                 count): from there on the chain may differ from an uncapped
                                 solve (-1: never) */
  int64_t n_simulated;        /* device simulations issued (states + candidate batches) */
} hesp_solver_result;

/* choose_p (solver.hpp:59-62): p = 1/k, k = clamp(ceil(sqrt(I+1)) + 1, 2,
 * min(k_max, d/min_block)) snapped down to a divisor grid of d; 0.0 when
 * d < 2*min_block or no grid exists (GrainTooSmall). */
double hesp_choose_p(double idle_avg, int64_t d, int64_t min_block, int32_t k_max);

/* select_candidate (solver.hpp:78-80) over bare scores: Hard = index of the
 * maximum score (first on ties: without target ids; hesp_solve breaks Hard
 * ties by the lowest target id); Soft = score-proportional draw
 * with hesp::Rng, whose splitmix64 state *rng_state advances.  -1 for an
 * empty list. */
int32_t hesp_select_candidate(const double* scores, int32_t n, int32_t sampling, uint64_t* rng_state);

/* Runs solve() from `initial` (NULL = the base tiling).  Returns 0, the
 * status of a failing initial state, or a negative HESP_E_* code. */
int hesp_solve(hesp_engine* e, const hesp_cand_desc* initial, const hesp_solver_config* cfg,
               hesp_solver_result* out);

/* n_chains independent solver chains (own config, seed, initial state and
 * result each) advanced in lockstep: per iteration ONE launch traces every
 * chain's state (one warp each) and ONE device batch validates every chain's
 * candidate mutations.  Chain c's result equals hesp_solve with cfgs[c]. */
int hesp_solve_batch(hesp_engine* e, int32_t n_chains, const hesp_cand_desc* initial /* n_chains or NULL */,
                     const hesp_solver_config* cfgs, hesp_solver_result* outs);

/* Cross-GPU winner: every rank passes its own batch
 * best; on return `best` holds the exact lexicographic (makespan, lowest
 * global index) argmin over all ranks of `nccl_comm` and the summed work
 * counters.  Two int64 MIN all-reduces (positive doubles order like their
 * bit patterns) + one int64 SUM, on the engine's stream, over the caller's
 * communicator (an ncclComm_t created by any NCCL in the process, e.g.
 * PyTorch's).  NCCL is resolved at run time (libnccl.so.2), not linked. */
int hesp_min_reduce(hesp_engine* e, void* nccl_comm, hesp_best* best);

/* ---------------------------------------------------------------------------
 * Neighbours of built states (local search, the solver's batches): candidate
 * k is bases[nbrs[k].base] followed by its own 1-2 extra ops.  Each base is
 * expanded once into a template slot; every neighbour copies it and applies
 * only its extra ops.  Outcomes equal hesp_eval_descs on the concatenated
 * descriptors (same ids, blocks and schedules), index k = first + k. */
typedef struct {
  int32_t base;    /* index into bases */
  int32_t n_ops;   /* 0..2 extra ops */
  hesp_op ops[2];
} hesp_neighbor;
int hesp_eval_neighbors(hesp_engine* e, const hesp_cand_desc* bases, int32_t n_bases, const hesp_neighbor* nbrs,
                        uint64_t count, hesp_outcome* out, hesp_best* best);

/* Engine facts: kernel launches issued so far, base tiling sizes, slots. */
typedef struct {
  int64_t kernel_launches;
  int32_t n_base_tasks, n_base_blocks, n_slots, sm_count;
  int64_t slot_bytes;
  int32_t warps_per_block, blocks_per_sm;
  int64_t chunk;   /* candidates per build/simulate chunk (0 = fused kernel) */
  int64_t last_h2d_bytes; /* bytes the last hesp_eval_descs copied host->device (packed descriptors) */
  int64_t min_reduces;    /* completed hesp_min_reduce exchanges on this handle */
} hesp_engine_info;
int hesp_engine_get_info(const hesp_engine* e, hesp_engine_info* info);

void hesp_engine_destroy(hesp_engine* e);

const char* hesp_last_error(void);
const char* hesp_status_name(int32_t status);

#ifdef __cplusplus
}
#endif

#endif /* HESP_ENGINE_H */
